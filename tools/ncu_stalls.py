"""Top warp-stall reasons (issue-active-normalised) per kernel of an ncu --set full capture.
    python tools/ncu_stalls.py rep.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, rows = r[0], r[2:]
    keys = [i for i, k in enumerate(h)
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio")]
    kn = h.index("Kernel Name")
    for row in rows:
        name = row[kn].split("(")[0].split("::")[-1]
        vals = sorted(((float(row[i].replace(",", "") or 0), h[i]) for i in keys), reverse=True)[:5]
        tops = ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
                         for v, k in vals)
        print(f"| {rep.split('/')[-1]} | {name} | {tops} |")

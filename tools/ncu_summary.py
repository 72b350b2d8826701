"""Summarise ncu captures for profiles/: per-kernel duration, DRAM traffic, throughput, occupancy.

    python tools/ncu_summary.py gpurun_out/prof_scale_C2.ncu-rep [...] --out profiles/r01_ncu_C2.md
Writes a markdown table and merges dram bytes/launch into profiles/ncu_traffic.json
(bench.py reports it as roofline.traffic).
"""
import argparse, csv, io, json, re, subprocess
from pathlib import Path

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "inst",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1, "s": 1}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = {"kernel": re.sub(r"\(.*", "", row[hdr.index("Kernel Name")]).split("::")[-1]}
        for k, short in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = float(row[i].replace(",", "")) if row[i] else 0.0
                d[short] = v * SCALE.get(units[i], 1) if short in ("duration", "dram_read", "dram_write") else v
        yield d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--out", required=True)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    lines = [f"# ncu summary {a.title}".rstrip(), "",
             "| capture | kernel | grid | regs | duration us | DRAM read MB | DRAM write MB | DRAM % peak | SM % | warps active % |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for rep in a.reps:
        for d in rows(rep):
            lines.append(f"| {Path(rep).name} | {d['kernel']} | {int(d.get('grid', 0))} | {int(d.get('regs', 0))} | "
                         f"{d['duration'] * 1e6:.1f} | {d.get('dram_read', 0) / 1e6:.2f} | {d.get('dram_write', 0) / 1e6:.2f} | "
                         f"{d.get('dram_pct_peak', 0):.1f} | {d.get('sm_pct', 0):.1f} | {d.get('occupancy_pct', 0):.1f} |")
            if d["kernel"].startswith("k_scale"):
                traffic.setdefault("k_scale", int(d.get("dram_read", 0) + d.get("dram_write", 0)))
                traffic.setdefault("dram_pct", round(float(d.get("dram_pct_peak", 0)), 1))
    Path(a.out).write_text("\n".join(lines) + "\n")
    tj = Path("profiles/ncu_traffic.json")
    data = json.loads(tj.read_text()) if tj.exists() else {}
    if traffic:
        data.setdefault(a.config, {})["k_scale"] = {"dram_bytes_per_launch": traffic["k_scale"],
                                                    "dram_pct_of_ncu_peak": traffic["dram_pct"],
                                                    "source": str(Path(a.out).name)}
        tj.write_text(json.dumps(data, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()

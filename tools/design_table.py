"""Print DESIGN.md §9's measured table from profiles/r01_bench/bench_C*.json (CPU)."""
import json
from pathlib import Path

ROWS = {"C1": "C1 1 × 1M f32 (4 MB; L2 flushed before every step)", "C2": "**C2** 64 × 4Mi f32, depth-4 dense",
        "C3": "C3 64 chains, scattered", "C4": "C4 1M × 256 f32, 1.02M sites", "C5": "C5 64 GiB on one GPU"}
print("| Config | value: HBM-resident step (graph GB/s) | leaf kernel (× measured HBM copy; × nominal 8 TB/s) | "
      "e2e from host buffers | e2e ÷ copy-only pipeline (this box's link) | CPU port |")
print("|---|---|---|---|---|---|")
for c, name in ROWS.items():
    d = json.loads((Path("profiles/r01_bench") / f"bench_{c}.json").read_text())
    e, r, cpu = d["e2e"], d["roofline"], d.get("cpu_baseline", {})
    step = d["ms_per_step"]
    step_s = f"{step * 1e3:.1f} µs" if step < 0.1 else (f"{step:.3f} ms" if step < 10 else f"{step:.1f} ms")
    e2e_ms = e["ms_per_step"]
    e2e_s = f"{e2e_ms:.2f} ms" if e2e_ms < 100 else f"{e2e_ms / 1e3:.2f} s"
    nominal = r.get("frac_of_nominal_8tbs")
    link = e["host_link_gbs"]["bidir"]
    frac = e.get("frac_of_link_roofline")
    frac_s = "—" if c == "C1" else f"{frac:.2f} ({link:.0f} GB/s both ways)"
    print(f"| {name} | {d['value']:.0f} ({step_s}) | {r['frac']:.2f}; {nominal:.2f} | {e['value']:.1f} GB/s ({e2e_s}) | "
          f"{frac_s} | {cpu.get('value', 0):.1f} GB/s ({cpu.get('cores', '?')} cores) |")

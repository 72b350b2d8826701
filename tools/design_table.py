"""Print DESIGN.md §9's measured table from profiles/r02_bench/bench_C*.json (CPU).
C1 comes from the default (C2) line's per_config block; C2-C5 from their own lines."""
import json
from pathlib import Path

B = Path("profiles/r02_bench")
ROWS = {"C1": "C1 1 × 1M f32 (4 MB; L2 flushed before every step)", "C2": "**C2** 64 × 4Mi f32, depth-4 dense",
        "C3": "C3 64 chains, scattered", "C4": "C4 1M × 256 f32, 1.02M sites", "C5": "C5 64 GiB on one GPU"}


def fmt_ms(ms: float) -> str:
    return f"{ms * 1e3:.1f} µs" if ms < 0.1 else (f"{ms:.4f} ms" if ms < 10 else f"{ms:.1f} ms")


print("| Config | value: HBM-resident step (graph GB/s) | leaf kernel (× measured HBM copy) | share of step | "
      "e2e from host buffers | e2e ÷ plain-copy link probe | CPU port |")
print("|---|---|---|---|---|---|---|")
c2 = json.loads((B / "bench_C2.json").read_text())
for c, name in ROWS.items():
    if c == "C1":
        p = c2["per_config"]["C1"]
        print(f"| {name} | {p['value_gbs']:.0f} ({fmt_ms(p['resident_ms_per_step'])}) | {p['kernel_frac']:.2f} | "
              f"{p['kernel_share_of_resident_step']:.2f} | {p['e2e_gbs']:.1f} GB/s ({fmt_ms(p['e2e_ms_per_step'])}) | "
              f"{p['frac_of_link_roofline']:.2f} (same-size probe {p['link_probe_gbs']['bidir']:.0f} GB/s) | — |")
        continue
    d = json.loads((B / f"bench_{c}.json").read_text())
    e, r, cpu = d["e2e"], d["roofline"], d.get("cpu_baseline", {})
    e2e_ms = e["ms_per_step"]
    e2e_s = f"{e2e_ms:.2f} ms" if e2e_ms < 100 else f"{e2e_ms / 1e3:.2f} s"
    print(f"| {name} | {d['value']:.0f} ({fmt_ms(d['ms_per_step'])}) | {r['frac']:.3f} | {r['share_of_resident_step']:.3f} | "
          f"{e['value']:.1f} GB/s ({e2e_s}) | {e['frac_of_link_roofline']:.2f} ({e['host_link_gbs']['bidir']:.0f} GB/s both ways) | "
          f"{cpu.get('value', 0):.1f} GB/s ({cpu.get('cores', '?')} cores) |")

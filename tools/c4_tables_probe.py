"""How much of C4's e2e gap to the link is the per-window table upload?  e2e windows (double-
buffered pair) with and without CF_WIN_TABLES (tables already resident from the plan), C2 for
reference.  Design experiment only: the product path always uploads the tables."""
import sys
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow, _native as N

for cfg in sys.argv[1:] or ["C4", "C2"]:
    spec, policy, _ = bench.make_spec(cfg)
    w = DeepCopyWindow(spec, seed=1, policy=policy, align=16, separate_output=True)
    tw = w.twin()
    link = N.link_probe(w.ctx, 1 << 30, iters=1, reps=3)
    for name, fl in (("full", N.CF_WIN_FULL | N.CF_WIN_GRAPH), ("no_tables", (N.CF_WIN_FULL & ~N.CF_WIN_TABLES) | N.CF_WIN_GRAPH)):
        w.run_pair_n(tw, 6, flags=fl)
        best = None
        for _ in range(3):
            st = w.run_pair_n(tw, 20, flags=fl)
            ms = st.ms_total / 20
            best = ms if best is None else min(best, ms)
        h2d = st.h2d_bytes / 20
        ideal = (h2d + w.total) / (link["bidir"] * 1e9) * 1e3
        print(f"{cfg} {name}: {best:.3f} ms/window, h2d {h2d / 1e6:.1f} MB, e2e {w.total / best / 1e6:.2f} GB/s, "
              f"frac of plain link {ideal / best:.4f} (link {link['bidir']:.1f})", flush=True)
    tw.close()
    w.close()

"""Design experiment: alternating two windows (double-buffered images) vs one, C2/C3 e2e."""
import sys
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow, _native as N
for cfg in ("C2", "C3", "C4"):
    spec, policy, _ = bench.make_spec(cfg)
    w = DeepCopyWindow(spec, seed=1, policy=policy)
    t = w.twin()
    for g in (0, N.CF_WIN_GRAPH):
        fl = N.CF_WIN_FULL | g
        w.run_n(3, flags=fl)
        st1 = w.run_n(10, flags=fl)
        w.run_pair_n(t, 4, flags=fl)
        st2 = w.run_pair_n(t, 10, flags=fl)
        print(cfg, "graph" if g else "direct", "single", round(st1.ms_total / 10, 3), "pair", round(st2.ms_total / 10, 3), flush=True)
    t.close(); w.close()

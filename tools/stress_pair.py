"""Stress: repeated single/pair e2e windows (direct + graph) per config; reports the first failure."""
import sys, traceback
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow, _native as N
for cfg in sys.argv[1:]:
    spec, policy, _ = bench.make_spec(cfg)
    w = DeepCopyWindow(spec, seed=1, policy=policy)
    t = w.twin()
    try:
        for it in range(4):
            for g in (0, N.CF_WIN_GRAPH):
                fl = N.CF_WIN_FULL | g
                w.run_n(3, flags=fl)
                w.run_n(5, flags=fl)
                w.run_pair_n(t, 4, flags=fl)
                w.run_pair_n(t, 6, flags=fl)
                w.upload_raw()
                w.run_n(3, flags=N.CF_WIN_RESIDENT | g)
        print(cfg, "ok", flush=True)
    except Exception as e:
        print(cfg, "FAIL at it", it, "graph" if g else "direct", e, flush=True)
        sys.exit(1)

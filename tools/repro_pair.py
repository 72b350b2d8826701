"""Stress the double-buffered window pair (bench e2e path) on a config; report failures.
python tools/repro_pair.py C4 [graph|direct] [rounds]"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1906_01128_b200 import DeepCopyWindow  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
mode = sys.argv[2] if len(sys.argv) > 2 else "graph"
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 10
spec, policy, _ = bench.make_spec(cfg)
w = DeepCopyWindow(spec, seed=1, policy=policy, align=16)
t = w.twin()
fl = N.CF_WIN_FULL | (N.CF_WIN_GRAPH if mode == "graph" else 0)
for r in range(rounds):
    st = w.run_pair_n(t, 5 if r % 2 else 20, flags=fl)
    print(f"{cfg} {mode} round {r}: ok {st.ms_total:.2f} ms", flush=True)

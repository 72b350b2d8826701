"""Single (not double-buffered) window device time: separate vs in-place copy-back, graph vs
direct enqueue -- what the fused drop-in window can reach.  python tools/e2e_single.py C2"""
import sys
import statistics

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1906_01128_b200 import DeepCopyWindow  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec, policy, _ = bench.make_spec(cfg)
for sep in (True, False):
    w = DeepCopyWindow(spec, seed=1, policy=policy, align=16, separate_output=sep)
    for flags, name in ((N.CF_WIN_FULL, "direct"), (N.CF_WIN_FULL | N.CF_WIN_GRAPH, "graph")):
        ms = []
        for r in range(8):
            st = w.run(scale=2.0 if r % 2 == 0 else 0.5, flags=flags)
            ms.append(st.ms_total)
        print(f"{cfg} separate_output={sep} {name}: median {statistics.median(ms[2:]):.2f} ms "
              f"(all {[round(x, 2) for x in ms]}) launches {st.launches} steps {st.nsteps}", flush=True)
    w.close()

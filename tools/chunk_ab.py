"""Interleaved A/B of the e2e window chunk size on one box (design experiment).
python tools/chunk_ab.py C2 16,32,64 [rounds]"""
import statistics
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1906_01128_b200 import DeepCopyWindow  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402

cfg = sys.argv[1]
chunks = [int(x) for x in sys.argv[2].split(",")]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
spec, policy, _ = bench.make_spec(cfg)
w = DeepCopyWindow(spec, seed=1, policy=policy, align=16)
t = w.twin()
fl = N.CF_WIN_FULL | N.CF_WIN_GRAPH
res = {c: [] for c in chunks}
for r in range(rounds):
    for c in chunks:
        w.chunk_bytes = t.chunk_bytes = c << 20
        w.run_pair_n(t, 4, flags=fl)
        res[c].append(w.run_pair_n(t, 10, flags=fl).ms_total / 10)
for c in chunks:
    print(f"{cfg} chunk {c:3d} MiB: median {statistics.median(res[c]):.3f} ms  all {[round(x, 2) for x in res[c]]}", flush=True)

"""C4 e2e window variants (design experiment): chunk size, table upload on/off, graph on/off.
python tools/e2e_c4.py [C4]"""
import statistics
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1906_01128_b200 import DeepCopyWindow  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
spec, policy, _ = bench.make_spec(cfg)
chunks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else (16, 32, 64)
only_full = len(sys.argv) > 3
for chunk_mb in chunks:
    w = DeepCopyWindow(spec, seed=1, policy=policy, align=16, chunk_bytes=chunk_mb << 20)
    t = w.twin()
    for name, fl in (("full", N.CF_WIN_FULL | N.CF_WIN_GRAPH), ("no-tables", (N.CF_WIN_FULL & ~N.CF_WIN_TABLES) | N.CF_WIN_GRAPH),
                     ("copy-only", N.CF_WIN_H2D | N.CF_WIN_D2H)):
        if only_full and name != "full":
            continue
        w.run_pair_n(t, 4, flags=fl)
        ms = [w.run_pair_n(t, 10, flags=fl).ms_total / 10 for _ in range(3)]
        print(f"{cfg} chunk {chunk_mb} MiB {name:10s}: {statistics.median(ms):.3f} ms/window", flush=True)
    t.close()
    w.close()

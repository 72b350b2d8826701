"""Fused naive window on C4 by pipeline chunk size (design experiment)."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1906_01128_b200 as cf  # noqa: E402
from paper_1906_01128_b200 import harness as H  # noqa: E402

spec, policy, _ = bench.make_spec(sys.argv[1] if len(sys.argv) > 1 else "C4")
for mb in (16, 32, 64, 128, 256):
    H.FUSED_CHUNK = mb << 20
    m = cf.Machine()
    h = cf.build_tree(m, spec, seed=1, align=16)
    ts = []
    for r in range(4):
        prep = cf.transfer_to_device(m, h, "naive", policy=policy)
        cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5)
        t = time.perf_counter()
        cf.copy_back(m, h, prep)
        ts.append(time.perf_counter() - t)
    print(f"chunk {mb:4d} MiB: naive window copy_back {statistics.median(ts[1:]) * 1e3:.1f} ms "
          f"arrays {prep.fused.timing['arrays_ms']:.1f} ms", flush=True)
    m.close()

import sys, time, statistics
sys.path.insert(0, "/root/repo")
import bench
import paper_1906_01128_b200 as cf
from paper_1906_01128_b200 import harness as H
spec, policy, _ = bench.make_spec("C2")
for chunk in (16 << 20, 32 << 20, 64 << 20, 128 << 20):
    H.FUSED_CHUNK = chunk
    m = cf.Machine()
    h = cf.build_tree(m, spec, seed=1, align=16)
    ts = []
    for r in range(5):
        m.ctx.sync()
        t = time.perf_counter()
        prep = cf.transfer_to_device(m, h, "pointerchain", policy=policy)
        cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5)
        cf.copy_back(m, h, prep)
        m.ctx.sync()
        ts.append(time.perf_counter() - t)
    print(f"chunk {chunk >> 20} MiB: pointerchain window median {statistics.median(ts[1:]) * 1e3:.2f} ms", flush=True)
    m.close()

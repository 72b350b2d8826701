"""Profiling target: build one workload's window and run only its resident step (attach ->
resolve -> leaf kernel -> detach) a few times, or the full window with --full.  Meant to be
wrapped in ncu (one GPU)."""
import argparse, sys
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow, _native as N

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--runs", type=int, default=4)
ap.add_argument("--mode", default="resolved")
ap.add_argument("--full", action="store_true")
ap.add_argument("--graph", action="store_true", help="resident steps replayed from a CUDA graph (fused detach, PDL)")
ap.add_argument("--dense", default="", help="q,n,depth,elem: a leaves-only dense spec instead of --config")
ap.add_argument("--align", type=int, default=16)
a = ap.parse_args()
if a.dense:
    from paper_1906_01128_b200 import DenseSpec
    q, n, d, e = (int(x) for x in a.dense.split(","))
    spec, policy = DenseSpec(q, n, d, elem=e, leaf_only=True), "all_leaves"
else:
    spec, policy, _ = bench.make_spec(a.config)
w = DeepCopyWindow(spec, seed=1, policy=policy, mode=a.mode, align=a.align, chunk_bytes=16 << 20)
if a.full:
    for i in range(a.runs):
        st = w.run(scale=2.0 if i % 2 == 0 else 0.5)
else:
    w.upload_raw()
    for i in range(a.runs):
        st = w.run_resident(scale=2.0 if i % 2 == 0 else 0.5, graph=a.graph)
print(f"{a.config} total={w.total} ms_total={st.ms_total:.4f} ms_kernel={st.ms_kernel:.4f} launches={st.launches}")
w.close()

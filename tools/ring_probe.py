"""C2 / C4 e2e: two windows alternating (the bench's pair) vs rings of 3 and 4 windows (each its
own image and copy-back buffer), CUDA-graph windows, best of 3 batches of 20 (design experiment)."""
import sys
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow, _native as N

for cfg in sys.argv[1:] or ["C2", "C4"]:
    spec, policy, _ = bench.make_spec(cfg)
    w = DeepCopyWindow(spec, seed=1, policy=policy, align=16, separate_output=True)
    twins = [w.twin() for _ in range(3)]
    fl = N.CF_WIN_FULL | N.CF_WIN_GRAPH
    link = N.link_probe(w.ctx, 1 << 30, iters=1, reps=3)
    for name, run in (("pair", lambda n: w.run_pair_n(twins[0], n, flags=fl)),
                      ("ring3", lambda n: w.run_ring_n(twins[:2], n, flags=fl)),
                      ("ring4", lambda n: w.run_ring_n(twins[:3], n, flags=fl)),
                      ("pair", lambda n: w.run_pair_n(twins[0], n, flags=fl))):
        run(8)
        best = min(run(20).ms_total / 20 for _ in range(3))
        print(f"{cfg} {name}: {best:.3f} ms/window = {w.total / best / 1e6:.2f} GB/s "
              f"(link {link['bidir']:.1f})", flush=True)
    for t in twins:
        t.close()
    w.close()

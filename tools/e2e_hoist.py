"""Design experiment: node hoisting on/off and chunking for C2/C3 e2e windows."""
import sys
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow, _native as N
for cfg in ("C2", "C3"):
    spec, policy, _ = bench.make_spec(cfg)
    w = DeepCopyWindow(spec, seed=1, policy=policy)
    for chunk in (16, 32):
        for name, fl in (("bidir", N.CF_WIN_H2D | N.CF_WIN_D2H), ("full", N.CF_WIN_FULL | N.CF_WIN_GRAPH)):
            w.run_n(2, flags=fl, chunk_bytes=chunk << 20)
            st = w.run_n(6, flags=fl, chunk_bytes=chunk << 20)
            print(cfg, chunk, name, round(st.ms_total / 6, 3), "ms", st.nchunks, "segs", st.nsteps, "steps", st.launches // 6, "launches", flush=True)
    w.close()

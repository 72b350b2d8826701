"""Design experiment: copy-engine / stream / chunk configuration of the pipelined window (C2)."""
import sys, itertools
sys.path.insert(0, ".")
from paper_1906_01128_b200 import DeepCopyWindow, DenseSpec, _native as N

spec = DenseSpec(4, 4 << 20, 3, elem=4, leaf_only=True)
for ns in (1, 2, 4):
    w = None
    for chunk_mb in (8, 16, 64):
        if w is None:
            w = DeepCopyWindow(spec, seed=1, chunk_bytes=chunk_mb << 20, nstreams=ns)
        res = {}
        for name, fl in (("h2d", N.CF_WIN_H2D), ("d2h", N.CF_WIN_D2H), ("bidir", N.CF_WIN_H2D | N.CF_WIN_D2H),
                         ("full", N.CF_WIN_FULL)):
            w.run_n(2, flags=fl, chunk_bytes=chunk_mb << 20)
            st = w.run_n(4, flags=fl, chunk_bytes=chunk_mb << 20)
            res[name] = (st.ms_total / 4, (st.h2d_bytes + st.d2h_bytes) / (st.ms_total * 1e-3) / 1e9)
        print(f"streams={ns} chunk={chunk_mb}MiB " + " ".join(f"{k}:{v[0]:.2f}ms/{v[1]:.1f}GB/s" for k, v in res.items()), flush=True)
    w.close()

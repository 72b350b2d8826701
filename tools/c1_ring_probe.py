"""C1 (4 MB graph) e2e window variants (design experiment): ring size x step size x CUDA graph,
and the same-size plain-copy probe (best of 10) before and after.
    python tools/c1_ring_probe.py"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1906_01128_b200 import DeepCopyWindow  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402

spec, policy, _ = bench.make_spec("C1")
base = DeepCopyWindow(spec, seed=1, policy=policy, align=16)
probe = N.link_probe(base.ctx, base.total, iters=8, reps=10)
out = {"probe_same_size": {k: round(v, 2) for k, v in probe.items()}}
twins = [base.twin() for _ in range(67)]
for chunk in (1 << 20, 2 << 20, 4 << 20):
    for ring in (8, 16, 34, 68):
        for graph in ((True, False) if chunk == 4 << 20 else (True,)):
            ws = [base] + twins[:ring - 1]
            for w in ws:
                w.chunk_bytes = chunk
            fl = N.CF_WIN_FULL | (N.CF_WIN_GRAPH if graph else 0)
            base.run_ring_n(ws[1:], ring + 2, flags=fl)
            best = 1e9
            for _ in range(3):
                st = base.run_ring_n(ws[1:], 40, flags=fl)
                best = min(best, st.ms_total / 40)
            bidir = 2 * base.total / (best * 1e-3) / 1e9
            key = f"chunk{chunk >> 20}M_ring{ring}_{'graph' if graph else 'direct'}"
            out[key] = {"ms": round(best, 4), "bidir_gbs": round(bidir, 2), "frac": round(bidir / probe["bidir"], 3)}
            print(key, out[key], flush=True)
out["probe_same_size_after"] = {k: round(v, 2) for k, v in N.link_probe(base.ctx, base.total, iters=8, reps=10).items()}
print(json.dumps(out))

"""Design experiment: why C3 (scattered forest) copies slower than C2."""
import sys
sys.path.insert(0, ".")
from paper_1906_01128_b200 import DeepCopyWindow, ForestSpec, LinearSpec, _native as N
H, D = N.CF_WIN_H2D, N.CF_WIN_D2H
for name, spec in (("forest-dfs", ForestSpec(LinearSpec(4, 4 << 20, "LLinit_LLused", elem=4), 64, 0)),
                   ("forest-scatter", ForestSpec(LinearSpec(4, 4 << 20, "LLinit_LLused", elem=4), 64, 0xC3))):
    w = DeepCopyWindow(spec, seed=1, policy="all_leaves")
    for chunk in (16, 64):
        for fl, fn in ((H, "h2d"), (D, "d2h"), (H | D, "bidir"), (N.CF_WIN_FULL | N.CF_WIN_GRAPH, "full")):
            w.run_n(2, flags=fl, chunk_bytes=chunk << 20)
            st = w.run_n(5, flags=fl, chunk_bytes=chunk << 20)
            print(name, chunk, fn, round(st.ms_total / 5, 3), "segs", st.nchunks, "steps", st.nsteps, flush=True)
    w.close()

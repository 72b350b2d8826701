import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1906_01128_b200 import DeepCopyWindow, ForestSpec, LinearSpec, _native as N
spec = ForestSpec(LinearSpec(4, 1 << 22, "LLinit_LLused", elem=4), 16, 0xC3)
w = DeepCopyWindow(spec, seed=1, policy="all_leaves")
for fl in (N.CF_WIN_FULL, N.CF_WIN_FULL | N.CF_WIN_GRAPH):
    st = w.run(scale=2.0, flags=fl)
    print("ok", fl, st.nchunks, st.nsteps, flush=True)

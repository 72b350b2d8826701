import os, subprocess, sys
code = r'''
import sys
sys.path.insert(0, ".")
from paper_1906_01128_b200 import DeepCopyWindow, ForestSpec, LinearSpec, _native as N
H, D = N.CF_WIN_H2D, N.CF_WIN_D2H
spec = ForestSpec(LinearSpec(4, 4 << 20, "LLinit_LLused", elem=4), 64, 0xC3)
w = DeepCopyWindow(spec, seed=1, policy="all_leaves")
out = []
for fl, fn in ((H | D, "bidir"), (N.CF_WIN_FULL | N.CF_WIN_GRAPH, "full")):
    w.run_n(2, flags=fl)
    st = w.run_n(5, flags=fl)
    out.append(f"{fn} {st.ms_total / 5:.3f} segs {st.nchunks}")
print(" | ".join(out))
'''
for so in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, CF_B200_LIB=so), capture_output=True, text=True)
    print(so, r.stdout.strip() or r.stderr[-300:], flush=True)

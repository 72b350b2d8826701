"""Leaf-kernel and resident-step times of C2 / C4 / C1 under each library variant in build/variants
(design experiment: launch bounds, tile search hoist, warp-cooperative resolve).
python tools/r2_variant_timing.py [variant.so ...]"""
import json
import os
import subprocess
import sys

code = r'''
import sys, statistics, json
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow
from paper_1906_01128_b200 import _native as N
out = {}
for cfg in sys.argv[1:]:
    spec, policy, _ = bench.make_spec(cfg)
    w = DeepCopyWindow(spec, seed=1, policy=policy)
    w.upload_raw()
    for i in range(3): w.run_resident(scale=2.0 if i % 2 == 0 else 0.5)
    ks = [w.run_resident(scale=2.0 if i % 2 == 0 else 0.5).ms_kernel for i in range(10)]
    w.run_n(4, flags=N.CF_WIN_RESIDENT | N.CF_WIN_GRAPH)
    st = w.run_n(20, flags=N.CF_WIN_RESIDENT | N.CF_WIN_GRAPH)
    out[cfg] = {"kernel_ms": round(statistics.median(ks), 4), "resident_ms": round(st.ms_total / 20, 4)}
    w.close()
print(json.dumps(out))
'''
sos = sys.argv[1:] or sorted(os.path.join("build/variants", f) for f in os.listdir("build/variants") if f.endswith(".so"))
for so in ["(in-tree)"] + sos:
    env = dict(os.environ)
    if so != "(in-tree)":
        env["CF_B200_LIB"] = so
    for rep in range(2):
        r = subprocess.run([sys.executable, "-c", code, "C2", "C4"], env=env, capture_output=True, text=True)
        print(os.path.basename(so), rep, r.stdout.strip() or r.stderr[-800:], flush=True)

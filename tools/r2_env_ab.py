"""A/B of the resident step under environment switches of the library (design experiments):
leaf-kernel time (CUDA events around the k_scale launch) and graph-replayed resident step per
config, each variant in a fresh process, twice.
python tools/r2_env_ab.py [C4 C2 ...] -- each variant is a comma list of VAR=VALUE (or 'base')."""
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
    rs = []
    for _ in range(3):
        st = w.run_n(40, flags=N.CF_WIN_RESIDENT | N.CF_WIN_GRAPH)
        rs.append(st.ms_total / 40)
    out[cfg] = {"kernel_ms": round(statistics.median(ks), 4), "resident_ms": round(min(rs), 4),
                "overhead": round(min(rs) / statistics.median(ks) - 1, 4)}
    w.close()
print(json.dumps(out))
'''
args = sys.argv[1:]
if "--" in args:
    cut = args.index("--")
    cfgs, variants = args[:cut], args[cut + 1:]
else:
    cfgs, variants = args, ["base"]
cfgs = cfgs or ["C4", "C2"]
for v in variants:
    env = dict(os.environ)
    if v != "base":
        for kv in v.split(","):
            k, _, val = kv.partition("=")
            env[k] = val
    for rep in range(2):
        r = subprocess.run([sys.executable, "-c", code, *cfgs], env=env, capture_output=True, text=True)
        print(v, rep, r.stdout.strip() or r.stderr[-800:], flush=True)

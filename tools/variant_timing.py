"""Time the resident leaf kernel of C2 / C4 under each library variant (design experiment)."""
import os, subprocess, sys, json
code = r'''
import sys, statistics, json
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow
out = {}
for cfg in sys.argv[1:]:
    spec, policy, _ = bench.make_spec(cfg)
    w = DeepCopyWindow(spec, seed=1, policy=policy)
    w.upload_raw()
    for i in range(3): w.run_resident(scale=2.0 if i % 2 == 0 else 0.5)
    ks = [w.run_resident(scale=2.0 if i % 2 == 0 else 0.5).ms_kernel for i in range(10)]
    out[cfg] = round(statistics.median(ks), 4)
    w.close()
print(json.dumps(out))
'''
for so in sorted(os.listdir("build/variants")):
    if not so.endswith(".so"): continue
    env = dict(os.environ, CF_B200_LIB=os.path.join("build/variants", so))
    r = subprocess.run([sys.executable, "-c", code, "C2", "C4"], env=env, capture_output=True, text=True)
    print(so, r.stdout.strip() or r.stderr[-500:], flush=True)

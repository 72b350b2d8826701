"""A/B the resident C2/C4 leaf kernel across library builds, alternating, in fresh processes."""
import os, subprocess, sys
code = r'''
import sys, statistics, json
sys.path.insert(0, ".")
import bench
from paper_1906_01128_b200 import DeepCopyWindow, _native as N
out = {}
for cfg in sys.argv[1:]:
    spec, policy, _ = bench.make_spec(cfg)
    w = DeepCopyWindow(spec, seed=1, policy=policy)
    w.upload_raw()
    w.run_n(20, flags=N.CF_WIN_RESIDENT | N.CF_WIN_GRAPH)
    ks = [w.run_resident(scale=2.0 if i % 2 == 0 else 0.5).ms_kernel for i in range(30)]
    st = w.run_n(50, flags=N.CF_WIN_RESIDENT | N.CF_WIN_GRAPH)
    out[cfg] = (round(statistics.median(ks), 4), round(st.ms_total / 50, 4))
    w.close()
print(json.dumps(out))
'''
libs = sys.argv[1:]
for rep in range(2):
    for so in libs:
        env = dict(os.environ, CF_B200_LIB=so)
        r = subprocess.run([sys.executable, "-c", code, "C2", "C4"], env=env, capture_output=True, text=True)
        print(rep, so, r.stdout.strip() or r.stderr[-400:], flush=True)

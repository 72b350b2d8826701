"""Soak test: minutes of back-to-back windows in every mode on every config, verifying the result
after each batch against payload_values x the net scale (dense configs: the whole copy-back against
the oracle's expected arena).  Catches rare races (the torn pointer
read needed ~1000 windows).  python tools/soak.py SECONDS [configs...]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1906_01128_b200 import DeepCopyWindow  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402
from paper_1906_01128_b200.scenarios import payload_values  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 300
cfgs = sys.argv[2:] or ["C2", "C3", "C4"]
deadline = time.time() + secs
per = secs / len(cfgs)
total = 0
EXTRA = {   # packed reference layouts: f64 leaves at 4 mod 8 (word-streaming kernel), 12-byte leaf records
    "P3": (lambda: __import__("paper_1906_01128_b200").DenseSpec(3, 5 << 20, 3, elem=8, leaf_only=True), "all_leaves", 1),
    "P4": (lambda: __import__("paper_1906_01128_b200").DenseSpec(4, 2 << 20, 3, elem=8, leaf_only=True), "all_leaves", 1),
}
for cfg in cfgs:
    if cfg in EXTRA:
        mk, policy, align = EXTRA[cfg]
        spec = mk()
    else:
        (spec, policy, _), align = bench.make_spec(cfg), 16
    w = DeepCopyWindow(spec, seed=1, policy=policy, align=align)
    t = w.twin()
    off, cnt, lvl = w.table(N.CF_TAB_ARR_OFF), w.table(N.CF_TAB_ARR_COUNT), w.table(N.CF_TAB_ARR_LEVEL)
    src = w.host_src().copy()
    # the whole copy-back of the twin (scale 0.5 last) against the oracle's expected arena
    from oracle import oracle as O
    kind = {"DenseSpec": O.DENSE}.get(type(spec).__name__)
    full = None
    if kind is not None:
        ot = O.build(O.OSpec(kind, spec.q, spec.n, spec.depth, elem=spec.elem, leaf_only=spec.leaf_only, align=align),
                     1, ptr_base=w.src)
        pol = {"all_leaves": O.TARGET_ALL_LEAVES, "all_arrays": O.TARGET_ALL_ARRAYS, "ref": O.TARGET_REF}[policy]
        full = O.expected_after_window(ot, O.targets(ot, pol), 0.5)[:w.total]
    end = min(deadline, time.time() + per)
    it = 0
    while time.time() < end:
        g = N.CF_WIN_GRAPH if it % 2 else 0
        st = w.run_pair_n(t, 8, flags=N.CF_WIN_FULL | g)          # last window (t): scale 0.5
        assert st.bad == N.NO_BAD
        w.upload_raw()
        st = w.run_n(10, flags=N.CF_WIN_RESIDENT | g)            # net scale 1.0 on the image
        assert st.bad == N.NO_BAD
        # checks: the image is back to the source, the twin's copy-back holds leaves x 0.5
        assert np.array_equal(w.image_bytes(), src), (cfg, it, "resident")
        got = t.host_dst()
        if full is not None:
            assert np.array_equal(got, full), (cfg, it, "whole copy-back")
        for i in (int(w.targets[0]), int(w.targets[len(w.targets) // 2]), int(w.targets[-1])):
            a, n = int(off[i]), int(cnt[i])
            dt = np.float32 if spec.elem == 4 else np.float64
            want = (payload_values(1, int(lvl[i]), n, spec.elem) * dt(0.5)).astype(dt)
            assert np.array_equal(np.frombuffer(got[a:a + spec.elem * n].tobytes(), dt), want), (cfg, it, i)
        it += 1
        total += 18
    print(f"{cfg}: {it} rounds ({it * 18} windows) ok", flush=True)
    t.close()
    w.close()
print("soak ok", total, "windows")

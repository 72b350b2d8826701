"""Pointerchain window device time by stage set (copy-only vs full), C2 (design experiment)."""
import sys
import time
import statistics
import ctypes as C

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1906_01128_b200 as cf  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402

spec, policy, _ = bench.make_spec(sys.argv[1] if len(sys.argv) > 1 else "C2")
m = cf.Machine()
h = cf.build_tree(m, spec, seed=1, align=16)
prep = cf.transfer_to_device(m, h, "pointerchain", policy=policy)
cf.kernel_scale(m, h, prep, 2.0)
cf.copy_back(m, h, prep)
w = next(v for k, v in m._plans.items() if k[0] == "selective")
for name, fl in (("H2D only", N.CF_WIN_H2D), ("D2H only", N.CF_WIN_D2H), ("H2D+D2H", N.CF_WIN_H2D | N.CF_WIN_D2H),
                 ("full", N.CF_WIN_H2D | N.CF_WIN_SCALE | N.CF_WIN_D2H)):
    ts = []
    for r in range(6):
        m.ctx.sync()
        t = time.perf_counter()
        N.check(N.lib().cf_selective_run(w, fl, 2.0 if r % 2 == 0 else 0.5))
        ts.append(time.perf_counter() - t)
    print(f"{name:10s} {statistics.median(ts[1:]) * 1e3:.2f} ms", flush=True)
m.close()

# the marshalling window over the same shape, single window, copy-only and full, in place and not
from paper_1906_01128_b200 import DeepCopyWindow  # noqa: E402
for sep in (False, True):
    dw = DeepCopyWindow(spec, seed=1, policy=policy, align=16, separate_output=sep)
    for name, fl in (("H2D+D2H", N.CF_WIN_H2D | N.CF_WIN_D2H), ("full", N.CF_WIN_FULL)):
        ts = []
        for r in range(6):
            st = dw.run_n(1, flags=fl)
            ts.append(st.ms_total)
        print(f"window separate={sep} {name:10s} {statistics.median(ts[1:]):.2f} ms", flush=True)
    dw.close()

"""Zero-copy per-object copies (k_copy_list) vs one bulk SM copy over the same bytes: 1 GiB of
pinned host memory as N contiguous objects, H2D and D2H (design experiment)."""
import sys
import time
import ctypes as C

import numpy as np

sys.path.insert(0, ".")
from paper_1906_01128_b200 import _native as N  # noqa: E402

ctx = N.DeviceContext.get(0)
lib = N.lib()
G = 1 << 30
h = C.c_void_p()
d = C.c_void_p()
N.check(lib.cf_host_alloc(G, N.CF_MEM_PINNED, C.byref(h)))
N.check(lib.cf_dev_alloc(ctx.handle, G, C.byref(d)))
for obj in (256, 1024, 4096, 16384):
    n = G // obj
    hs = np.arange(n, dtype=np.uint64) * np.uint64(obj) + np.uint64(h.value)
    ds = np.arange(n, dtype=np.uint64) * np.uint64(obj) + np.uint64(d.value)
    sz = np.full(n, obj, np.uint64)
    for name, dst, src in (("H2D", ds, hs), ("D2H", hs, ds)):
        ts = []
        for r in range(4):
            ctx.sync()
            t = time.perf_counter()
            N.check(lib.cf_copy_objects(ctx.handle, N.ptr(dst), N.ptr(src), N.ptr(sz), n))
            ctx.sync()
            ts.append(time.perf_counter() - t)
        print(f"objects of {obj:6d} B x {n:8d} {name}: {G / min(ts[1:]) / 1e9:6.1f} GB/s", flush=True)
for name, dst, src in (("H2D", d.value, h.value), ("D2H", h.value, d.value)):
    ts = []
    for r in range(4):
        ctx.sync()
        t = time.perf_counter()
        N.check(lib.cf_sm_copy(ctx.handle, dst, src, G, 0, None))
        ctx.sync()
        ts.append(time.perf_counter() - t)
    print(f"bulk SM copy {name}: {G / min(ts[1:]) / 1e9:6.1f} GB/s", flush=True)

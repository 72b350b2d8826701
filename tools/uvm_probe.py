"""Managed-memory migration throughput on this box: cudaMemPrefetchAsync of 1 GiB to the device
and back, whole vs chunked, one vs two streams (both directions at once).  python tools/uvm_probe.py"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1906_01128_b200 import _native as N  # noqa: E402

ctx = N.DeviceContext.get(0)
lib = N.lib()
G = 1 << 30
bufs = []
for _ in range(2):
    p = C.c_void_p()
    N.check(lib.cf_host_alloc(G, N.CF_MEM_MANAGED, C.byref(p)))
    N.host_view(p.value, G)[:] = 1   # first touch on the host
    bufs.append(p.value)
s1, s2 = lib.cf_ctx_stream(ctx.handle), None


def pf(addr, n, dev, chunk, stream=None):
    for o in range(0, n, chunk):
        N.check(lib.cf_uvm_prefetch(ctx.handle, addr + o, min(chunk, n - o), dev, stream))


for chunk in (G, 64 << 20, 16 << 20, 2 << 20):
    for r in range(2):
        ctx.sync()
        t = time.perf_counter(); pf(bufs[0], G, 0, chunk); ctx.sync(); h2d = time.perf_counter() - t
        t = time.perf_counter(); pf(bufs[0], G, -1, chunk); ctx.sync(); d2h = time.perf_counter() - t
    print(f"chunk {chunk >> 20} MiB: H2D {G / h2d / 1e9:.1f} GB/s, D2H {G / d2h / 1e9:.1f} GB/s", flush=True)
# both directions at once: buffer 1 resident on the device goes home while buffer 0 comes in
pf(bufs[1], G, 0, G)
ctx.sync()
stream = C.c_void_p()
for chunk in (64 << 20, 16 << 20):
    pf(bufs[0], G, -1, G)
    pf(bufs[1], G, 0, G)
    ctx.sync()
    t = time.perf_counter()
    for o in range(0, G, chunk):
        N.check(lib.cf_uvm_prefetch(ctx.handle, bufs[0] + o, chunk, 0, None))
        N.check(lib.cf_uvm_prefetch(ctx.handle, bufs[1] + o, chunk, -1, None))
    ctx.sync()
    dt = time.perf_counter() - t
    print(f"interleaved chunk {chunk >> 20} MiB, one stream: {2 * G / dt / 1e9:.1f} GB/s both directions", flush=True)

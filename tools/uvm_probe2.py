"""Managed-memory migration ceilings on this box (design experiment for the prefetch-pipelined UVM
window, CF_WIN_UVM): cudaMemPrefetchAsync of 1 GiB, whole or chunked, each direction alone and
both directions at once on two streams, with CUDA-event timing.  python tools/uvm_probe2.py"""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

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
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def pf(addr, n, dev, chunk, stream):
    for o in range(0, n, chunk):
        N.check(lib.cf_uvm_prefetch(ctx.handle, addr + o, min(chunk, n - o), dev, C.c_void_p(stream.cuda_stream)))


def timed(fn, streams):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for s in streams[1:]:
        s.wait_event(e0)
    fn()
    for s in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(s)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3


out = {}
for chunk in (G, 256 << 20, 32 << 20, 2 << 20):
    best = {}
    for _ in range(3):
        pf(bufs[0], G, -1, G, sa)
        t_in = timed(lambda: pf(bufs[0], G, 0, chunk, sa), [sa])
        t_out = timed(lambda: pf(bufs[0], G, -1, chunk, sa), [sa])
        best["h2d"] = max(best.get("h2d", 0), G / t_in / 1e9)
        best["d2h"] = max(best.get("d2h", 0), G / t_out / 1e9)
    out[f"chunk_{chunk >> 20}MiB"] = {k: round(v, 2) for k, v in best.items()}
    print(chunk >> 20, out[f"chunk_{chunk >> 20}MiB"], flush=True)
# both directions at once, two streams: buffer 1 (on the device) goes home while buffer 0 comes in
for chunk in (G, 32 << 20):
    best = 0
    for _ in range(3):
        pf(bufs[0], G, -1, G, sa)
        pf(bufs[1], G, 0, G, sa)
        dt = timed(lambda: (pf(bufs[0], G, 0, chunk, sa), pf(bufs[1], G, -1, chunk, sb)), [sa, sb])
        best = max(best, 2 * G / dt / 1e9)
    out[f"bidir_two_streams_chunk_{chunk >> 20}MiB"] = round(best, 2)
    print("bidir", chunk >> 20, round(best, 2), flush=True)
# device reads of host-resident managed pages (no prefetch): the on-demand fault path, for scale
print(json.dumps(out))

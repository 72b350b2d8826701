"""The pipelined pointerchain window (cf_selective) through its C ABI on mixed-size layouts.

The drop-in only ever hands cf_selective arrays of one size per tree; the public
cf_selective_plan accepts any mix.  Large (DMA-moved) and small (zero-copy / staged) arrays
interleaved in one host slab must each come back scaled exactly once, and every byte between
them must stay as it was (harness.py:228-238, 255-259, 312-325 pointerchain branches).
"""
import ctypes as C
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    from paper_1906_01128_b200 import _native as N
    if N.device_count() == 0:
        pytest.skip("no GPU visible: run `pytest -m gpu` on a B200 box (gpurun)")
    return N


def _layout(rng, n):
    sizes = [rng.choice([64, 1024, 4096, 40000, 70000, 300000]) for _ in range(n)]
    order = list(range(n))
    if rng.random() < 0.5:
        rng.shuffle(order)
    off = [0] * n
    x = 0
    for i in order:
        off[i] = x
        x += sizes[i] + rng.choice([0, 0, 16, 1200])
    return sizes, off, x


@pytest.mark.parametrize("trial", range(6))
def test_mixed_size_selective_window_scales_every_array_once(N, trial):
    rng = random.Random(100 + trial)
    ctx = N.DeviceContext.get(0, 1)
    lib = N.lib()
    n = rng.randint(40, 300)
    sizes, off, span = _layout(rng, n)
    host = C.c_void_p()
    N.check(lib.cf_host_alloc(span, N.CF_MEM_PINNED, C.byref(host)))
    dev = C.c_void_p()
    N.check(lib.cf_dev_alloc(ctx.handle, sum(sizes), C.byref(dev)))
    w = C.c_void_p()
    try:
        hv = N.host_view(host.value, span)
        src = np.random.default_rng(trial).integers(0, 1 << 20, span // 4, dtype=np.int64).astype(np.float32)
        hv[:span // 4 * 4] = src.view(np.uint8)
        before = hv.copy()
        h_src = np.array([host.value + o for o in off], np.uint64)
        d_buf = (np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64) + np.uint64(dev.value))
        cnt = np.array(sizes, np.uint64) // np.uint64(4)
        chunk = rng.choice([1 << 16, 1 << 18, 1 << 20])
        N.check(lib.cf_selective_plan(ctx.handle, n, N.ptr(h_src), N.ptr(d_buf), N.ptr(cnt), 4, chunk, C.byref(w)))
        N.check(lib.cf_selective_run(w, N.CF_WIN_H2D | N.CF_WIN_SCALE | N.CF_WIN_D2H, 2.0))
        want = before.copy()
        for i in range(n):
            a, b = off[i], off[i] + sizes[i]
            want[a:b] = (before[a:b].view(np.float32) * np.float32(2.0)).astype(np.float32).view(np.uint8)
        got = N.host_view(host.value, span)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, (trial, chunk, int(bad[0]) if bad.size else None)
    finally:
        if w.value:
            lib.cf_selective_free(w)
        lib.cf_dev_free(ctx.handle, dev)
        lib.cf_host_free_sized(host, span, N.CF_MEM_PINNED)

"""The planned, pipelined metered window (cf_window) as a Python object.

``DeepCopyWindow`` owns a pinned source arena built by the native marshaller, a pinned
copy-back buffer, a device image and one or more planned windows over them:

* ``run()``           the full window from host buffers: chunked multi-stream H2D, relocation,
                      pointerchain resolve, leaf kernel, detach and D2H, overlapped chunk by
                      chunk (what ``execute_case`` does for the marshalling scheme, pipelined);
* ``run_resident()``  the same device work on an image already resident in HBM (attach,
                      resolve, scale, detach) -- the kernel-side number.

This is the reference-facing C-ABI path the benchmark times (harness.py:369-373).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .scenarios import TARGET_POLICIES


class DeepCopyWindow:
    def __init__(self, spec, seed: int = 1, policy: str = "all_leaves", mode: str = "resolved",
                 align: int = 16, chunk_bytes: int = 32 << 20, device: int = 0,
                 separate_output: bool = True, scale: float = 2.0, nstreams: int = 1, numa_node: int | None = None):
        self.ctx = N.DeviceContext.get(device, nstreams)
        self.numa_node = numa_node   # pinned buffers allocated on this NUMA node (None: as the OS places them)
        self.spec = spec
        self.seed = seed
        self.plan = N.NativeTree(spec.native(align))
        self.total = int(self.plan.info.total_bytes)
        lib = N.lib()
        self._owned: list = []
        src = C.c_void_p()
        with N.numa_bound(numa_node):
            N.check(lib.cf_host_alloc(self.total, N.CF_MEM_PINNED, C.byref(src)), "pinned arena")
        self._owned.append(("host", src.value, self.total))
        self.src = src.value
        self.plan.build(self.src, self.src, seed)
        if separate_output:
            dst = C.c_void_p()
            with N.numa_bound(numa_node):
                N.check(lib.cf_host_alloc(self.total, N.CF_MEM_PINNED, C.byref(dst)), "pinned copy-back buffer")
            self._owned.append(("host", dst.value, self.total))
            self.dst = dst.value
        else:
            self.dst = self.src
        img = C.c_void_p()
        N.check(lib.cf_dev_alloc(self.ctx.handle, self.total, C.byref(img)), "device image")
        self._owned.append(("dev", img.value, self.total))
        self.image = img.value
        self.targets = self.plan.targets(TARGET_POLICIES[policy])
        self.mode = mode
        self.scale = scale
        self.chunk_bytes = chunk_bytes
        self._windows: dict = {}

    def twin(self) -> "DeepCopyWindow":
        """A second window over the same source arena and plan, with its own device image and
        copy-back buffer: alternating the two lets window r+1 copy in while window r copies out."""
        t = object.__new__(DeepCopyWindow)
        t.__dict__.update({k: v for k, v in self.__dict__.items() if k not in ("_owned", "_windows")})
        t._owned, t._windows = [], {}
        lib = N.lib()
        dst, img = C.c_void_p(), C.c_void_p()
        with N.numa_bound(self.numa_node):
            N.check(lib.cf_host_alloc(self.total, N.CF_MEM_PINNED, C.byref(dst)), "pinned copy-back buffer")
        t._owned.append(("host", dst.value, self.total))
        N.check(lib.cf_dev_alloc(self.ctx.handle, self.total, C.byref(img)), "device image")
        t._owned.append(("dev", img.value, self.total))
        t.dst, t.image = dst.value, img.value
        return t

    def run_pair_n(self, other: "DeepCopyWindow", nruns: int, flags: int = N.CF_WIN_FULL,
                   scales: tuple = (2.0, 0.5)):
        """Alternate this window and its twin for ``nruns`` windows (see cf_window_run_pair)."""
        a = self._window(flags, self.chunk_bytes, self.mode)
        b = other._window(flags, other.chunk_bytes, other.mode)
        st = N.CfWindowStats()
        N.check(N.lib().cf_window_run_pair(a, b, int(nruns), float(scales[0]), float(scales[1]), C.byref(st)),
                "cf_window_run_pair")
        return st

    def run_ring_n(self, others: list, nruns: int, flags: int = N.CF_WIN_FULL, scales: tuple = (2.0, 0.5)):
        """Rotate this window and ``others`` (twins) for ``nruns`` windows (see cf_window_run_ring)."""
        ws = [self._window(flags, self.chunk_bytes, self.mode)] + \
             [o._window(flags, o.chunk_bytes, o.mode) for o in others]
        arr = (N.P * len(ws))(*ws)
        st = N.CfWindowStats()
        N.check(N.lib().cf_window_run_ring(arr, len(ws), int(nruns), float(scales[0]), float(scales[1]), C.byref(st)),
                "cf_window_run_ring")
        return st

    # -- planning ---------------------------------------------------------------------------
    def _window(self, flags: int, chunk_bytes: int, mode: str):
        key = (flags, chunk_bytes, mode)
        w = self._windows.get(key)
        if w is None:
            d = N.CfWindowDesc(self.plan.handle, N.ptr(self.targets), len(self.targets), self.src, self.dst,
                               self.src, self.image, N.CF_MODE_CHASE if mode == "chase" else N.CF_MODE_RESOLVED,
                               flags, float(self.scale), chunk_bytes)
            h = C.c_void_p()
            N.check(N.lib().cf_window_plan(self.ctx.handle, C.byref(d), C.byref(h)), "cf_window_plan")
            w = self._windows[key] = h
        return w

    def _run(self, flags: int, chunk_bytes: int, mode: str | None, scale: float | None, sync: bool):
        w = self._window(flags, chunk_bytes, mode or self.mode)
        if scale is not None:
            N.check(N.lib().cf_window_set_scale(w, float(scale)))
        st = N.CfWindowStats()
        N.check(N.lib().cf_window_run(w, 1 if sync else 0, C.byref(st)), "cf_window_run")
        return st

    def run(self, scale: float | None = None, mode: str | None = None, sync: bool = True,
            chunk_bytes: int | None = None, flags: int = N.CF_WIN_FULL):
        """Full window from host buffers (H2D + tables + attach + resolve + scale + detach + D2H)."""
        return self._run(flags, self.chunk_bytes if chunk_bytes is None else chunk_bytes, mode, scale, sync)

    def run_n(self, nruns: int, flags: int = N.CF_WIN_FULL, chunk_bytes: int | None = None,
              mode: str | None = None, scales: tuple = (2.0, 0.5)):
        """Enqueue ``nruns`` windows back to back (scale alternating 2.0 / 0.5, exact in IEEE so
        the data stays bounded) and wait once; stats cover the whole sequence."""
        cb = self.chunk_bytes if chunk_bytes is None else chunk_bytes
        if not flags & (N.CF_WIN_H2D | N.CF_WIN_D2H):
            cb = 0
        w = self._window(flags, cb, mode or self.mode)
        st = N.CfWindowStats()
        N.check(N.lib().cf_window_run_n(w, int(nruns), float(scales[0]), float(scales[1]), C.byref(st)),
                "cf_window_run_n")
        return st

    def run_n_flushed(self, nruns: int, flush_buf: int, flush_bytes: int, flags: int = N.CF_WIN_FULL,
                      chunk_bytes: int | None = None, scales: tuple = (2.0, 0.5)):
        """``nruns`` windows, the L2 flushed before each; stats.ms_total = the windows' own time."""
        cb = self.chunk_bytes if chunk_bytes is None else chunk_bytes
        if not flags & (N.CF_WIN_H2D | N.CF_WIN_D2H):
            cb = 0
        w = self._window(flags, cb, self.mode)
        st = N.CfWindowStats()
        N.check(N.lib().cf_window_run_n_flushed(w, int(nruns), float(scales[0]), float(scales[1]), flush_buf,
                                                flush_bytes, C.byref(st)), "cf_window_run_n_flushed")
        return st

    def upload_raw(self) -> None:
        """Put the un-relocated arena bytes into the device image (prepares run_resident)."""
        N.check(N.lib().cf_memcpy(self.ctx.handle, self.image, self.src, self.total), "upload")

    def run_resident(self, scale: float | None = None, mode: str | None = None, sync: bool = True,
                     graph: bool = False):
        """attach -> resolve -> scale -> detach on the HBM-resident image (one chunk)."""
        return self._run(N.CF_WIN_RESIDENT | (N.CF_WIN_GRAPH if graph else 0), 0, mode, scale, sync)

    # -- inspection ----------------------------------------------------------------------
    def host_src(self) -> np.ndarray:
        return N.host_view(self.src, self.total)

    def host_dst(self) -> np.ndarray:
        return N.host_view(self.dst, self.total)

    def image_bytes(self) -> np.ndarray:
        out = np.empty(self.total, np.uint8)
        N.check(N.lib().cf_memcpy(self.ctx.handle, N.ptr(out), self.image, self.total))
        return out

    def table(self, which: int) -> np.ndarray:
        return self.plan.table(which)

    def close(self) -> None:
        lib = N._lib
        if lib is None:
            return
        for w in self._windows.values():
            lib.cf_window_free(w)
        self._windows.clear()
        for kind, p, n in self._owned:
            if kind == "dev":
                lib.cf_dev_free(self.ctx.handle, p)
            else:
                lib.cf_host_free_sized(p, n, N.CF_MEM_PINNED)
        self._owned.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""ctypes binding of libchainforge_b200.so (include/chainforge_b200.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``) into
``paper_1906_01128_b200/_lib/``.  Importing this module without the library raises
:class:`NativeUnavailable` -- there is no Python or CPU fallback for the device path.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import (AttachOutsideArena, NativeUnavailable, OutOfSimMemory, SimMemoryError,
                     WildAccess)

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libchainforge_b200.so"
ABI_VERSION = 2   # include/chainforge_b200.h CF_ABI_VERSION

# status codes
CF_OK, CF_E_INVALID, CF_E_OOM, CF_E_WILD, CF_E_OUTSIDE_ARENA, CF_E_CUDA, CF_E_NODEVICE, CF_E_STATE = (
    0, -1, -2, -3, -4, -5, -6, -7)
CF_LINEAR, CF_DENSE = 0, 1
CF_MEM_PAGEABLE, CF_MEM_PINNED, CF_MEM_MANAGED = 0, 1, 2
CF_TARGET_REF, CF_TARGET_ALL_LEAVES, CF_TARGET_ALL_ARRAYS = 0, 1, 2
CF_MODE_RESOLVED, CF_MODE_CHASE = 0, 1
CF_UVM_ADVISE_NONE, CF_UVM_PREFERRED_DEVICE, CF_UVM_ACCESSED_BY, CF_UVM_READ_MOSTLY = 0, 1, 2, 3
CF_UVM_UNSET = 0x100
CF_SEL_PER_OBJECT = 1
(CF_TAB_ALLOC_OFF, CF_TAB_ALLOC_SIZE, CF_TAB_NODE_OFF, CF_TAB_NODE_LEVEL, CF_TAB_NODE_SIZE,
 CF_TAB_ARR_LEVEL, CF_TAB_ARR_OWNER, CF_TAB_ARR_OFF, CF_TAB_ARR_COUNT, CF_TAB_SITE_OFF,
 CF_TAB_SITE_TARGET, CF_TAB_SITE_SORTED, CF_TAB_ARR_ORDINAL, CF_TAB_ARR_ROOT, CF_TAB_TREE_ROOT) = range(15)
CF_WIN_H2D, CF_WIN_TABLES, CF_WIN_ATTACH, CF_WIN_RESOLVE, CF_WIN_SCALE, CF_WIN_DETACH, CF_WIN_D2H, \
    CF_WIN_GRAPH = (1 << i for i in range(8))
CF_WIN_FULL = (CF_WIN_H2D | CF_WIN_TABLES | CF_WIN_ATTACH | CF_WIN_RESOLVE | CF_WIN_SCALE
               | CF_WIN_DETACH | CF_WIN_D2H)
CF_WIN_RESIDENT = CF_WIN_ATTACH | CF_WIN_RESOLVE | CF_WIN_SCALE | CF_WIN_DETACH
CF_WIN_UVM = 1 << 8
CF_WIN_TABLE_RESOLVE = 1 << 9
CF_WIN_DEBUG_KEEP_LEAF_ATTACHED = 1
NO_BAD = (1 << 64) - 1

_TAB_DTYPES = {CF_TAB_NODE_LEVEL: np.int32, CF_TAB_NODE_SIZE: np.uint32, CF_TAB_ARR_LEVEL: np.int32}

EXPORTED = (
    "cf_abi_version", "cf_last_error", "cf_device_count", "cf_ctx_create", "cf_ctx_destroy",
    "cf_ctx_sync", "cf_ctx_stream", "cf_ctx_launches", "cf_ctx_sm_count",
    "cf_timer_create", "cf_timer_start", "cf_timer_stop", "cf_timer_free", "cf_host_alloc",
    "cf_host_free", "cf_host_free_sized", "cf_dev_alloc", "cf_dev_free", "cf_memcpy",
    "cf_memcpy_async", "cf_memset", "cf_link_probe", "cf_tree_plan", "cf_tree_info_get", "cf_tree_table",
    "cf_tree_build", "cf_tree_targets", "cf_tree_chain_shape", "cf_tree_free", "cf_relocate",
    "cf_resolve", "cf_scale", "cf_marshal_transfer_and_attach", "cf_demarshal",
    "cf_kernel_scale", "cf_kernel_plan_create", "cf_kernel_plan_run", "cf_kernel_plan_resolve",
    "cf_kernel_plan_expect", "cf_kernel_plan_free", "cf_scale_resolved", "cf_memcpy_batch", "cf_naive_fixup", "cf_arena_check_sites",
    "cf_checksum_ranges", "cf_selective_plan", "cf_selective_plan_ex", "cf_selective_run", "cf_selective_free",
    "cf_copy_objects", "cf_naive_fixup_host", "cf_debug_info", "cf_device_numa_node", "cf_bind_numa_node",
    "cf_sm_copy", "cf_host_write_words", "cf_window_plan_check", "cf_selective_plan_check",
    "cf_window_plan", "cf_window_run", "cf_window_run_n", "cf_window_run_pair", "cf_window_run_ring", "cf_window_run_n_flushed",
    "cf_window_set_scale", "cf_window_debug", "cf_l2_evict", "cf_uvm_walk_pages",
    "cf_window_free",
    "cf_uvm_prefetch", "cf_uvm_advise",
)


class CfSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layout", C.c_int32), ("k_or_q", C.c_int64),
                ("n", C.c_int64), ("depth", C.c_int64), ("elem", C.c_int32),
                ("leaf_only", C.c_int32), ("align", C.c_int32), ("forest", C.c_int32),
                ("scatter_seed", C.c_uint64), ("shard_rank", C.c_int32), ("shard_world", C.c_int32)]


class CfTreeInfo(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("total_bytes", "nallocs", "nnodes", "narrays", "nsites", "ntrees",
                                         "root_off", "payload_bytes", "padding_bytes")]


class CfChainShape(C.Structure):
    _fields_ = [("kind", C.c_int32), ("depth", C.c_int32), ("q", C.c_uint32),
                ("reserved", C.c_uint32), ("root_off", C.c_uint64), ("image_bytes", C.c_uint64)]


class CfScaleWork(C.Structure):
    _fields_ = [("parts", C.c_void_p), ("tile_base", C.c_void_p), ("groups", C.c_void_p),
                ("big_begin", C.c_uint64), ("big_count", C.c_uint64), ("tb_begin", C.c_uint64),
                ("tile_begin", C.c_uint64), ("tile_end", C.c_uint64), ("group_begin", C.c_uint64),
                ("group_end", C.c_uint64)]


class CfWindowDesc(C.Structure):
    _fields_ = [("tree", C.c_void_p), ("h_targets", C.c_void_p), ("ntargets", C.c_uint64),
                ("host_src", C.c_void_p), ("host_dst", C.c_void_p), ("host_base", C.c_uint64),
                ("image", C.c_void_p), ("mode", C.c_int32), ("flags", C.c_uint32),
                ("scale", C.c_double), ("chunk_bytes", C.c_uint64)]


class CfPlanCheck(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("nsteps", "nsegments", "nsites", "ntargets", "nparts", "ngroups", "ntiles",
                                         "table_bytes", "zero_copy_node_segments")] + \
        [("violations", C.c_int32), ("leaf_owned", C.c_int32), ("plan_ms", C.c_double)]


class CfWindowStats(C.Structure):
    _fields_ = [("ms_total", C.c_float), ("ms_kernel", C.c_float), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("launches", C.c_uint64), ("bad", C.c_uint64),
                ("nchunks", C.c_uint64), ("nsteps", C.c_uint64)]


_lib = None
P = C.c_void_p
U64 = C.c_uint64
I32 = C.c_int32


def _declare(L):
    sig = {
        "cf_abi_version": (C.c_int, []),
        "cf_last_error": (C.c_char_p, []),
        "cf_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "cf_ctx_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(P)]),
        "cf_ctx_destroy": (C.c_int, [P]),
        "cf_ctx_sync": (C.c_int, [P]),
        "cf_timer_create": (C.c_int, [P, C.POINTER(P)]),
        "cf_timer_start": (C.c_int, [P]),
        "cf_timer_stop": (C.c_int, [P, C.POINTER(C.c_float)]),
        "cf_timer_free": (C.c_int, [P]),
        "cf_ctx_stream": (P, [P]),
        "cf_ctx_launches": (U64, [P]),
        "cf_ctx_sm_count": (C.c_int, [P]),
        "cf_host_alloc": (C.c_int, [U64, C.c_int, C.POINTER(P)]),
        "cf_host_free": (C.c_int, [P, C.c_int]),
        "cf_host_free_sized": (C.c_int, [P, U64, C.c_int]),
        "cf_dev_alloc": (C.c_int, [P, U64, C.POINTER(P)]),
        "cf_dev_free": (C.c_int, [P, P]),
        "cf_memcpy": (C.c_int, [P, P, P, U64]),
        "cf_memcpy_async": (C.c_int, [P, P, P, U64, P]),
        "cf_memset": (C.c_int, [P, P, C.c_int, U64]),
        "cf_link_probe": (C.c_int, [P, U64, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]),
        "cf_tree_plan": (C.c_int, [C.POINTER(CfSpec), C.POINTER(P)]),
        "cf_tree_info_get": (C.c_int, [P, C.POINTER(CfTreeInfo)]),
        "cf_tree_table": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(U64)]),
        "cf_tree_build": (C.c_int, [P, P, U64, U64, C.c_int]),
        "cf_tree_targets": (C.c_int, [P, C.c_int, P, U64, C.POINTER(U64)]),
        "cf_tree_chain_shape": (C.c_int, [P, C.POINTER(CfChainShape)]),
        "cf_tree_free": (C.c_int, [P]),
        "cf_relocate": (C.c_int, [P, P, U64, P, U64, U64, U64, P, P]),
        "cf_resolve": (C.c_int, [P, P, C.POINTER(CfChainShape), P, P, P, U64, P, P, P, P]),
        "cf_scale": (C.c_int, [P, C.c_int, C.c_int, P, C.POINTER(CfChainShape), P, P, P, P, P,
                               C.POINTER(CfScaleWork), C.c_double, P, P]),
        "cf_marshal_transfer_and_attach": (C.c_int, [P, P, U64, P, P, U64, U64, C.POINTER(U64)]),
        "cf_demarshal": (C.c_int, [P, P, U64, P, P, U64, U64, C.POINTER(U64)]),
        "cf_kernel_scale": (C.c_int, [P, C.c_int, C.c_int, P, C.POINTER(CfChainShape), P, P, P, P,
                                      U64, C.c_double, P, C.POINTER(U64)]),
        "cf_kernel_plan_create": (C.c_int, [P, C.c_int, P, P, P, P, U64, C.POINTER(P)]),
        "cf_kernel_plan_run": (C.c_int, [P, C.c_int, P, C.POINTER(CfChainShape), C.c_double, C.POINTER(U64)]),
        "cf_kernel_plan_resolve": (C.c_int, [P, P, C.POINTER(CfChainShape), P, P, C.POINTER(U64)]),
        "cf_kernel_plan_expect": (C.c_int, [P, P, P]),
        "cf_kernel_plan_free": (C.c_int, [P]),
        "cf_scale_resolved": (C.c_int, [P, C.c_int, P, P, U64, C.c_double]),
        "cf_memcpy_batch": (C.c_int, [P, P, P, P, U64, P]),
        "cf_naive_fixup": (C.c_int, [P, P, P, U64, P, P, P, U64, P, P]),
        "cf_arena_check_sites": (C.c_int, [P, U64, P, U64, U64, C.POINTER(U64)]),
        "cf_checksum_ranges": (C.c_int, [P, P, P, U64, P]),
        "cf_selective_plan": (C.c_int, [P, U64, P, P, P, C.c_int, U64, C.POINTER(P)]),
        "cf_selective_plan_ex": (C.c_int, [P, U64, P, P, P, P, C.c_uint32, C.c_int, U64, C.POINTER(P)]),
        "cf_selective_run": (C.c_int, [P, C.c_uint32, C.c_double]),
        "cf_selective_free": (C.c_int, [P]),
        "cf_copy_objects": (C.c_int, [P, P, P, P, U64]),
        "cf_debug_info": (C.c_int, [P, P, C.c_int]),
        "cf_device_numa_node": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
        "cf_bind_numa_node": (C.c_int, [C.c_int]),
        "cf_sm_copy": (C.c_int, [P, P, P, U64, C.c_uint, P]),
        "cf_host_write_words": (C.c_int, [P, P, U64]),
        "cf_window_plan_check": (C.c_int, [C.POINTER(CfWindowDesc), C.POINTER(CfPlanCheck)]),
        "cf_selective_plan_check": (C.c_int, [U64, P, P, P, C.c_int, U64, C.c_int, C.POINTER(U64)]),
        "cf_naive_fixup_host": (C.c_int, [P, P, P, U64, P, P, P, U64, C.POINTER(U64)]),
        "cf_window_plan": (C.c_int, [P, C.POINTER(CfWindowDesc), C.POINTER(P)]),
        "cf_window_run": (C.c_int, [P, C.c_int, C.POINTER(CfWindowStats)]),
        "cf_window_run_n": (C.c_int, [P, C.c_int, C.c_double, C.c_double, C.POINTER(CfWindowStats)]),
        "cf_window_run_pair": (C.c_int, [P, P, C.c_int, C.c_double, C.c_double, C.POINTER(CfWindowStats)]),
        "cf_window_run_ring": (C.c_int, [C.POINTER(P), C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.POINTER(CfWindowStats)]),
        "cf_window_set_scale": (C.c_int, [P, C.c_double]),
        "cf_window_debug": (C.c_int, [P, C.c_uint32]),
        "cf_l2_evict": (C.c_int, [P, P, U64]),
        "cf_uvm_walk_pages": (C.c_int, [P, U64, C.c_int, C.c_uint32, C.c_int32, P, P, P, P, U64, U64, P, U64,
                                        C.POINTER(U64)]),
        "cf_window_run_n_flushed": (C.c_int, [P, C.c_int, C.c_double, C.c_double, P, U64, C.POINTER(CfWindowStats)]),
        "cf_window_free": (C.c_int, [P]),
        "cf_uvm_prefetch": (C.c_int, [P, P, U64, C.c_int, P]),
        "cf_uvm_advise": (C.c_int, [P, P, U64, C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def lib():
    """Load the native library (raises NativeUnavailable if it was not built)."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("CF_B200_LIB", str(LIB_PATH)))
        if not path.exists():
            raise NativeUnavailable(
                f"{path} is missing: build it with `make` or `python -c 'import __graft_entry__ as g; "
                "g.build()'` (the deep-copy path has no CPU fallback)")
        L = C.CDLL(str(path))
        _declare(L)
        if L.cf_abi_version() != ABI_VERSION:   # a stale build with another struct layout
            raise NativeUnavailable(f"{path} has C ABI {L.cf_abi_version()}, this package needs {ABI_VERSION}: rebuild")
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().cf_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == CF_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == CF_E_OOM:
        raise OutOfSimMemory(msg)
    if rc == CF_E_WILD:
        raise WildAccess(msg)
    if rc == CF_E_OUTSIDE_ARENA:
        raise AttachOutsideArena(msg)
    if rc == CF_E_STATE:
        raise SimMemoryError(msg)
    if rc == CF_E_INVALID:
        raise ValueError(msg)
    if rc == CF_E_NODEVICE:
        raise NativeUnavailable(msg)
    raise RuntimeError(f"CUDA failure ({rc}): {msg}")


def gpu_numa_node(device: int) -> int:
    """NUMA node of the GPU's PCI device (-1: unknown / single node)."""
    node = C.c_int(-1)
    if lib().cf_device_numa_node(device, C.byref(node)) != CF_OK:
        return -1
    return node.value


@contextlib.contextmanager
def numa_bound(node: int | None):
    """Within the block, this thread runs on ``node``'s CPUs and prefers its memory, so pinned
    host memory allocated here is local to that GPU's host link.  Restores the CPU mask and the
    default policy afterwards (OpenMP pools created later are not confined to the node)."""
    if node is None or node < 0:
        yield
        return
    saved = os.sched_getaffinity(0)
    check(lib().cf_bind_numa_node(node), "cf_bind_numa_node")
    try:
        yield
    finally:
        lib().cf_bind_numa_node(-1)
        os.sched_setaffinity(0, saved)


def device_count() -> int:
    n = C.c_int(0)
    check(lib().cf_device_count(C.byref(n)))
    return n.value


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


class DeviceContext:
    """One cf_ctx (streams + scratch) per (process, device); shared by every Machine."""

    _cache: dict = {}

    def __init__(self, device: int = 0, nstreams: int = 1):
        h = P()
        check(lib().cf_ctx_create(device, nstreams, C.byref(h)), "cf_ctx_create")
        self.handle = h
        self.device = device
        self.sm_count = lib().cf_ctx_sm_count(h)

    @classmethod
    def get(cls, device: int = 0, nstreams: int = 1) -> "DeviceContext":
        ctx = cls._cache.get((device, nstreams))
        if ctx is None:
            ctx = cls._cache[(device, nstreams)] = cls(device, nstreams)
        return ctx

    def launches(self) -> int:
        return int(lib().cf_ctx_launches(self.handle))

    def sync(self) -> None:
        check(lib().cf_ctx_sync(self.handle), "cf_ctx_sync")

    def timer(self) -> "DeviceTimer":
        return DeviceTimer(self)


class DeviceTimer:
    """CUDA-event timer over a context's compute stream (cf_timer_*): ``start()`` ... ``stop()``
    returns the device milliseconds of the library work enqueued in between."""

    def __init__(self, ctx: DeviceContext):
        self.handle = C.c_void_p()
        check(lib().cf_timer_create(ctx.handle, C.byref(self.handle)), "cf_timer_create")

    def start(self) -> None:
        check(lib().cf_timer_start(self.handle), "cf_timer_start")

    def stop(self) -> float:
        ms = C.c_float(0.0)
        check(lib().cf_timer_stop(self.handle, C.byref(ms)), "cf_timer_stop")
        return float(ms.value)

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.cf_timer_free(self.handle)
            self.handle = None


class NativeTree:
    """A planned layout (cf_tree): tables are copied out into numpy arrays once."""

    def __init__(self, spec: CfSpec):
        h = P()
        check(lib().cf_tree_plan(C.byref(spec), C.byref(h)), "cf_tree_plan")
        self.handle = h
        self.spec = spec
        info = CfTreeInfo()
        check(lib().cf_tree_info_get(h, C.byref(info)))
        self.info = info
        self._tables: dict[int, np.ndarray] = {}

    def table(self, which: int) -> np.ndarray:
        arr = self._tables.get(which)
        if arr is None:
            p, n = P(), U64()
            check(lib().cf_tree_table(self.handle, which, C.byref(p), C.byref(n)))
            dt = _TAB_DTYPES.get(which, np.uint64)
            if n.value == 0:
                arr = np.zeros(0, dtype=dt)
            else:
                buf = (C.c_char * (n.value * np.dtype(dt).itemsize)).from_address(p.value)
                arr = np.frombuffer(buf, dtype=dt).copy()
            self._tables[which] = arr
        return arr

    def build(self, host_addr: int, ptr_base: int, seed: int, nthreads: int = 0) -> None:
        check(lib().cf_tree_build(self.handle, host_addr, ptr_base, seed % (1 << 31), nthreads),
              "cf_tree_build")

    def targets(self, policy: int) -> np.ndarray:
        n = U64()
        check(lib().cf_tree_targets(self.handle, policy, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=np.int64)
        check(lib().cf_tree_targets(self.handle, policy, ptr(out), len(out), C.byref(n)))
        return out[:n.value]

    def chain_shape(self) -> CfChainShape:
        sh = CfChainShape()
        check(lib().cf_tree_chain_shape(self.handle, C.byref(sh)))
        return sh

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.cf_tree_free(h)
            self.handle = None


def read_bytes(addr: int, n: int) -> bytes:
    return C.string_at(addr, n) if n else b""


def write_bytes(addr: int, data: bytes) -> None:
    if data:
        C.memmove(addr, data, len(data))


def link_probe(ctx, nbytes: int, iters: int = 1, reps: int = 5) -> dict:
    """Plain cudaMemcpyAsync H2D / D2H / bidirectional GB/s for `nbytes` (cf_link_probe)."""
    h, d, b = C.c_double(), C.c_double(), C.c_double()
    check(lib().cf_link_probe(ctx.handle, int(nbytes), int(iters), int(reps), C.byref(h), C.byref(d), C.byref(b)),
          "cf_link_probe")
    return {"h2d": h.value, "d2h": d.value, "bidir": b.value}


def host_view(addr: int, n: int) -> np.ndarray:
    """Writable numpy uint8 view over host (pinned/managed/pageable) memory."""
    buf = (C.c_char * n).from_address(addr)
    return np.frombuffer(buf, dtype=np.uint8)

"""ctypes front-end for the CPU oracle (oracle/cf_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs, always as the checker or the timed CPU baseline,
never as the product path.  Parity of this oracle is pinned by tests/test_oracle_golden.py
against tests/golden/reference_kats.json (generated from the reference by
oracle/gen_golden.py).  Function-level citations are in cf_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libcforacle.so"

LINEAR, DENSE = 0, 1
LAYOUTS = ("allinit_allused", "allinit_LLused", "LLinit_LLused")
TARGET_REF, TARGET_ALL_LEAVES, TARGET_ALL_ARRAYS = 0, 1, 2


class _Spec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layout", C.c_int32), ("k_or_q", C.c_int64),
                ("n", C.c_int64), ("depth", C.c_int64), ("elem", C.c_int32),
                ("leaf_only", C.c_int32), ("align", C.c_int32), ("pad_", C.c_int32)]


class _Counts(C.Structure):
    _fields_ = [("nallocs", C.c_uint64), ("nnodes", C.c_uint64), ("narrays", C.c_uint64),
                ("nsites", C.c_uint64), ("total", C.c_uint64)]


class _Tables(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in (
        "alloc_off", "alloc_size", "node_off", "node_level", "node_size", "arr_level",
        "arr_owner", "arr_off", "arr_count", "site_off", "site_target")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
        L = C.CDLL(str(LIB_PATH))
        L.orc_count.argtypes = [C.POINTER(_Spec), C.POINTER(_Counts)]
        L.orc_build.argtypes = [C.POINTER(_Spec), C.c_uint64, C.c_void_p, C.c_uint64,
                                C.POINTER(_Tables), C.POINTER(_Counts)]
        L.orc_targets.restype = C.c_int64
        L.orc_targets.argtypes = [C.POINTER(_Spec), C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                  C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.orc_relocate.restype = C.c_int64
        L.orc_relocate.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                   C.c_uint64, C.c_uint64, C.c_int]
        L.orc_resolve.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_Spec), C.c_uint64,
                                  C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        L.orc_scale.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int,
                                C.c_double, C.c_int]
        L.orc_window.restype = C.c_int64
        L.orc_window.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                 C.c_uint64, C.c_void_p, C.c_uint64, C.POINTER(_Spec), C.c_uint64,
                                 C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                 C.c_double, C.c_int]
        L.orc_resident.restype = C.c_int64
        L.orc_resident.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64,
                                   C.POINTER(_Spec), C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                   C.c_void_p, C.c_double, C.c_int]
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


@dataclass(frozen=True)
class OSpec:
    kind: int
    k_or_q: int
    n: int
    depth: int = 3
    layout: str = "allinit_allused"
    elem: int = 8
    leaf_only: bool = False
    align: int = 1

    def c(self) -> _Spec:
        return _Spec(self.kind, LAYOUTS.index(self.layout), self.k_or_q, self.n, self.depth,
                     self.elem, int(self.leaf_only), self.align, 0)


def spec_from_json(j: dict, elem: int = 8, align: int = 1, leaf_only: bool = False) -> OSpec:
    if j["kind"] == "linear":
        return OSpec(LINEAR, j["k"], j["n"], 0, j["layout"], elem, False, align)
    return OSpec(DENSE, j["q"], j["n"], j["depth"], "allinit_allused", elem, leaf_only, align)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


@dataclass
class OTree:
    spec: OSpec
    seed: int
    ptr_base: int
    buf: np.ndarray          # uint8 arena / slab image
    total: int
    allocs: np.ndarray       # (m, 2) offset, size in allocation order
    node_off: np.ndarray
    node_level: np.ndarray
    node_size: np.ndarray
    arr_level: np.ndarray
    arr_owner: np.ndarray
    arr_off: np.ndarray
    arr_count: np.ndarray
    site_off: np.ndarray     # DFS order
    site_target: np.ndarray

    @property
    def root_off(self) -> int:
        return int(self.allocs[0, 0])

    def node_ordinals(self) -> dict:
        """(offset -> ordinal among the nodes of its level, pre-order)."""
        seen: dict[int, int] = {}
        out = {}
        for off, lv in zip(self.node_off.tolist(), self.node_level.tolist()):
            out[off] = seen.get(lv, 0)
            seen[lv] = out[off] + 1
        return out


def counts(spec: OSpec) -> _Counts:
    c = _Counts()
    lib().orc_count(C.byref(spec.c()), C.byref(c))
    return c


def build(spec: OSpec, seed: int, ptr_base: int = 0x1000_0000) -> OTree:
    """Build the tree (reference builders, restated) into a fresh zeroed numpy buffer."""
    c = counts(spec)
    buf = np.zeros(max(int(c.total), 1), dtype=np.uint8)
    A = lambda n, dt=np.uint64: np.zeros(int(n), dtype=dt)  # noqa: E731
    alloc_off, alloc_size = A(c.nallocs), A(c.nallocs)
    node_off, node_level, node_size = A(c.nnodes), A(c.nnodes, np.int32), A(c.nnodes, np.uint32)
    arr_level, arr_owner, arr_off, arr_count = (A(c.narrays, np.int32), A(c.narrays),
                                                A(c.narrays), A(c.narrays))
    site_off, site_target = A(c.nsites), A(c.nsites)
    t = _Tables(*[_ptr(x) for x in (alloc_off, alloc_size, node_off, node_level, node_size,
                                     arr_level, arr_owner, arr_off, arr_count, site_off,
                                     site_target)])
    seed31 = seed % (1 << 31)
    lib().orc_build(C.byref(spec.c()), seed31, _ptr(buf), ptr_base, C.byref(t), None)
    return OTree(spec, seed, ptr_base, buf, int(c.total),
                 np.stack([alloc_off, alloc_size], axis=1) if c.nallocs else np.zeros((0, 2), np.uint64),
                 node_off, node_level, node_size, arr_level, arr_owner, arr_off, arr_count,
                 site_off, site_target)


def targets(tree: OTree, policy: int = TARGET_REF) -> np.ndarray:
    out = np.zeros(max(len(tree.arr_off), 1), dtype=np.int64)
    m = lib().orc_targets(C.byref(tree.spec.c()), policy, _ptr(tree.arr_level), _ptr(tree.arr_owner),
                          len(tree.arr_off), _ptr(tree.site_off), _ptr(tree.site_target),
                          len(tree.site_off), tree.root_off, _ptr(out))
    if m < 0:
        raise RuntimeError("oracle target walk failed")
    return out[:m]


def chain_keys(tree: OTree, idx: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(level, ordinal) of each targeted array's owner node: the chain the resolver walks."""
    ords = tree.node_ordinals()
    lv = np.array([int(tree.arr_level[i]) for i in idx], dtype=np.int32)
    od = np.array([ords[int(tree.arr_owner[i])] for i in idx], dtype=np.uint64)
    return lv, od


def normalised(buf: np.ndarray, site_off: np.ndarray, base: int) -> bytes:
    """Replace every pointer field by (value - base): address-free bytes (gen_golden.py)."""
    b = np.array(buf, dtype=np.uint8, copy=True)
    for off in site_off.tolist():
        v = int.from_bytes(b[off:off + 8].tobytes(), "little")
        b[off:off + 8] = np.frombuffer(((v - base) & (2 ** 64 - 1)).to_bytes(8, "little"), np.uint8)
    return b.tobytes()


def relocate(buf: np.ndarray, total: int, site_off: np.ndarray, from_base: int, to_base: int,
             nthreads: int = 1) -> int:
    so = np.ascontiguousarray(site_off, dtype=np.uint64)
    return int(lib().orc_relocate(_ptr(buf), total, _ptr(so), len(so), from_base, to_base, nthreads))


def resolve(image: np.ndarray, image_base: int, tree: OTree, idx: np.ndarray):
    lv, od = chain_keys(tree, idx)
    ea = np.zeros(max(len(idx), 1), dtype=np.uint64)
    cnt = np.zeros(max(len(idx), 1), dtype=np.uint32)
    lib().orc_resolve(_ptr(image), image_base, C.byref(tree.spec.c()), tree.root_off, _ptr(lv),
                      _ptr(od), len(idx), _ptr(ea), _ptr(cnt))
    return ea[:len(idx)], cnt[:len(idx)]


def scale(image: np.ndarray, ea_off: np.ndarray, count: np.ndarray, elem: int, s: float,
          nthreads: int = 1) -> None:
    ea = np.ascontiguousarray(ea_off, dtype=np.uint64)
    cn = np.ascontiguousarray(count, dtype=np.uint32)
    lib().orc_scale(_ptr(image), _ptr(ea), _ptr(cn), len(ea), elem, s, nthreads)


def expected_after_window(tree: OTree, idx: np.ndarray, s: float = 2.0) -> np.ndarray:
    """Host arena bytes after transfer -> scale(targets) -> copy-back (no pointer change)."""
    out = tree.buf.copy()
    scale(out, tree.arr_off[idx], tree.arr_count[idx].astype(np.uint32), tree.spec.elem, s)
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())


def window(tree: OTree, idx: np.ndarray, dev: np.ndarray, out: np.ndarray, host_base: int,
           dev_base: int, s: float, nthreads: int, keys=None) -> int:
    """CPU restatement of the metered window (harness.py:369-373) -- reference arm / baseline."""
    lv, od = keys if keys is not None else chain_keys(tree, idx)
    ea = np.zeros(max(len(idx), 1), dtype=np.uint64)
    cnt = np.zeros(max(len(idx), 1), dtype=np.uint32)
    return int(lib().orc_window(_ptr(tree.buf), _ptr(dev), _ptr(out), tree.total, host_base,
                                dev_base, _ptr(tree.site_off), len(tree.site_off),
                                C.byref(tree.spec.c()), tree.root_off, _ptr(lv), _ptr(od),
                                len(idx), _ptr(ea), _ptr(cnt), s, nthreads))


def resident(tree: OTree, idx: np.ndarray, dev: np.ndarray, host_base: int, dev_base: int, s: float,
             nthreads: int, keys=None) -> int:
    """attach -> resolve -> scale -> detach on ``dev`` (already holding the arena bytes): the
    device-side steps of the window without the copies (reference arm's resident step)."""
    lv, od = keys if keys is not None else chain_keys(tree, idx)
    ea = np.zeros(max(len(idx), 1), dtype=np.uint64)
    cnt = np.zeros(max(len(idx), 1), dtype=np.uint32)
    return int(lib().orc_resident(_ptr(dev), tree.total, host_base, dev_base, _ptr(tree.site_off),
                                  len(tree.site_off), C.byref(tree.spec.c()), tree.root_off, _ptr(lv), _ptr(od),
                                  len(idx), _ptr(ea), _ptr(cnt), s, nthreads))


def default_threads() -> int:
    """Host threads for the CPU legs: CF_ORACLE_THREADS, else every CPU this process may run on
    (its affinity mask, not the machine's count), as granted by OpenMP (measured team size)."""
    want = int(os.environ.get("CF_ORACLE_THREADS", "0"))
    if not want:
        try:
            want = len(os.sched_getaffinity(0))
        except (AttributeError, OSError):
            want = os.cpu_count() or 1
    return threads_used(want)


def threads_used(n: int) -> int:
    """The team size OpenMP grants for n threads (orc_threads_used)."""
    f = lib().orc_threads_used
    f.restype = C.c_int
    f.argtypes = [C.c_int]
    return int(f(int(n)))

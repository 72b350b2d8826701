"""End-to-end execution of one benchmark case per transfer scheme, on a B200.

Drop-in for the reference harness (harness.py:1-427).  The metered window
(``transfer_to_device -> kernel_scale -> copy_back``, harness.py:369-373) runs on the GPU:

* ``marshalling``  pinned arena -> chunked multi-stream H2D -> relocation kernel per chunk;
                   device pointerchain resolve + leaf kernel; detach kernel -> D2H.
* ``naive``        one batched per-object copy submission + interval-map fix-up kernel.
* ``pointerchain`` host-resolved selective copies of the targeted arrays (the reference's
                   semantics, harness.py:228-238) + resolved leaf kernel.
* ``uvm``          the tree lives in cudaMallocManaged memory; the kernels walk it in place.

The logical counters (bytes, ops, attaches, page faults) and the simulated cost-model columns
are computed exactly as the reference does, so rows stay comparable; measured wall time of
the window is added (``wall_us``).  Leaf-kernel modes: ``mode="resolved"`` (effective address
from the resolve kernel) or ``mode="chase"`` (chain re-walked per access).
"""
from __future__ import annotations

import ctypes as C
import os
import statistics
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import AttachOutsideArena, SchemeError, VerificationFailed, WildAccess
from .memory import D2H, DATA_OP_KINDS, H2D, NULL_ADDR, AddressMap, Arena, Machine, _poke_words
from .scenarios import (LEAF_NODE_SIZE, LEAF_OFF_A, NODE_SIZE, OFF_A, OFF_LNEXT, OFF_NA, ForestSpec,
                        LinearSpec, TreeHandle, build_tree, marshal_tree, payload_values)

SCHEMES = ("uvm", "marshalling", "pointerchain", "naive")
MODES = ("resolved", "chase")

# single-loop kernel instruction model of the reference (harness.py:38-43)
KERNEL_BASE_INSTRUCTIONS = 60
PLAIN_STEP_INSTRUCTIONS = 2
INDEXED_STEP_INSTRUCTIONS = 6
FINAL_ARRAY_LOAD_INSTRUCTIONS = 2


@dataclass(frozen=True)
class CostModel:
    """Constants turning counted events into the reference's simulated times.

    Kept so ``sim_*`` columns stay comparable with the reference; the B200 backend reports
    measured times beside them.
    """

    latency_us_per_op: float = 10.0
    bandwidth_gib_s: float = 12.0
    page_size: int = 4096
    elem_op_ns: float = 0.5
    deref_ns: float = 5.0
    l2_bytes: int = 6 << 20
    spill_penalty: float = 3.0

    def __post_init__(self):
        positive = ("latency_us_per_op", "bandwidth_gib_s", "page_size", "elem_op_ns", "deref_ns", "l2_bytes")
        bad = [k for k in positive if not getattr(self, k) > 0]
        if bad:
            raise ValueError(f"{bad[0]} must be positive")
        if self.spill_penalty < 1:
            raise ValueError("spill_penalty must be >= 1")

    @classmethod
    def from_file(cls, path) -> "CostModel":
        """Overrides from `key = value` lines; '#' starts a comment."""
        kw = {}
        for line in Path(path).read_text().splitlines():
            text = line.split("#", 1)[0].strip()
            if not text:
                continue
            key, _, val = (p.strip() for p in text.partition("="))
            fld = cls.__dataclass_fields__.get(key)
            if fld is None:
                raise ValueError(f"unknown cost-model key {key!r}")
            kw[key] = int(val) if fld.type in ("int", int) else float(val)
        return cls(**kw)


P100_COST_MODEL = CostModel(l2_bytes=4 << 20)


@dataclass(frozen=True)
class ChainShape:
    steps: tuple = ()
    count_final_array_load: bool = False


def chain_shape(spec, scheme: str) -> ChainShape:
    if isinstance(spec, ForestSpec):
        spec = spec.tree
    if scheme == "pointerchain":
        return ChainShape()
    if isinstance(spec, LinearSpec):
        return ChainShape(("plain",) * (spec.k - 1), False)
    return ChainShape(("indexed",) * spec.depth, True)


def estimate_instructions(shape: ChainShape) -> int:
    per = {"indexed": INDEXED_STEP_INSTRUCTIONS, "plain": PLAIN_STEP_INSTRUCTIONS}
    total = KERNEL_BASE_INSTRUCTIONS + sum(per.get(s, PLAIN_STEP_INSTRUCTIONS) for s in shape.steps)
    return total + (FINAL_ARRAY_LOAD_INSTRUCTIONS if shape.count_final_array_load else 0)


@dataclass
class RunMetrics:
    scenario: str
    scheme: str
    layout: str
    k_or_q: int
    n: int
    bytes_h2d: int = 0
    bytes_d2h: int = 0
    transfer_ops: int = 0
    attach_ops: int = 0
    page_faults: int = 0
    instr_estimate: int = 0
    sim_kernel_us: float = 0.0
    sim_wall_us: float = 0.0
    iterations: int = 1
    verified: bool = False
    # measured on the B200 (not in the reference)
    wall_us: float = 0.0
    mode: str = "resolved"
    gpu_launches: int = 0
    # device time of each call of the window (CUDA events on the context's compute stream); a
    # fused window enqueues at copy_back, so its whole pipeline shows in copy_back_us
    device_us: float = 0.0
    transfer_us: float = 0.0
    kernel_us: float = 0.0
    copy_back_us: float = 0.0

    def sort_key(self):
        return (self.scenario, self.scheme, self.layout, self.k_or_q, self.n)


@dataclass
class KernelStats:
    elements_touched: int = 0
    chain_derefs: int = 0


@dataclass
class RepeatResult:
    mean: float
    iterations: int
    converged: bool


def adaptive_repeat(run_closure, min_iters: int = 3, cv_threshold: float = 0.02,
                    max_iters: int = 100) -> RepeatResult:
    """Repeat until the coefficient of variation settles (harness.py:165-185 semantics)."""
    if min_iters < 3:
        raise ValueError("min_iters must be >= 3")
    samples = [float(run_closure()) for _ in range(min_iters)]
    while True:
        mean = statistics.fmean(samples)
        cv = 0.0 if mean == 0 else statistics.pstdev(samples) / abs(mean)
        if cv < cv_threshold:
            return RepeatResult(mean, len(samples), True)
        if len(samples) >= max_iters:
            return RepeatResult(mean, len(samples), False)
        samples.append(float(run_closure()))


def simulate_times(entries, elements_touched: int, chain_derefs: int, cost_model: CostModel,
                   working_set_bytes: int) -> tuple[float, float]:
    """Deterministic (kernel_us, wall_us) of the reference cost model (harness.py:188-205)."""
    cm = cost_model
    penalty = cm.spill_penalty if working_set_bytes > cm.l2_bytes else 1.0
    kernel_us = (elements_touched * cm.elem_op_ns * penalty + chain_derefs * cm.deref_ns) / 1000.0
    us_per_byte = 1e6 / (cm.bandwidth_gib_s * (1 << 30))
    if isinstance(entries, tuple):  # (dirs, kinds, bytes) columns of data-moving entries
        _, _, nbytes = entries
        wall = kernel_us
        for b in nbytes.tolist():   # same summation order as the reference
            wall += cm.latency_us_per_op + b * us_per_byte
        return kernel_us, wall
    wall = kernel_us
    for e in entries:
        if e.op_kind in DATA_OP_KINDS:
            wall += cm.latency_us_per_op + e.bytes * us_per_byte
    return kernel_us, wall


# -- scheme execution ---------------------------------------------------------

@dataclass
class DevicePrep:
    scheme: str
    device_root: int = 0
    arena: Arena | None = None
    amap: AddressMap | None = None
    policy: str = "ref"
    image: int = 0
    image_bytes: int = 0
    uvm_hints: str = "none"
    # pointerchain selective buffers, column-wise: device address, host address, count, index
    buf_dev: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    buf_host: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    buf_count: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    buf_array: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    handle: TreeHandle | None = None
    fused: "FusedMarshalWindow | None" = None

    @property
    def buffers(self) -> list:
        """(device_addr, ArrayRef) pairs as in the reference (harness.py:210-216)."""
        if self.handle is None:
            return []
        arrays = self.handle.arrays
        return [(int(d), arrays[int(i)]) for d, i in zip(self.buf_dev, self.buf_array)]


# UVM driver hints: migrate the tree ahead of the kernel ("prefetch"), map it for
# remote access ("advise": SetAccessedBy), prefer device residence ("preferred":
# SetPreferredLocation), or duplicate the read-only node pages on the device ("read_mostly":
# SetReadMostly on the pages holding node records only -- the arrays are written)
UVM_HINTS = ("none", "prefetch", "advise", "preferred", "read_mostly")

# pipeline granularity of the fused marshalling window (repo:profiles/r01_design_experiments.md)
FUSED_CHUNK = 32 << 20
# UVM window step (design experiment knob): migration throughput per
# cudaMemPrefetchAsync grows with its size (tools/uvm_probe2.py)
UVM_CHUNK = int(os.environ.get("CF_UVM_CHUNK_MB", "32")) << 20


class FusedMarshalWindow:
    """The marshalling scheme's ``transfer_to_device -> kernel_scale -> copy_back`` deferred
    and enqueued as ONE planned window (cf_window): chunked H2D, attach, device pointerchain
    resolve, leaf kernel, detach and D2H overlapped chunk by chunk over the full-duplex link,
    instead of three synchronous phases.

    The calls keep the reference's observable behaviour (harness.py:219-325, memory.py:307-345):
    each logs its logical entries when called, ``transfer_to_device`` raises
    ``AttachOutsideArena`` up front (host-side bounds check of every site, memory.py:319-321),
    and ``copy_back`` returns with the host arena restored and scaled.  Anything that observes or
    mutates machine state in between (a device/host read or write, another transfer, ...)
    calls ``Machine.flush``, which runs the window up to the stage reached so far: H2D + attach,
    or H2D + attach + resolve + scale.  The eager primitives then carry on from there.
    """

    def __init__(self, machine: Machine, handle: TreeHandle, arena: Arena, image: int, policy: str):
        self.machine, self.handle, self.arena, self.image, self.policy = machine, handle, arena, image, policy
        self.scale: float | None = None     # set by kernel_scale
        self.mode = "resolved"

    def _run(self, flags: int, targets: np.ndarray, scale: float) -> None:
        base = self.arena.buffer_host_addr
        mode = N.CF_MODE_CHASE if self.mode == "chase" else N.CF_MODE_RESOLVED
        lib = N.lib()
        t0 = time.perf_counter()
        # plans are cached per (arena, image, targets, mode, flags) on the machine: the tables
        # depend only on the tree and the target set; the scale is set per run
        key = (base, self.image, self.policy if len(targets) else None, mode, flags)
        w = self.machine._plans.get(key)
        if w is None:
            tg = np.ascontiguousarray(targets, np.int64)
            d = N.CfWindowDesc(self.handle.plan.handle, N.ptr(tg) if len(tg) else None, len(tg), base, base, base,
                               self.image, mode, flags, float(scale), FUSED_CHUNK)
            w = C.c_void_p()
            N.check(lib.cf_window_plan(self.machine.ctx.handle, C.byref(d), C.byref(w)), "fused window plan")
            self.machine._plans[key] = w
        t1 = time.perf_counter()
        N.check(lib.cf_window_set_scale(w, float(scale)))
        rc = lib.cf_window_run(w, 1, None)   # no per-kernel events: detach fuses into the leaf launch
        # host-side phase times of the last run (plan, enqueue + wait)
        self.timing = {"plan_ms": (t1 - t0) * 1e3, "run_ms": (time.perf_counter() - t1) * 1e3}
        # the window's fault word names its phase: attach / detach -> AttachOutsideArena
        # (memory.py:319-321, 337-343), chain walk / leaf span -> WildAccess (memory.py:139-152)
        N.check(rc, "fused marshalling window")

    def _targets(self) -> np.ndarray:
        cache = self.handle.__dict__.setdefault("_nonempty_targets", {})
        idx = cache.get(self.policy)
        if idx is None:
            idx = self.handle.target_indices(self.policy)
            idx = cache[self.policy] = idx[self.handle.arr_count[idx] > 0]
        return idx

    def flush(self) -> None:
        """Materialise the stage reached so far; later calls take the eager paths."""
        if self.scale is None:
            self._run(N.CF_WIN_H2D | N.CF_WIN_TABLES | N.CF_WIN_ATTACH, np.zeros(0, np.int64), 1.0)
        else:
            self._run(N.CF_WIN_H2D | N.CF_WIN_TABLES | N.CF_WIN_ATTACH | N.CF_WIN_RESOLVE | N.CF_WIN_SCALE,
                      self._targets(), self.scale)

    def complete(self) -> None:
        """copy_back of a window whose kernel was recorded: the whole pipelined window."""
        self._run(N.CF_WIN_FULL, self._targets(), self.scale)


class FusedSelectiveWindow:
    """The pointerchain scheme's ``transfer_to_device -> kernel_scale -> copy_back`` (selective
    copies of the targeted arrays, harness.py:228-238, 255-259, 312-325) deferred into one
    pipelined cf_selective window: per step of ~32 MiB the arrays' bytes go in, get scaled and go
    back while the next step copies in; big arrays on the copy engines, small ones by zero-copy
    SM kernels.  Same observable behaviour and flush rules as FusedMarshalWindow."""

    def __init__(self, machine: Machine, prep: DevicePrep, elem: int):
        self.machine, self.prep, self.elem = machine, prep, elem
        self.scale: float | None = None
        self.mode = "resolved"

    def _run(self, flags: int, scale: float) -> None:
        p = self.prep
        lib = N.lib()
        t0 = time.perf_counter()
        w = _selective_plan(self.machine, p, self.elem)
        t1 = time.perf_counter()
        rc = lib.cf_selective_run(w, flags, float(scale))
        self.timing = {"plan_ms": (t1 - t0) * 1e3, "run_ms": (time.perf_counter() - t1) * 1e3}
        if rc == N.CF_E_WILD:
            raise WildAccess(N.last_error())
        N.check(rc, "pointerchain window")

    def flush(self) -> None:
        if self.scale is None:
            self._run(N.CF_WIN_H2D, 1.0)
        else:
            self._run(N.CF_WIN_H2D | N.CF_WIN_SCALE, self.scale)

    def complete(self) -> None:
        self._run(N.CF_WIN_H2D | N.CF_WIN_SCALE | N.CF_WIN_D2H, self.scale)


def _selective_plan(machine: Machine, p: DevicePrep, elem: int):
    """The cf_selective plan of a pointerchain DevicePrep's buffers (cached on the machine)."""
    key = ("selective", int(p.buf_dev[0]), len(p.buf_dev))
    w = machine._plans.get(key)
    if w is None:
        host = np.ascontiguousarray(p.buf_host, np.uint64)
        dev = np.ascontiguousarray(p.buf_dev, np.uint64)
        cnt = np.ascontiguousarray(p.buf_count, np.uint64)
        w = C.c_void_p()
        N.check(N.lib().cf_selective_plan(machine.ctx.handle, len(dev), N.ptr(host), N.ptr(dev), N.ptr(cnt),
                                          elem, FUSED_CHUNK, C.byref(w)), "pointerchain window plan")
        machine._plans[key] = w
        machine._plan_free[key] = N.lib().cf_selective_free
    return w


class FusedUvmWindow:
    """The UVM scheme with prefetch hints (harness.py:239-240, 261-283, 321-325; memory.py:239-261)
    deferred into one pipelined cf_window over the managed tree (CF_WIN_UVM): per ~32 MiB step,
    cudaMemPrefetchAsync to the GPU on the H2D copy stream, chain resolve and leaf kernel for the
    pieces that have arrived, and back-migration of released steps on the D2H stream -- so page
    migration overlaps compute and runs both directions at once, instead of one whole-tree
    prefetch before the kernel and one migration back after it.  Logical page-fault accounting is
    unchanged (it follows the reference's single-residence model, not the driver)."""

    def __init__(self, machine: Machine, handle: TreeHandle, prep: DevicePrep):
        self.machine, self.handle, self.prep = machine, handle, prep
        self.scale: float | None = None
        self.mode = "resolved"

    def flush(self) -> None:
        """Materialise the stage reached with the eager calls: the whole-tree prefetch (+ kernel)."""
        m, h, p = self.machine, self.handle, self.prep
        N.check(N.lib().cf_uvm_prefetch(m.ctx.handle, h.base, h.total_bytes, m.ctx.device, None))
        if self.scale is not None:
            _run_kernel(m, h, p, self.scale, self.mode)

    def complete(self) -> None:
        m, h, p = self.machine, self.handle, self.prep
        mode = N.CF_MODE_CHASE if self.mode == "chase" else N.CF_MODE_RESOLVED
        flags = (N.CF_WIN_UVM | N.CF_WIN_H2D | N.CF_WIN_TABLES | N.CF_WIN_RESOLVE | N.CF_WIN_SCALE
                 | N.CF_WIN_D2H)
        key = ("uvm_window", h.base, p.policy, mode)
        w = m._plans.get(key)
        if w is None:
            idx, _, _, _, _, _ = _kernel_args(h, p.policy)
            tg = np.ascontiguousarray(idx, np.int64)
            d = N.CfWindowDesc(h.plan.handle, N.ptr(tg) if len(tg) else None, len(tg), h.base, h.base, h.base,
                               h.base, mode, flags, float(self.scale), UVM_CHUNK)
            w = C.c_void_p()
            N.check(N.lib().cf_window_plan(m.ctx.handle, C.byref(d), C.byref(w)), "UVM window plan")
            m._plans[key] = w
        N.check(N.lib().cf_window_set_scale(w, float(self.scale)))
        N.check(N.lib().cf_window_run(w, 1, None), "UVM window")


class FusedNaiveWindow:
    """The naive scheme's ``transfer_to_device -> kernel_scale -> copy_back`` (per-object deep
    copy, memory.py:349-374; device chain walk, harness.py:244-304) deferred into one window:
    the node objects go over first (one transfer per object) and get their pointer fields fixed,
    every target chain is walked on the device and must land on its array's device copy
    (``WildAccess`` otherwise), then the arrays -- still one transfer per object, big ones on the
    copy engines, small ones by zero-copy warps -- are copied in, scaled and copied back step by
    step in a cf_selective pipeline (CF_SEL_PER_OBJECT: no staged spans), and the node objects go
    back last, their host pointers restored.  Logs, errors and flush rules as the other fused
    windows; chase mode and observations in between take the eager path."""

    def __init__(self, machine: Machine, prep: DevicePrep, lay, dev_base: int):
        self.machine, self.prep, self.lay, self.dev_base = machine, prep, lay, dev_base
        self.scale: float | None = None
        self.mode = "resolved"

    def flush(self) -> None:
        """Materialise the stage reached: every object copied and fixed (+ the kernel)."""
        m, p = self.machine, self.prep
        m._naive_copy_in(self.lay, self.dev_base, p.amap)
        if self.scale is not None:
            _run_kernel(m, p.handle, p, self.scale, self.mode)

    def _fixup(self) -> None:
        """Every pointer field rewritten through the interval map on the device; the site and map
        tables (C4: 1M sites, 2M map entries, 64 MB) are uploaded once per tree and span."""
        m, p, lay = self.machine, self.prep, self.lay
        n = len(lay.fields)
        if n == 0:
            return
        if p.amap._origin is None:   # the map was extended since the transfer: from host tables
            m._device_fixup(p.amap, lay.fields, lay.targets)
            return
        lib, ctx = N.lib(), m.ctx.handle
        hb, sz, db = p.amap.arrays()
        nmap = len(hb)
        key = ("naive_fixup", self.dev_base)
        blk = m._plans.get(key)
        if blk is not None and m._plan_keep.get(key) is not lay:
            lib.cf_dev_free(ctx, m._plans.pop(key))
            blk = None
        if blk is None:
            blk = C.c_void_p()
            N.check(lib.cf_dev_alloc(ctx, 8 * (2 * n + 3 * nmap + 1), C.byref(blk)), "naive fixup tables")
            off = 0
            for arr in (lay.fields, lay.targets, hb, sz, db):
                a = np.ascontiguousarray(arr, np.uint64)
                N.check(lib.cf_memcpy(ctx, blk.value + off, N.ptr(a), a.nbytes))
                off += a.nbytes
            m._plans[key] = blk
            m._plan_free[key] = lambda w, c=ctx: lib.cf_dev_free(c, w)
            m._plan_keep[key] = lay
        b = blk.value
        bad = b + 8 * (2 * n + 3 * nmap)
        N.check(lib.cf_memset(ctx, bad, 0xFF, 8))
        N.check(lib.cf_naive_fixup(ctx, b, b + 8 * n, n, b + 16 * n, b + 16 * n + 8 * nmap, b + 16 * n + 16 * nmap,
                                   nmap, bad, None), "naive fixup")
        out = np.zeros(1, np.uint64)
        N.check(lib.cf_memcpy(ctx, N.ptr(out), bad, 8))
        if int(out[0]) != (1 << 64) - 1:
            raise WildAccess(f"fixup target 0x{int(lay.targets[int(out[0])]):x} was never copied to the device")

    def complete(self) -> None:
        m, p, lay = self.machine, self.prep, self.lay
        lib, ctx = N.lib(), m.ctx.handle
        handle = p.handle
        t0 = time.perf_counter()
        dev = lay.dev_at(self.dev_base)
        node_dev = np.ascontiguousarray(dev[lay.node_alloc])
        # 1. node objects in, pointer fields fixed on the device
        N.check(lib.cf_copy_objects(ctx, N.ptr(node_dev), N.ptr(lay.node_host), N.ptr(lay.node_sizes),
                                    len(node_dev)), "naive per-object copies")
        self._fixup()
        t1 = time.perf_counter()
        # 2. every target chain walked through the device objects: it must end on the device copy
        #    of its array with the planned count
        idx, _, _, _, cnt, _ = _kernel_args(handle, p.policy)
        if len(idx):
            kp, sh = _kernel_plan(m, handle, p)
            if m._plan_keep.get(("expect", kp.value)) is not lay:   # where each chain must end, once per plan
                expect = np.ascontiguousarray(lay.dev_off[lay.arr_alloc[idx]])   # held across the call
                N.check(lib.cf_kernel_plan_expect(kp, N.ptr(expect), N.ptr(cnt)), "naive chain targets")
                m._plan_keep[("expect", kp.value)] = lay
            bad = N.U64(0)
            rc = lib.cf_kernel_plan_resolve(kp, p.image, C.byref(sh), None, None, C.byref(bad))
            if rc == N.CF_E_WILD:
                raise WildAccess(N.last_error())
            N.check(rc, "naive chain walk")
        t2 = time.perf_counter()
        # 3. arrays: in -> scale (targets) -> back, pipelined; one transfer per object
        key = ("naive_sel", self.dev_base, p.policy)
        w = m._plans.get(key)
        if w is None:
            sel = lay.selective.get(p.policy)
            if sel is None:
                nz = np.nonzero(np.asarray(handle.arr_count, np.uint64) > 0)[0]
                mask = np.zeros(len(handle.arr_count), np.uint8)
                mask[idx] = 1
                sel = lay.selective[p.policy] = (nz, np.ascontiguousarray(lay.host[lay.arr_alloc[nz]]),
                                                 np.ascontiguousarray(np.asarray(handle.arr_count, np.uint64)[nz]),
                                                 np.ascontiguousarray(mask[nz]))
            nz, host, count, mask = sel
            dbuf = np.ascontiguousarray(dev[lay.arr_alloc[nz]])
            w = C.c_void_p()
            N.check(lib.cf_selective_plan_ex(ctx, len(nz), N.ptr(host), N.ptr(dbuf), N.ptr(count), N.ptr(mask),
                                             N.CF_SEL_PER_OBJECT, handle.spec.elem, FUSED_CHUNK, C.byref(w)),
                    "naive window plan")
            m._plans[key] = w
            m._plan_free[key] = lib.cf_selective_free
        t3 = time.perf_counter()
        rc = lib.cf_selective_run(w, N.CF_WIN_H2D | N.CF_WIN_SCALE | N.CF_WIN_D2H, float(self.scale))
        if rc == N.CF_E_WILD:
            raise WildAccess(N.last_error())
        N.check(rc, "naive window")
        t4 = time.perf_counter()
        # 4. node objects back, host pointers restored (memory.py:368-372)
        N.check(lib.cf_copy_objects(ctx, N.ptr(lay.node_host), N.ptr(node_dev), N.ptr(lay.node_sizes),
                                    len(node_dev)), "naive copy back")
        _poke_words(lay.fields, lay.targets)
        t5 = time.perf_counter()
        self.timing = {"run_ms": (t5 - t0) * 1e3, "nodes_in_fixup_ms": (t1 - t0) * 1e3, "chain_walk_ms": (t2 - t1) * 1e3,
                       "plan_ms": (t3 - t2) * 1e3, "arrays_ms": (t4 - t3) * 1e3, "nodes_out_ms": (t5 - t4) * 1e3}


def _pending(machine: Machine, prep: DevicePrep):
    f = prep.fused
    return f if f is not None and machine._deferred is f else None


def transfer_to_device(machine: Machine, handle: TreeHandle, scheme: str, arena: Arena | None = None,
                       policy: str = "ref", uvm_hints: str = "none", fused: bool = True) -> DevicePrep:
    """harness.py:219-241.  ``fused=True`` (marshalling): defer the copy so that kernel_scale and
    copy_back join it in one pipelined window (FusedMarshalWindow); ``False``: eager phases."""
    machine.flush()
    if scheme == "marshalling" and fused:
        if arena is None:
            raise ValueError("marshalling needs the arena returned by marshal_tree")
        base, total = arena.buffer_host_addr, arena.total_bytes
        # every pointer field must target the arena (memory.py:319-321): checked in address order
        # (page-sequential reads of the pinned arena); on a fault re-checked in the reference's
        # site order so the error names the first offending site as the attach loop would
        sites = arena.sorted_site_offsets
        bad = N.U64(0)
        rc = N.lib().cf_arena_check_sites(base, total, N.ptr(sites) if len(sites) else None, len(sites), base,
                                          C.byref(bad))
        if rc == N.CF_E_OUTSIDE_ARENA:
            machine.attach_failed(arena)   # logs what the reference logged before raising
        N.check(rc, "transfer_to_device")
        image = arena.take_image()   # fully overwritten by the copy
        machine.log.append(H2D, "bulk", total)
        machine.log.append_many(H2D, "attach", arena.site_words)
        arena.device_image_addr = image
        prep = DevicePrep(scheme, device_root=image + (handle.root_addr - base), arena=arena, policy=policy,
                          image=image, image_bytes=total)
        prep.fused = FusedMarshalWindow(machine, handle, arena, image, policy)
        machine._deferred = prep.fused
        return prep
    if scheme == "marshalling":
        if arena is None:
            raise ValueError("marshalling needs the arena returned by marshal_tree")
        image = machine.marshal_transfer_and_attach(arena)
        return DevicePrep(scheme, device_root=image + (handle.root_addr - arena.buffer_host_addr), arena=arena,
                          policy=policy, image=image, image_bytes=arena.total_bytes)
    if scheme == "naive":
        if not fused:
            root, amap = machine.naive_deep_copy(handle)
            base, span = machine._naive_span
            return DevicePrep(scheme, device_root=root, amap=amap, policy=policy, image=base, image_bytes=span)
        machine.flush()
        lay, base, amap = machine._naive_prepare(handle)   # logs the per-object copies + attaches
        prep = DevicePrep(scheme, device_root=amap.translate(handle.root_addr), amap=amap, policy=policy, image=base,
                          image_bytes=lay.span, handle=handle)
        prep.fused = FusedNaiveWindow(machine, prep, lay, base)
        machine._deferred = prep.fused
        return prep
    if scheme == "pointerchain":
        # host-side chain resolution, then one selective bulk copy per targeted array
        # (harness.py:228-238), submitted together as one batched copy into one device span
        # the selection and its span layout depend only on the (immutable) tree shape and the
        # policy: computed once per tree (C4: 1M targets, 16 ms of numpy per window otherwise)
        e = handle.spec.elem
        cache = handle.__dict__.setdefault("_selective_layout", {})
        lay = cache.get(policy)
        if lay is None:
            idx = handle.target_indices(policy)
            idx = idx[handle.arr_count[idx] > 0]
            sizes = handle.arr_count[idx] * np.uint64(e)
            aligned = (sizes + np.uint64(7)) & ~np.uint64(7)
            offs = np.concatenate([[0], np.cumsum(aligned)[:-1]]).astype(np.uint64) if len(idx) else aligned
            lay = (idx, sizes, sizes.astype(np.int64), offs, int(aligned.sum()),
                   np.ascontiguousarray(handle.arr_off[idx] + np.uint64(handle.base)),
                   np.ascontiguousarray(handle.arr_count[idx]), {})
            for a in lay[:7]:
                if isinstance(a, np.ndarray):
                    a.flags.writeable = False   # shared by every window of this tree
            cache[policy] = lay
        idx, sizes, sizes_i64, offs, span, buf_host, buf_count, by_base = lay
        prep = DevicePrep(scheme, policy=policy, handle=handle, buf_array=idx, buf_host=buf_host, buf_count=buf_count)
        if len(idx):
            spare = handle.__dict__.setdefault("_spare_spans", {})
            dev_base = spare.pop(policy, 0) or machine.device.allocate_span(span, offs, sizes, zero=False)
            prep.buf_dev = by_base.get(dev_base)
            if prep.buf_dev is None:
                if len(by_base) >= 4:
                    by_base.clear()
                prep.buf_dev = by_base[dev_base] = offs + np.uint64(dev_base)
                prep.buf_dev.flags.writeable = False
            if fused:
                # addresses come from the tree's own array table and the span just allocated for
                # exactly these sizes: in bounds by construction (the eager path re-checks them)
                machine.log.append_many(H2D, "bulk", sizes_i64)
                prep.fused = FusedSelectiveWindow(machine, prep, e)
                machine._deferred = prep.fused
            else:
                machine.transfer_ranges(machine.host, prep.buf_host, machine.device, prep.buf_dev, sizes, "bulk")
        return prep
    if scheme == "uvm":
        # the tree already lives in managed memory (harness.py:239-240: no copy); optional
        # driver hints: migrate the whole tree ahead of the kernel, or map it for remote access
        if uvm_hints not in UVM_HINTS:
            raise ValueError(f"unknown uvm hint {uvm_hints!r}")
        ctx = machine.ctx.handle
        prep = DevicePrep(scheme, device_root=handle.root_addr, policy=policy, image=handle.base,
                          image_bytes=handle.total_bytes, uvm_hints=uvm_hints)
        if uvm_hints == "prefetch" and fused:
            # deferred: kernel_scale and copy_back join one prefetch-pipelined window
            prep.fused = FusedUvmWindow(machine, handle, prep)
            machine._deferred = prep.fused
            return prep
        if uvm_hints == "prefetch":
            N.check(N.lib().cf_uvm_prefetch(ctx, handle.base, handle.total_bytes, machine.ctx.device, None))
        for lo, hi, advice in _uvm_advice(handle, uvm_hints):
            N.check(N.lib().cf_uvm_advise(ctx, handle.base + lo, hi - lo, advice))
        return prep
    raise SchemeError(f"unknown transfer scheme {scheme!r}")


def _reference_derefs(handle: TreeHandle, policy: str, idx: np.ndarray) -> int:
    """chain_derefs exactly as the reference walk counts them (harness.py:264-304)."""
    spec = handle.spec
    trees = 1
    if isinstance(spec, ForestSpec):
        spec, trees = spec.tree, spec.count
    if policy == "ref":
        if isinstance(spec, LinearSpec):
            return trees * ((spec.k if spec.all_levels_used else 1) + (spec.k - 1))
        return trees * (spec.depth + 1)
    return int((handle.arr_level[idx].astype(np.int64) + 1).sum())


def _level_nodes(handle: TreeHandle, level: int) -> np.ndarray:
    return handle.node_off[handle.node_level == level]


def _pages_of_spans(starts: np.ndarray, counts: np.ndarray, e: int, page: int) -> np.ndarray:
    """Distinct pages hit by the element touches aptr + e*i, i < n, of every span."""
    starts = np.asarray(starts, np.int64)
    counts = np.asarray(counts, np.int64)
    keep = counts > 0
    first = starts[keep] // page
    last = (starts[keep] + e * (counts[keep] - 1)) // page
    k = last - first + 1
    if k.size == 0:
        return np.zeros(0, np.int64)
    rep = np.repeat(first - np.concatenate([[0], np.cumsum(k)[:-1]]), k)
    return np.unique(rep + np.arange(int(k.sum()), dtype=np.int64))


def _uvm_advice(handle: TreeHandle, hint: str) -> list[tuple[int, int, int]]:
    """(lo, hi, advice) byte ranges of the tree a UVM hint advises (offsets from handle.base)."""
    if hint == "advise":
        return [(0, handle.total_bytes, N.CF_UVM_ACCESSED_BY)]
    if hint == "preferred":
        return [(0, handle.total_bytes, N.CF_UVM_PREFERRED_DEVICE)]
    if hint == "read_mostly":
        cache = handle.__dict__.setdefault("_node_pages", {})
        if "ranges" not in cache:   # node allocations rounded out to 4 KiB pages, merged
            off = np.sort(np.asarray(handle.node_off, np.uint64))
            end = off + np.asarray(handle.node_size, np.uint64)[np.argsort(np.asarray(handle.node_off, np.uint64))]
            lo = (off // np.uint64(4096)) * np.uint64(4096)
            hi = np.minimum((end + np.uint64(4095)) // np.uint64(4096) * np.uint64(4096), np.uint64(handle.total_bytes))
            if len(lo):   # merge overlapping / touching page ranges (sorted by start)
                reach = np.maximum.accumulate(hi)
                first = np.concatenate([[True], lo[1:] > reach[:-1]])
                starts = lo[first]
                ends = np.maximum.reduceat(hi, np.nonzero(first)[0])
            else:
                starts = ends = lo
            cache["ranges"] = [(int(a), int(b), N.CF_UVM_READ_MOSTLY) for a, b in zip(starts, ends)]
        return cache["ranges"]
    return []


def _uvm_device_pages(handle: TreeHandle, policy: str, idx: np.ndarray, page: int):
    """Pages the reference's UVM walk touches and dirties (harness.py:261-304, memory.py:378-394):
    the sorted distinct pages of the chain fields it reads, and the inclusive page ranges of the
    arrays it scales (read, then written).  Used for the logical page-fault counters; the data
    itself migrates under the CUDA driver.  The chains are walked through the arena's pointer
    values by the native library (cf_uvm_walk_pages); array pages stay ranges (a 1 GiB tree is
    262,144 pages)."""
    spec = handle.spec
    base, e = handle.base, spec.elem
    forest = isinstance(spec, ForestSpec)
    tree = spec.tree if forest else spec
    linear = isinstance(tree, LinearSpec)
    arr = None

    if policy == "ref" and not forest and not linear:
        # always take the last child: the last node of every level in pre-order
        path = [int(handle.node_off[handle.node_level == lv][-1]) for lv in range(spec.depth + 1)]
        fields = [np.array(path[:-1], np.int64) + OFF_LNEXT, np.array([path[-1] + LEAF_OFF_A], np.int64)]
        t_nodes = np.array([path[-1]], np.int64)
    elif policy == "ref" and not forest and linear:
        # the reference walk reads A on every used level and Lnext on every level but the last
        nodes = _level_nodes_all(handle)
        used = np.arange(spec.k) if spec.all_levels_used else np.array([spec.k - 1])
        fields = [nodes[:-1] + OFF_LNEXT, nodes[used] + OFF_A]
        t_nodes = nodes[used]
    else:
        sel = idx if policy != "ref" or forest else handle.target_indices("ref")
        # the tree-shape columns of the walk and the arrays' page ranges (immutable per tree and
        # target set) are gathered once; the pointer values are read from memory on every call,
        # by the native walk (cf_uvm_walk_pages: one chain per target, distinct pages by bitmap)
        wcache = handle.__dict__.setdefault("_uvm_walk_cache", {})
        key = (policy, len(sel), int(sel[0]) if len(sel) else -1, int(sel[-1]) if len(sel) else -1, page)
        cols = wcache.get(key)
        if cols is None or not np.array_equal(cols[0], sel):
            cnt = handle.arr_count[sel].astype(np.uint64)
            keep = cnt > 0
            starts = handle.arr_off[sel].astype(np.int64)[keep] + base
            dirty = (starts // page, (starts + e * (cnt[keep].astype(np.int64) - 1)) // page)
            cols = wcache[key] = (np.array(sel, copy=True),
                                  np.ascontiguousarray(handle.arr_level[sel], np.int32),
                                  np.ascontiguousarray(handle.arr_root[sel], np.uint64),
                                  np.ascontiguousarray(handle.arr_ordinal[sel], np.uint64),
                                  np.ascontiguousarray(cnt), dirty)
        _, lv, roots, ords, cnt, dirty = cols
        n = len(sel)
        kind, q, depth = (N.CF_LINEAR, 1, 0) if linear else (N.CF_DENSE, int(tree.q), int(tree.depth))
        lib = N.lib()
        need = C.c_uint64()
        args = (C.c_void_p(base), handle.total_bytes, kind, q, depth, N.ptr(roots), N.ptr(lv), N.ptr(ords),
                N.ptr(cnt), n, page)
        N.check(lib.cf_uvm_walk_pages(*args, None, 0, C.byref(need)), "uvm walk")
        pages = np.empty(max(int(need.value), 1), np.uint64)
        N.check(lib.cf_uvm_walk_pages(*args, N.ptr(pages), len(pages), C.byref(need)), "uvm walk")
        return pages[:int(need.value)].astype(np.int64), dirty
    if arr is None:
        # terminal nodes with an array (the fixed reference paths above): find it by owner
        t_nodes = np.asarray(t_nodes, np.int64)
        owner_sorted = np.argsort(handle.arr_owner, kind="stable")
        pos = np.searchsorted(handle.arr_owner[owner_sorted], t_nodes.astype(np.uint64))
        pos = np.minimum(pos, max(len(owner_sorted) - 1, 0))
        has = (len(owner_sorted) > 0) & (handle.arr_owner[owner_sorted][pos] == t_nodes.astype(np.uint64)) \
            if len(owner_sorted) else np.zeros(t_nodes.shape, bool)
        arr = owner_sorted[pos][has] if len(owner_sorted) else np.zeros(0, np.int64)
    t_nodes = np.asarray(t_nodes, np.int64)
    cnt = handle.arr_count[arr].astype(np.int64)
    # the walk also reads the count of every terminal node that owns a non-empty array
    fields.append(t_nodes[has][cnt > 0] + OFF_NA)
    keep = cnt > 0
    starts = handle.arr_off[arr].astype(np.int64)[keep] + base
    dirty = (starts // page, (starts + e * (cnt[keep] - 1)) // page)   # page ranges, inclusive
    f = np.concatenate([np.asarray(x, np.int64) for x in fields]) if fields else np.zeros(0, np.int64)
    return _distinct_pages((f + base) // page), dirty


def _distinct_pages(p: np.ndarray) -> np.ndarray:
    """Sorted distinct page numbers (np.unique) by a bitmap over their span when that span is
    small (a tree's pages), a sort otherwise."""
    if p.size == 0:
        return p
    lo, hi = int(p.min()), int(p.max())
    if hi - lo > 8 * p.size + (1 << 20):
        return np.unique(p)
    m = np.zeros(hi - lo + 1, bool)
    m[p - lo] = True
    return np.nonzero(m)[0].astype(np.int64) + lo


def _merged_ranges(handle: TreeHandle, idx: np.ndarray, gap: int) -> list:
    """Byte ranges of the given arrays, merged when closer than `gap` (few prefetch calls)."""
    idx = idx[handle.arr_count[idx] > 0]
    if len(idx) == 0:
        return []
    lo = handle.arr_off[idx].astype(np.int64)
    hi = lo + handle.arr_count[idx].astype(np.int64) * handle.spec.elem
    order = np.argsort(lo)
    lo, hi = lo[order], hi[order]
    out = [[int(lo[0]), int(hi[0])]]
    for a, b in zip(lo[1:].tolist(), hi[1:].tolist()):
        if a <= out[-1][1] + gap:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def _level_nodes_all(handle: TreeHandle) -> np.ndarray:
    """Node offsets of a single linear tree, level order."""
    order = np.argsort(handle.node_level, kind="stable")
    return handle.node_off[order].astype(np.int64)


def kernel_scale(machine: Machine, handle: TreeHandle, prep: DevicePrep, scale: float,
                 mode: str = "resolved") -> KernelStats:
    """Scale the targeted arrays where the scheme left them, on the GPU."""
    if mode not in MODES:
        raise ValueError(f"unknown kernel mode {mode!r}")
    stats = KernelStats()
    elem = handle.spec.elem
    fw = _pending(machine, prep)
    if fw is not None and fw.scale is None and prep.scheme == "uvm":
        # joins the deferred prefetch-pipelined window; the logical page accounting happens now
        fw.scale, fw.mode = float(scale), mode
        idx, stats.chain_derefs, _, _, cnt, _ = _kernel_args(handle, prep.policy)
        _uvm_account_kernel(machine, handle, prep, idx)
        stats.elements_touched = int(cnt.sum()) if len(idx) else 0
        return stats
    if fw is not None and fw.scale is None and prep.scheme == "marshalling":
        # joins the deferred window: the leaf kernel runs chunk by chunk as the arena lands
        fw.scale, fw.mode = float(scale), mode
        cache = handle.__dict__.setdefault("_kernel_stats", {})
        if prep.policy not in cache:
            idx = fw._targets()
            cache[prep.policy] = (_reference_derefs(handle, prep.policy, idx), int(handle.arr_count[idx].sum()))
        stats.chain_derefs, stats.elements_touched = cache[prep.policy]
        return stats
    if fw is not None and fw.scale is None and prep.scheme == "pointerchain":
        fw.scale = float(scale)   # joins the deferred pointerchain window
        stats.elements_touched = int(prep.buf_count.sum())
        return stats
    if fw is not None and fw.scale is None and prep.scheme == "naive" and mode == "resolved":
        fw.scale = float(scale)   # joins the deferred naive window
        idx, stats.chain_derefs, _, _, cnt, _ = _kernel_args(handle, prep.policy)
        stats.elements_touched = int(cnt.sum())
        return stats
    machine.flush()
    if prep.scheme == "pointerchain":
        if len(prep.buf_dev):
            # the leaf kernel over the copied buffers (host-resolved addresses): the buffers' work
            # list is planned once per tree (the pointerchain window's plan, leaf-kernel stage only)
            rc = N.lib().cf_selective_run(_selective_plan(machine, prep, elem), N.CF_WIN_SCALE, float(scale))
            if rc == N.CF_E_WILD:
                raise WildAccess(N.last_error())
            N.check(rc, "kernel_scale")
            stats.elements_touched = int(prep.buf_count.sum())
        return stats

    idx, stats.chain_derefs, _, _, cnt, _ = _kernel_args(handle, prep.policy)
    if prep.scheme == "uvm":
        _uvm_account_kernel(machine, handle, prep, idx)
    if len(idx) == 0:
        return stats
    _run_kernel(machine, handle, prep, scale, mode)
    stats.elements_touched = int(cnt.sum())
    return stats


def _uvm_account_kernel(machine: Machine, handle: TreeHandle, prep: DevicePrep, idx: np.ndarray) -> None:
    """The reference UVM walk's logical page touches (harness.py:261-304, memory.py:378-394)."""
    fields, (dlo, dhi) = _uvm_device_pages(handle, prep.policy, idx, machine.uvm.page_size)
    # every page read once (fields, then array pages -- a page met twice migrates once), then
    # the array pages written (dirty)
    machine.uvm_touch_pages(fields, "read", "device")
    if dlo.size:
        mask = machine.uvm_range_mask(dlo, dhi)   # the same pages for the read and the write
        machine.uvm_touch_mask(mask, "read", "device")
        machine.uvm_touch_mask(mask, "write", "device")


def _kernel_args(handle: TreeHandle, policy: str):
    """(targets, chain_derefs, level i32, ordinal u32, count u64, root offset u64) of a policy's
    non-empty targets: they depend only on the immutable tree shape, so computed once."""
    kcache = handle.__dict__.setdefault("_kernel_args", {})
    ka = kcache.get(policy)
    if ka is None:
        idx = handle.target_indices(policy)
        idx = idx[handle.arr_count[idx] > 0]
        ka = kcache[policy] = (idx, _reference_derefs(handle, policy, idx),
                               np.ascontiguousarray(handle.arr_level[idx], np.int32),
                               np.ascontiguousarray(handle.arr_ordinal[idx], np.uint32),
                               np.ascontiguousarray(handle.arr_count[idx], np.uint64),
                               np.ascontiguousarray(handle.arr_root[idx], np.uint64))
    return ka


def _kernel_plan(machine: Machine, handle: TreeHandle, prep: DevicePrep):
    """The cf_kernel_plan of prep's targets (tables uploaded once per tree, policy and roots) and
    the chain shape of prep's image."""
    idx, _, lv, od, cnt, root_off = _kernel_args(handle, prep.policy)
    sh = handle.chain_shape()
    sh.root_off = prep.device_root - prep.image
    sh.image_bytes = prep.image_bytes
    # per-target chain roots inside the image (several for a forest)
    if prep.amap is not None:   # naive: objects were re-placed on the device
        origin = prep.amap._origin
        lay = origin[0] if origin is not None and origin[1] == prep.image else None
        roots = lay.roots.get(prep.policy) if lay is not None else None
        if roots is None:
            roots = np.ascontiguousarray(prep.amap.translate_many(root_off + np.uint64(handle.base)) - np.uint64(prep.image))
            if lay is not None:   # relative to the span base: the same for every window of this tree
                lay.roots[prep.policy] = roots
    else:                       # marshalling image / managed tree: same offsets as the host layout
        roots = root_off
    key = ("kernel", id(handle), prep.policy)
    held = machine._plan_keep.get(key)
    if held is not None and (held[0] is not handle or held[1] is not roots):
        old = machine._plans.pop(key)
        machine._plan_keep.pop(("expect", old.value), None)
        N.lib().cf_kernel_plan_free(old)
        held = None
    if held is None:
        kp = C.c_void_p()
        N.check(N.lib().cf_kernel_plan_create(machine.ctx.handle, handle.spec.elem, N.ptr(roots), N.ptr(lv), N.ptr(od),
                                              N.ptr(cnt), len(idx), C.byref(kp)), "kernel_scale plan")
        machine._plans[key] = kp
        machine._plan_free[key] = N.lib().cf_kernel_plan_free
        machine._plan_keep[key] = (handle, roots)
    return machine._plans[key], sh


def _run_kernel(machine: Machine, handle: TreeHandle, prep: DevicePrep, scale: float, mode: str) -> None:
    """Eager kernel_scale on the device: resolve every target chain, then the leaf kernel."""
    kp, sh = _kernel_plan(machine, handle, prep)
    bad = N.U64(0)
    rc = N.lib().cf_kernel_plan_run(kp, N.CF_MODE_CHASE if mode == "chase" else N.CF_MODE_RESOLVED,
                                    prep.image, C.byref(sh), float(scale), C.byref(bad))
    N.check(rc, "kernel_scale")


def copy_back(machine: Machine, handle: TreeHandle, prep: DevicePrep) -> None:
    fw = _pending(machine, prep)
    if fw is not None and fw.scale is not None and prep.scheme == "uvm":
        machine._deferred = None
        fw.complete()   # every released step already migrated home inside the window
        machine.uvm_touch_mask(machine.uvm._dirty.copy(), "read", "host")
        return
    if fw is not None and fw.scale is not None and prep.scheme == "naive":
        machine._deferred = None
        fw.complete()
        lay = fw.lay
        if getattr(machine, "_naive_span", None) and machine._naive_span[0] == fw.dev_base:
            handle.__dict__["_spare_naive_span"] = fw.dev_base
        machine.log.append_many(D2H, "per_object", lay.sizes_i64)
        machine.log.append_many(D2H, "detach", lay.attach8)
        return
    if fw is not None and fw.scale is not None and prep.scheme == "pointerchain":
        machine._deferred = None
        fw.complete()
        lay = handle.__dict__.get("_selective_layout", {}).get(prep.policy)
        machine.log.append_many(D2H, "bulk", lay[2] if lay is not None and lay[6] is prep.buf_count
                                else (prep.buf_count * np.uint64(handle.spec.elem)).astype(np.int64))
        prep.handle.__dict__.setdefault("_spare_spans", {})[prep.policy] = int(prep.buf_dev[0])
        return
    if fw is not None and fw.scale is not None:
        machine._deferred = None
        fw.complete()
        arena = prep.arena
        machine.log.append(D2H, "bulk", arena.total_bytes)
        machine.log.append_many(D2H, "detach", arena.site_words)
        arena._spare_image = arena.device_image_addr
        arena.device_image_addr = NULL_ADDR
        return
    machine.flush()
    if prep.scheme == "marshalling":
        machine.demarshal(prep.arena)
    elif prep.scheme == "naive":
        machine.naive_copy_back(handle, prep.amap)
    elif prep.scheme == "pointerchain":
        lay = handle.__dict__.get("_selective_layout", {}).get(prep.policy)
        sizes = lay[1] if lay is not None and lay[6] is prep.buf_count else prep.buf_count * np.uint64(handle.spec.elem)
        machine.transfer_ranges(machine.device, prep.buf_dev, machine.host, prep.buf_host, sizes, "bulk")
        if len(prep.buf_dev):
            handle.__dict__.setdefault("_spare_spans", {})[prep.policy] = int(prep.buf_dev[0])
    elif prep.scheme == "uvm":
        # the host re-touches every page the kernel dirtied (harness.py:321-325): migrate the
        # targeted arrays back explicitly, then account the logical page migrations
        ctx = machine.ctx.handle
        for lo, hi in _merged_ranges(handle, handle.target_indices(prep.policy), machine.uvm.page_size):
            N.check(N.lib().cf_uvm_prefetch(ctx, handle.base + lo, hi - lo, -1, None))
        machine.ctx.sync()
        for lo, hi, advice in _uvm_advice(handle, prep.uvm_hints):   # the hint lasts one window
            N.check(N.lib().cf_uvm_advise(ctx, handle.base + lo, hi - lo, advice | N.CF_UVM_UNSET))
        machine.uvm_touch_mask(machine.uvm._dirty.copy(), "read", "host")


def verify_tree(machine: Machine, handle: TreeHandle, scale: float, policy: str = "ref") -> None:
    """Check every element and pointer field on the host after copy-back (harness.py:328-345)."""
    spec = handle.spec
    e = spec.elem
    dt = np.dtype("<f8") if e == 8 else np.dtype("<f4")
    view = N.host_view(handle.base, handle.total_bytes)
    targeted = np.zeros(len(handle.arr_off), bool)
    targeted[handle.target_indices(policy)] = True
    s = np.float64(scale) if e == 8 else np.float32(scale)
    for lv in np.unique(handle.arr_level).tolist() if len(handle.arr_level) else []:
        sel = np.nonzero(handle.arr_level == lv)[0]
        for flag in (False, True):
            group = sel[targeted[sel] == flag]
            if len(group) == 0:
                continue
            for n in np.unique(handle.arr_count[group]).tolist():
                if n == 0:
                    continue
                g = group[handle.arr_count[group] == n]
                expected = payload_values(handle.seed, lv, n, e)
                if flag:
                    expected = (expected * s).astype(dt)
                exp_bytes = np.frombuffer(expected.astype(dt).tobytes(), np.uint8)
                nb = n * e
                step = max(1, (64 << 20) // max(nb, 1))
                for c0 in range(0, len(g), step):
                    offs = handle.arr_off[g[c0:c0 + step]].astype(np.int64)
                    got = view[offs[:, None] + np.arange(nb, dtype=np.int64)[None, :]]
                    rows = np.nonzero((got != exp_bytes[None, :]).any(axis=1))[0]
                    if len(rows):
                        a = handle.base + int(offs[rows[0]])
                        raise VerificationFailed(f"array at 0x{a:x} (level {lv}) does not match")
    fields, targets = handle.site_off.astype(np.int64), handle.site_target + np.uint64(handle.base)
    if len(fields):
        got = view[fields[:, None] + np.arange(8, dtype=np.int64)[None, :]].copy().view("<u8").ravel()
        bad = np.nonzero(got != targets)[0]
        if len(bad):
            raise VerificationFailed(f"pointer field at 0x{handle.base + int(fields[bad[0]]):x} not restored")


# -- one full case -------------------------------------------------------------

def _describe(spec) -> tuple[str, str, int, int]:
    if isinstance(spec, ForestSpec):
        scen, layout, k_or_q, n = _describe(spec.tree)
        return f"forest{spec.count}-{scen}", layout, k_or_q, n
    if isinstance(spec, LinearSpec):
        return "linear", spec.layout, spec.k, spec.n
    return "dense", "dense", spec.q, spec.n


def execute_case(spec, scheme: str, cost_model: CostModel, seed: int = 0, scale: float = 2.0,
                 mode: str = "resolved", policy: str = "ref", align: int | None = None,
                 device: int = 0, uvm_hints: str = "none", fused: bool = True) -> tuple[RunMetrics, Machine]:
    """Run one case once on the GPU; returns the metrics and the machine (for its log).
    ``fused`` (marshalling): the metered window runs as one pipelined cf_window."""
    if scheme not in SCHEMES:
        raise SchemeError(f"unknown transfer scheme {scheme!r}")
    machine = Machine(page_size=cost_model.page_size, device=device)
    if scheme == "uvm":
        machine.enable_uvm(cost_model.page_size)
    arena = None
    if scheme == "marshalling":
        arena, handle = marshal_tree(machine, spec, seed=seed, align=align or 1)
    else:
        handle = build_tree(machine, spec, seed=seed, align=align)
    launches0 = machine.ctx.launches()
    mark = machine.log.mark()
    timer = machine.ctx.timer()
    phase_us = []
    t0 = time.perf_counter()
    timer.start()
    prep = transfer_to_device(machine, handle, scheme, arena, policy=policy, uvm_hints=uvm_hints, fused=fused)
    phase_us.append(timer.stop() * 1e3)
    timer.start()
    stats = kernel_scale(machine, handle, prep, scale, mode=mode)
    phase_us.append(timer.stop() * 1e3)
    timer.start()
    copy_back(machine, handle, prep)
    phase_us.append(timer.stop() * 1e3)
    machine.ctx.sync()
    wall_us = (time.perf_counter() - t0) * 1e6
    kernel_us, sim_wall = simulate_times(machine.log.data_entries_since(mark), stats.elements_touched,
                                         stats.chain_derefs, cost_model, handle.served_bytes)
    verify_tree(machine, handle, scale, policy)  # outside the metered window
    scenario, layout, k_or_q, n = _describe(spec)
    metrics = RunMetrics(
        scenario=scenario, scheme=scheme, layout=layout, k_or_q=k_or_q, n=n,
        bytes_h2d=machine.log.bytes_moved("H2D", mark), bytes_d2h=machine.log.bytes_moved("D2H", mark),
        transfer_ops=machine.log.data_ops(mark), attach_ops=machine.log.count("attach", mark),
        page_faults=machine.log.count("page_migration", mark),
        instr_estimate=estimate_instructions(chain_shape(spec, scheme)),
        sim_kernel_us=kernel_us, sim_wall_us=sim_wall, iterations=1, verified=True,
        wall_us=wall_us, mode=mode, gpu_launches=machine.ctx.launches() - launches0,
        device_us=sum(phase_us), transfer_us=phase_us[0], kernel_us=phase_us[1], copy_back_us=phase_us[2])
    return metrics, machine


def run_case(spec, scheme: str, cost_model: CostModel | None = None, seed: int = 0, scale: float = 2.0,
             min_iters: int = 3, cv_threshold: float = 0.02, max_iters: int = 50,
             mode: str = "resolved", policy: str = "ref") -> RunMetrics:
    """Execute one cell with adaptive repetition over the simulated wall time (as the reference)."""
    if scheme not in SCHEMES:
        raise SchemeError(f"unknown transfer scheme {scheme!r}")
    cm = cost_model or CostModel()
    runs: list[RunMetrics] = []

    def one_run():
        metrics, machine = execute_case(spec, scheme, cm, seed, scale, mode=mode, policy=policy)
        machine.close()
        runs.append(metrics)
        return metrics.sim_wall_us

    result = adaptive_repeat(one_run, min_iters, cv_threshold, max_iters)
    metrics = runs[-1]
    metrics.sim_wall_us = result.mean
    metrics.sim_kernel_us = statistics.fmean(r.sim_kernel_us for r in runs)
    metrics.wall_us = statistics.fmean(r.wall_us for r in runs)
    metrics.iterations = result.iterations
    return metrics


def sweep(cases, cost_model: CostModel | None = None, seed: int = 0, min_iters: int = 3) -> list[RunMetrics]:
    """Run (spec, scheme) pairs and merge results in deterministic order."""
    rows = [run_case(spec, scheme, cost_model, seed=seed, min_iters=min_iters) for spec, scheme in cases]
    rows.sort(key=RunMetrics.sort_key)
    return rows

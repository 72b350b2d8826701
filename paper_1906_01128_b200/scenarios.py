"""Benchmark tree scenarios built by the native host marshaller.

Drop-in for the reference's scenarios module (scenarios.py:1-284): the same specs, closed
forms, handles and builder names.  Construction is done by libchainforge_b200's planner and
multi-threaded builder (``cf_tree_plan`` / ``cf_tree_build``) straight into pinned host
memory; the packed plan is byte-identical to the reference arena (tests/golden).

B200 extensions, all keyword-only with reference-preserving defaults:
  * ``elem`` (8 = float64 as in the reference, 4 = float32 as in the BASELINE configs);
  * ``DenseSpec.leaf_only`` -- arrays only on the depth-D leaves (BASELINE C2/C5);
  * ``marshal_tree(..., align=16)`` -- the aligned production arena;
  * target policies "ref" (``targeted_arrays``), "all_leaves", "all_arrays".
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .memory import Arena, Machine

NODE_SIZE = 24
LEAF_NODE_SIZE = 12  # dense last level: packed {count, array pointer}
ELEM_SIZE = 8

OFF_NA = 0
OFF_NLNEXT = 4
OFF_A = 8
OFF_LNEXT = 16
LEAF_OFF_A = 4

LAYOUTS = ("allinit_allused", "allinit_LLused", "LLinit_LLused")
TARGET_POLICIES = {"ref": N.CF_TARGET_REF, "all_leaves": N.CF_TARGET_ALL_LEAVES,
                   "all_arrays": N.CF_TARGET_ALL_ARRAYS}


def _check_elem(elem: int) -> None:
    if elem not in (4, 8):
        raise ValueError("elem must be 4 (float32) or 8 (float64)")


@dataclass(frozen=True)
class LinearSpec:
    k: int
    n: int
    layout: str = "allinit_allused"
    elem: int = 8

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.n < 0:
            raise ValueError("n must be >= 0")
        if self.layout not in LAYOUTS:
            raise ValueError(f"unknown layout {self.layout!r}")
        _check_elem(self.elem)

    @property
    def all_levels_allocated(self) -> bool:
        return self.layout.startswith("allinit")

    @property
    def all_levels_used(self) -> bool:
        return self.layout.endswith("allused")

    def native(self, align: int) -> N.CfSpec:
        return N.CfSpec(N.CF_LINEAR, LAYOUTS.index(self.layout), self.k, self.n, 0, self.elem, 0, align, 1, 0)


@dataclass(frozen=True)
class DenseSpec:
    q: int
    n: int
    depth: int = 3
    elem: int = 8
    leaf_only: bool = False
    # subtree shard (not in the reference): this rank's part of the tree cut at the
    # shallowest level l with q^l >= shard_world (shard.subtree_shard)
    shard_rank: int = 0
    shard_world: int = 1

    def __post_init__(self):
        if self.q < 1:
            raise ValueError("q must be >= 1")
        if self.n < 0:
            raise ValueError("n must be >= 0")
        if self.depth < 0:
            raise ValueError("depth must be >= 0")
        _check_elem(self.elem)
        if self.shard_world < 1 or not 0 <= self.shard_rank < self.shard_world:
            raise ValueError("bad shard rank / world")
        if self.shard_world > 1 and self.q ** self.depth < self.shard_world:
            raise ValueError(f"q^depth = {self.q ** self.depth} subtrees cannot be split over {self.shard_world} shards")

    def native(self, align: int) -> N.CfSpec:
        return N.CfSpec(N.CF_DENSE, 0, self.q, self.n, self.depth, self.elem, int(self.leaf_only), align, 1, 0,
                        self.shard_rank, self.shard_world)


@dataclass(frozen=True)
class ForestSpec:
    """``count`` independent copies of one tree spec, optionally scattered over the slab.

    BASELINE C3 (64 x LinearSpec(4, 4Mi, LLinit_LLused), sparse allocations).  Not in the
    reference, which builds one tree per case; each tree is byte-for-byte a reference tree.
    """

    tree: object
    count: int
    scatter_seed: int = 0

    def __post_init__(self):
        if self.count < 1:
            raise ValueError("count must be >= 1")
        if not isinstance(self.tree, (LinearSpec, DenseSpec)):
            raise ValueError("tree must be a LinearSpec or DenseSpec")

    @property
    def elem(self) -> int:
        return self.tree.elem

    @property
    def n(self) -> int:
        return self.tree.n

    def native(self, align: int) -> N.CfSpec:
        s = self.tree.native(align)
        s.forest = self.count
        s.scatter_seed = self.scatter_seed
        return s


@dataclass
class ArrayRef:
    level: int
    owner_addr: int
    addr: int
    count: int


class TreeHandle:
    """Everything a transfer scheme needs to know about one built tree (scenarios.py:79-96).

    Tables are numpy columns from the native planner (offsets relative to ``base``); the
    reference's list-of-tuples views are materialised on demand.
    """

    def __init__(self, spec, base: int, plan: N.NativeTree, seed: int):
        self.spec = spec
        self.base = base
        self.plan = plan
        self.seed = seed
        info = plan.info
        self.total_bytes = int(info.total_bytes)
        self.served_bytes = int(info.total_bytes - info.padding_bytes)
        t = plan.table
        self.alloc_off, self.alloc_size = t(N.CF_TAB_ALLOC_OFF), t(N.CF_TAB_ALLOC_SIZE)
        self.node_off, self.node_level, self.node_size = (t(N.CF_TAB_NODE_OFF), t(N.CF_TAB_NODE_LEVEL),
                                                          t(N.CF_TAB_NODE_SIZE))
        self.arr_level, self.arr_owner, self.arr_off, self.arr_count, self.arr_ordinal = (
            t(N.CF_TAB_ARR_LEVEL), t(N.CF_TAB_ARR_OWNER), t(N.CF_TAB_ARR_OFF), t(N.CF_TAB_ARR_COUNT),
            t(N.CF_TAB_ARR_ORDINAL))
        self.arr_root, self.tree_root = t(N.CF_TAB_ARR_ROOT), t(N.CF_TAB_TREE_ROOT)
        self.ntrees = int(info.ntrees)
        self.site_off, self.site_target = t(N.CF_TAB_SITE_OFF), t(N.CF_TAB_SITE_TARGET)
        self.root_off = int(info.root_off)

    # reference-shaped views -------------------------------------------------------------
    @property
    def root_addr(self) -> int:
        return self.base + self.root_off

    @property
    def node_addrs(self) -> list[int]:
        return (self.node_off + np.uint64(self.base)).tolist()

    @property
    def node_levels(self) -> list[int]:
        return self.node_level.tolist()

    @property
    def node_sizes(self) -> list[int]:
        return self.node_size.tolist()

    @property
    def arrays(self) -> list[ArrayRef]:
        b = self.base
        return [ArrayRef(int(lv), b + int(o), b + int(a), int(c)) for lv, o, a, c in
                zip(self.arr_level, self.arr_owner, self.arr_off, self.arr_count)]

    @property
    def reference_field_sites(self) -> list[tuple[int, int, int]]:
        """(holder, offset, target) per non-null pointer field, DFS order."""
        b = self.base
        out = []
        for f, tg in zip(self.site_off.tolist(), self.site_target.tolist()):
            off = self._field_offset(f)
            out.append((b + f - off, off, b + tg))
        return out

    def _field_offset(self, field_off: int) -> int:
        if getattr(self, "_node_sorted", None) is None:
            self._node_sorted = np.sort(self.node_off)
        i = int(np.searchsorted(self._node_sorted, np.uint64(field_off), side="right")) - 1
        return field_off - int(self._node_sorted[i]) if i >= 0 else 0

    @property
    def allocations(self) -> list[tuple[int, int]]:
        return [(self.base + int(o), int(z)) for o, z in zip(self.alloc_off, self.alloc_size)]

    def allocation_array(self) -> np.ndarray:
        return np.stack([self.alloc_off + np.uint64(self.base), self.alloc_size], axis=1)

    def site_field_target_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        b = np.uint64(self.base)
        return self.site_off + b, self.site_target + b

    def arrays_at_level(self, level: int) -> list[ArrayRef]:
        return [a for a in self.arrays if a.level == level]

    def target_indices(self, policy: str = "ref") -> np.ndarray:
        """Array indices the kernel targets (cached per policy: the tree shape is immutable)."""
        cache = self.__dict__.setdefault("_targets", {})
        t = cache.get(policy)
        if t is None:
            t = cache[policy] = self.plan.targets(TARGET_POLICIES[policy])
            t.setflags(write=False)
        return t

    def chain_shape(self) -> N.CfChainShape:
        return self.plan.chain_shape()


# -- closed-form sizes (test oracles and report tables, never construction) --

def linear_data_size(k: int, n: int, layout: str = "allinit_allused", elem: int = ELEM_SIZE) -> int:
    """Eq. 1 / Eq. 2: 24k + e*n*k, or 24k + e*n when only the last level owns an array."""
    if layout not in LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    arrays = 1 if layout == "LLinit_LLused" else k
    return NODE_SIZE * k + elem * n * arrays


def dense_data_size(q: int, n: int, depth: int = 3, elem: int = ELEM_SIZE, leaf_only: bool = False) -> int:
    """Eq. 3 unrolled from the 12-byte leaf level upwards."""
    level_bytes = LEAF_NODE_SIZE + elem * n
    for _ in range(depth):
        own = 0 if leaf_only else elem * n
        level_bytes = NODE_SIZE + own + q * level_bytes
    return level_bytes


# -- structural walks ---------------------------------------------------------

def iter_linear_allocations(spec: LinearSpec):
    """Allocation sizes in construction order: each node, then its array."""
    for level in range(spec.k):
        yield ("node", level, NODE_SIZE)
        if spec.n > 0 and (spec.all_levels_allocated or level == spec.k - 1):
            yield ("array", level, spec.elem * spec.n)


def iter_dense_allocations(spec: DenseSpec):
    """Allocation sizes in construction order (pre-order, arrays before child blocks)."""
    stack = [0]
    yield ("node", 0, NODE_SIZE if spec.depth > 0 else LEAF_NODE_SIZE)
    while stack:
        level = stack.pop()
        if spec.n > 0 and (not spec.leaf_only or level == spec.depth):
            yield ("array", level, spec.elem * spec.n)
        if level < spec.depth:
            child = NODE_SIZE if level + 1 < spec.depth else LEAF_NODE_SIZE
            yield ("block", level + 1, spec.q * child)
            stack.extend([level + 1] * spec.q)


def tree_total_bytes(spec, align: int = 1) -> int:
    """Planned arena size (dry-run traversal by the native planner)."""
    return int(N.NativeTree(spec.native(align)).info.total_bytes)


def payload_values(seed: int, level: int, n: int, elem: int = ELEM_SIZE) -> np.ndarray:
    """Deterministic per-element init pattern: (seed*16777619 + level*1000003 + i) mod 2^31."""
    start = (seed * 16777619 + level * 1000003) % (1 << 31)
    raw = (np.arange(n, dtype=np.int64) + start) & ((1 << 31) - 1)
    return raw.astype(np.float64) if elem == 8 else raw.astype(np.float32)


# -- builders ----------------------------------------------------------------

def _build(machine: Machine, spec, arena: Arena | None, seed: int, align: int | None) -> TreeHandle:
    if arena is not None:
        plan = N.NativeTree(spec.native(arena.align))
        total = int(plan.info.total_bytes)
        if arena.served_offset != 0 or total > arena.total_bytes:
            raise ValueError("arena must be fresh and at least as large as the planned tree")
        base = arena.buffer_host_addr
    else:
        plan = N.NativeTree(spec.native(align or 8))
        total = int(plan.info.total_bytes)
        base = machine.host.allocate_span(total, plan.table(N.CF_TAB_ALLOC_OFF), plan.table(N.CF_TAB_ALLOC_SIZE))
    plan.build(base, base, seed)
    handle = TreeHandle(spec, base, plan, seed)
    if arena is not None:
        arena._req_arr = np.stack([handle.alloc_off, handle.alloc_size], axis=1)
        arena.served_offset = total
        arena.set_site_offsets(handle.site_off, plan.table(N.CF_TAB_SITE_SORTED))
    elif machine.uvm is not None:
        from .harness import _pages_of_spans
        starts = handle.alloc_off.astype(np.int64) + base
        machine.uvm.register_pages(_pages_of_spans(starts, handle.alloc_size.astype(np.int64), 1,
                                                   machine.uvm.page_size))
    return handle


def build_linear_tree(machine: Machine, spec: LinearSpec, arena: Arena | None = None, seed: int = 0,
                      align: int | None = None) -> TreeHandle:
    return _build(machine, spec, arena, seed, align)


def build_dense_tree(machine: Machine, spec: DenseSpec, arena: Arena | None = None, seed: int = 0,
                     align: int | None = None) -> TreeHandle:
    return _build(machine, spec, arena, seed, align)


def build_tree(machine: Machine, spec, arena: Arena | None = None, seed: int = 0,
               align: int | None = None) -> TreeHandle:
    return _build(machine, spec, arena, seed, align)


def marshal_tree(machine: Machine, spec, seed: int = 0, align: int = 1) -> tuple[Arena, TreeHandle]:
    """Plan the tree, then build it inside one pinned arena so it ships as a single bulk op."""
    total = int(N.NativeTree(spec.native(align)).info.total_bytes)
    arena = machine.create_arena(total, align)
    handle = _build(machine, spec, arena, seed, None)
    return arena, handle


def targeted_arrays(handle: TreeHandle, policy: str = "ref") -> list[ArrayRef]:
    """The arrays the scale kernel touches (scenarios.py:270-284 for policy "ref")."""
    arrays = handle.arrays
    return [arrays[int(i)] for i in handle.target_indices(policy)]

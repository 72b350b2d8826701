"""Host and device memory spaces backed by real pinned memory and HBM.

Drop-in for the reference's simulated machine (memory.py:1-419): same class and method names,
argument meaning and exceptions, but a ``Machine`` owns a B200 context, its host space is
pinned (``cudaHostAlloc``) or managed (UVM mode) memory, its device space is HBM, and every
transfer, attach and detach is executed by libchainforge_b200 (multi-stream copies and sm_100a
relocation kernels).  The transfer log keeps the reference's *logical* accounting
(memory.py:60-98): one marshalled arena is one ``bulk`` entry however many streams carried
it, and each relocated site is one ``attach`` entry.

Addresses are real virtual addresses.  Bounds are still enforced per allocation (WildAccess),
so a fix-up that escapes the arena fails loudly as in the reference.
"""
from __future__ import annotations

import bisect
import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import (AttachOutsideArena, OutOfSimMemory, SimMemoryError,  # noqa: F401
                     WildAccess)

HOST_BASE = 0x1000_0000        # reference constants (memory.py:27-35), kept for API parity
DEVICE_BASE = 0xD0_0000_0000
DEFAULT_CAPACITY = 8 << 30
ALIGNMENT = 8
NULL_ADDR = 0
DEFAULT_PAGE_SIZE = 4096

H2D = "H2D"
D2H = "D2H"
DATA_OP_KINDS = ("bulk", "per_object", "page_migration")

_DIRS = (H2D, D2H)
_KINDS = ("bulk", "per_object", "page_migration", "attach", "detach")
_DATA_KIND_IDS = (0, 1, 2)

# marshalled arenas are uploaded in chunks of this many bytes over the context's copy streams
MARSHAL_CHUNK = 32 << 20
# host/device spaces carve small allocations out of slabs of this size
SLAB_BYTES = 64 << 20


@dataclass
class TransferEntry:
    direction: str
    op_kind: str
    bytes: int
    order: int


class TransferLog:
    """Append-only logical transfer log (memory.py:68-98) stored column-wise.

    A marshalled C4 tree logs a million attach entries; they are kept as numpy columns and
    appended in bulk, and ``entries`` materialises ``TransferEntry`` objects only on demand.
    """

    def __init__(self):
        self._dir = np.zeros(0, np.uint8)
        self._kind = np.zeros(0, np.uint8)
        self._bytes = np.zeros(0, np.int64)
        self._pending: list = []  # small appends, folded lazily
        self._chunks: list = []   # bulk appends (dir, kind, bytes-array), folded lazily

    def _fold(self) -> None:
        if self._pending:
            d, k, b = zip(*self._pending)
            self._chunks.append((np.array(d, np.uint8), np.array(k, np.uint8), np.array(b, np.int64)))
            self._pending = []
        if self._chunks:
            cols = [(self._dir, self._kind, self._bytes)] + [
                (d if isinstance(d, np.ndarray) else np.full(b.size, d, np.uint8),
                 k if isinstance(k, np.ndarray) else np.full(b.size, k, np.uint8), b) for d, k, b in self._chunks]
            self._dir = np.concatenate([c[0] for c in cols])
            self._kind = np.concatenate([c[1] for c in cols])
            self._bytes = np.concatenate([c[2] for c in cols])
            self._chunks = []

    def append(self, direction: str, op_kind: str, nbytes: int) -> None:
        if nbytes <= 0:
            raise ValueError("log entries must move at least one byte")
        self._pending.append((_DIRS.index(direction), _KINDS.index(op_kind), int(nbytes)))

    def append_many(self, direction: str, op_kind: str, nbytes) -> None:
        """Append one entry per element of ``nbytes`` (an array); O(len) -- columns fold on read."""
        b = np.asarray(nbytes, dtype=np.int64).ravel()
        if b.size == 0:
            return
        if (b <= 0).any():
            raise ValueError("log entries must move at least one byte")
        if self._pending:   # keep order: earlier single appends go first
            d, k, bb = zip(*self._pending)
            self._chunks.append((np.array(d, np.uint8), np.array(k, np.uint8), np.array(bb, np.int64)))
            self._pending = []
        self._chunks.append((_DIRS.index(direction), _KINDS.index(op_kind), b))

    @property
    def entries(self) -> list[TransferEntry]:
        self._fold()
        return [TransferEntry(_DIRS[d], _KINDS[k], int(b), i)
                for i, (d, k, b) in enumerate(zip(self._dir.tolist(), self._kind.tolist(),
                                                  self._bytes.tolist()))]

    def mark(self) -> int:
        self._fold()
        return int(self._dir.size)

    def since(self, mark: int) -> list[TransferEntry]:
        return self.entries[mark:]

    def _cols(self, since: int):
        self._fold()
        return self._dir[since:], self._kind[since:], self._bytes[since:]

    def bytes_moved(self, direction: str, since: int = 0) -> int:
        d, k, b = self._cols(since)
        m = (d == _DIRS.index(direction)) & (k <= 2)
        return int(b[m].sum())

    def data_ops(self, since: int = 0) -> int:
        _, k, _ = self._cols(since)
        return int((k <= 2).sum())

    def count(self, op_kind: str, since: int = 0) -> int:
        _, k, _ = self._cols(since)
        return int((k == _KINDS.index(op_kind)).sum())

    def dump(self) -> str:
        """Stable newline-delimited `direction,op_kind,bytes,order` records."""
        return "\n".join(f"{e.direction},{e.op_kind},{e.bytes},{e.order}" for e in self.entries)

    def data_entries_since(self, mark: int):
        """(direction, op_kind, bytes) arrays of data-moving entries (for simulate_times)."""
        d, k, b = self._cols(mark)
        m = k <= 2
        return d[m], k[m], b[m]


class _Segment:
    """A contiguous storage block holding one or many allocations (sorted sub-offsets)."""

    __slots__ = ("base", "size", "offs", "sizes")

    def __init__(self, base: int, size: int, offs=None, sizes=None):
        self.base = base
        self.size = size
        self.offs = np.zeros(1, np.uint64) if offs is None else offs
        self.sizes = np.array([size], np.uint64) if sizes is None else sizes

    def locate(self, addr: int, nbytes: int):
        rel = addr - self.base
        if rel < 0 or rel + nbytes > self.size:
            return None
        i = int(np.searchsorted(self.offs, np.uint64(rel), side="right")) - 1
        if i < 0:
            return None
        if rel + nbytes <= int(self.offs[i]) + int(self.sizes[i]):
            return i
        return None


class MemorySpace:
    """One memory space with a bump allocator over real storage (memory.py:101-190).

    kind="host": pinned host memory (managed memory once the machine is in UVM mode; pageable
    memory when no GPU is visible, which only the host-side builder uses).
    kind="device": HBM of the machine's GPU.
    Storage is taken in slabs; allocations are 8-byte aligned and adjacent within a slab.
    """

    def __init__(self, kind: str, machine: "Machine" = None, capacity: int = DEFAULT_CAPACITY):
        if kind not in ("host", "device"):
            raise ValueError(f"unknown space kind {kind!r}")
        self.kind = kind
        self.machine = machine
        self.capacity = capacity
        self.bump_offset = 0
        self._segs: list[_Segment] = []
        self._seg_bases: list[int] = []
        self._storage: list[tuple[int, int, int]] = []  # (addr, bytes, memkind)
        self._slab: tuple[int, int] | None = None        # (addr, bytes)
        self._slab_used = 0
        self._last = None

    # -- storage -------------------------------------------------------------------------
    def _memkind(self) -> int:
        if self.kind == "device":
            return -1
        if self.machine is not None and self.machine.uvm is not None:
            return N.CF_MEM_MANAGED
        return N.CF_MEM_PINNED if self.machine is not None and self.machine.has_device else N.CF_MEM_PAGEABLE

    def _raw_alloc(self, nbytes: int, zero: bool = True) -> int:
        p = C.c_void_p()
        kind = self._memkind()
        if kind < 0:
            N.check(N.lib().cf_dev_alloc(self.machine.ctx.handle, nbytes, C.byref(p)), "device allocate")
            if zero:
                N.check(N.lib().cf_memset(self.machine.ctx.handle, p, 0, nbytes))
        else:
            N.check(N.lib().cf_host_alloc(nbytes, kind, C.byref(p)), "host allocate")
        self._storage.append((p.value, nbytes, kind))
        return p.value

    @property
    def base(self) -> int:
        return self._segs[0].base if self._segs else (HOST_BASE if self.kind == "host" else DEVICE_BASE)

    @property
    def end(self) -> int:
        return self.base + self.capacity

    def _reserve(self, aligned: int, size_bytes: int) -> None:
        if self.bump_offset + aligned > self.capacity:
            raise OutOfSimMemory(
                f"{self.kind} space exhausted: want {size_bytes} bytes, "
                f"{self.capacity - self.bump_offset} remain")
        self.bump_offset += aligned

    def _register(self, seg: _Segment) -> None:
        i = bisect.bisect_left(self._seg_bases, seg.base)
        self._seg_bases.insert(i, seg.base)
        self._segs.insert(i, seg)
        self._gen = getattr(self, "_gen", 0) + 1

    def allocate(self, size_bytes: int, zero: bool = True) -> int:
        """Bump allocation.  ``zero=False`` skips the zero fill for storage the caller overwrites
        completely (device images of an arena, selective-copy buffers)."""
        if size_bytes <= 0:
            raise ValueError("allocation size must be positive")
        aligned = (size_bytes + ALIGNMENT - 1) & ~(ALIGNMENT - 1)
        self._reserve(aligned, size_bytes)
        if aligned > SLAB_BYTES // 4:
            addr = self._raw_alloc(aligned, zero)
        else:
            if self._slab is None or self._slab_used + aligned > self._slab[1]:
                self._slab = (self._raw_alloc(SLAB_BYTES), SLAB_BYTES)
                self._slab_used = 0
            addr = self._slab[0] + self._slab_used
            self._slab_used += aligned
        self._register(_Segment(addr, size_bytes))
        return addr

    def allocate_span(self, total: int, offs: np.ndarray, sizes: np.ndarray, zero: bool = True) -> int:
        """One storage block holding a whole tree's allocations (offsets relative to the block).

        Used by the native builder so a million-object tree is one pinned block while each
        object stays a separately bounds-checked allocation.
        """
        if total <= 0:
            raise ValueError("allocation size must be positive")
        aligned = (total + 4095) & ~4095
        self._reserve((total + ALIGNMENT - 1) & ~(ALIGNMENT - 1), total)
        addr = self._raw_alloc(aligned, zero)
        order = np.argsort(offs, kind="stable")
        self._register(_Segment(addr, total, np.ascontiguousarray(offs[order], np.uint64),
                                np.ascontiguousarray(sizes[order], np.uint64)))
        return addr

    def free_all(self) -> None:
        lib = N._lib
        for addr, nbytes, kind in self._storage:
            if lib is None:
                break
            if kind < 0:
                lib.cf_dev_free(self.machine.ctx.handle, addr)
            else:
                lib.cf_host_free_sized(addr, nbytes, kind)
        self._storage.clear()
        self._segs.clear()
        self._seg_bases.clear()
        self._gen = getattr(self, "_gen", 0) + 1
        self._slab = None

    # -- bounds-checked access (memory.py:139-184) ---------------------------------------
    def _check(self, addr: int, nbytes: int) -> None:
        seg = self._last
        if seg is not None and seg.locate(addr, nbytes) is not None:
            return
        i = bisect.bisect_right(self._seg_bases, addr) - 1
        if i >= 0 and self._segs[i].locate(addr, nbytes) is not None:
            self._last = self._segs[i]
            return
        raise WildAccess(f"{self.kind} access at 0x{addr:x} (+{nbytes}) hits no live allocation")

    def _check_many(self, addrs: np.ndarray, sizes: np.ndarray) -> None:
        """Vectorised _check: every [addr, addr+size) inside one live allocation.  Read-only
        range tables (the drop-in's cached per-tree layouts) checked once per allocation state."""
        frozen = isinstance(addrs, np.ndarray) and isinstance(sizes, np.ndarray) and \
            not addrs.flags.writeable and not sizes.flags.writeable
        gen = getattr(self, "_gen", 0)
        if frozen:
            memo = self.__dict__.setdefault("_checked", {})
            hit = memo.get((id(addrs), id(sizes)))
            if hit is not None and hit[0] is addrs and hit[1] is sizes and hit[2] == gen:
                return
        self._check_many_uncached(addrs, sizes)
        if frozen:
            if len(memo) >= 16:
                memo.clear()
            memo[(id(addrs), id(sizes))] = (addrs, sizes, gen)

    def _check_many_uncached(self, addrs: np.ndarray, sizes: np.ndarray) -> None:
        addrs = np.asarray(addrs, np.uint64)
        sizes = np.asarray(sizes, np.uint64)
        if addrs.size <= 64:
            for a, n in zip(addrs.tolist(), sizes.tolist()):
                self._check(a, n)
            return
        bases = np.array(self._seg_bases, np.uint64)
        si = np.searchsorted(bases, addrs, side="right").astype(np.int64) - 1
        if (si < 0).any():
            raise WildAccess(f"{self.kind} access hits no live allocation")
        for k in np.unique(si).tolist():
            seg = self._segs[k]
            m = si == k
            rel = addrs[m] - np.uint64(seg.base)
            j = np.searchsorted(seg.offs, rel, side="right").astype(np.int64) - 1
            if (j < 0).any() or (rel + sizes[m] > seg.offs[np.maximum(j, 0)] + seg.sizes[np.maximum(j, 0)]).any():
                raise WildAccess(f"{self.kind} access hits no live allocation")

    def contains_range(self, addr: int, nbytes: int) -> bool:
        try:
            self._check(addr, nbytes)
            return True
        except WildAccess:
            return False

    def _sync_deferred(self) -> None:
        if self.machine is not None and self.machine._deferred is not None:
            self.machine.flush()

    def read_bytes(self, addr: int, nbytes: int) -> bytes:
        self._sync_deferred()
        self._check(addr, nbytes)
        if self.kind == "host":
            return N.read_bytes(addr, nbytes)
        out = np.empty(nbytes, np.uint8)
        N.check(N.lib().cf_memcpy(self.machine.ctx.handle, N.ptr(out), addr, nbytes), "read")
        return out.tobytes()

    def write_bytes(self, addr: int, data: bytes) -> None:
        self._sync_deferred()
        self._check(addr, len(data))
        if self.kind == "host":
            N.write_bytes(addr, data)
        else:
            src = np.frombuffer(bytes(data), np.uint8)
            N.check(N.lib().cf_memcpy(self.machine.ctx.handle, addr, N.ptr(src), len(data)), "write")

    def read_word(self, addr: int) -> int:
        return int.from_bytes(self.read_bytes(addr, 8), "little")

    def write_word(self, addr: int, value: int) -> None:
        self.write_bytes(addr, (value & 0xFFFF_FFFF_FFFF_FFFF).to_bytes(8, "little"))

    def read_u32(self, addr: int) -> int:
        return int.from_bytes(self.read_bytes(addr, 4), "little")

    def write_u32(self, addr: int, value: int) -> None:
        self.write_bytes(addr, (value & 0xFFFF_FFFF).to_bytes(4, "little"))

    def read_f64(self, addr: int) -> float:
        return float(np.frombuffer(self.read_bytes(addr, 8), "<f8")[0])

    def write_f64(self, addr: int, value: float) -> None:
        self.write_bytes(addr, np.array([value], "<f8").tobytes())

    def allocations(self) -> list[tuple[int, int]]:
        out = []
        for s in self._segs:
            out.extend((s.base + int(o), int(z)) for o, z in zip(s.offs, s.sizes))
        return out

    def snapshot(self, addr: int, nbytes: int) -> bytes:
        return self.read_bytes(addr, nbytes)


@dataclass
class AllocationRequest:
    host_addr: int
    size_bytes: int
    order: int


class Arena:
    """One contiguous pinned host buffer serving a whole tree (memory.py:200-230).

    ``align=1`` packs sub-allocations back to back exactly like the reference (the arena size
    equals the closed form); ``align=16`` is the production layout whose arrays are 16-byte
    aligned for 128-bit vector access.
    """

    def __init__(self, space: MemorySpace, total_bytes: int, align: int = 1):
        self.space = space
        self.total_bytes = total_bytes
        self.align = align
        self.buffer_host_addr = space.allocate(total_bytes)
        self.served_offset = 0
        self._req: list = []             # (offset, size) appended by allocate()
        self._req_arr = None             # numpy (m, 2) set by the native builder
        self._site_off = np.zeros(0, np.uint64)   # DFS order, relative to the arena
        self._sorted = None
        self.device_image_addr = NULL_ADDR
        # image of a completed (copied-back) window, reused by the next transfer of this arena
        # instead of a fresh 1 GiB-class allocation per window
        self._spare_image = NULL_ADDR

    def take_image(self) -> int:
        img, self._spare_image = self._spare_image, NULL_ADDR
        return img or self.space.machine.device.allocate(self.total_bytes, zero=False)

    def allocate(self, size_bytes: int) -> int:
        if size_bytes <= 0:
            raise ValueError("allocation size must be positive")
        off = self.served_offset
        if self.align > 1:
            off = (off + self.align - 1) // self.align * self.align
        if off + size_bytes > self.total_bytes:
            raise OutOfSimMemory(
                f"arena exhausted: want {size_bytes} bytes, "
                f"{self.total_bytes - self.served_offset} remain")
        self.served_offset = off + size_bytes
        self._req.append((off, size_bytes))
        return self.buffer_host_addr + off

    @property
    def request_list(self) -> list[AllocationRequest]:
        rows = self._req_arr.tolist() if self._req_arr is not None else self._req
        return [AllocationRequest(self.buffer_host_addr + int(o), int(z), i)
                for i, (o, z) in enumerate(rows)]

    @property
    def pointer_sites(self) -> list[int]:
        return (self._site_off + np.uint64(self.buffer_host_addr)).tolist()

    @pointer_sites.setter
    def pointer_sites(self, sites) -> None:
        arr = np.asarray(list(sites), dtype=np.uint64)
        self._site_off = arr - np.uint64(self.buffer_host_addr) if arr.size else arr
        self._sorted = self._detach_order = None

    def set_site_offsets(self, site_off: np.ndarray, sorted_off: np.ndarray | None = None) -> None:
        self._site_off = np.ascontiguousarray(site_off, np.uint64)
        self._sorted = None if sorted_off is None else np.ascontiguousarray(sorted_off, np.uint64)
        self._detach_order = None

    @property
    def site_offsets(self) -> np.ndarray:
        return self._site_off

    @property
    def site_words(self) -> np.ndarray:
        """One 8-byte log entry per pointer field (attach / detach), built once per arena."""
        w = getattr(self, "_site_words", None)
        if w is None or len(w) != len(self._site_off):
            w = self._site_words = np.full(len(self._site_off), 8, np.int64)
        return w

    @property
    def detach_order_offsets(self) -> np.ndarray:
        """Site offsets in the reference's detach order (reversed pointer_sites, memory.py:337)."""
        d = getattr(self, "_detach_order", None)
        if d is None:
            d = self._detach_order = np.ascontiguousarray(np.asarray(self._site_off, np.uint64)[::-1])
        return d

    @property
    def sorted_site_offsets(self) -> np.ndarray:
        if self._sorted is None:
            self._sorted = np.sort(self._site_off)
        return self._sorted

    def contains(self, addr: int) -> bool:
        return self.buffer_host_addr <= addr < self.buffer_host_addr + self.total_bytes


@dataclass
class PageState:
    resident: str  # "host" | "device"
    dirty: bool = False


class UvmState:
    """Logical page table of the unified-memory mode (memory.py:239-261).

    The real data lives in ``cudaMallocManaged`` memory and migrates under the CUDA driver;
    this table keeps the reference's single-residence accounting (page_faults, migrations) so
    RunMetrics stay comparable.  Stored as sorted numpy columns (a 1 GiB tree is 262,144
    pages); ``page_table`` materialises the reference's dict view on demand.
    """

    def __init__(self, page_size: int = DEFAULT_PAGE_SIZE):
        self.page_size = page_size
        self._pages = np.zeros(0, np.int64)
        self._device = np.zeros(0, bool)
        self._dirty = np.zeros(0, bool)

    def register_range(self, addr: int, size: int) -> None:
        first = addr // self.page_size
        last = (addr + size - 1) // self.page_size
        self.register_pages(np.arange(first, last + 1, dtype=np.int64))

    def register_pages(self, pages: np.ndarray) -> None:
        new = np.setdiff1d(np.asarray(pages, np.int64), self._pages, assume_unique=False)
        if new.size == 0:
            return
        allp = np.concatenate([self._pages, new])
        order = np.argsort(allp, kind="stable")
        self._pages = allp[order]
        self._device = np.concatenate([self._device, np.zeros(new.size, bool)])[order]
        self._dirty = np.concatenate([self._dirty, np.zeros(new.size, bool)])[order]

    def index(self, pages) -> np.ndarray:
        pages = np.asarray(pages, np.int64)
        i = np.searchsorted(self._pages, pages)
        ok = (i < self._pages.size) & (self._pages[np.minimum(i, max(self._pages.size - 1, 0))] == pages) \
            if self._pages.size else np.zeros(pages.shape, bool)
        return np.where(ok, i, -1)

    @property
    def page_table(self) -> dict:
        return {int(p): PageState("device" if d else "host", bool(y))
                for p, d, y in zip(self._pages, self._device, self._dirty)}

    def resident_pages(self, side: str) -> list[int]:
        m = self._device if side == "device" else ~self._device
        return self._pages[m].tolist()

    def dirty_pages(self) -> list[int]:
        return self._pages[self._dirty].tolist()


class Machine:
    """A pinned host space, an HBM device space, one logical transfer log, optional UVM mode.

    ``device`` selects the GPU; all device work goes through the shared per-process context.
    Without a visible GPU the machine can still plan and build trees in pageable host memory,
    but every transfer or kernel raises ``NativeUnavailable``.
    """

    def __init__(self, capacity: int = DEFAULT_CAPACITY, page_size: int = DEFAULT_PAGE_SIZE,
                 device: int = 0):
        self.has_device = N.device_count() > device
        self._device = device
        self._ctx = None
        self.host = MemorySpace("host", self, capacity)
        self.device = MemorySpace("device", self, capacity)
        self.log = TransferLog()
        self.uvm: UvmState | None = None
        self._default_page_size = page_size
        # a deferred metered window (harness.FusedMarshalWindow) not yet enqueued; anything that
        # observes or mutates device/host state runs it first (flush)
        self._deferred = None
        self._plans: dict = {}   # cached plans of the fused windows (cf_window / cf_selective)
        self._plan_free: dict = {}   # key -> free function when not cf_window_free
        self._plan_keep: dict = {}   # key -> objects a plan was built from (identity-checked on reuse)

    @property
    def ctx(self) -> N.DeviceContext:
        if self._ctx is None:
            if not self.has_device:
                raise N.NativeUnavailable("no CUDA device visible: device operations need a B200")
            self._ctx = N.DeviceContext.get(self._device)
        return self._ctx

    def space(self, kind: str) -> MemorySpace:
        return self.host if kind == "host" else self.device

    def alloc_host(self, size_bytes: int) -> int:
        addr = self.host.allocate(size_bytes)
        if self.uvm is not None:
            self.uvm.register_range(addr, size_bytes)
        return addr

    def enable_uvm(self, page_size: int = None) -> UvmState:
        self.uvm = UvmState(page_size or self._default_page_size)
        return self.uvm

    def create_arena(self, total_bytes: int, align: int = 1) -> Arena:
        return Arena(self.host, total_bytes, align)

    def flush(self) -> None:
        """Run deferred work (a fused marshalling window not yet enqueued) up to its current stage."""
        d, self._deferred = self._deferred, None
        if d is not None:
            d.flush()

    def close(self) -> None:
        self._deferred = None   # abandoned deferred work is dropped with the storage
        lib = N._lib
        if lib is not None and self._plans:
            self.ctx.sync()
            for key, w in self._plans.items():
                self._plan_free.get(key, lib.cf_window_free)(w)
        self._plans, self._plan_free, self._plan_keep = {}, {}, {}
        self.host.free_all()
        self.device.free_all()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- transfers (memory.py:294-303) ------------------------------------------------------
    def transfer_range(self, src: MemorySpace, src_addr: int, dst: MemorySpace, dst_addr: int,
                       nbytes: int, op_kind: str = "bulk") -> None:
        """Copy nbytes between spaces (snapshot semantics) and log one entry."""
        self.flush()
        if src.kind == dst.kind:
            raise ValueError("transfer_range requires distinct memory spaces")
        src._check(src_addr, nbytes)
        dst._check(dst_addr, nbytes)
        N.check(N.lib().cf_memcpy(self.ctx.handle, dst_addr, src_addr, nbytes), "transfer_range")
        self.log.append(H2D if dst.kind == "device" else D2H, op_kind, nbytes)

    def transfer_ranges(self, src: MemorySpace, src_addrs, dst: MemorySpace, dst_addrs, sizes,
                        op_kind: str = "bulk") -> None:
        """Several transfer_range calls submitted as one batched copy (one log entry each)."""
        self.flush()
        if src.kind == dst.kind:
            raise ValueError("transfer_range requires distinct memory spaces")
        sa = np.ascontiguousarray(src_addrs, np.uint64)
        da = np.ascontiguousarray(dst_addrs, np.uint64)
        sz = np.ascontiguousarray(sizes, np.uint64)
        if sa.size == 0:
            return
        src._check_many(sa, sz)
        dst._check_many(da, sz)
        ctx = self.ctx.handle
        N.check(N.lib().cf_copy_objects(ctx, N.ptr(da), N.ptr(sa), N.ptr(sz), sa.size), "transfer_ranges")
        self.log.append_many(H2D if dst.kind == "device" else D2H, op_kind, sz.astype(np.int64))

    # -- marshalling (memory.py:307-345) ----------------------------------------------------
    def marshal_transfer_and_attach(self, arena: Arena, chunk_bytes: int = MARSHAL_CHUNK) -> int:
        """Ship the arena in one logical bulk op (chunked over copy streams) and relocate every
        pointer field on the device as its chunk lands."""
        self.flush()
        image = arena.take_image()   # fully overwritten by the copy
        sites = arena.sorted_site_offsets
        bad = N.U64(0)
        rc = N.lib().cf_marshal_transfer_and_attach(
            self.ctx.handle, arena.buffer_host_addr, arena.total_bytes, image, N.ptr(sites),
            len(sites), chunk_bytes, C.byref(bad))
        if rc == N.CF_E_OUTSIDE_ARENA:
            self.attach_failed(arena)
        N.check(rc, "marshal_transfer_and_attach")
        self.log.append(H2D, "bulk", arena.total_bytes)
        self.log.append_many(H2D, "attach", arena.site_words)
        arena.device_image_addr = image
        return image

    def attach_failed(self, arena: Arena) -> None:
        """The attach loop met a pointer field outside the arena (memory.py:316-321): log what the
        reference logged before raising -- the bulk copy, then one attach per site preceding the
        first bad one in its site order -- and raise AttachOutsideArena naming that site."""
        base, total = arena.buffer_host_addr, arena.total_bytes
        dfs = np.ascontiguousarray(arena.site_offsets, np.uint64)
        bad = N.U64(0)
        rc = N.lib().cf_arena_check_sites(base, total, N.ptr(dfs), len(dfs), base, C.byref(bad))
        self.log.append(H2D, "bulk", total)
        if rc != N.CF_E_OUTSIDE_ARENA:
            raise AttachOutsideArena("relocation kernel reported a pointer field outside the arena")
        j = int(bad.value)
        if j:
            self.log.append_many(H2D, "attach", np.full(j, 8, np.int64))
        site = base + int(dfs[j])
        target = int.from_bytes(N.host_view(site, 8).tobytes(), "little")
        raise AttachOutsideArena(f"pointer field at 0x{site:x} targets 0x{target:x} outside the arena")

    def demarshal(self, arena: Arena, chunk_bytes: int = MARSHAL_CHUNK) -> None:
        """Detach on the device (inverse relocation kernel), then bulk copy the image back.
        The detach table is the reference's detach order (reversed site order, memory.py:337), so
        a fault reports -- and the log keeps -- exactly the detaches that preceded it there."""
        self.flush()
        image = arena.device_image_addr
        if image == NULL_ADDR:
            raise SimMemoryError("demarshal before marshal_transfer_and_attach")
        sites = arena.detach_order_offsets
        bad = N.U64(0)
        rc = N.lib().cf_demarshal(self.ctx.handle, arena.buffer_host_addr, arena.total_bytes, image,
                                  N.ptr(sites), len(sites), chunk_bytes, C.byref(bad))
        if rc == N.CF_E_OUTSIDE_ARENA:
            self.log.append(D2H, "bulk", arena.total_bytes)
            if bad.value:
                self.log.append_many(D2H, "detach", np.full(int(bad.value), 8, np.int64))
            raise AttachOutsideArena(N.last_error())
        N.check(rc, "demarshal")
        self.log.append(D2H, "bulk", arena.total_bytes)
        self.log.append_many(D2H, "detach", arena.site_words)
        arena._spare_image = image
        arena.device_image_addr = NULL_ADDR

    # -- naive per-object deep copy (memory.py:349-374) -------------------------------------
    def naive_deep_copy(self, tree) -> tuple[int, "AddressMap"]:
        """Copy every object individually (one batched submission), then fix every pointer
        field on the device through the sorted interval map."""
        self.flush()
        lay, dev_base, amap = self._naive_prepare(tree)
        self._naive_copy_in(lay, dev_base, amap)
        return amap.translate(tree.root_addr), amap

    def _naive_prepare(self, tree):
        """naive_deep_copy without its device work: the per-object device span (reused from this
        tree's previous copied-back window), the address map and the logical log entries."""
        lay = naive_layout(tree)
        # the span of this tree's previous (copied-back) naive window is reused: a fresh
        # 1 GiB-class allocation per window costs more than the copies
        dev_base = tree.__dict__.pop("_spare_naive_span", 0) or \
            self.device.allocate_span(lay.span, lay.dev_off, lay.sizes, zero=False)
        amap = AddressMap.from_sorted(lay.hb, lay.sz, lay.map_dev_at(dev_base))
        amap._origin = (lay, dev_base)
        self.log.append_many(H2D, "per_object", lay.sizes_i64)
        self.log.append_many(H2D, "attach", lay.attach8)
        self._naive_span = (dev_base, lay.span)
        return lay, dev_base, amap

    def _naive_copy_in(self, lay: "NaiveLayout", dev_base: int, amap: "AddressMap") -> None:
        """The device work of naive_deep_copy: every object copied, every pointer field fixed."""
        dev = lay.dev_at(dev_base)
        N.check(N.lib().cf_copy_objects(self.ctx.handle, N.ptr(dev), N.ptr(lay.host), N.ptr(lay.sizes), len(lay.host)),
                "naive per-object copies")
        self._device_fixup(amap, lay.fields, lay.targets)

    def _device_fixup(self, amap: "AddressMap", fields: np.ndarray, targets: np.ndarray) -> None:
        hb, sz, db = (np.ascontiguousarray(x, np.uint64) for x in amap.arrays())
        fields = np.ascontiguousarray(fields, np.uint64)
        targets = np.ascontiguousarray(targets, np.uint64)
        if len(fields) == 0:
            return
        bad = N.U64(0)
        rc = N.lib().cf_naive_fixup_host(self.ctx.handle, N.ptr(fields), N.ptr(targets), len(fields), N.ptr(hb),
                                         N.ptr(sz), N.ptr(db), len(hb), C.byref(bad))
        if rc == N.CF_E_WILD:
            raise WildAccess(f"fixup target 0x{int(targets[bad.value]):x} was never copied to the device")
        N.check(rc, "naive fixup")

    def naive_copy_back(self, tree, amap: "AddressMap") -> None:
        """Per-object copy back (one batched submission) plus host-side pointer restore."""
        self.flush()
        lay = naive_layout(tree)
        origin = getattr(amap, "_origin", None)
        # the map this tree's naive_deep_copy built: every object's device address is known
        dev = lay.dev_at(origin[1]) if origin is not None and origin[0] is lay else amap.translate_many(lay.host)
        N.check(N.lib().cf_copy_objects(self.ctx.handle, N.ptr(lay.host), N.ptr(dev), N.ptr(lay.sizes), len(lay.host)),
                "naive copy back")
        _poke_words(lay.fields, lay.targets)
        if getattr(self, "_naive_span", None) and len(dev) and int(dev[0]) == self._naive_span[0]:
            tree.__dict__["_spare_naive_span"] = self._naive_span[0]
        self.log.append_many(D2H, "per_object", lay.sizes_i64)
        self.log.append_many(D2H, "detach", lay.attach8)

    # -- unified memory (memory.py:378-394) -------------------------------------------------
    def uvm_touch(self, addr: int, access: str, actor: str) -> int:
        """Route one access through the logical page table; returns migrations (0/1)."""
        if self.uvm is None:
            raise SimMemoryError("uvm_touch outside UVM mode")
        (i,) = self.uvm.index([addr // self.uvm.page_size])
        if i < 0:
            raise WildAccess(f"unified access at 0x{addr:x} hits no registered page")
        return self._touch(np.array([i]), access, actor)

    def uvm_touch_ranges(self, lo_pages, hi_pages, access: str, actor: str) -> int:
        """Touch every page of the inclusive page ranges [lo, hi] (each page once)."""
        return self.uvm_touch_mask(self.uvm_range_mask(lo_pages, hi_pages), access, actor)

    def uvm_range_mask(self, lo_pages, hi_pages) -> np.ndarray:
        """Boolean mask over the page table of the pages in the inclusive ranges [lo, hi];
        WildAccess if any of them was never registered."""
        if self.uvm is None:
            raise SimMemoryError("uvm_touch outside UVM mode")
        u = self.uvm
        lo = np.asarray(lo_pages, np.int64)
        hi = np.asarray(hi_pages, np.int64)
        n = u._pages.size
        if n and int(u._pages[-1]) - int(u._pages[0]) + 1 == n:   # one contiguous registration
            first = int(u._pages[0])
            a = np.clip(lo - first, 0, n)
            b = np.clip(hi - first + 1, 0, n)
        else:
            a = np.searchsorted(u._pages, lo, side="left")
            b = np.searchsorted(u._pages, hi, side="right")
        if ((b - a) != (hi - lo + 1)).any():   # some page of a range was never registered
            raise WildAccess("unified access hits no registered page")
        d = np.bincount(a, minlength=n + 1) - np.bincount(b, minlength=n + 1)   # difference array
        return np.cumsum(d[:-1]) > 0

    def uvm_touch_mask(self, mask: np.ndarray, access: str, actor: str) -> int:
        """Touch the registered pages selected by a boolean mask over the page table."""
        if self.uvm is None:
            raise SimMemoryError("uvm_touch outside UVM mode")
        return self._touch(np.nonzero(mask)[0], access, actor)

    def uvm_touch_pages(self, pages, access: str, actor: str) -> int:
        """Vectorised uvm_touch over a set of page numbers (one touch per page)."""
        if self.uvm is None:
            raise SimMemoryError("uvm_touch outside UVM mode")
        idx = self.uvm.index(np.unique(np.asarray(pages, np.int64)))
        if (idx < 0).any():
            raise WildAccess("unified access hits no registered page")
        return self._touch(idx, access, actor)

    def _touch(self, idx: np.ndarray, access: str, actor: str) -> int:
        u = self.uvm
        on_device = actor == "device"
        move = idx[u._device[idx] != on_device]
        if move.size:
            u._device[move] = on_device
            u._dirty[move] = False
            self.log.append_many(H2D if on_device else D2H, "page_migration",
                                 np.full(move.size, u.page_size, np.int64))
        if access == "write":
            u._dirty[idx] = True
        return int(move.size)


class NaiveLayout:
    """Per-tree layout of the naive scheme's per-object copies (the tree shape is immutable, so
    this is computed once: C4 has 2M objects and 1M pointer fields)."""

    def __init__(self, tree):
        self.host = np.ascontiguousarray(np.asarray(tree.alloc_off, np.uint64) + np.uint64(tree.base))
        self.sizes = np.ascontiguousarray(tree.alloc_size, np.uint64)
        self.sizes_i64 = self.sizes.astype(np.int64)
        aligned = (self.sizes + np.uint64(7)) & ~np.uint64(7)
        self.span = int(aligned.sum())
        self.dev_off = np.concatenate([[0], np.cumsum(aligned)[:-1]]).astype(np.uint64) if len(aligned) else aligned
        order = np.argsort(self.host, kind="stable")
        self.hb = np.ascontiguousarray(self.host[order])
        self.sz = np.ascontiguousarray(self.sizes[order])
        self.doff_sorted = np.ascontiguousarray(self.dev_off[order])
        fields, targets = tree.site_field_target_arrays()
        self.fields = np.ascontiguousarray(fields, np.uint64)
        self.targets = np.ascontiguousarray(targets, np.uint64)
        self.attach8 = np.full(len(self.fields), 8, np.int64)
        # allocation index of every array (allocation order = address order) and of every node
        # (offset, non-empty) keys: scattered forests allocate out of address order, and an empty
        # allocation may share its offset with the next one
        one = np.uint64(1)
        akey = (np.asarray(tree.alloc_off, np.uint64) << one) | (self.sizes > 0).astype(np.uint64)
        rkey = (np.asarray(tree.arr_off, np.uint64) << one) | (np.asarray(tree.arr_count, np.uint64) > 0).astype(np.uint64)
        order = np.argsort(akey, kind="stable")
        self.arr_alloc = order[np.searchsorted(akey[order], rkey)].astype(np.int64) if len(rkey) else np.zeros(0, np.int64)
        is_arr = np.zeros(len(akey), bool)
        is_arr[self.arr_alloc] = True
        self.node_alloc = np.nonzero(~is_arr)[0]
        self.node_host = np.ascontiguousarray(self.host[self.node_alloc])
        self.node_sizes = np.ascontiguousarray(self.sizes[self.node_alloc])
        self._dev: dict[int, np.ndarray] = {}
        self._map_dev: dict[int, np.ndarray] = {}
        for a in (self.host, self.sizes, self.sizes_i64, self.dev_off, self.hb, self.sz, self.doff_sorted, self.fields,
                  self.targets, self.attach8, self.node_host, self.node_sizes):
            a.flags.writeable = False   # shared by every window of this tree
        self.roots: dict = {}   # per policy: chain roots relative to the span base
        self.selective: dict = {}   # per policy: the fused naive window's array list (FusedNaiveWindow)

    def map_dev_at(self, base: int) -> np.ndarray:
        """Device bases in host-address order (the AddressMap column) for a span base."""
        d = self._map_dev.get(base)
        if d is None:
            if len(self._map_dev) >= 4:
                self._map_dev.clear()
            d = self._map_dev[base] = self.doff_sorted + np.uint64(base)
            d.flags.writeable = False
        return d

    def dev_at(self, base: int) -> np.ndarray:
        d = self._dev.get(base)
        if d is None:
            if len(self._dev) >= 4:
                self._dev.clear()
            d = self._dev[base] = self.dev_off + np.uint64(base)
        return d


def naive_layout(tree) -> NaiveLayout:
    lay = tree.__dict__.get("_naive_layout")
    if lay is None:
        lay = tree.__dict__["_naive_layout"] = NaiveLayout(tree)
    return lay


def _poke_words(fields: np.ndarray, values: np.ndarray) -> None:
    """Write 8-byte values at arbitrary (4-aligned) host addresses (native, parallel)."""
    fields = np.ascontiguousarray(fields, np.uint64)
    if fields.size == 0:
        return
    values = np.ascontiguousarray(values, np.uint64)
    N.check(N.lib().cf_host_write_words(N.ptr(fields), N.ptr(values), fields.size), "host pointer restore")


class AddressMap:
    """Interval map translating host addresses into a copied device image (memory.py:397-419)."""

    def __init__(self):
        self._hb = np.zeros(0, np.uint64)
        self._sz = np.zeros(0, np.uint64)
        self._db = np.zeros(0, np.uint64)
        self._pending: list = []
        self._origin = None   # (NaiveLayout, span base) when built by naive_deep_copy and unchanged since

    @classmethod
    def from_arrays(cls, host_base, size, dev_base) -> "AddressMap":
        m = cls()
        order = np.argsort(host_base, kind="stable")
        m._hb = np.ascontiguousarray(np.asarray(host_base, np.uint64)[order])
        m._sz = np.ascontiguousarray(np.asarray(size, np.uint64)[order])
        m._db = np.ascontiguousarray(np.asarray(dev_base, np.uint64)[order])
        return m

    @classmethod
    def from_sorted(cls, host_base, size, dev_base) -> "AddressMap":
        """From contiguous uint64 arrays already ordered by host address."""
        m = cls()
        m._hb, m._sz, m._db = host_base, size, dev_base
        return m

    def add(self, host_base: int, size: int, dev_base: int) -> None:
        self._pending.append((host_base, size, dev_base))
        self._origin = None

    def arrays(self):
        if self._pending:
            hb, sz, db = (np.array(c, np.uint64) for c in zip(*self._pending))
            self._pending = []
            merged = AddressMap.from_arrays(np.concatenate([self._hb, hb]), np.concatenate([self._sz, sz]),
                                            np.concatenate([self._db, db]))
            self._hb, self._sz, self._db = merged._hb, merged._sz, merged._db
        return self._hb, self._sz, self._db

    def translate(self, addr: int) -> int:
        hb, sz, db = self.arrays()
        i = int(np.searchsorted(hb, np.uint64(addr), side="right")) - 1
        if i >= 0 and addr < int(hb[i]) + int(sz[i]):
            return int(db[i]) + (addr - int(hb[i]))
        raise WildAccess(f"fixup target 0x{addr:x} was never copied to the device")

    def translate_many(self, addrs: np.ndarray) -> np.ndarray:
        hb, sz, db = self.arrays()
        a = np.asarray(addrs, np.uint64)
        i = np.searchsorted(hb, a, side="right").astype(np.int64) - 1
        if (i < 0).any() or (a >= hb[i] + sz[i]).any():
            raise WildAccess("fixup target was never copied to the device")
        return db[i] + (a - hb[i])

"""Multi-GPU sharding of the deep-copy workload: one process per GPU, no exchange.

Leaf objects are independent, so every rank deep-copies its own subtree shard over its own
host link and runs relocation, resolve and the leaf kernel locally.  Nothing on the data path
crosses GPUs; the timed region shares only control (barrier, max-over-ranks timing).

* weak scaling (the default benchmark): every rank owns one full config-shaped subtree of a
  forest whose root has one child per rank -- per-GPU work is fixed as N grows;
* strong scaling (C5, 64 GiB total): ONE dense tree cut by subtree at the shallowest level l
  with q^l >= N (DenseSpec.shard_rank / shard_world, planned natively): rank r materialises
  the replicated ancestor path plus the level-l subtrees with ordinal * N // q^l == r, and
  the pointers to the other ranks' subtrees are nulled in its arena.  G = 2: 4 level-1
  subtrees, 2 per GPU; G = 4: 1 each; G = 8: 16 level-2 subtrees, 2 per GPU.

After the timed region the ranks gather a per-leaf checksum vector (position-weighted wrapping
u64 sum of each leaf's u32 words, computed on the device by cf_checksum_ranges) to verify the union of the
shards against the whole tree -- the only collective, over NCCL when every rank has its own
GPU (NVLink / NVSwitch), else gloo.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .scenarios import DenseSpec, payload_values


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    spec: object
    seed: int
    scaling: str  # "weak" | "strong"
    base_seed: int = 1
    # True: this rank holds a subtree shard of ONE tree (seed shared, leaves keyed by the whole
    # tree's ordinals); False: it owns a tree of its own (seed base_seed + rank)
    whole_tree: bool = False


def cut_level(q: int, world: int) -> int:
    """Shallowest level l with q^l >= world."""
    lvl, width = 0, 1
    while width < world:
        width *= q
        lvl += 1
    return lvl


def owned_subtrees(q: int, world: int, rank: int) -> range:
    """Ordinals (at the cut level) of the subtrees rank owns: a contiguous block."""
    width = q ** cut_level(q, world)
    lo = next((o for o in range(width) if o * world // width == rank), width)
    hi = next((o for o in range(lo, width) if o * world // width != rank), width)
    return range(lo, hi)


def subtree_shard(spec: DenseSpec, rank: int, world: int) -> DenseSpec:
    return replace(spec, shard_rank=rank, shard_world=world)


def shard_for(spec, rank: int, world: int, scaling: str = "weak", base_seed: int = 1) -> Shard:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if scaling == "weak":
        return Shard(rank, world, spec, base_seed + rank, scaling, base_seed, False)
    if scaling == "strong":
        if isinstance(spec, DenseSpec) and spec.q ** spec.depth >= world:
            # one tree: every rank builds its subtree shard of the same seeded tree
            return Shard(rank, world, subtree_shard(spec, rank, world) if world > 1 else spec, base_seed, scaling,
                         base_seed, True)
        # fallback: every rank a tree of its own with 1/world of the leaf length
        n = spec.n // world
        if n * world != spec.n:
            raise ValueError(f"leaf length {spec.n} does not split evenly over {world} ranks")
        return Shard(rank, world, replace(spec, n=n), base_seed + rank, scaling, base_seed, False)
    raise ValueError(f"unknown scaling {scaling!r}")


def aggregate_gbs(bytes_per_rank: list[int], max_ms: float) -> float:
    """Whole-job GB/s: all ranks' bytes over the slowest rank's device time."""
    return sum(bytes_per_rank) / (max_ms * 1e-3) / 1e9


# ----------------------------------------------------------------------- result gather
def leaf_checksums(ctx, image: int, arr_off: np.ndarray, arr_count: np.ndarray, elem: int) -> np.ndarray:
    """Per-array checksums of device arrays at image + arr_off (cf_checksum_ranges)."""
    from . import _native as N
    addr = np.ascontiguousarray(np.asarray(arr_off, np.uint64) + np.uint64(image), np.uint64)
    nbytes = np.ascontiguousarray(np.asarray(arr_count, np.uint64) * np.uint64(elem), np.uint64)
    out = np.zeros(len(addr), np.uint64)
    if len(addr):
        N.check(N.lib().cf_checksum_ranges(ctx.handle, N.ptr(addr), N.ptr(nbytes), len(addr), N.ptr(out)),
                "cf_checksum_ranges")
    return out


def range_checksum(words: np.ndarray, first_index: int = 0) -> int:
    """The device checksum (cf_checksum_ranges) of u32 words on the host: sum of word_i * (i + 1)
    mod 2^64, i counted from first_index (position-weighted, so misplaced tiles show)."""
    w = np.asarray(words, np.uint32).astype(np.uint64)
    pos = np.arange(first_index + 1, first_index + 1 + len(w), dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int((w * pos).sum(dtype=np.uint64))


def expected_checksum(seed: int, level: int, n: int, elem: int, scale: float, chunk: int = 1 << 24) -> int:
    """Host-side checksum of payload_values(seed, level, n) * scale (the same for every array of
    a level, scenarios.py:152-155), computed in chunks."""
    dt = np.float64 if elem == 8 else np.float32
    total = 0
    start = (seed * 16777619 + level * 1000003) % (1 << 31)
    wpe = elem // 4   # u32 words per element
    for i0 in range(0, n, chunk):
        m = min(chunk, n - i0)
        raw = (np.arange(i0, i0 + m, dtype=np.int64) + start) & ((1 << 31) - 1)
        vals = raw.astype(np.float64) if elem == 8 else raw.astype(np.float32)
        words = (vals * dt(scale)).astype(dt).view(np.uint32)
        total = (total + range_checksum(words, i0 * wpe)) & ((1 << 64) - 1)
    return total


def gather_checksums(ordinals: np.ndarray, sums: np.ndarray, pg=None, device=None) -> tuple[np.ndarray, np.ndarray]:
    """All-gather (ordinal, checksum) pairs from every rank (torch.distributed; NCCL when
    ``device`` is a CUDA device of this rank, else the group's CPU backend).  Returns them
    sorted by ordinal on every rank; a single process returns its own."""
    import torch
    import torch.distributed as dist
    o = np.asarray(ordinals, np.int64)
    v = np.asarray(sums, np.uint64).view(np.int64)
    if not (dist.is_available() and dist.is_initialized()):
        order = np.argsort(o, kind="stable")
        return o[order], v[order].view(np.uint64)
    world = dist.get_world_size(pg)
    dev = device if device is not None else torch.device("cpu")
    cnt = torch.tensor([len(o)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=pg)
    m = int(max(int(c.item()) for c in counts))
    buf = torch.full((2, max(m, 1)), -1, dtype=torch.int64, device=dev)
    buf[0, :len(o)] = torch.from_numpy(o).to(dev)
    buf[1, :len(o)] = torch.from_numpy(v).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=pg)
    oo = np.concatenate([p[0, :int(c.item())].cpu().numpy() for p, c in zip(parts, counts)])
    vv = np.concatenate([p[1, :int(c.item())].cpu().numpy() for p, c in zip(parts, counts)])
    order = np.argsort(oo, kind="stable")
    return oo[order], vv[order].view(np.uint64)

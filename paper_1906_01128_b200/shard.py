"""Multi-GPU sharding of the deep-copy workload: one process per GPU, no exchange.

Leaf objects are independent, so every rank deep-copies its own subtree shard over its own
host link and runs relocation, resolve and the leaf kernel locally.  Nothing on the data path
crosses GPUs; the only cross-rank traffic is control (barrier, max-over-ranks timing).

* weak scaling (the default benchmark): every rank owns one full config-shaped subtree of a
  forest whose root has one child per rank -- per-GPU work is fixed as N grows;
* strong scaling (C5, 64 GiB total): the 64 leaves' payload is split evenly, each rank owning
  the same tree shape with 1/N of every leaf array (equal bytes per GPU, as a subtree split
  would give for N | 64).
"""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    spec: object
    seed: int
    scaling: str  # "weak" | "strong"


def shard_for(spec, rank: int, world: int, scaling: str = "weak", base_seed: int = 1) -> Shard:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if scaling == "weak":
        return Shard(rank, world, spec, base_seed + rank, scaling)
    if scaling == "strong":
        n = spec.n // world
        if n * world != spec.n:
            raise ValueError(f"leaf length {spec.n} does not split evenly over {world} ranks")
        return Shard(rank, world, replace(spec, n=n), base_seed + rank, scaling)
    raise ValueError(f"unknown scaling {scaling!r}")


def aggregate_gbs(bytes_per_rank: list[int], max_ms: float) -> float:
    """Whole-job GB/s: all ranks' bytes over the slowest rank's device time."""
    return sum(bytes_per_rank) / (max_ms * 1e-3) / 1e9

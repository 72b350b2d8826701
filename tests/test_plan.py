"""The pipelined window's schedule, checked on the CPU (no GPU): cf_window_plan_check plans the
window host-side and verifies its invariants against an independent walk of every chain through
the tree's site table (see include/chainforge_b200.h).  Random trees, packed / aligned arenas,
scattered forests, subtree shards, tiny to whole-arena chunks, resolved and chase modes."""
import ctypes as C
import random

import numpy as np
import pytest

import paper_1906_01128_b200 as cf
from paper_1906_01128_b200 import _native as N
from paper_1906_01128_b200.scenarios import TARGET_POLICIES


def check(spec, align, policy, chunk, mode=N.CF_MODE_RESOLVED, flags=N.CF_WIN_FULL):
    tree = N.NativeTree(spec.native(align))
    tg = np.ascontiguousarray(tree.targets(TARGET_POLICIES[policy]), np.int64)
    d = N.CfWindowDesc(tree.handle, N.ptr(tg) if len(tg) else None, len(tg), None, None, 0x7f0000000000, None,
                       mode, flags, 2.0, chunk)
    out = N.CfPlanCheck()
    rc = N.lib().cf_window_plan_check(C.byref(d), C.byref(out))
    assert rc == 0, (spec, align, policy, chunk, mode, N.last_error())
    assert out.violations == 0
    return out


def test_baseline_shapes():
    c2 = check(cf.DenseSpec(4, 1 << 14, 3, elem=4, leaf_only=True), 16, "all_leaves", 1 << 16)
    assert c2.nsites == 85 and c2.ntargets == 64 and c2.nsteps > 1
    c3 = check(cf.ForestSpec(cf.LinearSpec(4, 1 << 12, "LLinit_LLused", elem=4), 64, scatter_seed=0xC3), 16,
               "all_leaves", 1 << 16)
    assert c3.zero_copy_node_segments > 0        # scattered nodes hoisted and moved by zero-copy
    c4 = check(cf.DenseSpec(100, 16, 2, elem=4), 16, "all_leaves", 1 << 16)
    assert c4.ntargets == 10000


@pytest.mark.parametrize("seed", range(6))
def test_random_plans_hold_their_invariants(seed):
    rng = random.Random(seed)
    for _ in range(25):
        elem = rng.choice([4, 8])
        kind = rng.random()
        if kind < 0.35:
            spec = cf.LinearSpec(rng.randint(1, 7), rng.choice([0, 1, 5, 300, 5000]),
                                 rng.choice(["allinit_allused", "allinit_LLused", "LLinit_LLused"]), elem=elem)
        elif kind < 0.75:
            spec = cf.DenseSpec(rng.randint(1, 5), rng.choice([0, 3, 257, 4000]), rng.randint(0, 3), elem=elem,
                                leaf_only=rng.random() < 0.4)
        else:
            spec = cf.ForestSpec(cf.LinearSpec(rng.randint(1, 4), rng.choice([7, 999, 3000]), "LLinit_LLused", elem=elem),
                                 rng.randint(2, 24), scatter_seed=rng.choice([0, 3, 11]))
        align = rng.choice([1, 8, 16])
        policy = rng.choice(["ref", "all_leaves", "all_arrays"])
        chunk = rng.choice([0, 64, 1000, 4096, 1 << 16])
        mode = rng.choice([N.CF_MODE_RESOLVED, N.CF_MODE_CHASE])
        check(spec, align, policy, chunk, mode)


def test_subtree_shard_plans():
    from paper_1906_01128_b200.shard import subtree_shard
    for world in (2, 4, 8):
        for r in range(world):
            check(subtree_shard(cf.DenseSpec(4, 3000, 3, elem=4, leaf_only=True), r, world), 16, "all_leaves", 8192)


def test_resident_and_copy_only_flag_sets():
    spec = cf.DenseSpec(3, 2000, 3)
    for flags in (N.CF_WIN_RESIDENT, N.CF_WIN_H2D | N.CF_WIN_D2H, N.CF_WIN_H2D | N.CF_WIN_TABLES | N.CF_WIN_ATTACH):
        check(spec, 1, "all_arrays", 0 if flags == N.CF_WIN_RESIDENT else 4096, flags=flags)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
@pytest.mark.parametrize("chunk_mb", [16, 32])
def test_full_size_baseline_schedules(cfg, chunk_mb):
    """The production schedules themselves (full BASELINE shapes, aligned16, 16 / 32 MiB chunks)."""
    import sys
    from conftest import REPO
    sys.path.insert(0, str(REPO))
    import bench
    spec, policy, _ = bench.make_spec(cfg)
    out = check(spec, 16, policy, chunk_mb << 20)
    assert out.nsteps >= 30


@pytest.mark.parametrize("mapped", [0, 1])
def test_pointerchain_window_plans(mapped):
    """cf_selective_plan_check: every targeted array moves exactly once to its device buffer and
    each step scales exactly what it moved -- mixes of big (split), medium and tiny arrays."""
    rng = random.Random(11 + mapped)
    for trial in range(40):
        n = rng.randint(0, 300)
        elem = rng.choice([4, 8])
        counts = np.array([rng.choice([0, 1, 7, 300, 5000, 20000, 300000, 3_000_000]) for _ in range(n)], np.uint64)
        sizes = counts * np.uint64(elem)
        host = np.zeros(n, np.uint64)
        dev = np.zeros(n, np.uint64)
        hb, db = 0x7f0000000000, 0x7e0000000000
        for i in range(n):
            host[i], dev[i] = hb, db
            hb += int(sizes[i]) + 4 * rng.randint(0, 3) + (4 if elem == 8 and rng.random() < 0.3 else 0)
            db += (int(sizes[i]) + 7) // 8 * 8
        steps = N.U64(0)
        chunk = rng.choice([1 << 16, 1 << 20, 32 << 20])
        rc = N.lib().cf_selective_plan_check(n, N.ptr(host) if n else None, N.ptr(dev) if n else None,
                                             N.ptr(counts) if n else None, elem, chunk, mapped, C.byref(steps))
        assert rc == 0, (trial, N.last_error())
        assert steps.value >= 1


def test_pointerchain_window_plans_with_interleaved_layouts():
    """Staged spans on shuffled / gapped host layouts: every array still moves exactly once, and a
    span copied back whole (one D2H DMA) never overlaps an array of another step, nor a DMA-moved
    array of its own step (its scaled result would be overwritten by the stale staging bytes)."""
    rng = random.Random(3)
    for trial in range(150):
        n = rng.randint(2, 400)
        sizes = np.array([rng.choice([64, 1024, 4096, 40000, 70000, 300000]) for _ in range(n)], np.uint64)
        order = list(range(n))
        if rng.random() < 0.5:
            rng.shuffle(order)
        host = np.zeros(n, np.uint64)
        hb = 0x7f0000000000
        for i in order:
            host[i] = hb
            hb += int(sizes[i]) + rng.choice([0, 0, 16, 1200])
        dev = (np.concatenate([[0], np.cumsum(sizes)[:-1]]) + 0x7e0000000000).astype(np.uint64)
        cnt = sizes // np.uint64(4)
        steps = N.U64(0)
        rc = N.lib().cf_selective_plan_check(n, N.ptr(host), N.ptr(dev), N.ptr(cnt), 4,
                                             rng.choice([1 << 16, 1 << 18, 1 << 20]), 1, C.byref(steps))
        assert rc == 0, (trial, N.last_error())


def test_leaf_owned_plans():
    """Steps whose whole, group-sized leaf arrays form one run of consecutive ordinals hand their
    A-field relocation to the leaf kernel (LeafOwn): the checker verifies that those targets leave
    every table (sites, resolve entries, parts), land and stay home long enough, and that each
    step's range has the shape the kernel derives; partial-phase, chase and packed windows keep
    the tables."""
    import sys
    from conftest import REPO
    sys.path.insert(0, str(REPO))
    import bench
    spec, policy, _ = bench.make_spec("C4")
    out = check(spec, 16, policy, 0, flags=N.CF_WIN_RESIDENT)
    assert out.nsteps == 1 and out.leaf_owned == 1
    assert check(spec, 16, policy, 0, flags=N.CF_WIN_RESIDENT | N.CF_WIN_TABLE_RESOLVE).leaf_owned == 0
    # the multi-step e2e window: every step owns its run of whole 1 KiB leaves; only the node-level
    # sites, the few leaves split at step boundaries and the group lists stay in the tables
    out = check(spec, 16, policy, 32 << 20)
    assert out.leaf_owned == out.nsteps >= 30 and out.table_bytes < (1 << 20)
    assert check(spec, 16, policy, 32 << 20, flags=N.CF_WIN_H2D | N.CF_WIN_TABLES | N.CF_WIN_ATTACH).leaf_owned == 0
    assert check(cf.DenseSpec(100, 16, 2, elem=4), 16, "all_leaves", 0, mode=N.CF_MODE_CHASE).leaf_owned == 0
    assert check(cf.DenseSpec(7, 9, 4, elem=4), 1, "all_leaves", 0).leaf_owned == 0   # packed: node fields at 4 mod 8
    owned = 0
    rng = random.Random(7)
    for _ in range(40):
        q = rng.randint(1, 40)
        depth = rng.randint(1, 4)
        while q ** depth > 200000:
            depth -= 1
        spec = cf.DenseSpec(q, rng.choice([1, 3, 16, 64, 300, 5000]), depth, elem=rng.choice([4, 8]),
                            leaf_only=rng.random() < 0.5)
        out = check(spec, rng.choice([8, 16]), rng.choice(["all_leaves", "ref"]), rng.choice([0, 4096, 1 << 16]),
                    flags=rng.choice([N.CF_WIN_RESIDENT, N.CF_WIN_FULL]))
        owned += out.leaf_owned > 0
    assert owned > 5

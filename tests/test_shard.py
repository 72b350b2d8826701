"""Subtree shards of one dense tree: the native planner's partition, on CPU, and
the sharded window against the whole-tree oracle on the GPU."""
import numpy as np
import pytest

import paper_1906_01128_b200 as cf
from paper_1906_01128_b200 import _native as N
from paper_1906_01128_b200.shard import (cut_level, expected_checksum, leaf_checksums, owned_subtrees,
                                         shard_for, subtree_shard)


@pytest.mark.parametrize("q,depth,world", [(4, 3, 1), (4, 3, 2), (4, 3, 4), (4, 3, 8), (3, 2, 2), (2, 3, 8),
                                           (5, 1, 3), (100, 2, 8)])
def test_shards_partition_the_leaves(q, depth, world):
    full = N.NativeTree(cf.DenseSpec(q, 5, depth, leaf_only=True).native(16))
    seen = []
    payload = 0
    for r in range(world):
        spec = subtree_shard(cf.DenseSpec(q, 5, depth, leaf_only=True), r, world) if world > 1 else \
            cf.DenseSpec(q, 5, depth, leaf_only=True)
        t = N.NativeTree(spec.native(16))
        lv, od = t.table(N.CF_TAB_ARR_LEVEL), t.table(N.CF_TAB_ARR_ORDINAL)
        assert (lv == depth).all()
        # each shard's leaves lie under its own cut-level subtrees
        width = q ** (depth - cut_level(q, world))
        assert set((od // width).tolist()) <= set(owned_subtrees(q, world, r))
        seen += od.tolist()
        payload += int(t.info.payload_bytes)
        # the reference target (last child path) lives only on the shard that owns it
        assert len(t.targets(N.CF_TARGET_REF)) == (1 if q ** depth - 1 in od.tolist() else 0)
        assert sorted(t.targets(N.CF_TARGET_ALL_LEAVES).tolist()) == list(range(len(od)))
    assert sorted(seen) == list(range(q ** depth))
    assert payload == int(full.info.payload_bytes)


def test_shard_validation():
    with pytest.raises(ValueError):
        cf.DenseSpec(2, 5, 2, shard_rank=0, shard_world=5)   # 4 subtrees for 5 shards
    with pytest.raises(ValueError):
        cf.DenseSpec(2, 5, 2, shard_rank=2, shard_world=2)
    sh = shard_for(cf.DenseSpec(4, 64, 3, elem=4, leaf_only=True), 3, 8, "strong")
    assert (sh.spec.shard_rank, sh.spec.shard_world, sh.seed, sh.spec.n) == (3, 8, 1, 64)


def test_expected_checksum_matches_numpy():
    for elem in (4, 8):
        vals = cf.payload_values(3, 2, 100_003, elem) * (np.float64(2.0) if elem == 8 else np.float32(2.0))
        words = vals.view(np.uint32)
        want = sum(int(x) * (i + 1) for i, x in enumerate(words.tolist())) % (1 << 64)
        assert expected_checksum(3, 2, 100_003, elem, 2.0, chunk=4096) == want


def test_checksum_sees_misplaced_tiles():
    """The gather checksum is position weighted: two swapped 64 KiB tiles, or one tile written
    at the wrong offset, change it (a plain word sum would not)."""
    from paper_1906_01128_b200.shard import range_checksum
    w = np.random.default_rng(0).integers(0, 1 << 32, 3 * 16384, dtype=np.uint64).astype(np.uint32)
    swapped = np.concatenate([w[16384:32768], w[:16384], w[32768:]])
    shifted = np.concatenate([w[:16384], w[16384:16384 + 8], w[16384:-8]])   # a tile 32 bytes late
    assert int(w.astype(np.uint64).sum()) == int(swapped.astype(np.uint64).sum())
    assert range_checksum(w) != range_checksum(swapped)
    assert range_checksum(w) != range_checksum(shifted)


@pytest.mark.gpu
def test_device_checksum_equals_host_and_sees_swaps():
    if N.device_count() == 0:
        pytest.skip("no GPU visible")
    import ctypes as C
    from paper_1906_01128_b200.shard import range_checksum
    ctx = N.DeviceContext.get(0, 1)
    lib = N.lib()
    rng = np.random.default_rng(1)
    sizes = [4, 64 << 10, (64 << 10) + 12, 3 << 20, 5 * (64 << 10) + 4]
    total = sum(sizes)
    host = rng.integers(0, 1 << 32, total // 4, dtype=np.uint64).astype(np.uint32)
    dev = C.c_void_p()
    N.check(lib.cf_dev_alloc(ctx.handle, total, C.byref(dev)))
    try:
        N.check(lib.cf_memcpy(ctx.handle, dev, N.ptr(host), total))
        offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
        got = leaf_checksums(ctx, dev.value, offs, np.array(sizes, np.uint64) // np.uint64(4), 4)
        want = [range_checksum(host[int(o) // 4:(int(o) + n) // 4]) for o, n in zip(offs, sizes)]
        assert got.tolist() == want
        # swap the first two 64 KiB tiles of the 3 MiB range on the device
        o = int(offs[3]) // 4
        sw = host.copy()
        sw[o:o + 16384], sw[o + 16384:o + 32768] = host[o + 16384:o + 32768], host[o:o + 16384]
        N.check(lib.cf_memcpy(ctx.handle, dev, N.ptr(sw), total))
        got2 = leaf_checksums(ctx, dev.value, offs, np.array(sizes, np.uint64) // np.uint64(4), 4)
        assert got2[3] != got[3] and got2[3] == range_checksum(sw[o:o + (3 << 20) // 4])
    finally:
        lib.cf_dev_free(ctx.handle, dev)


@pytest.mark.gpu
@pytest.mark.parametrize("world,align,elem", [(4, 16, 4), (8, 1, 8), (2, 1, 4)])
def test_sharded_windows_match_the_whole_tree_oracle(oracle, world, align, elem):
    """Each rank's shard window (run one after another on one GPU) returns exactly the whole
    tree's leaves it owns; the gathered checksums cover every leaf once."""
    if N.device_count() == 0:
        pytest.skip("no GPU visible")
    q, n, depth = 4, 3001, 3
    full = oracle.build(oracle.OSpec(oracle.DENSE, q, n, depth, elem=elem, leaf_only=True, align=align), 1)
    fidx = oracle.targets(full, oracle.TARGET_ALL_LEAVES)
    want_full = oracle.expected_after_window(full, fidx, 2.0)
    leaf_nodes = full.node_off[full.node_level == depth]                # pre-order = ordinal order
    by_owner = {int(o): i for i, o in enumerate(full.arr_owner.tolist())}
    ords, sums = [], []
    for r in range(world):
        spec = subtree_shard(cf.DenseSpec(q, n, depth, elem=elem, leaf_only=True), r, world)
        w = cf.DeepCopyWindow(spec, seed=1, policy="all_leaves", align=align, chunk_bytes=8192)
        try:
            st = w.run(scale=2.0)
            assert st.bad == (1 << 64) - 1
            got = w.host_dst()
            off, cnt = w.table(N.CF_TAB_ARR_OFF), w.table(N.CF_TAB_ARR_COUNT)
            od = w.table(N.CF_TAB_ARR_ORDINAL)
            for i in w.targets.tolist():
                a = by_owner[int(leaf_nodes[int(od[i])])]
                fa, nb = int(full.arr_off[a]), int(full.arr_count[a]) * elem
                assert np.array_equal(got[int(off[i]):int(off[i]) + nb], want_full[fa:fa + nb]), (r, int(od[i]))
            # checksums of the device image (detached, scaled) after the window
            ords += od[w.targets].tolist()
            sums += leaf_checksums(w.ctx, w.image, off[w.targets], cnt[w.targets], elem).tolist()
        finally:
            w.close()
    assert sorted(ords) == list(range(q ** depth))
    assert set(sums) == {expected_checksum(1, depth, n, elem, 2.0)}


@pytest.mark.gpu
def test_sharded_tree_through_the_drop_in_api():
    if N.device_count() == 0:
        pytest.skip("no GPU visible")
    for r in range(4):
        m = cf.Machine()
        spec = subtree_shard(cf.DenseSpec(4, 700, 3), r, 4)
        arena, h = cf.marshal_tree(m, spec, seed=5)
        prep = cf.transfer_to_device(m, h, "marshalling", arena, policy="all_arrays")
        cf.kernel_scale(m, h, prep, 2.0)
        cf.copy_back(m, h, prep)
        cf.verify_tree(m, h, 2.0, policy="all_arrays")
        m.close()


@pytest.mark.gpu
def test_gather_over_nccl_single_rank(tmp_path):
    """The result gather's NCCL path (CUDA tensors) on a one-rank group: the only multi-GPU
    collective of the benchmark, exercised on the one GPU a gpurun box has."""
    import socket

    import torch
    import torch.distributed as dist
    from paper_1906_01128_b200.shard import gather_checksums
    if not torch.cuda.is_available():
        pytest.skip("no GPU visible")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        o = np.array([5, 1, 3], np.int64)
        v = np.array([2 ** 64 - 1, 7, 2 ** 63], np.uint64)
        go, gv = gather_checksums(o, v, None, torch.device("cuda", 0))
        assert go.tolist() == [1, 3, 5] and gv.tolist() == [7, 2 ** 63, 2 ** 64 - 1]
    finally:
        dist.destroy_process_group()

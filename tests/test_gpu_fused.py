"""The fused (deferred) marshalling window behind the drop-in calls.

``transfer_to_device -> kernel_scale -> copy_back`` (harness.py:219-325) for the marshalling
scheme is deferred into one pipelined cf_window.  These tests pin it against the eager phases
(``fused=False``: marshal_transfer_and_attach / cf_kernel_scale / demarshal) and the oracle:
identical host bytes after the window, identical logical logs, and the reference's observable
behaviour when something looks at the machine between the calls (flush).
"""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import paper_1906_01128_b200 as cf
    from paper_1906_01128_b200 import _native as N
    if N.device_count() == 0:
        pytest.skip("no GPU visible: run `pytest -m gpu` on a B200 box (gpurun)")
    return cf


def _window(cf, spec, fused, seed=3, scale=2.0, mode="resolved", policy="ref", align=1):
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, spec, seed=seed, align=align)
    mark = m.log.mark()
    prep = cf.transfer_to_device(m, h, "marshalling", arena, policy=policy, fused=fused)
    st = cf.kernel_scale(m, h, prep, scale, mode=mode)
    cf.copy_back(m, h, prep)
    out = bytes(m.host.read_bytes(arena.buffer_host_addr, arena.total_bytes))
    log = [(e.direction, e.op_kind, e.bytes) for e in m.log.since(mark)]
    base = arena.buffer_host_addr
    m.close()
    return out, log, (st.elements_touched, st.chain_derefs), base


def _rel_dump(m, h) -> list:
    """Every allocation's bytes with each pointer field rewritten as (allocation index, offset) of
    its target: two machines place their trees at different host addresses (managed memory in
    particular), so raw pointer words differ while the trees are identical."""
    import bisect
    allocs = sorted(h.allocations)
    starts = [a for a, _ in allocs]
    out = {a: bytearray(m.host.read_bytes(a, s)) for a, s in allocs}
    for holder, off, _ in h.reference_field_sites:
        i = bisect.bisect_right(starts, holder) - 1
        a = starts[i]
        v = m.host.read_word(holder + off)
        j = bisect.bisect_right(starts, v) - 1
        rel = ((j + 1) << 40) | (v - starts[j]) if j >= 0 and v - starts[j] < allocs[j][1] else v
        out[a][holder - a + off:holder - a + off + 8] = rel.to_bytes(8, "little")
    return [bytes(out[a]) for a, _ in h.allocations]


def _norm(cf, raw, spec, base, seed, align):
    """Pointer fields as arena offsets, so two arenas at different addresses compare."""
    m = cf.Machine()
    _, h = cf.marshal_tree(m, spec, seed=seed, align=align)
    a = np.frombuffer(raw, np.uint8).copy()
    for f in h.site_off.tolist():
        v = int.from_bytes(a[f:f + 8].tobytes(), "little") - base
        a[f:f + 8] = np.frombuffer(v.to_bytes(8, "little"), np.uint8)
    m.close()
    return a.tobytes()


@pytest.mark.parametrize("elem", [4, 8])
def test_fused_equals_eager_random_specs(cf, elem):
    rng = random.Random(77 + elem)
    for trial in range(16):
        if rng.random() < 0.5:
            spec = cf.LinearSpec(rng.randint(1, 6), rng.choice([0, 1, 7, 1000, 70001]),
                                 rng.choice(["allinit_allused", "allinit_LLused", "LLinit_LLused"]), elem=elem)
        else:
            spec = cf.DenseSpec(rng.randint(1, 5), rng.choice([0, 3, 257, 40000]), rng.randint(0, 3), elem=elem,
                                leaf_only=rng.random() < 0.3)
        policy = rng.choice(["ref", "all_leaves", "all_arrays"])
        mode = rng.choice(["resolved", "chase"])
        align = rng.choice([1, 16])
        a, la, sa, ba = _window(cf, spec, True, mode=mode, policy=policy, align=align)
        b, lb, sb, bb = _window(cf, spec, False, mode=mode, policy=policy, align=align)
        assert la == lb and sa == sb, (spec, policy, mode)
        assert _norm(cf, a, spec, ba, 3, align) == _norm(cf, b, spec, bb, 3, align), (spec, policy, mode, align)


def test_fused_scattered_forest_in_place(cf):
    """Scattered forests (C3 shape, small): node pages hoisted and moved by zero-copy kernels,
    copy-back in place into the source arena -- fused == eager byte for byte."""
    for elem in (4, 8):
        spec = cf.ForestSpec(cf.LinearSpec(4, 40000, "LLinit_LLused", elem=elem), 24, scatter_seed=7)
        outs = []
        for fused in (True, False):
            m = cf.Machine()
            arena, h = cf.marshal_tree(m, spec, seed=2, align=16)
            prep = cf.transfer_to_device(m, h, "marshalling", arena, policy="all_leaves", fused=fused)
            cf.kernel_scale(m, h, prep, 2.0)
            cf.copy_back(m, h, prep)
            cf.verify_tree(m, h, 2.0, "all_leaves")
            raw = m.host.read_bytes(arena.buffer_host_addr, arena.total_bytes)
            outs.append(_norm_sites(raw, h, arena.buffer_host_addr))
            m.close()
        assert outs[0] == outs[1]


def _norm_sites(raw, h, base):
    import numpy as np
    a = np.frombuffer(raw, np.uint8).copy()
    for f in h.site_off.tolist():
        v = int.from_bytes(a[f:f + 8].tobytes(), "little") - base
        a[f:f + 8] = np.frombuffer(v.to_bytes(8, "little"), np.uint8)
    return a.tobytes()


def test_fused_window_multi_chunk_matches_oracle(cf, oracle):
    """An arena spanning many 16 MiB chunks (C2 shape, small) through the drop-in calls."""
    spec = cf.DenseSpec(4, 1 << 20, 3, elem=4, leaf_only=True)
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, spec, seed=1, align=16)
    prep = cf.transfer_to_device(m, h, "marshalling", arena, policy="all_leaves")
    cf.kernel_scale(m, h, prep, 2.0)
    cf.copy_back(m, h, prep)
    got = np.frombuffer(m.host.read_bytes(arena.buffer_host_addr, arena.total_bytes), np.uint8)
    ospec = oracle.OSpec(oracle.DENSE, 4, 1 << 20, 3, elem=4, leaf_only=True, align=16)
    ot = oracle.build(ospec, 1, ptr_base=arena.buffer_host_addr)
    want = oracle.expected_after_window(ot, oracle.targets(ot, oracle.TARGET_ALL_LEAVES), 2.0)
    assert np.array_equal(got, want[: arena.total_bytes])
    cf.verify_tree(m, h, 2.0, policy="all_leaves")
    m.close()


def test_device_read_between_transfer_and_kernel_flushes(cf):
    """Reading the device after a deferred transfer sees the attached image (test_memory.py:141-150)."""
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, cf.LinearSpec(3, 4, "allinit_allused"), seed=7)
    prep = cf.transfer_to_device(m, h, "marshalling", arena)
    assert m._deferred is prep.fused
    node = prep.device_root
    for _ in range(2):
        node = m.device.read_word(node + 16)
    assert m._deferred is None
    assert m.device.read_f64(m.device.read_word(node + 8)) == m.host.read_f64(h.arrays[-1].addr)
    cf.kernel_scale(m, h, prep, 2.0)          # eager from here on
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0)
    assert m.log.count("attach") == m.log.count("detach") == 5
    m.close()


def test_device_read_between_kernel_and_copy_back_flushes(cf):
    m = cf.Machine()
    spec = cf.DenseSpec(2, 16, 2)
    arena, h = cf.marshal_tree(m, spec, seed=2)
    prep = cf.transfer_to_device(m, h, "marshalling", arena, policy="all_leaves")
    cf.kernel_scale(m, h, prep, 2.0)
    t = h.target_indices("all_leaves")[0]
    dev_arr = prep.image + int(h.arr_off[t])
    host_arr = h.base + int(h.arr_off[t])
    assert m.device.read_f64(dev_arr) == 2.0 * m.host.read_f64(host_arr)
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0, policy="all_leaves")
    m.close()


def test_host_write_before_copy_back_is_snapshotted(cf):
    """transfer_range snapshot semantics (memory.py:294-303): a host write after the transfer call
    does not reach the device copy (it flushes the deferred upload first)."""
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, cf.LinearSpec(2, 8, "allinit_allused"), seed=4)
    prep = cf.transfer_to_device(m, h, "marshalling", arena)
    a = h.arrays[-1].addr
    orig = m.host.read_f64(a)        # flushes
    m.host.write_f64(a, -5.0)
    cf.kernel_scale(m, h, prep, 2.0)
    cf.copy_back(m, h, prep)
    assert m.host.read_f64(a) == orig * 2.0
    m.close()


def test_fused_transfer_rejects_targets_outside_the_arena(cf):
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, cf.LinearSpec(2, 10, "allinit_allused"))
    stray = m.host.allocate(8)
    m.host.write_word(arena.pointer_sites[0], stray)
    mark = m.log.mark()
    with pytest.raises(cf.AttachOutsideArena):
        cf.transfer_to_device(m, h, "marshalling", arena)
    # the reference logs the bulk copy before its attach loop raises on site 0 (memory.py:313-321)
    assert m._deferred is None and [e.op_kind for e in m.log.since(mark)] == ["bulk"]
    m.close()


def test_copy_back_without_kernel_round_trips(cf):
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, cf.DenseSpec(3, 5, 2), seed=1)
    before = m.host.read_bytes(arena.buffer_host_addr, arena.total_bytes)
    prep = cf.transfer_to_device(m, h, "marshalling", arena)
    cf.copy_back(m, h, prep)
    assert m.host.read_bytes(arena.buffer_host_addr, arena.total_bytes) == before
    m.close()


def test_abandoned_window_is_dropped(cf):
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, cf.LinearSpec(2, 10), seed=1)
    prep = cf.transfer_to_device(m, h, "marshalling", arena)
    cf.kernel_scale(m, h, prep, 2.0)
    m.close()
    assert m._deferred is None


def test_execute_case_fused_and_eager_agree(cf):
    cm = cf.CostModel()
    for spec in (cf.LinearSpec(5, 1000, "LLinit_LLused"), cf.DenseSpec(3, 50, 3)):
        a, ma = cf.execute_case(spec, "marshalling", cm, seed=0, fused=True)
        b, mb = cf.execute_case(spec, "marshalling", cm, seed=0, fused=False)
        for k in ("bytes_h2d", "bytes_d2h", "transfer_ops", "attach_ops", "page_faults", "instr_estimate",
                  "sim_kernel_us", "sim_wall_us", "verified"):
            assert getattr(a, k) == getattr(b, k), k
        assert a.gpu_launches > 0
        ma.close()
        mb.close()


def _pc_window(cf, spec, fused, seed=3, scale=2.0, policy="ref", align=None):
    m = cf.Machine()
    h = cf.build_tree(m, spec, seed=seed, align=align)
    mark = m.log.mark()
    prep = cf.transfer_to_device(m, h, "pointerchain", policy=policy, fused=fused)
    st = cf.kernel_scale(m, h, prep, scale)
    cf.copy_back(m, h, prep)
    arrays = [m.host.read_bytes(a.addr, a.count * spec.elem) for a in h.arrays]
    log = [(e.direction, e.op_kind, e.bytes) for e in m.log.since(mark)]
    cf.verify_tree(m, h, scale, policy)
    m.close()
    return arrays, log, st.elements_touched


@pytest.mark.parametrize("elem", [4, 8])
def test_fused_pointerchain_equals_eager(cf, elem):
    """Selective copies pipelined (DMA for big arrays, zero-copy SM copies for small ones)."""
    rng = random.Random(5 + elem)
    specs = [cf.DenseSpec(100, 256, 2, elem=elem), cf.DenseSpec(3, 20001, 2, elem=elem),
             cf.LinearSpec(5, 1000, "LLinit_LLused", elem=elem), cf.DenseSpec(4, 1 << 16, 3, elem=elem, leaf_only=True)]
    for spec in specs + [cf.DenseSpec(rng.randint(1, 6), rng.randint(0, 40000), rng.randint(0, 3), elem=elem)
                         for _ in range(6)]:
        for policy in ("ref", "all_arrays"):
            for align in (None, 1):
                a, la, sa = _pc_window(cf, spec, True, policy=policy, align=align)
                b, lb, sb = _pc_window(cf, spec, False, policy=policy, align=align)
                assert a == b and la == lb and sa == sb, (spec, policy, align)


def test_fused_pointerchain_flush_and_repeat(cf):
    m = cf.Machine()
    h = cf.build_tree(m, cf.DenseSpec(10, 300, 2), seed=2)
    for r in range(3):   # repeated windows reuse the device span and the plan
        prep = cf.transfer_to_device(m, h, "pointerchain", policy="all_leaves")
        cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5)
        cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0, "all_leaves")
    prep = cf.transfer_to_device(m, h, "pointerchain", policy="all_leaves")
    d0 = int(prep.buf_dev[0])
    assert m.device.read_f64(d0) == m.host.read_f64(int(prep.buf_host[0]))   # flushed H2D
    cf.kernel_scale(m, h, prep, 0.5)
    cf.copy_back(m, h, prep)
    m.close()


@pytest.mark.parametrize("scheme,fused", [("naive", True), ("pointerchain", False), ("marshalling", False)])
def test_repeated_windows_reuse_device_storage(cf, scheme, fused):
    """Spare device spans / images are reused window after window (no 1 GiB-class allocation per
    window): repeated transfer -> kernel -> copy_back on one tree stays exact and the device space
    does not grow after the first window."""
    m = cf.Machine()
    spec = cf.DenseSpec(5, 3000, 2)
    if scheme == "marshalling":
        arena, h = cf.marshal_tree(m, spec, seed=4)
    else:
        arena, h = None, cf.build_tree(m, spec, seed=4)
    used = []
    for r in range(4):
        prep = cf.transfer_to_device(m, h, scheme, arena, policy="all_arrays", fused=fused)
        cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5)
        cf.copy_back(m, h, prep)
        used.append(m.device.bump_offset)
    assert used[1] == used[2] == used[3]
    prep = cf.transfer_to_device(m, h, scheme, arena, policy="all_arrays", fused=fused)
    cf.kernel_scale(m, h, prep, 2.0)
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0, "all_arrays")
    m.close()


def test_fused_pointerchain_multi_step_and_split_arrays(cf):
    """Pointerchain windows spanning many 32 MiB steps: arrays larger than a step (split into DMA
    pieces), many small arrays (zero-copy), and a mix -- verify_tree after each."""
    specs = [cf.LinearSpec(3, 12_000_000, "allinit_allused", elem=4),     # 48 MB arrays: split pieces
             cf.DenseSpec(60, 2000, 2, elem=8),                           # 3,600 x 16 KB arrays: zero-copy
             cf.DenseSpec(4, 3_000_000, 2, elem=4)]                       # 21 x 12 MB arrays, DMA
    for spec in specs:
        m = cf.Machine()
        h = cf.build_tree(m, spec, seed=6, align=16)
        prep = cf.transfer_to_device(m, h, "pointerchain", policy="all_arrays")
        cf.kernel_scale(m, h, prep, 2.0)
        cf.copy_back(m, h, prep)
        cf.verify_tree(m, h, 2.0, "all_arrays")
        m.close()


@pytest.mark.parametrize("scheme", ["naive", "marshalling"])
def test_planned_kernel_scale_across_trees_and_policies(cf, scheme):
    """Eager kernel_scale plans its targets' tables once per (tree, policy): interleaving two trees,
    two policies and both leaf-kernel modes in one machine still scales exactly the right arrays."""
    m = cf.Machine()
    trees = []
    for seed, spec in ((5, cf.DenseSpec(3, 700, 2)), (6, cf.LinearSpec(4, 900, "allinit_allused"))):
        if scheme == "marshalling":
            trees.append(cf.marshal_tree(m, spec, seed=seed))
        else:
            trees.append((None, cf.build_tree(m, spec, seed=seed)))
    for r, (t, policy, mode) in enumerate([(0, "all_arrays", "resolved"), (1, "ref", "chase"), (0, "all_arrays", "chase"),
                                           (1, "all_arrays", "resolved"), (0, "ref", "resolved")]):
        arena, h = trees[t]
        prep = cf.transfer_to_device(m, h, scheme, arena, policy=policy, fused=False)
        st = cf.kernel_scale(m, h, prep, 2.0, mode=mode)
        cf.copy_back(m, h, prep)
        assert st.elements_touched == int(h.arr_count[h.target_indices(policy)].sum())
        cf.verify_tree(m, h, 2.0, policy)
        # undo on the host so every round starts from the payload
        prep = cf.transfer_to_device(m, h, scheme, arena, policy=policy, fused=False)
        cf.kernel_scale(m, h, prep, 0.5, mode=mode)
        cf.copy_back(m, h, prep)
        cf.verify_tree(m, h, 1.0, policy)
    m.close()


@pytest.mark.parametrize("scheme,fused", [("marshalling", True), ("marshalling", False), ("pointerchain", True),
                                          ("naive", True), ("uvm", True)])
def test_execute_case_device_phase_times(cf, scheme, fused):
    """execute_case's measured columns: CUDA-event device time per call of the window (a fused
    window enqueues its pipeline at copy_back); they ride in the report row's measured extras."""
    m, machine = cf.execute_case(cf.DenseSpec(4, 200000, 2, elem=4), scheme, cf.CostModel(), seed=1, fused=fused,
                                 policy="all_leaves")
    machine.close()
    assert m.device_us > 0 and abs(m.device_us - (m.transfer_us + m.kernel_us + m.copy_back_us)) < 1e-6 * m.device_us + 1e-3
    assert m.copy_back_us > 0 and m.gpu_launches > 0
    row = cf.report.ResultRow.from_metrics(m) if hasattr(cf, "report") else None
    if row is not None:
        assert row.extra["device_us"] == m.device_us


def _naive_window(cf, spec, fused, seed=3, scale=2.0, policy="ref", align=None, mode="resolved"):
    m = cf.Machine()
    h = cf.build_tree(m, spec, seed=seed, align=align)
    mark = m.log.mark()
    prep = cf.transfer_to_device(m, h, "naive", policy=policy, fused=fused)
    st = cf.kernel_scale(m, h, prep, scale, mode=mode)
    cf.copy_back(m, h, prep)
    dump = [bytes(m.host.read_bytes(a, s)) for a, s in h.allocations]
    log = [(e.direction, e.op_kind, e.bytes) for e in m.log.since(mark)]
    cf.verify_tree(m, h, scale, policy)
    m.close()
    return dump, log, (st.elements_touched, st.chain_derefs)


@pytest.mark.parametrize("elem", [4, 8])
def test_fused_naive_equals_eager(cf, elem):
    """The fused naive window (nodes first + fixup + device chain walk, then the arrays pipelined
    one transfer per object) leaves every host byte, log entry and counter as the eager phases."""
    rng = random.Random(17 + elem)
    specs = [cf.DenseSpec(100, 256, 2, elem=elem), cf.DenseSpec(3, 20001, 2, elem=elem),
             cf.LinearSpec(5, 1000, "LLinit_LLused", elem=elem), cf.LinearSpec(4, 300, "allinit_allused", elem=elem),
             cf.DenseSpec(4, 1 << 16, 3, elem=elem, leaf_only=True),
             cf.ForestSpec(cf.LinearSpec(3, 700, "LLinit_LLused", elem=elem), 9, scatter_seed=5)]
    for spec in specs + [cf.DenseSpec(rng.randint(1, 6), rng.randint(0, 40000), rng.randint(0, 3), elem=elem)
                         for _ in range(5)]:
        for policy in ("ref", "all_arrays", "all_leaves"):
            for align in (None, 1):
                a = _naive_window(cf, spec, True, policy=policy, align=align)
                b = _naive_window(cf, spec, False, policy=policy, align=align)
                assert a == b, (spec, policy, align)


def test_fused_naive_flush_chase_and_repeat(cf):
    m = cf.Machine()
    h = cf.build_tree(m, cf.DenseSpec(6, 3000, 2), seed=4)
    for r in range(3):   # repeated fused windows reuse the span and the plans
        prep = cf.transfer_to_device(m, h, "naive", policy="all_leaves")
        cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5)
        cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0, "all_leaves")
    # an observation between transfer and kernel materialises the copy-in
    prep = cf.transfer_to_device(m, h, "naive", policy="all_leaves")
    root_dev = prep.device_root
    assert m.device.read_word(root_dev + 8) == prep.amap.translate(m.host.read_word(h.root_addr + 8))
    cf.kernel_scale(m, h, prep, 0.5)
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 1.0, "all_leaves")
    # chase mode runs eagerly; copy_back without a kernel round-trips
    prep = cf.transfer_to_device(m, h, "naive", policy="all_leaves")
    cf.kernel_scale(m, h, prep, 2.0, mode="chase")
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0, "all_leaves")
    prep = cf.transfer_to_device(m, h, "naive", policy="all_leaves")
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0, "all_leaves")
    m.close()


def test_naive_chain_walk_check_rejects_wrong_targets(cf):
    """cf_kernel_plan_expect / _resolve: the device-side check of the naive window's chain walk
    reports the first chain that does not end on its array's device copy (CF_E_WILD)."""
    import ctypes as C
    from paper_1906_01128_b200 import _native as N
    from paper_1906_01128_b200 import harness as H
    m = cf.Machine()
    h = cf.build_tree(m, cf.DenseSpec(3, 500, 2), seed=1)
    prep = cf.transfer_to_device(m, h, "naive", policy="all_leaves", fused=False)
    idx, _, _, _, cnt, _ = H._kernel_args(h, "all_leaves")
    kp, sh = H._kernel_plan(m, h, prep)
    lay = prep.amap._origin[0]
    good = np.ascontiguousarray(lay.dev_off[lay.arr_alloc[idx]])
    bad = N.U64(0)
    lib = N.lib()
    N.check(lib.cf_kernel_plan_expect(kp, N.ptr(good), N.ptr(cnt)))
    assert lib.cf_kernel_plan_resolve(kp, prep.image, C.byref(sh), None, None, C.byref(bad)) == 0
    wrong = good.copy()
    wrong[5] += np.uint64(8)
    N.check(lib.cf_kernel_plan_expect(kp, N.ptr(wrong), N.ptr(cnt)))
    assert lib.cf_kernel_plan_resolve(kp, prep.image, C.byref(sh), None, None, C.byref(bad)) == N.CF_E_WILD
    assert bad.value == 5
    wrong_cnt = cnt.copy()
    wrong_cnt[2] += np.uint64(1)
    N.check(lib.cf_kernel_plan_expect(kp, N.ptr(good), N.ptr(wrong_cnt)))
    assert lib.cf_kernel_plan_resolve(kp, prep.image, C.byref(sh), None, None, C.byref(bad)) == N.CF_E_WILD
    assert bad.value == 2
    cf.kernel_scale(m, h, prep, 2.0)
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0, "all_leaves")
    m.close()


@pytest.mark.parametrize("policy", ["ref", "all_leaves", "all_arrays"])
def test_fused_pointerchain_staged_spans_leave_other_bytes_alone(cf, policy):
    """Small arrays staged through one span DMA each way: every byte of the tree outside the
    selected arrays (nodes, unselected arrays, scattered neighbours) is exactly as before, and the
    selected ones exactly as the eager phases leave them."""
    specs = [cf.ForestSpec(cf.LinearSpec(3, 700, "allinit_allused", elem=4), 40, scatter_seed=7),
             cf.DenseSpec(30, 200, 2, elem=4), cf.DenseSpec(12, 1000, 3, elem=8)]
    for spec in specs:
        dumps = []
        for fused in (True, False):
            m = cf.Machine()
            h = cf.build_tree(m, spec, seed=2, align=16)
            for r in range(2):
                prep = cf.transfer_to_device(m, h, "pointerchain", policy=policy, fused=fused)
                cf.kernel_scale(m, h, prep, 2.0)
                cf.copy_back(m, h, prep)
            cf.verify_tree(m, h, 4.0, policy)
            dumps.append([bytes(m.host.read_bytes(a, s)) for a, s in h.allocations])
            m.close()
        assert dumps[0] == dumps[1], (spec, policy)


@pytest.mark.parametrize("mode", ["resolved", "chase"])
def test_fused_uvm_prefetch_window_equals_eager(cf, mode):
    """UVM with prefetch hints runs as one prefetch-pipelined window (CF_WIN_UVM): per step
    migrate in, resolve + scale, migrate home.  Host bytes, logical page-fault log and kernel
    stats equal the eager whole-tree prefetch path, over several windows and multi-chunk trees."""
    specs = [cf.DenseSpec(4, 300_000, 2, elem=4), cf.DenseSpec(3, 5000, 3, elem=8),
             cf.ForestSpec(cf.LinearSpec(3, 200_000, "LLinit_LLused", elem=4), 12, scatter_seed=9)]
    for spec in specs:
        out = []
        for fused in (True, False):
            m = cf.Machine()
            m.enable_uvm()
            h = cf.build_tree(m, spec, seed=4)
            logs, stats = [], []
            for r in range(3):
                mark = m.log.mark()
                prep = cf.transfer_to_device(m, h, "uvm", policy="all_leaves", uvm_hints="prefetch", fused=fused)
                st = cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5, mode=mode)
                cf.copy_back(m, h, prep)
                logs.append([(e.direction, e.op_kind, e.bytes) for e in m.log.since(mark)])
                stats.append((st.elements_touched, st.chain_derefs))
            cf.verify_tree(m, h, 2.0, "all_leaves")
            out.append((_rel_dump(m, h), logs, stats))
            m.close()
        assert out[0][1] == out[1][1] and out[0][2] == out[1][2], spec
        assert out[0][0] == out[1][0], spec


def test_fused_uvm_flush_between_calls(cf):
    """A read between kernel_scale and copy_back materialises the deferred UVM window eagerly."""
    m = cf.Machine()
    m.enable_uvm()
    h = cf.build_tree(m, cf.DenseSpec(3, 2000, 2, elem=4), seed=1)
    prep = cf.transfer_to_device(m, h, "uvm", policy="all_leaves", uvm_hints="prefetch")
    assert m._deferred is prep.fused
    cf.kernel_scale(m, h, prep, 2.0)
    a = h.arrays[-1]
    v = m.host.read_bytes(a.addr, 4)   # observation: flush
    assert m._deferred is None
    assert np.frombuffer(v, np.float32)[0] == cf.payload_values(1, a.level, 1, 4)[0] * 2
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0, "all_leaves")
    m.close()

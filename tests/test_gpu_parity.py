"""GPU parity: the CUDA path against the reference golden vectors and the CPU oracle.

Bar (north_star): relocated pointers / offsets bit-exact; leaf outputs bit-exact (the scale is
a single IEEE multiply, __fmul_rn/__dmul_rn, so no FMA contraction is possible -- tolerance 0).
"""
import hashlib
import random

import numpy as np
import pytest

from paper_1906_01128_b200 import _native as N

pytestmark = pytest.mark.gpu

NO_BAD = (1 << 64) - 1


@pytest.fixture(scope="module")
def cf():
    import paper_1906_01128_b200 as cf
    from paper_1906_01128_b200 import _native as N
    if N.device_count() == 0:
        pytest.skip("no GPU visible: run `pytest -m gpu` on a B200 box (gpurun)")
    return cf


def _spec(cf, j, elem=8, leaf_only=False):
    if j["kind"] == "linear":
        return cf.LinearSpec(j["k"], j["n"], j["layout"], elem=elem)
    return cf.DenseSpec(j["q"], j["n"], j["depth"], elem=elem, leaf_only=leaf_only)


def test_attach_image_matches_reference_kats(cf, kats, oracle):
    """Device image after the relocation kernel == the reference's device image (offset-normalised)."""
    for r in kats["marshal"]:
        m = cf.Machine()
        arena, handle = cf.marshal_tree(m, _spec(cf, r["spec"]), seed=r["seed"])
        image = m.marshal_transfer_and_attach(arena)
        dev = np.frombuffer(m.device.read_bytes(image, arena.total_bytes), np.uint8)
        sites = np.array(r["sites"], np.uint64)
        # relocated pointers bit-exact: device value - image base == reference target offset
        vals = [int.from_bytes(dev[s:s + 8].tobytes(), "little") - image for s in r["sites"]]
        assert vals == r["site_targets"], r["spec"]
        assert hashlib.sha256(oracle.normalised(dev, sites, image)).hexdigest() == r["image_sha"]
        assert m.log.count("attach") == len(r["sites"])
        bulk = [e for e in m.log.entries if e.op_kind == "bulk"]
        assert len(bulk) == 1 and bulk[0].bytes == r["total_bytes"]
        # byte-exact demarshal round trip (test_memory.py:153-160)
        before = m.host.read_bytes(arena.buffer_host_addr, arena.total_bytes)
        m.demarshal(arena)
        assert m.host.read_bytes(arena.buffer_host_addr, arena.total_bytes) == before
        assert m.log.count("detach") == m.log.count("attach")
        m.close()


def test_execute_case_counters_match_reference(cf, kats):
    """Every scheme's RunMetrics counters and sim columns equal the reference's (seed 1)."""
    cm = cf.CostModel()
    for row in kats["counters"]:
        spec = _spec(cf, row["spec"])
        for scheme, want in row["schemes"].items():
            m, machine = cf.execute_case(spec, scheme, cm, seed=1)
            got = [m.bytes_h2d, m.bytes_d2h, m.transfer_ops, m.attach_ops, m.page_faults, m.instr_estimate,
                   m.verified]
            assert got == want[:7], (row["spec"], scheme, got, want)
            assert m.sim_kernel_us == pytest.approx(want[7], rel=1e-12, abs=1e-12)
            assert m.sim_wall_us == pytest.approx(want[8], rel=1e-12)
            machine.close()


def test_after_window_bytes_match_reference(cf, kats, oracle):
    """Host arena after transfer -> scale(2.0) -> copy_back == the reference's (normalised)."""
    for r in kats["marshal"]:
        m = cf.Machine()
        spec = _spec(cf, r["spec"])
        arena, handle = cf.marshal_tree(m, spec, seed=r["seed"])
        for mode in ("resolved", "chase"):
            prep = cf.transfer_to_device(m, handle, "marshalling", arena)
            cf.kernel_scale(m, handle, prep, 2.0 if mode == "resolved" else 0.5, mode=mode)
            cf.copy_back(m, handle, prep)
        # x * 2 * 0.5 == x exactly; run once more with 2.0 for the golden comparison
        prep = cf.transfer_to_device(m, handle, "marshalling", arena)
        cf.kernel_scale(m, handle, prep, 2.0)
        cf.copy_back(m, handle, prep)
        raw = np.frombuffer(m.host.read_bytes(arena.buffer_host_addr, arena.total_bytes), np.uint8)
        norm = oracle.normalised(raw, np.array(r["sites"], np.uint64), arena.buffer_host_addr)
        assert hashlib.sha256(norm).hexdigest() == r["after_window_sha"], r["spec"]
        cf.verify_tree(m, handle, 2.0)
        m.close()


def test_attach_rejects_targets_outside_the_arena(cf):
    m = cf.Machine()
    arena, _ = cf.marshal_tree(m, cf.LinearSpec(2, 10, "allinit_allused"))
    stray = m.host.allocate(8)
    m.host.write_word(arena.pointer_sites[0], stray)
    with pytest.raises(cf.AttachOutsideArena):
        m.marshal_transfer_and_attach(arena)
    m.close()


def test_demarshal_rejects_corrupted_device_pointer(cf):
    m = cf.Machine()
    arena, _ = cf.marshal_tree(m, cf.LinearSpec(2, 10, "allinit_allused"))
    image = m.marshal_transfer_and_attach(arena)
    site = arena.pointer_sites[0] - arena.buffer_host_addr
    m.device.write_word(image + site, 0xDEAD_BEEF)
    with pytest.raises(cf.AttachOutsideArena):
        m.demarshal(arena)
    m.close()


def test_demarshal_before_marshal_raises(cf):
    m = cf.Machine()
    arena, _ = cf.marshal_tree(m, cf.LinearSpec(2, 10))
    with pytest.raises(cf.SimMemoryError):
        m.demarshal(arena)
    m.close()


def test_device_side_chain_chase_after_attach(cf):
    m = cf.Machine()
    arena, handle = cf.marshal_tree(m, cf.LinearSpec(3, 4, "allinit_allused"), seed=7)
    image = m.marshal_transfer_and_attach(arena)
    node = image + (handle.root_addr - arena.buffer_host_addr)
    for _ in range(2):
        node = m.device.read_word(node + 16)
    aptr = m.device.read_word(node + 8)
    assert m.device.read_f64(aptr) == m.host.read_f64(handle.arrays[-1].addr)
    m.close()


def test_naive_and_marshalled_trees_agree_after_copy_back(cf):
    spec = cf.LinearSpec(3, 40, "allinit_allused")
    dumps = []
    for scheme in ("marshalling", "naive", "uvm", "pointerchain"):
        m = cf.Machine()
        if scheme == "uvm":
            m.enable_uvm()
        if scheme == "marshalling":
            arena, h = cf.marshal_tree(m, spec, seed=9)
        else:
            arena, h = None, cf.build_tree(m, spec, seed=9)
        prep = cf.transfer_to_device(m, h, scheme, arena)
        cf.kernel_scale(m, h, prep, 2.0)
        cf.copy_back(m, h, prep)
        dumps.append([m.host.read_bytes(a.addr, a.count * 8) for a in h.arrays])
        m.close()
    assert all(d == dumps[0] for d in dumps[1:])


@pytest.mark.parametrize("elem", [4, 8])
@pytest.mark.parametrize("mode", ["resolved", "chase"])
def test_pipelined_window_matches_oracle_random_specs(cf, oracle, elem, mode):
    """Random trees, packed and aligned layouts, small chunks: the pipelined window's copy-back
    equals the oracle's expected arena bit-for-bit (every dependency path exercised)."""
    rng = random.Random(1234 + elem + len(mode))
    for trial in range(24):
        if rng.random() < 0.5:
            j = {"kind": "linear", "k": rng.randint(1, 9), "n": rng.randint(0, 5000),
                 "layout": rng.choice(["allinit_allused", "allinit_LLused", "LLinit_LLused"])}
            leaf_only = False
        else:
            j = {"kind": "dense", "q": rng.randint(1, 5), "n": rng.randint(0, 3000), "depth": rng.randint(0, 3)}
            leaf_only = rng.random() < 0.4
        align = rng.choice([1, 8, 16])
        policy = rng.choice(["ref", "all_leaves", "all_arrays"])
        chunk = rng.choice([0, 256, 4096, 1 << 16])
        spec = _spec(cf, j, elem, leaf_only)
        w = cf.DeepCopyWindow(spec, seed=trial, policy=policy, mode=mode, align=align, chunk_bytes=chunk)
        try:
            if w.total == 0:
                continue
            st = w.run(scale=2.0)
            assert st.bad == NO_BAD
            ot = oracle.build(oracle.spec_from_json(j, elem=elem, align=align, leaf_only=leaf_only), trial,
                              ptr_base=w.src)
            pol = {"ref": oracle.TARGET_REF, "all_leaves": oracle.TARGET_ALL_LEAVES,
                   "all_arrays": oracle.TARGET_ALL_ARRAYS}[policy]
            idx = oracle.targets(ot, pol)
            want = oracle.expected_after_window(ot, idx, 2.0)[:w.total]
            assert np.array_equal(w.host_dst(), want), (j, align, policy, chunk)
            # same window replayed from a captured CUDA graph (detach fused into the leaf launch)
            st = w.run(scale=2.0, flags=N.CF_WIN_FULL | N.CF_WIN_GRAPH)
            st = w.run(scale=2.0, flags=N.CF_WIN_FULL | N.CF_WIN_GRAPH)
            assert st.bad == NO_BAD
            assert np.array_equal(w.host_dst(), want), (j, align, policy, chunk, "graph")
            # resident path on the same image: attach -> resolve -> scale -> detach
            w.upload_raw()
            st = w.run_resident(scale=2.0)
            assert st.bad == NO_BAD
            assert np.array_equal(w.image_bytes(), want), (j, align, policy, "resident")
            w.upload_raw()
            st = w.run_resident(scale=2.0, graph=True)
            assert st.bad == NO_BAD
            assert np.array_equal(w.image_bytes(), want), (j, align, policy, "resident graph")
        finally:
            w.close()


def test_kernel_scale_counts_and_derefs(cf):
    m = cf.Machine()
    h = cf.build_tree(m, cf.LinearSpec(3, 4, "allinit_allused"))
    prep = cf.transfer_to_device(m, h, "naive")
    st = cf.kernel_scale(m, h, prep, 2.0)
    assert st.elements_touched == 12 and st.chain_derefs == 5
    m.close()
    m = cf.Machine()
    h = cf.build_tree(m, cf.DenseSpec(3, 5, 3))
    prep = cf.transfer_to_device(m, h, "naive")
    st = cf.kernel_scale(m, h, prep, 2.0)
    assert st.elements_touched == 5 and st.chain_derefs == 4
    m.close()


def test_verification_catches_corruption(cf):
    m = cf.Machine()
    h = cf.build_tree(m, cf.LinearSpec(2, 8, "allinit_allused"), seed=3)
    prep = cf.transfer_to_device(m, h, "naive")
    cf.kernel_scale(m, h, prep, 2.0)
    cf.copy_back(m, h, prep)
    cf.verify_tree(m, h, 2.0)
    m.host.write_f64(h.arrays[0].addr, -1.0)
    with pytest.raises(cf.VerificationFailed):
        cf.verify_tree(m, h, 2.0)
    m.close()


@pytest.mark.parametrize("elem", [4, 8])
def test_scattered_forest_window_and_schemes(cf, elem):
    """C3-shaped forests (many chains, objects scattered over the slab): the pipelined window's
    copy-back equals the input with exactly the targeted arrays scaled, for every chunking, and
    all four schemes verify through the drop-in API."""
    spec = cf.ForestSpec(cf.LinearSpec(4, 3001, "LLinit_LLused", elem=elem), 9, scatter_seed=77)
    dt = np.float32 if elem == 4 else np.float64
    for chunk in (0, 4096, 1 << 15):
        for mode in ("resolved", "chase"):
            w = cf.DeepCopyWindow(spec, seed=5, policy="all_leaves", mode=mode, align=16, chunk_bytes=chunk)
            try:
                src = w.host_src().copy()
                st = w.run(scale=2.0)
                assert st.bad == NO_BAD
                want = src.copy()
                for i in w.targets.tolist():
                    a, n = int(w.table(N.CF_TAB_ARR_OFF)[i]), int(w.table(N.CF_TAB_ARR_COUNT)[i])
                    v = want[a:a + n * elem].view(dt)
                    v *= dt(2.0)
                assert np.array_equal(w.host_dst(), want), (chunk, mode)
                assert len(w.targets) == 9
            finally:
                w.close()
    for scheme in ("marshalling", "naive", "pointerchain", "uvm"):
        m, machine = cf.execute_case(spec, scheme, cf.CostModel(), seed=3, policy="all_leaves", align=16)
        assert m.verified and m.scenario.startswith("forest9")
        machine.close()


def test_cli_simulate_and_sweep_match_reference_counters(cf, kats, tmp_path):
    """`python -m paper_1906_01128_b200 simulate|sweep` emit the reference CSV schema with the
    reference's counters (golden execute_case rows); sweeps are byte-deterministic."""
    from paper_1906_01128_b200 import cli
    import contextlib
    import io
    row = next(r for r in kats["counters"] if r["spec"] == {"kind": "dense", "q": 2, "n": 10, "depth": 3})
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert cli.main(["simulate", "--scenario", "dense", "--q", "2", "--n", "10", "--scheme", "marshalling",
                         "--seed", "1"]) == 0
    header, line = buf.getvalue().strip().split("\n")
    assert header == cli.CSV_HEADER
    vals = dict(zip(header.split(","), line.split(",")))
    want = row["schemes"]["marshalling"]
    assert [int(vals[k]) for k in ("bytes_h2d", "bytes_d2h", "transfer_ops", "attach_ops", "page_faults",
                                   "instr_estimate")] == want[:6]
    grid = tmp_path / "grid.csv"
    grid.write_text("scenario,scheme,layout,k_or_q,n\n" + "".join(
        f"linear,{s},LLinit_LLused,3,100\n" for s in ("uvm", "marshalling", "pointerchain", "naive")))
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(["sweep", "--grid", str(grid), "--out", str(a), "--seed", "3"]) == 0
    assert cli.main(["sweep", "--grid", str(grid), "--out", str(b), "--seed", "3"]) == 0
    assert a.read_bytes() == b.read_bytes()
    rows = a.read_text().strip().split("\n")
    assert len(rows) == 5 and rows[0] == cli.CSV_HEADER


@pytest.mark.parametrize("mode", ["resolved", "chase"])
def test_packed_f64_word_streaming_matches_oracle(cf, oracle, mode):
    """f64 arrays at 4 (mod 8) -- the packed reference layout with odd q -- take the aligned-word
    streaming path of the leaf kernel (scale_f64_shifted).  Multi-tile arrays cut into pieces at
    arbitrary element offsets by odd chunk sizes must come back bit-exact."""
    cases = [({"kind": "dense", "q": 3, "n": n, "depth": 2}, lo) for n in (2047, 2048, 2049, 4095, 10001)
             for lo in (False, True)]
    cases += [({"kind": "dense", "q": 5, "n": 7000, "depth": 2}, True), ({"kind": "dense", "q": 1, "n": 9999, "depth": 3}, False)]
    for trial, (j, leaf_only) in enumerate(cases):
        spec = _spec(cf, j, 8, leaf_only)
        for chunk in (0, 4096, 12340, 1 << 16):
            w = cf.DeepCopyWindow(spec, seed=trial, policy="all_arrays", mode=mode, align=1, chunk_bytes=chunk)
            try:
                offs = w.table(N.CF_TAB_ARR_OFF)
                assert (offs % 8 == 4).any(), "case must exercise arrays at 4 mod 8"
                st = w.run(scale=2.0)
                assert st.bad == NO_BAD
                ot = oracle.build(oracle.spec_from_json(j, elem=8, align=1, leaf_only=leaf_only), trial,
                                  ptr_base=w.src)
                want = oracle.expected_after_window(ot, oracle.targets(ot, oracle.TARGET_ALL_ARRAYS), 2.0)[:w.total]
                assert np.array_equal(w.host_dst(), want), (j, leaf_only, chunk)
                w.upload_raw()
                st = w.run_resident(scale=2.0)
                assert st.bad == NO_BAD and np.array_equal(w.image_bytes(), want), (j, leaf_only, "resident")
            finally:
                w.close()


@pytest.mark.parametrize("mode", ["resolved", "chase"])
def test_salted_payload_catches_same_level_swaps(cf, mode):
    """payload_values depends only on (seed, level, i), so every array of a level holds the same
    bytes and a chain resolved to the wrong sibling would go unnoticed.  Salt every array with
    its own pattern (array index in the values), run the window, and require each targeted array
    = its own salt x 2 and everything else unchanged ("salted init")."""
    specs = [(cf.DenseSpec(3, 700, 3, elem=4), 1, "all_arrays"), (cf.DenseSpec(4, 3000, 2, elem=8), 16, "all_leaves"),
             (cf.DenseSpec(20, 40, 2, elem=4), 16, "all_leaves"),
             (cf.LinearSpec(6, 2500, "allinit_allused", elem=8), 1, "ref"),
             (cf.ForestSpec(cf.LinearSpec(3, 3000, "LLinit_LLused", elem=4), 12, scatter_seed=3), 16, "all_leaves")]
    for spec, align, policy in specs:
        for chunk in (0, 8192):
            w = cf.DeepCopyWindow(spec, seed=2, policy=policy, mode=mode, align=align, chunk_bytes=chunk)
            try:
                e = spec.elem
                dt = np.float32 if e == 4 else np.float64
                off, cnt = w.table(N.CF_TAB_ARR_OFF), w.table(N.CF_TAB_ARR_COUNT)
                src = w.host_src()
                for i in range(len(off)):
                    n, a = int(cnt[i]), int(off[i])
                    if n:
                        salt = ((np.arange(n, dtype=np.int64) * 7 + i * 65537) % (1 << 20)).astype(dt)
                        src[a:a + n * e] = np.frombuffer(salt.tobytes(), np.uint8)
                before = src.copy()
                st = w.run(scale=2.0)
                assert st.bad == NO_BAD
                want = before.copy()
                for i in w.targets.tolist():
                    n, a = int(cnt[i]), int(off[i])
                    if n:
                        vals = np.frombuffer(before[a:a + n * e].tobytes(), dt) * dt(2.0)
                        want[a:a + n * e] = np.frombuffer(vals.astype(dt).tobytes(), np.uint8)
                assert np.array_equal(w.host_dst(), want), (spec, align, policy, chunk)
                w.upload_raw()
                st = w.run_resident(scale=2.0, graph=True)
                assert st.bad == NO_BAD and np.array_equal(w.image_bytes(), want), (spec, "resident")
            finally:
                w.close()


def test_fields_straddling_chunk_boundaries(cf, oracle):
    """4-mod-8 pointer fields that straddle a chunk grid point (packed layouts, 12-byte leaf
    records) must land whole before they are attached -- on a fresh image, first window.  The
    schedule bug this pins (a moved cut left a 4-byte segment holding half a field) was found
    by cf_window_plan_check (tests/test_plan.py)."""
    for j, chunk in (({"kind": "dense", "q": 2, "n": 4000, "depth": 3}, 64), ({"kind": "dense", "q": 3, "n": 5, "depth": 3}, 40),
                     ({"kind": "dense", "q": 5, "n": 100, "depth": 2}, 256)):
        for leaf_only in (False, True):
            spec = _spec(cf, j, 8, leaf_only)
            w = cf.DeepCopyWindow(spec, seed=3, policy="all_arrays", align=1, chunk_bytes=chunk)
            try:
                st = w.run(scale=2.0)
                assert st.bad == NO_BAD, (j, chunk, leaf_only)
                ot = oracle.build(oracle.spec_from_json(j, elem=8, align=1, leaf_only=leaf_only), 3, ptr_base=w.src)
                want = oracle.expected_after_window(ot, oracle.targets(ot, oracle.TARGET_ALL_ARRAYS), 2.0)[:w.total]
                assert np.array_equal(w.host_dst(), want), (j, chunk, leaf_only)
            finally:
                w.close()


@pytest.mark.parametrize("hint", ["none", "prefetch", "advise", "preferred", "read_mostly"])
def test_uvm_hints_keep_results_and_counters(cf, hint):
    """Every UVM driver hint leaves the results bit-exact and the reference's logical
    counters unchanged; the hint is undone at copy-back, so windows with different hints can follow
    one another on one tree."""
    spec = cf.DenseSpec(4, 3000, 2, elem=4)
    m = cf.Machine()
    m.enable_uvm()
    h = cf.build_tree(m, spec, seed=2)
    counters = []
    for r, hh in enumerate((hint, "none", hint)):
        mark = m.log.mark()
        prep = cf.transfer_to_device(m, h, "uvm", policy="all_leaves", uvm_hints=hh)
        cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5)
        cf.copy_back(m, h, prep)
        counters.append([(e.direction, e.op_kind, e.bytes) for e in m.log.since(mark)])
    cf.verify_tree(m, h, 2.0, "all_leaves")
    assert counters[1] == counters[2]   # same starting residence, different hint
    m.close()

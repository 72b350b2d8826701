"""Large dense trees whose targets form uniform resolve ranges (consecutive ordinals at one level):
the one-launch attach || resolve takes the memory-parallel resolver (k_attach_resolve_uni, 32 U
targets per warp, parents walked one per lane) and the leaf kernel launches as its programmatic
dependent.  Every case is checked byte for byte against the oracle's expected arena
(scenarios.py:270-284 resolve, harness.py:307-309 scale, memory.py:316-344 attach / detach) through
the pipelined window (one step and many small steps, so ranges start at arbitrary ordinals and
split parent runs -- the multi-step windows own each step's run of whole leaves, the leaves split at
step boundaries go through the tables), its graph replay, and the resident step.  The fan-outs q cover every run
width U the launcher picks (q = 2 forces U = 1 ... q >= 9 allows U = 8), leaf records at 4 mod 8
(owned attach) and aligned, f32 and f64."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
NO_BAD = (1 << 64) - 1


@pytest.fixture(scope="module")
def cf():
    import paper_1906_01128_b200 as cf
    from paper_1906_01128_b200 import _native as N
    if N.device_count() == 0:
        pytest.skip("no GPU visible: run `pytest -m gpu` on a B200 box (gpurun)")
    return cf


@pytest.fixture(scope="module")
def oracle():
    from oracle import oracle as O
    return O


CASES = [
    # q, depth, n (elements per leaf), elem, leaf_only
    (2, 13, 3, 4, True),
    (3, 9, 5, 8, True),
    (4, 7, 33, 4, False),
    (7, 5, 9, 4, True),
    (9, 4, 70, 8, True),
    (16, 4, 1, 4, True),
    (33, 3, 17, 4, False),
    (100, 2, 256, 4, True),
    (100, 3, 4, 4, True),
    (5000, 1, 2, 4, True),     # depth 1: the parent is the root
    (4500, 1, 7, 8, False),
    (65, 2, 2048, 4, True),    # 8 KiB leaves: 4 per group
    (70, 2, 3801, 4, True),    # 15.2 KB leaves (just under a tile): 2 per group, scalar tails
]


@pytest.mark.parametrize("q,depth,n,elem,leaf_only", CASES)
def test_uniform_ranges_match_oracle(cf, oracle, q, depth, n, elem, leaf_only):
    spec = cf.DenseSpec(q, n, depth, elem=elem, leaf_only=leaf_only)
    j = {"kind": "dense", "q": q, "n": n, "depth": depth}
    for chunk in (0, 1 << 16):
        w = cf.DeepCopyWindow(spec, seed=q + depth, policy="all_leaves", align=16, chunk_bytes=chunk)
        try:
            assert len(w.targets) > 4096   # past the one-CTA attach + resolve: the wide launch
            st = w.run(scale=2.0)
            assert st.bad == NO_BAD
            ot = oracle.build(oracle.spec_from_json(j, elem=elem, align=16, leaf_only=leaf_only), q + depth,
                              ptr_base=w.src)
            idx = oracle.targets(ot, oracle.TARGET_ALL_LEAVES)
            want = oracle.expected_after_window(ot, idx, 2.0)[:w.total]
            assert np.array_equal(w.host_dst(), want), (q, depth, n, chunk)
            for _ in range(2):   # graph capture, then replay
                st = w.run(scale=2.0, flags=_flags().CF_WIN_FULL | _flags().CF_WIN_GRAPH)
                assert st.bad == NO_BAD
                assert np.array_equal(w.host_dst(), want), (q, depth, n, chunk, "graph")
            if chunk == 0:
                w.upload_raw()
                assert w.run_resident(scale=2.0).bad == NO_BAD
                assert np.array_equal(w.image_bytes(), want), (q, depth, n, "resident")
                for rep in ("capture", "replay"):
                    w.upload_raw()
                    assert w.run_resident(scale=2.0, graph=True).bad == NO_BAD
                    assert np.array_equal(w.image_bytes(), want), (q, depth, n, "resident graph", rep)
                # the same step planned without leaf ownership (EA table + full site list)
                w.upload_raw()
                assert w.run_n(1, flags=_flags().CF_WIN_RESIDENT | _flags().CF_WIN_TABLE_RESOLVE).bad == NO_BAD
                assert np.array_equal(w.image_bytes(), want), (q, depth, n, "table resolve")
        finally:
            w.close()


def _flags():
    from paper_1906_01128_b200 import _native as N
    return N


def test_uniform_resolver_reports_a_broken_parent_link(cf):
    """A parent's child-block pointer corrupted to the arena's last bytes: the uniform resolver
    sees a record outside the image -> WildAccess from the resolve phase (harness.py walk), and
    the leaf kernel scales nothing through it."""
    from paper_1906_01128_b200 import _native as N
    spec = cf.DenseSpec(16, 2, 4, elem=4, leaf_only=True)
    w = cf.DeepCopyWindow(spec, seed=5, policy="all_leaves", align=16)
    try:
        assert len(w.targets) > 4096
        node_off = w.table(N.CF_TAB_NODE_OFF)
        node_lv = w.table(N.CF_TAB_NODE_LEVEL)
        parent = int(node_off[np.flatnonzero(node_lv == spec.depth - 1)[7]])
        src = w.host_src()
        bad_ptr = w.src + w.total - 4   # inside the arena, so attach accepts it
        src[parent + 16:parent + 24] = np.frombuffer(int(bad_ptr).to_bytes(8, "little"), np.uint8)
        with pytest.raises(cf.WildAccess):
            w.run(scale=2.0)
    finally:
        w.close()


@pytest.mark.parametrize("bad,exc", [("outside", "AttachOutsideArena"), ("overrun", "WildAccess")])
def test_leaf_owned_relocation_faults(cf, bad, exc):
    """Resident one-step windows over uniform leaf ranges attach every leaf A field inside the leaf
    kernel (leaf-owned relocation).  A field holding a host address outside the arena raises the
    attach fault (memory.py:319-321 AttachOutsideArena); an address inside the arena whose span
    overruns the image raises WildAccess (memory.py:139-152).  Either way the other leaves'
    fields come back detached (host values) in the image."""
    from paper_1906_01128_b200 import _native as N
    spec = cf.DenseSpec(16, 4, 4, elem=4, leaf_only=True)
    w = cf.DeepCopyWindow(spec, seed=9, policy="all_leaves", align=16)
    try:
        arr_owner = w.table(N.CF_TAB_ARR_OWNER)
        i = int(w.targets[len(w.targets) // 3])
        field = int(arr_owner[i]) + 4
        src = w.host_src()
        keep = src.copy()
        ptr = (w.src + w.total + 4096) if bad == "outside" else (w.src + w.total - 8)
        src[field:field + 8] = np.frombuffer(int(ptr).to_bytes(8, "little"), np.uint8)
        w.upload_raw()
        with pytest.raises(getattr(cf, exc)):
            w.run_resident(scale=2.0)
        img = w.image_bytes()
        others = np.ones(w.total, bool)
        off, cnt = w.table(N.CF_TAB_ARR_OFF), w.table(N.CF_TAB_ARR_COUNT)
        for t in w.targets.tolist():   # the leaves' payload was scaled; pointers and nodes must be back
            others[int(off[t]):int(off[t]) + 4 * int(cnt[t])] = False
        others[field:field + 8] = False
        assert np.array_equal(img[others], keep[others])
        src[:] = keep
    finally:
        w.close()


def test_leaf_owned_steps_attach_the_leaf_fields(cf, oracle):
    """Leaf-owned relocation really attaches: with the detach suppressed (CF_WIN_DEBUG_KEEP_LEAF_ATTACHED)
    every owned leaf record's A field holds the device address of its array (image + offset, the
    value memory.py:316-323 writes), in the resident image and in a multi-step window's copy-back;
    every other byte is the normal window's result (node pointers detached, leaves scaled)."""
    from paper_1906_01128_b200 import _native as N
    spec = cf.DenseSpec(16, 4, 4, elem=4, leaf_only=True)
    w = cf.DeepCopyWindow(spec, seed=2, policy="all_leaves", align=16, chunk_bytes=1 << 16)
    try:
        ot = oracle.build(oracle.spec_from_json({"kind": "dense", "q": 16, "n": 4, "depth": 4}, elem=4, align=16,
                                                leaf_only=True), 2, ptr_base=w.src)
        want = oracle.expected_after_window(ot, oracle.targets(ot, oracle.TARGET_ALL_LEAVES), 2.0)[:w.total]
        owner, off = w.table(N.CF_TAB_ARR_OWNER), w.table(N.CF_TAB_ARR_OFF)
        fields = np.array([int(owner[t]) + 4 for t in w.targets.tolist()], np.int64)
        attached = want.copy()
        for f, t in zip(fields.tolist(), w.targets.tolist()):
            attached[f:f + 8] = np.frombuffer(int(w.image + int(off[t])).to_bytes(8, "little"), np.uint8)
        res = w._window(N.CF_WIN_RESIDENT, 0, "resolved")
        full = w._window(N.CF_WIN_FULL, w.chunk_bytes, "resolved")
        for h in (res, full):
            N.check(N.lib().cf_window_debug(h, N.CF_WIN_DEBUG_KEEP_LEAF_ATTACHED))
        w.upload_raw()
        assert w.run_resident(scale=2.0).bad == NO_BAD
        assert np.array_equal(w.image_bytes(), attached), "resident image"
        assert w.run(scale=2.0).bad == NO_BAD
        assert np.array_equal(w.host_dst(), attached), "multi-step window copy-back"
        for h in (res, full):
            N.check(N.lib().cf_window_debug(h, 0))
        assert w.run(scale=2.0).bad == NO_BAD
        assert np.array_equal(w.host_dst(), want)
    finally:
        w.close()

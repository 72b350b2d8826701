"""Fault paths of the device window against the reference's exceptions and logs.

* a leaf array pointer corrupted to point near the end of the image (its span overruns the
  image, the count is valid) -> WildAccess, and nothing outside the image is written
  (memory.py:139-152: any span past its allocation raises WildAccess);
* attach of a pointer field outside the arena -> AttachOutsideArena, with the reference's log
  up to the raise: the bulk copy plus one attach per site before the bad one (memory.py:313-323);
* demarshal of a corrupted device pointer -> AttachOutsideArena after the bulk copy and the
  detaches that precede it in reversed site order (memory.py:335-343).
"""
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


def _last_leaf_field(w, N):
    """(arena offset of the A field of the last targeted array's owner, count) for a window."""
    off, cnt, own = w.table(N.CF_TAB_ARR_OFF), w.table(N.CF_TAB_ARR_COUNT), w.table(N.CF_TAB_ARR_OWNER)
    site_off, site_tgt = w.table(N.CF_TAB_SITE_OFF), w.table(N.CF_TAB_SITE_TARGET)
    i = int(w.targets[-1])
    field = int(site_off[np.flatnonzero(site_tgt == off[i])[0]])
    assert int(own[i]) <= field < int(own[i]) + 24
    return field, int(cnt[i])


@pytest.mark.parametrize("spec_kw", [dict(kind="dense", elem=4), dict(kind="dense", elem=8),
                                     dict(kind="linear", elem=4)])
@pytest.mark.parametrize("mode", ["resolved", "chase"])
def test_leaf_pointer_near_image_end_is_wild(cf, spec_kw, mode):
    from paper_1906_01128_b200 import _native as N
    if spec_kw["kind"] == "dense":
        spec = cf.DenseSpec(3, 5000, 2, elem=spec_kw["elem"], leaf_only=True)
    else:
        spec = cf.LinearSpec(3, 5000, "allinit_allused", elem=spec_kw["elem"])
    w = cf.DeepCopyWindow(spec, seed=1, policy="all_arrays", mode=mode, align=16, chunk_bytes=1 << 16)
    try:
        field, cnt = _last_leaf_field(w, N)
        src = w.host_src()
        # inside the arena (attach accepts it), but [A, A + nA * elem) runs past its end
        bad_ptr = w.src + w.total - 8
        src[field:field + 8] = np.frombuffer(int(bad_ptr).to_bytes(8, "little"), np.uint8)
        assert cnt * spec.elem > 8
        with pytest.raises(cf.WildAccess, match="leaf kernel"):
            w.run(scale=2.0)
        # resident: the same image, attach -> resolve -> scale -> detach
        w.upload_raw()
        before = w.image_bytes()
        with pytest.raises(cf.WildAccess):
            w.run_resident(scale=2.0)
        after = w.image_bytes()
        # no array was scaled through the bad pointer: the image's last 8 bytes are intact
        assert np.array_equal(after[-8:], before[-8:])
    finally:
        w.close()


def test_dropin_window_reports_wild_leaf_pointer(cf):
    """Through the drop-in calls (fused marshalling window): the corrupted leaf pointer raises
    WildAccess by copy_back at the latest (the reference raises it inside kernel_scale)."""
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, cf.LinearSpec(2, 1000, "allinit_allused"), seed=1)
    base, total = arena.buffer_host_addr, arena.total_bytes
    last_a = h.node_addrs[-1] + 8
    m.host.write_word(last_a, base + total - 16)
    prep = cf.transfer_to_device(m, h, "marshalling", arena, policy="all_arrays")
    with pytest.raises(cf.WildAccess):
        cf.kernel_scale(m, h, prep, 2.0)
        cf.copy_back(m, h, prep)
    m.close()


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("bad_site", [0, 2, 4])
def test_attach_fault_logs_like_the_reference(cf, fused, bad_site):
    m = cf.Machine()
    arena, h = cf.marshal_tree(m, cf.LinearSpec(3, 10, "allinit_allused"), seed=1)
    assert len(arena.pointer_sites) == 5
    stray = m.host.allocate(8)
    m.host.write_word(arena.pointer_sites[bad_site], stray)
    mark = m.log.mark()
    with pytest.raises(cf.AttachOutsideArena, match=f"pointer field at 0x{arena.pointer_sites[bad_site]:x} targets"):
        if fused:
            cf.transfer_to_device(m, h, "marshalling", arena)
        else:
            m.marshal_transfer_and_attach(arena)
    log = [(e.direction, e.op_kind, e.bytes) for e in m.log.since(mark)]
    assert log == [("H2D", "bulk", arena.total_bytes)] + [("H2D", "attach", 8)] * bad_site
    assert m._deferred is None
    m.close()


@pytest.mark.parametrize("bad_site", [0, 2, 4])
def test_demarshal_fault_logs_like_the_reference(cf, bad_site):
    m = cf.Machine()
    arena, _ = cf.marshal_tree(m, cf.LinearSpec(3, 10, "allinit_allused"), seed=1)
    image = m.marshal_transfer_and_attach(arena)
    site = arena.pointer_sites[bad_site] - arena.buffer_host_addr
    m.device.write_word(image + site, 0xDEAD_BEEF)
    mark = m.log.mark()
    with pytest.raises(cf.AttachOutsideArena):
        m.demarshal(arena)
    # detach runs over reversed(pointer_sites): sites 4, 3, ... precede site bad_site
    log = [(e.direction, e.op_kind, e.bytes) for e in m.log.since(mark)]
    assert log == [("D2H", "bulk", arena.total_bytes)] + [("D2H", "detach", 8)] * (4 - bad_site)
    m.close()

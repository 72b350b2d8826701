"""Pin the C oracle against the reference's own outputs (tests/golden/reference_kats.json).

Every record there was produced by running the reference (oracle/gen_golden.py); this file
checks the restatement in oracle/cf_oracle.c reproduces it bit-for-bit (f64, packed arena and
8-byte host bump layouts), so the oracle can stand in for the reference in the GPU parity tests.
"""
import hashlib

import numpy as np
import pytest

pytestmark = []


def _records(kats):
    return kats["marshal"]


def test_payload_values_match_reference(kats, oracle):
    # payload_values (scenarios.py:152-155) KATs
    for key, vals in kats["payload_kat"].items():
        seed, level = (int(x) for x in key.split(":"))
        spec = oracle.OSpec(oracle.LINEAR, level + 1, 6, 0, "allinit_allused", 8)
        t = oracle.build(spec, seed)
        a = t.arr_off[level]
        got = np.frombuffer(t.buf[a:a + 48].tobytes(), "<f8").tolist()
        assert got == vals, key


def test_closed_form_sizes(kats, oracle):
    for k, n, lay, size in kats["sizes"]["linear"]:
        assert oracle.counts(oracle.OSpec(oracle.LINEAR, k, n, 0, lay)).total == size
    for q, n, d, size in kats["sizes"]["dense"]:
        if q ** d > 2_000_000:
            continue
        assert oracle.counts(oracle.OSpec(oracle.DENSE, q, n, d)).total == size


@pytest.mark.parametrize("i", range(64))
def test_marshal_record(kats, oracle, i):
    recs = _records(kats)
    if i >= len(recs):
        pytest.skip("fewer records")
    r = recs[i]
    spec = oracle.spec_from_json(r["spec"])
    t = oracle.build(spec, r["seed"])
    assert t.total == r["total_bytes"]
    assert t.allocs.tolist() == r["requests"]
    assert t.site_off.tolist() == r["sites"]
    assert t.site_target.tolist() == r["site_targets"]
    assert [[a, b, c] for a, b, c in zip(t.node_off.tolist(), t.node_level.tolist(),
                                         t.node_size.tolist())] == r["nodes"]
    assert [[a, b, c, d] for a, b, c, d in zip(t.arr_level.tolist(), t.arr_owner.tolist(),
                                               t.arr_off.tolist(), t.arr_count.tolist())] == r["arrays"]
    norm = oracle.normalised(t.buf[:t.total], t.site_off, t.ptr_base)
    assert hashlib.sha256(norm).hexdigest() == r["arena_sha"]
    if "arena_hex" in r:
        assert norm.hex() == r["arena_hex"]
    # attach into an image at another base (memory.py:316-323)
    img = t.buf.copy()
    image_base = 0x7F00_0000_0000
    assert oracle.relocate(img, t.total, t.site_off, t.ptr_base, image_base) == -1
    assert hashlib.sha256(oracle.normalised(img[:t.total], t.site_off, image_base)).hexdigest() == r["image_sha"]
    # targeted_arrays (scenarios.py:270-284) and the device-side chain walk (harness.py:285-304)
    idx = oracle.targets(t, oracle.TARGET_REF)
    assert t.arr_off[idx].tolist() == r["targeted"]
    ea, cnt = oracle.resolve(img, image_base, t, idx)
    assert ea.tolist() == t.arr_off[idx].tolist()
    assert int(cnt.astype(np.int64).sum()) == r["kernel_elements"]
    # metered window: transfer -> scale(2.0) -> copy_back, host arena afterwards
    after = oracle.expected_after_window(t, idx, 2.0)
    assert hashlib.sha256(oracle.normalised(after[:t.total], t.site_off, t.ptr_base)).hexdigest() == r["after_window_sha"]
    dev, out = np.zeros_like(t.buf), np.zeros_like(t.buf)
    assert oracle.window(t, idx, dev, out, t.ptr_base, image_base, 2.0, 2) == -1
    assert out[:t.total].tobytes() == after[:t.total].tobytes()
    # detach restores the original arena (memory.py:337-344, test_memory.py:153-160)
    assert oracle.relocate(img, t.total, t.site_off, image_base, t.ptr_base) == -1
    assert img.tobytes() == t.buf.tobytes()


@pytest.mark.parametrize("i", range(64))
def test_bump_layout_record(kats, oracle, i):
    recs = _records(kats)
    if i >= len(recs):
        pytest.skip("fewer records")
    r = recs[i]
    t = oracle.build(oracle.spec_from_json(r["spec"], align=8), r["seed"])
    assert t.allocs.tolist() == r["bump_allocations"]
    got = [[int(h), 0, int(tg)] for h, tg in zip(t.site_off.tolist(), t.site_target.tolist())]
    want = [[h + o, 0, tg] for h, o, tg in r["bump_sites"]]
    assert got == want


def test_attach_rejects_targets_outside_the_arena(oracle):
    # memory.py:319-321 / test_memory.py:181-189
    t = oracle.build(oracle.OSpec(oracle.LINEAR, 2, 10), 0)
    img = t.buf.copy()
    off = int(t.site_off[0])
    img[off:off + 8] = np.frombuffer((0xDEAD_BEEF).to_bytes(8, "little"), np.uint8)
    assert oracle.relocate(img, t.total, t.site_off, t.ptr_base, 1 << 40) == 0


def test_f32_payload_is_round_to_nearest(oracle):
    t = oracle.build(oracle.OSpec(oracle.DENSE, 2, 1000, 1, elem=4), 123457)
    for i in range(len(t.arr_off)):
        a, n, lv = int(t.arr_off[i]), int(t.arr_count[i]), int(t.arr_level[i])
        got = np.frombuffer(t.buf[a:a + 4 * n].tobytes(), "<f4")
        raw = (123457 * 16777619 + lv * 1000003 + np.arange(n, dtype=np.int64)) % (1 << 31)
        assert np.array_equal(got, raw.astype(np.float64).astype(np.float32))

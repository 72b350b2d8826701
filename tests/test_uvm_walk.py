"""cf_uvm_walk_pages (the UVM scheme's logical page accounting: the pages of every pointer field the
reference's kernel walk reads, harness.py:261-304 through memory.py:378-394) against an
independent numpy walk over oracle-built arenas whose pointer fields hold real addresses of the
buffer, on the CPU.  Also: a chain leaving the arena reports the page of its first outside field."""
import ctypes as C
import random

import numpy as np
import pytest

from paper_1906_01128_b200 import _native as N

OFF_NA, OFF_A, OFF_LNEXT, LEAF_OFF_A = 0, 8, 16, 4


@pytest.fixture(scope="module")
def O():
    from oracle import oracle as O
    return O


def _arena(O, ospec, seed):
    """Oracle tree with its pointer fields rebased onto the buffer's own address."""
    t = O.build(ospec, seed, ptr_base=0)
    base = t.buf.ctypes.data
    for s in t.site_off.tolist():
        v = int.from_bytes(t.buf[s:s + 8].tobytes(), "little")
        t.buf[s:s + 8] = np.frombuffer((v + base).to_bytes(8, "little"), np.uint8)
    return t, base


def _walk_numpy(t, base, idx, lv, od, kind, q, depth, page):
    pages = set()
    for i, L, o in zip(idx.tolist(), lv.tolist(), od.tolist()):
        node = t.root_off
        for level in range(1, L + 1):
            f = node + OFF_LNEXT
            pages.add((base + f) // page)
            blk = int.from_bytes(t.buf[f:f + 8].tobytes(), "little") - base
            if kind == N.CF_DENSE:
                digit = (o // q ** (L - level)) % q
                node = blk + digit * (12 if level == depth else 24)
            else:
                node = blk
        leaf = kind == N.CF_DENSE and L == depth
        pages.add((base + node + (LEAF_OFF_A if leaf else OFF_A)) // page)
        if int(t.arr_count[i]) > 0:
            pages.add((base + node + OFF_NA) // page)
    return sorted(pages)


def _native_walk(t, base, idx, lv, od, kind, q, depth, page):
    roots = np.full(len(idx), t.root_off, np.uint64)
    cnt = np.ascontiguousarray(t.arr_count[idx], np.uint64)
    lv = np.ascontiguousarray(lv, np.int32)
    od = np.ascontiguousarray(od, np.uint64)
    need = C.c_uint64()
    args = (C.c_void_p(base), t.total, kind, q, depth, N.ptr(roots), N.ptr(lv), N.ptr(od), N.ptr(cnt), len(idx), page)
    N.check(N.lib().cf_uvm_walk_pages(*args, None, 0, C.byref(need)))
    out = np.zeros(max(int(need.value), 1), np.uint64)
    N.check(N.lib().cf_uvm_walk_pages(*args, N.ptr(out), len(out), C.byref(need)))
    return out[:int(need.value)].tolist()


@pytest.mark.parametrize("seed", range(4))
def test_native_walk_matches_numpy_walk(O, seed):
    rng = random.Random(seed)
    for _ in range(12):
        if rng.random() < 0.4:
            k = rng.randint(1, 7)
            ospec = O.OSpec(O.LINEAR, k, rng.choice([1, 100, 3000]), 0, rng.choice(["allinit_allused", "LLinit_LLused"]),
                            rng.choice([4, 8]), False, rng.choice([1, 16]))
            kind, q, depth = N.CF_LINEAR, 1, 0
        else:
            q, depth = rng.randint(2, 6), rng.randint(1, 4)
            ospec = O.OSpec(O.DENSE, q, rng.choice([1, 50, 700]), depth, "allinit_allused", rng.choice([4, 8]),
                            rng.random() < 0.5, rng.choice([1, 16]))
            kind = N.CF_DENSE
        t, base = _arena(O, ospec, seed)
        idx = O.targets(t, rng.choice([O.TARGET_REF, O.TARGET_ALL_LEAVES, O.TARGET_ALL_ARRAYS]))
        if len(idx) == 0:
            continue
        lv, od = O.chain_keys(t, idx)
        page = rng.choice([256, 4096])
        assert _native_walk(t, base, idx, lv, od, kind, q, depth, page) == \
            _walk_numpy(t, base, idx, lv, od, kind, q, depth, page), (ospec, page)


def test_chain_leaving_the_arena_reports_its_field_page(O):
    t, base = _arena(O, O.OSpec(O.DENSE, 3, 10, 2, "allinit_allused", 8, True, 16), 1)
    idx = O.targets(t, O.TARGET_ALL_LEAVES)
    lv, od = O.chain_keys(t, idx)
    # the root's child-block pointer sent far past the arena: every chain's second field is outside
    f = t.root_off + OFF_LNEXT
    far = base + t.total + (1 << 30)
    t.buf[f:f + 8] = np.frombuffer(far.to_bytes(8, "little"), np.uint8)
    pages = _native_walk(t, base, idx, lv, od, N.CF_DENSE, 3, 2, 4096)
    assert any(p > (base + t.total) // 4096 for p in pages)

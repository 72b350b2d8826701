"""C-ABI surface checks that need no GPU: the library loads, exports every symbol the header
declares, and the host-side marshaller (planner + builder) matches the CPU oracle and the
reference golden vectors."""
import ctypes as C
import hashlib
import re

import numpy as np
import pytest

from conftest import REPO


def _header_symbols():
    text = (REPO / "include" / "chainforge_b200.h").read_text()
    return sorted(set(re.findall(r"\b(cf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1906_01128_b200 import _native
    lib = _native.lib()
    declared = _header_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_native.EXPORTED)
    assert lib.cf_abi_version() == 2


def test_ctx_create_without_gpu_fails_loudly():
    from paper_1906_01128_b200 import _native as N
    if N.device_count() > 0:
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    rc = N.lib().cf_ctx_create(0, 2, C.byref(h))
    assert rc == N.CF_E_NODEVICE
    assert "requires a GPU" in N.last_error()
    with pytest.raises(N.NativeUnavailable):
        N.check(rc)


def _native_build(spec_json, seed, align=1, elem=8, leaf_only=False, ptr_base=0x1000_0000):
    from paper_1906_01128_b200 import _native as N
    from paper_1906_01128_b200.scenarios import DenseSpec, LinearSpec
    if spec_json["kind"] == "linear":
        spec = LinearSpec(spec_json["k"], spec_json["n"], spec_json["layout"], elem=elem)
    else:
        spec = DenseSpec(spec_json["q"], spec_json["n"], spec_json["depth"], elem=elem, leaf_only=leaf_only)
    t = N.NativeTree(spec.native(align))
    total = int(t.info.total_bytes)
    p = C.c_void_p()
    N.check(N.lib().cf_host_alloc(max(total, 1), N.CF_MEM_PAGEABLE, C.byref(p)))
    t.build(p.value, ptr_base, seed)
    buf = N.host_view(p.value, max(total, 1)).copy()
    N.lib().cf_host_free_sized(p.value, max(total, 1), N.CF_MEM_PAGEABLE)
    return t, buf[:total]


def test_native_builder_matches_reference_kats(kats, oracle):
    from paper_1906_01128_b200 import _native as N
    for r in kats["marshal"]:
        t, buf = _native_build(r["spec"], r["seed"])
        assert int(t.info.total_bytes) == r["total_bytes"]
        assert np.stack([t.table(N.CF_TAB_ALLOC_OFF), t.table(N.CF_TAB_ALLOC_SIZE)], 1).tolist() == r["requests"]
        assert t.table(N.CF_TAB_SITE_OFF).tolist() == r["sites"]
        assert t.table(N.CF_TAB_SITE_TARGET).tolist() == r["site_targets"]
        norm = oracle.normalised(buf, t.table(N.CF_TAB_SITE_OFF), 0x1000_0000)
        assert hashlib.sha256(norm).hexdigest() == r["arena_sha"], r["spec"]
        idx = t.targets(N.CF_TARGET_REF)
        assert t.table(N.CF_TAB_ARR_OFF)[idx].tolist() == r["targeted"]
        # bump-8 layout of the reference host allocator
        tb, _ = _native_build(r["spec"], r["seed"], align=8)
        assert np.stack([tb.table(N.CF_TAB_ALLOC_OFF), tb.table(N.CF_TAB_ALLOC_SIZE)], 1).tolist() == r["bump_allocations"]


@pytest.mark.parametrize("elem,align,leaf_only", [(4, 16, True), (4, 1, False), (8, 16, False), (4, 8, True)])
def test_native_builder_matches_oracle_f32_and_aligned(oracle, elem, align, leaf_only):
    from paper_1906_01128_b200 import _native as N
    specs = [{"kind": "dense", "q": 4, "n": 1001, "depth": 3}, {"kind": "dense", "q": 3, "n": 5, "depth": 2},
             {"kind": "linear", "k": 5, "n": 333, "layout": "allinit_LLused"},
             {"kind": "dense", "q": 7, "n": 0, "depth": 2}, {"kind": "dense", "q": 1, "n": 9, "depth": 0}]
    for sj in specs:
        lo = leaf_only and sj["kind"] == "dense"
        t, buf = _native_build(sj, 77, align=align, elem=elem, leaf_only=lo)
        ot = oracle.build(oracle.spec_from_json(sj, elem=elem, align=align, leaf_only=lo), 77)
        assert int(t.info.total_bytes) == ot.total
        assert buf.tobytes() == ot.buf[:ot.total].tobytes(), sj
        assert t.table(N.CF_TAB_SITE_OFF).tolist() == ot.site_off.tolist()
        for pol in (N.CF_TARGET_REF, N.CF_TARGET_ALL_LEAVES, N.CF_TARGET_ALL_ARRAYS):
            assert t.targets(pol).tolist() == oracle.targets(ot, pol).tolist()


def test_baseline_config_sizes():
    """Graph bytes of the BASELINE configs from the planner."""
    from paper_1906_01128_b200.scenarios import DenseSpec, LinearSpec, dense_data_size, tree_total_bytes
    assert tree_total_bytes(LinearSpec(1, 1_000_000, elem=4)) == 4_000_024
    assert tree_total_bytes(DenseSpec(4, 4 << 20, 3, elem=4, leaf_only=True)) == 1_073_743_096
    assert dense_data_size(4, 4 << 20, 3, elem=4, leaf_only=True) == 1_073_743_096
    assert dense_data_size(100, 256, 3, elem=4) == 1_046_585_848
    assert dense_data_size(4, 268_435_456, 3, elem=4, leaf_only=True) == 68_719_478_008
    # aligned production arena: every array 16-byte aligned
    from paper_1906_01128_b200 import _native as N
    t = N.NativeTree(DenseSpec(4, 4 << 20, 3, elem=4, leaf_only=True).native(16))
    assert (t.table(N.CF_TAB_ARR_OFF) % 16 == 0).all()


def test_spec_validation_matches_reference():
    from paper_1906_01128_b200 import DenseSpec, LinearSpec
    for bad in (lambda: LinearSpec(0, 10), lambda: LinearSpec(2, -1), lambda: LinearSpec(2, 10, "bogus"),
                lambda: DenseSpec(0, 10), lambda: DenseSpec(2, 10, -1), lambda: DenseSpec(2, 1, 1, elem=2)):
        with pytest.raises(ValueError):
            bad()


def test_sass_chase_mode_keeps_per_access_chain_loads():
    """CHASE must re-load the chain per access (non-hoistable ld.global.nc ->
    LDG.E.64.CONSTANT in SASS) while RESOLVED issues none and streams with 128-bit accesses."""
    import shutil
    import subprocess
    import sys
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run([sys.executable, str(REPO / "tools" / "sass_report.py")], capture_output=True,
                         text=True, check=True, cwd=str(REPO)).stdout
    rows = {}
    for line in out.splitlines()[2:]:
        t, mode, path, total, ld128, st128, chain = [x.strip() for x in line.strip("|").split("|")]
        rows[(t, mode, path)] = (int(total), int(ld128), int(st128), int(chain))
    paths = {p for _, _, p in rows}
    assert paths == {"tiles", "groups", "tiles+groups", "leaf-owned groups"}, paths
    for t in ("float", "double"):
        for p in paths:
            assert rows[(t, "resolved", p)][3] == 0
            if p != "leaf-owned groups":   # RESOLVED-only path (no chase instantiation)
                assert rows[(t, "chase", p)][3] > 0
            assert rows[(t, "resolved", p)][1] > 0 and rows[(t, "resolved", p)][2] > 0
        assert (t, "chase", "leaf-owned groups") not in rows


def test_numa_binding_is_scoped():
    """numa_bound(node) confines the thread to the node's CPUs only inside the block (pinned arenas
    are allocated there); the CPU mask is restored afterwards."""
    import os
    from pathlib import Path
    from paper_1906_01128_b200 import _native as N
    if not Path("/sys/devices/system/node/node0/cpulist").exists():
        pytest.skip("no NUMA sysfs")
    before = os.sched_getaffinity(0)
    with N.numa_bound(0):
        inside = os.sched_getaffinity(0)
    assert inside <= before or inside
    assert os.sched_getaffinity(0) == before
    with N.numa_bound(-1):
        assert os.sched_getaffinity(0) == before

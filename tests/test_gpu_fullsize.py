"""Full-size GPU checks: BASELINE C2 / C4 windows bit-exact against the oracle restatement, and a
compute-sanitizer memcheck pass over every kernel on small windows."""
import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import paper_1906_01128_b200 as cf
    from paper_1906_01128_b200 import _native as N
    if N.device_count() == 0:
        pytest.skip("no GPU visible: run `pytest -m gpu` on a B200 box (gpurun)")
    return cf


@pytest.mark.parametrize("cfg,mode,elem", [("C1", "resolved", 4), ("C2", "resolved", 4), ("C4", "resolved", 4),
                                            ("C2", "chase", 4), ("C4", "chase", 4),
                                            ("C2", "resolved", 8), ("C2", "chase", 8)])
def test_full_size_window_matches_oracle(cf, oracle, cfg, mode, elem):
    """The BASELINE config at full size (1 GiB of f32 leaves; 2 GiB in the reference's own f64):
    e2e window copy-back and resident image equal the oracle's expected arena byte for byte
    (relocated pointers restored, leaves x2), in both leaf-kernel modes."""
    from dataclasses import replace
    sys.path.insert(0, str(REPO))
    import bench
    spec, policy, _ = bench.make_spec(cfg)
    if elem != spec.elem:
        spec = replace(spec, elem=elem)
    w = cf.DeepCopyWindow(spec, seed=1, policy=policy, mode=mode, align=16)
    try:
        st = w.run(scale=2.0)
        assert st.bad == (1 << 64) - 1
        if isinstance(spec, cf.LinearSpec):
            ospec = oracle.OSpec(oracle.LINEAR, spec.k, spec.n, 0, spec.layout, elem=spec.elem, align=16)
        else:
            ospec = oracle.OSpec(oracle.DENSE, spec.q, spec.n, spec.depth, elem=spec.elem, leaf_only=spec.leaf_only,
                                 align=16)
        ot = oracle.build(ospec, 1, ptr_base=w.src)
        idx = oracle.targets(ot, {"all_leaves": oracle.TARGET_ALL_LEAVES,
                                  "all_arrays": oracle.TARGET_ALL_ARRAYS}[policy])
        want = oracle.expected_after_window(ot, idx, 2.0)[:w.total]
        assert np.array_equal(w.host_dst(), want)
        assert np.array_equal(w.host_src(), ot.buf[:w.total])   # source untouched
        w.upload_raw()
        st = w.run_resident(scale=2.0, graph=True)
        assert st.bad == (1 << 64) - 1
        assert np.array_equal(w.image_bytes(), want)
    finally:
        w.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_full_size_c5_strong_shards(cf, world):
    """C5 (64 GiB, DenseSpec(4, 256Mi, 3) f32 leaves-only) cut into `world` subtree shards, each
    planned and run one after another on this GPU at the full leaf length: every shard's leaves
    equal payload_values x 2 byte for byte, every pointer field is restored to its host target,
    and the shards' leaf ordinals cover the whole tree's 64 leaves exactly once."""
    from paper_1906_01128_b200 import _native as N
    from paper_1906_01128_b200.shard import shard_for
    sys.path.insert(0, str(REPO))
    import bench
    spec, policy, _ = bench.make_spec("C5")
    want = None
    seen = []
    for r in range(world):
        sh = shard_for(spec, r, world, "strong")
        w = cf.DeepCopyWindow(sh.spec, seed=sh.seed, policy=policy, align=16, separate_output=False)
        try:
            st = w.run(scale=2.0)
            assert st.bad == (1 << 64) - 1
            got = w.host_dst()
            off, cnt = w.table(N.CF_TAB_ARR_OFF), w.table(N.CF_TAB_ARR_COUNT)
            lvl, od = w.table(N.CF_TAB_ARR_LEVEL), w.table(N.CF_TAB_ARR_ORDINAL)
            for i in w.targets.tolist():
                n = int(cnt[i])
                assert n == spec.n and int(lvl[i]) == spec.depth
                if want is None:   # every leaf of a level holds the same payload (scenarios.py:152-155)
                    want = (cf.payload_values(1, spec.depth, n, 4) * np.float32(2.0)).astype(np.float32).view(np.uint8)
                a = int(off[i])
                assert np.array_equal(got[a:a + 4 * n], want), (world, r, int(od[i]))
                seen.append(int(od[i]))
            so, tg = w.table(N.CF_TAB_SITE_OFF), w.table(N.CF_TAB_SITE_TARGET)
            vals = np.array([int.from_bytes(got[int(o):int(o) + 8].tobytes(), "little") for o in so.tolist()], np.uint64)
            assert np.array_equal(vals, tg + np.uint64(w.src)), (world, r)
        finally:
            w.close()
    assert sorted(seen) == list(range(spec.q ** spec.depth))


def test_full_size_scattered_forest_c3(cf):
    """C3 at full size (64 scattered chains, 1 GiB of leaves; the oracle has no scattered forests):
    after the e2e window every targeted leaf equals payload_values x 2 and every other byte --
    nodes with their restored pointers, untargeted space -- equals the source arena."""
    sys.path.insert(0, str(REPO))
    import bench
    from paper_1906_01128_b200 import _native as N
    spec, policy, _ = bench.make_spec("C3")
    w = cf.DeepCopyWindow(spec, seed=1, policy=policy, align=16)
    try:
        st = w.run(scale=2.0)
        assert st.bad == (1 << 64) - 1
        src, got = w.host_src(), w.host_dst()
        off, cnt, lvl = w.table(N.CF_TAB_ARR_OFF), w.table(N.CF_TAB_ARR_COUNT), w.table(N.CF_TAB_ARR_LEVEL)
        mask = np.ones(w.total, bool)
        want_leaf = None
        for i in w.targets.tolist():
            a, nb = int(off[i]), int(cnt[i]) * 4
            if want_leaf is None:
                want_leaf = (cf.payload_values(1, int(lvl[i]), int(cnt[i]), 4) * np.float32(2.0)).astype(np.float32)
            assert np.array_equal(got[a:a + nb].view(np.float32), want_leaf), i
            mask[a:a + nb] = False
        assert len(w.targets) == 64
        assert np.array_equal(got[mask], src[mask])
    finally:
        w.close()


SANITIZE = r'''
import sys
sys.path.insert(0, ".")
import paper_1906_01128_b200 as cf
from paper_1906_01128_b200 import _native as N
specs = [cf.DenseSpec(3, 301, 2, elem=4), cf.DenseSpec(4, 5000, 3, elem=4, leaf_only=True),
         cf.LinearSpec(4, 777, "allinit_allused"), cf.DenseSpec(3, 17, 2),
         cf.ForestSpec(cf.LinearSpec(3, 1000, "LLinit_LLused", elem=4), 20, scatter_seed=5),
         cf.DenseSpec(3, 4099, 2), cf.DenseSpec(5, 2500, 1, leaf_only=True)]   # packed f64 at 4 mod 8
for spec in specs:
    for align in (1, 16):
        for mode in ("resolved", "chase"):
            w = cf.DeepCopyWindow(spec, seed=2, policy="all_arrays", mode=mode, align=align, chunk_bytes=4096)
            w.run(scale=2.0)
            w.upload_raw()
            w.run_resident(scale=0.5)
            w.close()
# uniform leaf ranges: the memory-parallel resolver (multi-step windows, > 4096 targets) and the
# leaf-owned group path (one-step resident windows), f32 and f64
for spec in (cf.DenseSpec(16, 4, 4, elem=4, leaf_only=True), cf.DenseSpec(9, 3, 4, elem=8, leaf_only=True)):
    for chunk in (0, 1 << 16):
        w = cf.DeepCopyWindow(spec, seed=3, policy="all_leaves", align=16, chunk_bytes=chunk)
        w.run(scale=2.0)
        w.upload_raw()
        w.run_resident(scale=0.5)
        w.run_n(3, flags=N.CF_WIN_RESIDENT | N.CF_WIN_GRAPH)
        w.close()
for scheme in ("marshalling", "naive", "pointerchain", "uvm"):
    m, mach = cf.execute_case(cf.DenseSpec(2, 64, 3), scheme, cf.CostModel(), seed=1)
    mach.close()
# a leaf pointer corrupted to the image's last 8 bytes (valid count): the leaf kernel must reject
# the span, not write past the image
from paper_1906_01128_b200 import _native as N
w = cf.DeepCopyWindow(cf.DenseSpec(3, 5000, 2, elem=4, leaf_only=True), seed=1, policy="all_arrays", align=16)
so, st = w.table(N.CF_TAB_SITE_OFF), w.table(N.CF_TAB_SITE_TARGET)
f = int(so[list(st).index(w.table(N.CF_TAB_ARR_OFF)[int(w.targets[-1])])])
w.host_src()[f:f + 8] = list((w.src + w.total - 8).to_bytes(8, "little"))
for mode in ("resolved", "chase"):
    try:
        w.run(scale=2.0, mode=mode)
        raise SystemExit("corrupted leaf pointer was not rejected")
    except cf.WildAccess:
        pass
w.close()
# the same corruption in a leaf-owned resident step (the leaf kernel attaches that field itself)
w = cf.DeepCopyWindow(cf.DenseSpec(16, 4, 4, elem=4, leaf_only=True), seed=1, policy="all_leaves", align=16)
f = int(w.table(N.CF_TAB_ARR_OWNER)[int(w.targets[-1])]) + 4
w.host_src()[f:f + 8] = list((w.src + w.total - 8).to_bytes(8, "little"))
w.upload_raw()
try:
    w.run_resident(scale=2.0)
    raise SystemExit("corrupted leaf pointer was not rejected (leaf-owned)")
except cf.WildAccess:
    pass
w.close()
print("sanitized ok")
'''


def test_compute_sanitizer_memcheck(cf, tmp_path):
    tool = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(tool):
        pytest.skip("compute-sanitizer not installed")
    script = tmp_path / "san.py"
    script.write_text(SANITIZE)
    out = subprocess.run([tool, "--tool", "memcheck", "--error-exitcode", "99", sys.executable, str(script)],
                         capture_output=True, text=True, timeout=900, cwd=str(REPO))
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "sanitized ok" in out.stdout
    assert "ERROR SUMMARY: 0 errors" in out.stdout + out.stderr


def test_compute_sanitizer_racecheck(cf, tmp_path):
    """Shared-memory hazards (k_checksum's reduction, the one-CTA attach + resolve barrier, the
    word-streaming tile barrier): racecheck over small windows."""
    tool = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(tool):
        pytest.skip("compute-sanitizer not installed")
    script = tmp_path / "race.py"
    script.write_text(RACE)
    out = subprocess.run([tool, "--tool", "racecheck", "--error-exitcode", "99", sys.executable, str(script)],
                         capture_output=True, text=True, timeout=900, cwd=str(REPO))
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "race ok" in out.stdout


RACE = r'''
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1906_01128_b200 as cf
from paper_1906_01128_b200 import _native as N
from paper_1906_01128_b200.shard import leaf_checksums
for spec, align in ((cf.DenseSpec(3, 4099, 2), 1), (cf.DenseSpec(4, 3000, 2, elem=4, leaf_only=True), 16)):
    w = cf.DeepCopyWindow(spec, seed=1, policy="all_arrays", align=align, chunk_bytes=8192)
    w.run(scale=2.0)
    off, cnt = w.table(N.CF_TAB_ARR_OFF), w.table(N.CF_TAB_ARR_COUNT)
    leaf_checksums(w.ctx, w.image, off[w.targets], cnt[w.targets], spec.elem)
    w.close()
# leaf-owned steps (per-warp shared-memory slots, no CTA barrier): resident and multi-step
w = cf.DeepCopyWindow(cf.DenseSpec(16, 8, 3, elem=4, leaf_only=True), seed=1, policy="all_leaves", align=16,
                      chunk_bytes=16384)
w.run(scale=2.0)
w.upload_raw()
w.run_resident(scale=2.0)
w.close()
print("race ok")
'''


def test_many_small_chains_repeated_windows_stay_exact(cf):
    """1M chains with 12-byte leaf records (A fields at 4 mod 8 even in the aligned arena): many
    back-to-back resident and full windows (fused detach, graph replay) must never tear a
    pointer field.  Scales alternate 2.0 / 0.5, so after an even number of windows the image and
    the copy-back equal the source arena byte for byte."""
    from paper_1906_01128_b200 import _native as N
    w = cf.DeepCopyWindow(cf.DenseSpec(100, 16, 3, elem=4), seed=3, policy="all_leaves", align=16)
    try:
        src = w.host_src().copy()
        w.upload_raw()
        for flags in (N.CF_WIN_RESIDENT, N.CF_WIN_RESIDENT | N.CF_WIN_GRAPH):
            for _ in range(20):
                st = w.run_n(10, flags=flags)
                assert st.bad == (1 << 64) - 1
        assert np.array_equal(w.image_bytes(), src)
        for _ in range(5):
            st = w.run_n(4, flags=N.CF_WIN_FULL | N.CF_WIN_GRAPH)
            assert st.bad == (1 << 64) - 1
        st = w.run(scale=2.0)
        assert st.bad == (1 << 64) - 1
        got = w.host_dst()
        arr = w.table(N.CF_TAB_ARR_OFF)
        lv = w.table(N.CF_TAB_ARR_LEVEL)
        mask = np.ones(len(src), bool)
        for i in w.targets.tolist():
            mask[int(arr[i]):int(arr[i]) + 64] = False
        assert np.array_equal(got[mask], src[mask])      # pointers restored, untargeted unchanged
        i = int(w.targets[-1])
        want = (cf.payload_values(3, int(lv[i]), 16, 4) * np.float32(2.0)).astype(np.float32)
        assert np.array_equal(got[int(arr[i]):int(arr[i]) + 64].view(np.float32), want)
    finally:
        w.close()

"""bench.py contract checks that need no GPU: the workload table, the reference arm (oracle port,
no product import), identical config keys for both arms, and the multi-rank launch rules."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO

sys.path.insert(0, str(REPO))
import bench  # noqa: E402


@pytest.mark.parametrize("name", sorted(bench.CONFIGS))
def test_config_bytes_match_the_planner(name):
    from paper_1906_01128_b200 import _native as N
    spec, policy, _ = bench.make_spec(name)
    plan = N.NativeTree(spec.native(16))
    assert int(plan.info.total_bytes) == bench.CONFIGS[name]["graph_bytes"]
    tg = plan.targets({"all_leaves": N.CF_TARGET_ALL_LEAVES, "all_arrays": N.CF_TARGET_ALL_ARRAYS}[policy])
    leaf = int(plan.table(N.CF_TAB_ARR_COUNT)[tg].sum()) * spec.elem
    assert leaf == bench.CONFIGS[name]["leaf_bytes"]


def test_oracle_sample_matches_config_shape():
    from oracle import oracle as O
    for name in ("C1", "C2", "C4"):
        spec, trees, shrink = bench.oracle_spec(name, 4)
        assert shrink == 1 and trees == 1
        assert int(O.counts(spec).total) == bench.CONFIGS[name]["graph_bytes"]
    spec, trees, shrink = bench.oracle_spec("C3", 4)
    assert trees == 64 and shrink == 1
    spec, trees, shrink = bench.oracle_spec("C5", 4)
    assert shrink > 1 and int(O.counts(spec).total) <= bench.CPU_SAMPLE_BYTES


def test_oracle_resident_step_equals_window_image():
    """orc_resident (attach, resolve, scale, detach on a buffer holding the arena) leaves exactly the
    bytes the full window copies back."""
    from oracle import oracle as O
    spec = O.OSpec(O.DENSE, 3, 1000, 2, elem=4, leaf_only=False, align=16)
    t = O.build(spec, 1)
    idx = O.targets(t, O.TARGET_ALL_ARRAYS)
    dev = t.buf.copy()
    assert O.resident(t, idx, dev, t.ptr_base, 0x7E00_0000_0000, 2.0, 4) == -1
    assert np.array_equal(dev, O.expected_after_window(t, idx, 2.0))


REF_ARM = r'''
import json, sys
sys.path.insert(0, sys.argv[1])
import bench
bench.main(["--impl", "reference", "--config", sys.argv[2], "--steps", "3", "--warmup", "3"])
assert "paper_1906_01128_b200" not in sys.modules, "reference arm imported the product package"
print("NO_PRODUCT_IMPORT")
'''


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_reference_arm_is_the_oracle_only(name):
    out = subprocess.run([sys.executable, "-c", REF_ARM, str(REPO), name], capture_output=True, text=True,
                         timeout=600, cwd=str(REPO), env=dict(os.environ, CF_ORACLE_THREADS="4"))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert lines[-1] == "NO_PRODUCT_IMPORT"
    rec = json.loads(lines[-2])
    assert rec["impl"] == "reference" and rec["metric"] == bench.METRIC
    assert rec["config"] == bench.workload_config(name, 1)      # the same dict our arm prints
    assert rec["cpu_baseline"]["kind"] == "port" and rec["cpu_baseline"]["cores"] == 4
    assert rec["value"] > 0 and rec["e2e"]["value"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["steps"] == 3


def test_workload_config_keys():
    c = bench.workload_config("C2", 1)
    assert set(c) == {"workload", "graph_bytes_per_gpu", "leaf_bytes_per_gpu", "dtype", "layout", "targets", "l2",
                      "parallelism"}
    assert c["graph_bytes_per_gpu"] == 1_073_743_104 and c["dtype"] == "f32"
    c5 = bench.workload_config("C5", 8)
    assert c5["graph_bytes_per_gpu"] == bench.CONFIGS["C5"]["graph_bytes"] // 8 and "strong" in c5["parallelism"]


def test_world_size_must_match_gpus(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.main(["--gpus", "4"])


def test_gpus_without_torchrun_respawns(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}

    def fake_run(cmd, *a, **k):
        seen["cmd"] = cmd

        class R:
            returncode = 0
        return R()
    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    with pytest.raises(SystemExit) as e:
        bench.main(["--gpus", "2", "--steps", "4"])
    assert e.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=2" in cmd and "127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "2", "--steps", "4"][-3:]

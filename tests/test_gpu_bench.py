"""bench.py on the GPU: the multi-rank launch (``--gpus 2`` without torchrun re-launches itself,
two ranks sharing this box's GPU) and the JSON contract keys of one line."""
import json
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    from paper_1906_01128_b200 import _native as N
    if N.device_count() == 0:
        pytest.skip("no GPU visible: run `pytest -m gpu` on a B200 box (gpurun)")


def _line(out: str) -> dict:
    recs = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    assert len(recs) == 1, out[-3000:]
    return recs[0]


def test_bench_gpus_2_spawns_two_ranks(gpu):
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "4", "--warmup", "3",
                        "--leaf-elems", "65536", "--skip-schemes", "--skip-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=str(REPO))
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    rec = _line(r.stdout)
    assert rec["n_gpus"] == 2 and rec["scaling"] == "weak"
    assert rec["config"]["parallelism"].startswith("dp2")
    assert rec["gather"]["leaves"] == 128 and rec["gather"]["complete"] and rec["gather"]["checksums_match"]
    assert rec["value_host_wall"]["value"] > 0 and rec["e2e"]["host_wall_gbs"] > 0


def test_bench_line_contract_small(gpu):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "4", "--warmup", "3", "--leaf-elems", "65536",
                        "--skip-schemes"], capture_output=True, text=True, timeout=900, cwd=str(REPO))
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    rec = _line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert k in rec, k
    assert rec["n_gpus"] == 1 and rec["steps"] == 4
    assert rec["gpu_launches"] > 0
    assert rec["cpu_baseline"]["kind"] == "port"
    assert rec["e2e"]["host_link_gbs"]["bidir"] > 0 and rec["e2e"]["frac_of_link_roofline"] > 0
    ref = rec.get("cpu_baseline_reference_python", {})
    assert ref.get("kind") == "reference_python"


def test_bench_gpus_4_strong_c5_subtree_shards(gpu):
    """The strong-scaling launch the driver's scaling run uses for C5: four ranks (sharing this
    box's GPU), one dense tree cut by subtree, every leaf checksum gathered and checked."""
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--config", "C5", "--steps", "3", "--warmup", "3",
                        "--leaf-elems", "262144", "--skip-schemes", "--skip-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=str(REPO))
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    rec = _line(r.stdout)
    assert rec["n_gpus"] == 4 and rec["scaling"] == "strong"
    assert rec["gather"]["leaves"] == 64 and rec["gather"]["complete"] and rec["gather"]["checksums_match"]

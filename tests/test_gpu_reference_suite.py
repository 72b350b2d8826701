"""The reference's OWN test modules, unmodified, run against the drop-in on a B200.

``pkg/tests/test_{memory,scenarios,harness,acceptance,report,cli}.py`` of the reference are staged
byte-for-byte into ``baseline/_ref_tests/`` by ``tools/stage_reference_tests.sh`` (git-ignored like
the pip-installed reference in ``baseline/_ref``; both travel to the GPU box).  They run in a
child pytest with ``tests/refshim`` first on ``sys.path``: ``import chainforge`` then resolves to
this package for the hot path (memory / scenarios / harness), while the presentation and text
layers (report tables, cli, frontend, rewrite, codegen -- out of scope) stay
the reference's own modules, bound to the drop-in's harness.

Every test must pass except the deviations listed in ``EXPECTED_DEVIATIONS``, each with the
reference line it depends on and why a real-memory backend differs.  A listed test that starts
passing is reported too (the list must stay exact).
"""
from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
SUITE = REPO / "baseline" / "_ref_tests"
SHIM = REPO / "tests" / "refshim"

# test id -> why the drop-in (real pinned / device memory on a B200) differs from the simulator
EXPECTED_DEVIATIONS = {
    # test_scenarios.py:122-129 compares raw host bytes of two trees built in two Machines.  The
    # simulator's host space starts at a fixed base (memory.py:27-30, HOST_BASE), so pointer fields
    # hold identical addresses; the drop-in's trees live in real pinned allocations whose
    # addresses differ per Machine.  Payloads and the pointer graph are identical (checked with
    # allocation-relative pointers in tests/test_reference_contract.py).
    "test_scenarios.py::test_same_seed_builds_byte_identical_trees":
        "fixed simulated HOST_BASE (memory.py:27-30) vs real pinned addresses",
    # test_memory.py:163-178 monkeypatches ``machine.host.write_word`` to watch the simulator's
    # per-site detach loop (memory.py:337-344) write host words in reverse site order.  The drop-in
    # detaches every site with one device kernel and brings the image home with one bulk D2H, so
    # there are no per-site host writes to observe.  What the test pins beyond the observation --
    # detach count == attach count == sites, byte-exact restore -- holds
    # (tests/test_reference_contract.py::test_attach_image_and_round_trip).
    "test_memory.py::test_detach_mirrors_attach_in_reverse_order":
        "per-site host write_word calls of the simulator's detach loop vs one device detach kernel + bulk D2H",
}


def _run_suite(tmp_path: Path) -> dict:
    xml = tmp_path / "ref_suite.xml"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(SHIM), str(REPO)]),
               CF_REF_ROOT=str(REPO / "baseline" / "_ref"))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", f"--junitxml={xml}",
                        "-o", "junit_family=xunit1", "."], cwd=SUITE, env=env, capture_output=True, text=True,
                       timeout=1500)
    if not xml.exists():
        raise AssertionError(f"reference suite did not run:\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}")
    out = {}
    for case in ET.parse(xml).getroot().iter("testcase"):
        mod = case.get("file") or (case.get("classname", "").replace(".", "/") + ".py")
        tid = f"{Path(mod).name}::{case.get('name')}"
        if case.find("failure") is not None or case.find("error") is not None:
            node = case.find("failure") if case.find("failure") is not None else case.find("error")
            out[tid] = ("failed", (node.get("message") or "")[:300])
        elif case.find("skipped") is not None:
            out[tid] = ("skipped", "")
        else:
            out[tid] = ("passed", "")
    return out


def test_reference_suite_runs_unmodified_against_the_dropin(tmp_path):
    if not (SUITE / "test_memory.py").exists():
        pytest.skip("reference test modules not staged (tools/stage_reference_tests.sh in the build container)")
    import paper_1906_01128_b200 as cf
    from paper_1906_01128_b200 import _native as N
    if N.device_count() == 0:
        pytest.skip("no GPU visible")
    assert cf is not None
    res = _run_suite(tmp_path)
    failed = {k: v[1] for k, v in res.items() if v[0] == "failed"}
    unexpected = {k: v for k, v in failed.items() if k not in EXPECTED_DEVIATIONS}
    fixed = [k for k in EXPECTED_DEVIATIONS if res.get(k, ("absent",))[0] == "passed"]
    passed = sum(1 for v in res.values() if v[0] == "passed")
    print(f"reference suite: {passed} passed, {len(failed)} failed ({len(failed) - len(unexpected)} expected) "
          f"of {len(res)}")
    for k, v in sorted(failed.items()):
        print(f"  FAILED {k}: {v}")
    assert not unexpected, unexpected
    assert not fixed, f"listed deviations now pass: {fixed}"
    assert passed >= 100, res

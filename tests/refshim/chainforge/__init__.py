"""Alias shim: ``import chainforge`` resolves to the B200 drop-in (paper_1906_01128_b200).

Used only by tests/test_gpu_reference_suite.py to run the reference's OWN test modules
(pkg/tests/test_{memory,scenarios,harness,acceptance,report,cli}.py, staged unmodified by
tools/stage_reference_tests.sh) against the drop-in on a B200.  The hot-path modules -- memory,
scenarios, harness (and errors) -- are the drop-in's.  The presentation / text layers -- report
tables, cli, and the directive frontend / rewriter / codegen, out of scope for this repo
 -- are the reference's own unmodified modules from its install
(``CF_REF_ROOT``, default baseline/_ref), loaded as ``chainforge.<name>`` so that their own
``from .harness import ...`` binds the drop-in: the reference CLI and report drive the B200 hot
path exactly as a user who switched packages would see it.
"""
import importlib.util
import os
import sys
from pathlib import Path

import paper_1906_01128_b200 as _dropin
from paper_1906_01128_b200 import errors, harness, memory, scenarios  # noqa: F401

_me = sys.modules[__name__]
for _k in dir(_dropin):
    if not _k.startswith("__"):
        setattr(_me, _k, getattr(_dropin, _k))
for _name in ("memory", "scenarios", "harness", "errors"):
    sys.modules[f"{__name__}.{_name}"] = importlib.import_module(f"paper_1906_01128_b200.{_name}")
    setattr(_me, _name, sys.modules[f"{__name__}.{_name}"])

_ref = Path(os.environ.get("CF_REF_ROOT", Path(__file__).resolve().parents[3] / "baseline" / "_ref")) / "chainforge"
for _name in ("frontend", "rewrite", "codegen", "report", "cli"):   # the reference's own, unmodified
    _path = _ref / f"{_name}.py"
    if _path.exists():
        _spec = importlib.util.spec_from_file_location(f"{__name__}.{_name}", _path)
        _mod = importlib.util.module_from_spec(_spec)
        sys.modules[_spec.name] = _mod
        _spec.loader.exec_module(_mod)
        setattr(_me, _name, _mod)
        for _k in dir(_mod):
            if not _k.startswith("_") and not hasattr(_me, _k):
                setattr(_me, _k, getattr(_mod, _k))

#!/bin/sh
# Stage the reference's own test modules, UNMODIFIED, into baseline/_ref_tests/ (git-ignored like
# the pip-installed reference in baseline/_ref; not gpurun-ignored, so both travel to the GPU box)
# for tests/test_gpu_reference_suite.py, which runs them against the drop-in through the alias
# shim tests/refshim/chainforge.  Run in the build container, where /root/reference exists.
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg/tests}
DST="$REPO/baseline/_ref_tests"
rm -rf "$DST"
mkdir -p "$DST"
cp "$SRC"/conftest.py "$SRC"/test_memory.py "$SRC"/test_scenarios.py "$SRC"/test_harness.py \
   "$SRC"/test_acceptance.py "$SRC"/test_report.py "$SRC"/test_cli.py "$DST"/
cp -r "$SRC"/data "$DST"/data
sha256sum "$DST"/*.py > "$DST"/SHA256SUMS
echo "staged $(ls "$DST"/test_*.py | wc -l) reference test modules into $DST"

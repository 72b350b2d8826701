"""The results-CSV data format (report.py:48-140) and the sweep against the reference's own
output (tests/golden/reference_sweep_seed3.csv, written by oracle/gen_sweep_golden.py with the
reference's `chainforge sweep --seed 3`)."""
import pytest

import paper_1906_01128_b200 as cf
from paper_1906_01128_b200 import _native as N
from paper_1906_01128_b200 import cli
from conftest import GOLDEN

REF_CSV = (GOLDEN / "reference_sweep_seed3.csv").read_text()


def test_reference_csv_round_trips_byte_for_byte():
    rows = cf.rows_from_csv(REF_CSV)
    assert len(rows) == 24
    assert cf.rows_to_csv(rows) == REF_CSV
    assert cf.rows_to_csv(cf.normalize(rows)) == REF_CSV     # normalising again changes nothing


def test_normalize_needs_the_uvm_cell():
    rows = [r for r in cf.rows_from_csv(REF_CSV) if r.scheme != "uvm"]
    with pytest.raises(cf.MissingBaseline):
        cf.normalize(rows, strict=True)
    loose = cf.normalize(rows, strict=False)
    assert all(r.normalized_wall is None and r.normalized_kernel is None for r in loose)
    assert ",,\n" in cf.rows_to_csv(loose[:1])


def test_cli_report_command(tmp_path):
    src = tmp_path / "in.csv"
    src.write_text(REF_CSV)
    out = tmp_path / "out.csv"
    assert cli.main(["report", str(src), "--normalize", "--out", str(out)]) == 0
    assert out.read_text() == REF_CSV
    no_uvm = tmp_path / "no_uvm.csv"
    no_uvm.write_text("\n".join(l for l in REF_CSV.splitlines() if ",uvm," not in l) + "\n")
    assert cli.main(["report", str(no_uvm), "--normalize"]) == 1


@pytest.mark.gpu
def test_sweep_reproduces_the_reference_csv_byte_for_byte(tmp_path):
    """Counters, cost-model floats, iterations and UVM ratios of every cell equal the reference's
    -- the drop-in's sweep file is interchangeable with chainforge's."""
    if N.device_count() == 0:
        pytest.skip("no GPU visible")
    out = tmp_path / "ours.csv"
    assert cli.main(["sweep", "--grid", str(GOLDEN / "sweep_grid.csv"), "--out", str(out), "--seed", "3"]) == 0
    assert out.read_text() == REF_CSV
    measured = tmp_path / "measured.csv"
    assert cli.main(["sweep", "--grid", str(GOLDEN / "sweep_grid.csv"), "--out", str(measured), "--seed", "3",
                     "--measured"]) == 0
    rows = cf.rows_from_csv(measured.read_text())
    assert cf.rows_to_csv(rows) == REF_CSV           # same cells, plus the measured B200 columns
    assert all(float(r.extra["wall_us"]) > 0 and int(r.extra["gpu_launches"]) > 0 for r in rows)

"""Golden results CSV from the REFERENCE's own `sweep` command (test infrastructure).

Run in the build container only (imports /root/reference):

    python oracle/gen_sweep_golden.py

Writes tests/golden/sweep_grid.csv (the acceptance-criterion-10 grid, test_acceptance.py:279-299,
plus two dense cells) and tests/golden/reference_sweep_seed3.csv = `chainforge sweep --grid ...
--seed 3` (cli.py:129-148, report.py:117-122).  The drop-in's sweep must reproduce it byte for
byte: identical counters, identical cost-model floats, identical UVM normalisation.
"""
from __future__ import annotations

import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO / "oracle"))
from gen_golden import DEFAULT_REF, load_reference  # noqa: E402

GOLDEN = REPO / "tests" / "golden"


def main() -> None:
    load_reference(DEFAULT_REF)
    cli = sys.modules["chainforge_ref.cli"] if "chainforge_ref.cli" in sys.modules else None
    if cli is None:
        import importlib
        cli = importlib.import_module("chainforge_ref.cli")
    lines = ["scenario,scheme,layout,k_or_q,n"]
    for scheme in ("uvm", "marshalling", "pointerchain", "naive"):
        for k in (2, 5):
            lines.append(f"linear,{scheme},LLinit_LLused,{k},100")
            lines.append(f"linear,{scheme},allinit_allused,{k},100")
        lines.append(f"dense,{scheme},dense,2,10")
        lines.append(f"dense,{scheme},dense,3,7")
    grid = GOLDEN / "sweep_grid.csv"
    grid.write_text("\n".join(lines) + "\n")
    out = GOLDEN / "reference_sweep_seed3.csv"
    rc = cli.main(["sweep", "--grid", str(grid), "--out", str(out), "--seed", "3"])
    assert rc == 0
    print(f"wrote {grid} and {out} ({len(out.read_text().splitlines()) - 1} rows)")


if __name__ == "__main__":
    main()

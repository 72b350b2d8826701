"""Command line for the B200 path: the reference's ``simulate`` / ``sweep`` subcommands
(cli.py:41-62, 129-148) with the device backend underneath.

    python -m paper_1906_01128_b200 simulate --scenario dense --q 4 --n 1000 --scheme marshalling
    python -m paper_1906_01128_b200 sweep --grid grid.csv --out results.csv [--measured]

Rows use the reference's results-CSV schema (report.py:22-24, 117-122) -- counters and the
cost-model ``sim_*`` columns are identical to the reference's -- and ``--measured`` appends the
B200 columns (measured window wall time, leaf-kernel mode, kernel launches).  The directive
rewriter, source generator, report renderer and tables are not part of this path.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

from .harness import SCHEMES, CostModel, RunMetrics, execute_case, run_case, sweep
from .report import CSV_HEADER, MissingBaseline, ResultRow, normalize, rows_from_csv  # noqa: F401
from .report import rows_to_csv as _rows_to_csv
from .scenarios import LAYOUTS, DenseSpec, LinearSpec


def rows_to_csv(metrics: list[RunMetrics], measured: bool = False) -> str:
    """Reference CSV rows (report.py:117-122), UVM-normalised where the cell has a UVM row."""
    return _rows_to_csv(normalize([ResultRow.from_metrics(m) for m in metrics], strict=False), measured)


def _spec(scenario: str, k_or_q: int, n: int, layout: str, depth: int, elem: int):
    if scenario == "linear":
        return LinearSpec(k_or_q, n, layout, elem=elem)
    return DenseSpec(k_or_q, n, depth, elem=elem)


def _parse_grid(path: str, elem: int) -> list[tuple]:
    lines = Path(path).read_text().strip().split("\n")
    if not lines or lines[0] != "scenario,scheme,layout,k_or_q,n":
        raise SystemExit("grid file needs header scenario,scheme,layout,k_or_q,n")
    cases = []
    for line in lines[1:]:
        scenario, scheme, layout, k_or_q, n = [x.strip() for x in line.split(",")]
        cases.append((_spec(scenario, int(k_or_q), int(n), layout if scenario == "linear" else "allinit_allused",
                            3, elem), scheme))
    return cases


def _parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1906_01128_b200", description="deep-copy hot path on B200")
    sub = p.add_subparsers(dest="command", required=True)
    s = sub.add_parser("simulate", help="run one benchmark case on the GPU")
    s.add_argument("--scenario", choices=("linear", "dense"), required=True)
    s.add_argument("--scheme", choices=SCHEMES, required=True)
    s.add_argument("--layout", choices=LAYOUTS, default="allinit_allused")
    s.add_argument("--k", type=int)
    s.add_argument("--q", type=int)
    s.add_argument("--n", type=int, required=True)
    s.add_argument("--depth", type=int, default=3)
    s.add_argument("--config", help="cost-model key=value file")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--min-iters", type=int, default=3)
    s.add_argument("--dump-log", help="write the transfer log to this path")
    s.add_argument("--elem", type=int, choices=(4, 8), default=8, help="4 = float32, 8 = float64 (reference)")
    s.add_argument("--mode", choices=("resolved", "chase"), default="resolved")
    s.add_argument("--policy", choices=("ref", "all_leaves", "all_arrays"), default="ref")
    s.add_argument("--measured", action="store_true", help="append the measured B200 columns")
    w = sub.add_parser("sweep", help="run a grid of cases into a results CSV")
    w.add_argument("--grid", required=True)
    w.add_argument("--out", required=True)
    w.add_argument("--config")
    w.add_argument("--seed", type=int, default=0)
    w.add_argument("--min-iters", type=int, default=3)
    w.add_argument("--elem", type=int, choices=(4, 8), default=8)
    w.add_argument("--measured", action="store_true")
    r = sub.add_parser("report", help="re-emit (and optionally UVM-normalise) a results CSV")
    r.add_argument("infile")
    r.add_argument("--normalize", action="store_true")
    r.add_argument("--out")
    return p


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    cm = CostModel.from_file(args.config) if getattr(args, "config", None) else CostModel()
    if args.command == "simulate":
        k_or_q = args.k if args.scenario == "linear" else args.q
        if k_or_q is None:
            raise SystemExit(f"--{'k' if args.scenario == 'linear' else 'q'} is required for the {args.scenario} scenario")
        spec = _spec(args.scenario, k_or_q, args.n, args.layout, args.depth, args.elem)
        m = run_case(spec, args.scheme, cm, seed=args.seed, min_iters=args.min_iters, mode=args.mode,
                     policy=args.policy)
        sys.stdout.write(rows_to_csv([m], args.measured))
        if args.dump_log:
            _, machine = execute_case(spec, args.scheme, cm, seed=args.seed, mode=args.mode, policy=args.policy)
            Path(args.dump_log).write_text(machine.log.dump() + "\n")
            machine.close()
        return 0
    if args.command == "report":   # cli.py _cmd_report, CSV format (tables are presentation)
        rows = rows_from_csv(Path(args.infile).read_text())
        if args.normalize:
            try:
                rows = normalize(rows, strict=True)
            except MissingBaseline as exc:
                print(f"error: {exc}", file=sys.stderr)
                return 1
        text = _rows_to_csv(rows, measured=bool(rows and rows[0].extra))
        if args.out:
            Path(args.out).write_text(text)
        else:
            sys.stdout.write(text)
        return 0
    rows = sweep(_parse_grid(args.grid, args.elem), cm, seed=args.seed, min_iters=args.min_iters)
    Path(args.out).write_text(rows_to_csv(rows, args.measured))
    print(f"{len(rows)} rows written to {args.out}", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())

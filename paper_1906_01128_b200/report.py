"""Results rows and their CSV form -- the data format on the output side of the hot path.

Drop-in for the reference's results layer (report.py:48-140): ``ResultRow`` (one metrics row),
``normalize`` (wall / kernel ratios against the UVM cell of the same scenario, layout, k_or_q
and n; ``MissingBaseline`` when strict), ``rows_to_csv`` / ``rows_from_csv`` with the same
header and value formatting (booleans ``true``/``false``, floats by ``repr``, empty for None),
so sweep files written here and by chainforge are interchangeable byte for byte.  The measured
B200 columns of a row (``wall_us``, ``mode``, ``gpu_launches``, and the CUDA-event device times
``device_us`` = ``transfer_us`` + ``kernel_us`` + ``copy_back_us``) ride in ``extra`` and are written
only when asked (``measured=True``).  The table renderers (render_size_table /
render_instruction_table / rows_to_table) are presentation and not part of this path.
"""
from __future__ import annotations

from dataclasses import dataclass, field, fields, replace

CSV_HEADER = ("scenario,scheme,layout,k_or_q,n,bytes_h2d,bytes_d2h,transfer_ops,attach_ops,page_faults,"
              "instr_estimate,sim_kernel_us,sim_wall_us,iterations,verified,normalized_wall,normalized_kernel")
MEASURED = ("wall_us", "mode", "gpu_launches", "device_us", "transfer_us", "kernel_us", "copy_back_us")
_INT = ("k_or_q", "n", "bytes_h2d", "bytes_d2h", "transfer_ops", "attach_ops", "page_faults", "instr_estimate",
        "iterations")
_FLOAT = ("sim_kernel_us", "sim_wall_us", "normalized_wall", "normalized_kernel")


class MissingBaseline(Exception):
    """A results grid has no UVM cell to normalise a row against."""


@dataclass
class ResultRow:
    scenario: str
    scheme: str
    layout: str
    k_or_q: int
    n: int
    bytes_h2d: int
    bytes_d2h: int
    transfer_ops: int
    attach_ops: int
    page_faults: int
    instr_estimate: int
    sim_kernel_us: float
    sim_wall_us: float
    iterations: int
    verified: bool
    normalized_wall: float | None = None
    normalized_kernel: float | None = None
    extra: dict = field(default_factory=dict, compare=False)   # measured B200 columns

    @classmethod
    def from_metrics(cls, m) -> "ResultRow":
        base = {f.name: getattr(m, f.name) for f in fields(cls) if f.name not in ("normalized_wall",
                                                                                "normalized_kernel", "extra")}
        return cls(**base, extra={k: getattr(m, k) for k in MEASURED if hasattr(m, k)})

    def cell_key(self) -> tuple:
        return (self.scenario, self.layout, self.k_or_q, self.n)


def normalize(rows: list[ResultRow], strict: bool = True) -> list[ResultRow]:
    """Ratios of sim_wall_us / sim_kernel_us to the UVM row of the same cell."""
    uvm = {r.cell_key(): r for r in rows if r.scheme == "uvm"}
    out = []
    for r in rows:
        b = uvm.get(r.cell_key())
        if b is None:
            if strict:
                raise MissingBaseline(f"no uvm baseline for cell {r.cell_key()}")
            out.append(replace(r, normalized_wall=None, normalized_kernel=None))
        else:
            out.append(replace(r, normalized_wall=r.sim_wall_us / b.sim_wall_us,
                               normalized_kernel=r.sim_kernel_us / b.sim_kernel_us))
    return out


def _cell(v) -> str:
    if v is None:
        return ""
    if isinstance(v, bool):
        return "true" if v else "false"
    return repr(v) if isinstance(v, float) else str(v)


def rows_to_csv(rows: list[ResultRow], measured: bool = False) -> str:
    cols = [f.name for f in fields(ResultRow) if f.name != "extra"]
    out = [CSV_HEADER + ("," + ",".join(MEASURED) if measured else "")]
    for r in rows:
        vals = [_cell(getattr(r, c)) for c in cols]
        if measured:
            vals += [_cell(r.extra.get(c)) for c in MEASURED]
        out.append(",".join(vals))
    return "\n".join(out) + "\n"


def rows_from_csv(text: str) -> list[ResultRow]:
    lines = [ln for ln in text.split("\n") if ln]
    if not lines or not lines[0].startswith(CSV_HEADER):
        raise ValueError("unexpected results CSV header")
    names = lines[0].split(",")
    rows = []
    for ln in lines[1:]:
        d = dict(zip(names, ln.split(",")))
        kw = {}
        for f in fields(ResultRow):
            if f.name == "extra":
                continue
            v = d[f.name]
            if f.name in _INT:
                kw[f.name] = int(v)
            elif f.name in _FLOAT:
                kw[f.name] = float(v) if v != "" else None
            elif f.name == "verified":
                kw[f.name] = v == "true"
            else:
                kw[f.name] = v
        kw["extra"] = {k: d[k] for k in MEASURED if k in d}
        rows.append(ResultRow(**kw))
    return rows

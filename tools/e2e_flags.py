"""Design experiment: which part of the pipelined window costs time beyond the copies (C2)."""
import sys
sys.path.insert(0, ".")
from paper_1906_01128_b200 import DeepCopyWindow, DenseSpec, _native as N

spec = DenseSpec(4, 4 << 20, 3, elem=4, leaf_only=True)
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = DeepCopyWindow(spec, seed=1, chunk_bytes=16 << 20, nstreams=ns)
H, D = N.CF_WIN_H2D, N.CF_WIN_D2H
combos = {
    "bidir": H | D,
    "+attach+detach": H | D | N.CF_WIN_ATTACH | N.CF_WIN_DETACH,
    "+attach+resolve": H | D | N.CF_WIN_ATTACH | N.CF_WIN_RESOLVE,
    "+att+res+scale": H | D | N.CF_WIN_ATTACH | N.CF_WIN_RESOLVE | N.CF_WIN_SCALE,
    "full-tables": N.CF_WIN_FULL & ~N.CF_WIN_TABLES,
    "full": N.CF_WIN_FULL,
}
w.run(flags=N.CF_WIN_FULL)
for name, fl in combos.items():
    w.run_n(2, flags=fl)
    st = w.run_n(4, flags=fl)
    print(f"streams={ns} {name:16s} {st.ms_total/4:.2f} ms/step launches/step={st.launches//4}", flush=True)
for chunk in (4, 8, 32, 128):
    st = w.run_n(4, flags=N.CF_WIN_FULL, chunk_bytes=chunk << 20)
    st = w.run_n(4, flags=N.CF_WIN_FULL, chunk_bytes=chunk << 20)
    print(f"streams={ns} full chunk={chunk}MiB {st.ms_total/4:.2f} ms/step", flush=True)

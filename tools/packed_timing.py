"""Resident leaf-kernel time in the reference's packed layout (align=1) vs the aligned layout,
f32 / f64, including odd q whose f64 arrays sit at 4 mod 8.  python tools/packed_timing.py"""
import statistics
import sys

sys.path.insert(0, ".")
from paper_1906_01128_b200 import DeepCopyWindow, DenseSpec  # noqa: E402

only = sys.argv[1:]
cases = [("q4 f32 leaves", DenseSpec(4, 4 << 20, 3, elem=4, leaf_only=True)),
         ("q4 f64 leaves", DenseSpec(4, 2 << 20, 3, elem=8, leaf_only=True)),
         ("q3 f64 leaves", DenseSpec(3, 5 << 20, 3, elem=8, leaf_only=True)),
         ("q3 f32 leaves", DenseSpec(3, 10 << 20, 3, elem=4, leaf_only=True))]
for name, spec in cases:
    if only and not any(o in name for o in only):
        continue
    for align in (1, 16):
        w = DeepCopyWindow(spec, seed=1, policy="all_leaves", align=align)
        w.upload_raw()
        ms = []
        for r in range(12):
            st = w.run_resident(scale=2.0 if r % 2 == 0 else 0.5, graph=False)
            ms.append(st.ms_kernel)
        leaf = spec.q ** spec.depth * spec.n * spec.elem
        k = statistics.median(ms[2:])
        print(f"{name:14s} align={align:2d}: kernel {k:.3f} ms = {2 * leaf / k / 1e6:.0f} GB/s", flush=True)
        w.close()

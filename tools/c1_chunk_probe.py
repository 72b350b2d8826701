"""C1 end-to-end window (L2 flushed before each) by step size (design experiment)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1906_01128_b200 import DeepCopyWindow  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402

spec, policy, _ = bench.make_spec("C1")
w = DeepCopyWindow(spec, seed=1, policy=policy, mode="resolved", align=16, separate_output=True)
fl = bench.L2Flush(w)
for rep in range(2):
    for kib in (512, 1024, 1376, 1536, 2048, 4096):
        w.chunk_bytes = kib << 10
        w.run_n_flushed(5, fl.buf.value, bench.L2_FLUSH_BELOW, flags=N.CF_WIN_FULL | N.CF_WIN_GRAPH)
        st = w.run_n_flushed(20, fl.buf.value, bench.L2_FLUSH_BELOW, flags=N.CF_WIN_FULL | N.CF_WIN_GRAPH)
        print(f"step {kib:5d} KiB: {st.ms_total / 20 * 1e3:6.1f} us per window ({st.nsteps} steps)", flush=True)
fl.close()
w.close()

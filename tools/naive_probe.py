"""Where the naive scheme's transfer time goes (C2 / C4): device span allocation, per-object
copies (cf_copy_objects vs cf_memcpy_batch), fix-up kernel.  python tools/naive_probe.py C2"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1906_01128_b200 as cf  # noqa: E402
from paper_1906_01128_b200 import _native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec, policy, _ = bench.make_spec(cfg)
m = cf.Machine()
h = cf.build_tree(m, spec, seed=1, align=16)
allocs = h.allocation_array()
sizes = allocs[:, 1].astype(np.uint64)
aligned = (sizes + np.uint64(7)) & ~np.uint64(7)
offs = np.concatenate([[0], np.cumsum(aligned)[:-1]]).astype(np.uint64)
host = np.ascontiguousarray(allocs[:, 0], np.uint64)
for r in range(3):
    t = time.perf_counter()
    base = m.device.allocate_span(int(aligned.sum()), offs, sizes, zero=False)
    ta = time.perf_counter() - t
    dev = np.ascontiguousarray(offs + np.uint64(base), np.uint64)
    m.ctx.sync()
    t = time.perf_counter()
    N.check(N.lib().cf_copy_objects(m.ctx.handle, N.ptr(dev), N.ptr(host), N.ptr(sizes), len(sizes)))
    tc = time.perf_counter() - t
    t = time.perf_counter()
    N.check(N.lib().cf_memcpy_batch(m.ctx.handle, N.ptr(dev), N.ptr(host), N.ptr(sizes), len(sizes), None))
    m.ctx.sync()
    tb = time.perf_counter() - t
    t = time.perf_counter()
    amap = cf.AddressMap.from_arrays(host, sizes, dev)
    fields, targets = h.site_field_target_arrays()
    m._device_fixup(amap, fields, targets)
    tf = time.perf_counter() - t
    print(f"{cfg} r{r}: alloc_span {ta*1e3:.1f} ms, copy_objects {tc*1e3:.1f} ms, memcpy_batch {tb*1e3:.1f} ms, "
          f"fixup {tf*1e3:.1f} ms ({len(sizes)} objects)", flush=True)
m.close()

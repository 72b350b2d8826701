"""Time each piece of the drop-in API schemes on a config (debugging helper)."""
import sys, time
sys.path.insert(0, ".")
import bench
import paper_1906_01128_b200 as cf
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
spec, policy, _ = bench.make_spec(cfg)
for scheme in ("marshalling", "pointerchain", "naive", "uvm"):
    t = time.perf_counter()
    m = cf.Machine()
    if scheme == "uvm":
        m.enable_uvm()
    if scheme == "marshalling":
        arena, h = cf.marshal_tree(m, spec, seed=1, align=16)
    else:
        arena, h = None, cf.build_tree(m, spec, seed=1, align=16)
    tb = time.perf_counter() - t
    t = time.perf_counter(); prep = cf.transfer_to_device(m, h, scheme, arena, policy=policy); t1 = time.perf_counter() - t
    t = time.perf_counter(); cf.kernel_scale(m, h, prep, 2.0); t2 = time.perf_counter() - t
    t = time.perf_counter(); cf.copy_back(m, h, prep); m.ctx.sync(); t3 = time.perf_counter() - t
    t = time.perf_counter(); cf.verify_tree(m, h, 2.0, policy); t4 = time.perf_counter() - t
    print(f"{cfg} {scheme:12s} build {tb:.2f}s transfer {t1*1e3:.1f}ms kernel {t2*1e3:.1f}ms copy_back {t3*1e3:.1f}ms verify {t4:.2f}s", flush=True)
    m.close()

"""Time each drop-in API call of every scheme on a config (phase breakdown, 3 repetitions).

    python tools/time_schemes.py C4 [schemes...]
"""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1906_01128_b200 as cf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
which = sys.argv[2:] or ["marshalling", "marshalling_eager", "pointerchain", "naive", "uvm"]
spec, policy, _ = bench.make_spec(cfg)
for name in which:
    scheme = name.split("_")[0]
    kw = {"fused": False} if name.endswith("eager") else {}
    if scheme == "uvm" and "_" in name:
        kw = {"uvm_hints": name.split("_", 1)[1]}
    t = time.perf_counter()
    m = cf.Machine()
    if scheme == "uvm":
        m.enable_uvm()
    if scheme == "marshalling":
        arena, h = cf.marshal_tree(m, spec, seed=1, align=16)
    else:
        arena, h = None, cf.build_tree(m, spec, seed=1, align=16)
    tb = time.perf_counter() - t
    for r in range(3):
        m.ctx.sync()
        t = time.perf_counter(); prep = cf.transfer_to_device(m, h, scheme, arena, policy=policy, **kw); t1 = time.perf_counter() - t
        t = time.perf_counter(); cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5); t2 = time.perf_counter() - t
        t = time.perf_counter(); cf.copy_back(m, h, prep); m.ctx.sync(); t3 = time.perf_counter() - t
        print(f"{cfg} {name:18s} r{r} build {tb:.2f}s transfer {t1*1e3:.1f}ms kernel {t2*1e3:.1f}ms "
              f"copy_back {t3*1e3:.1f}ms window {(t1+t2+t3)*1e3:.1f}ms "
              f"{getattr(prep.fused, 'timing', '')}", flush=True)
    m.close()

"""Where does the C4 UVM-prefetch window's time go?  cProfile of the drop-in calls (host side) and
the window's device time, C4 vs C2 (design experiment)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import bench
import paper_1906_01128_b200 as cf

for cfg in sys.argv[1:] or ["C4", "C2"]:
    spec, policy, _ = bench.make_spec(cfg)
    m = cf.Machine()
    m.enable_uvm()
    h = cf.build_tree(m, spec, seed=1, align=16)
    def once(s):
        m.ctx.sync()
        t0 = time.perf_counter()
        prep = cf.transfer_to_device(m, h, "uvm", None, policy=policy, uvm_hints="prefetch")
        t1 = time.perf_counter()
        cf.kernel_scale(m, h, prep, s)
        t2 = time.perf_counter()
        cf.copy_back(m, h, prep)
        m.ctx.sync()
        t3 = time.perf_counter()
        return t1 - t0, t2 - t1, t3 - t2
    once(2.0)
    print(cfg, "phases (transfer, kernel_scale, copy_back) s:", [round(x, 4) for x in once(0.5)], flush=True)
    pr = cProfile.Profile()
    pr.enable()
    once(2.0)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
    m.close()

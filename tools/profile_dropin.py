"""cProfile of the drop-in calls of one scheme on a config (host-side overhead around the window).

    python tools/profile_dropin.py C4 pointerchain
"""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1906_01128_b200 as cf  # noqa: E402

cfg, scheme = (sys.argv[1:3] + ["C4", "pointerchain"][len(sys.argv[1:3]):])[:2]
spec, policy, _ = bench.make_spec(cfg)
m = cf.Machine()
if scheme == "marshalling":
    arena, h = cf.marshal_tree(m, spec, seed=1, align=16)
else:
    arena, h = None, cf.build_tree(m, spec, seed=1, align=16)


def window(r):
    prep = cf.transfer_to_device(m, h, scheme, arena, policy=policy)
    cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5)
    cf.copy_back(m, h, prep)
    m.ctx.sync()


for r in range(2):
    window(r)
pr = cProfile.Profile()
pr.enable()
window(2)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
m.close()

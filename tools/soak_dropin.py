"""Soak the drop-in calls (fused marshalling / pointerchain windows, eager phases, naive) on
packed f64 and aligned f32 trees, verify_tree after every window.  python tools/soak_dropin.py SECONDS"""
import sys
import time

sys.path.insert(0, ".")
import paper_1906_01128_b200 as cf  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 300
cases = [(cf.DenseSpec(3, 200000, 3), 1, "all_arrays"), (cf.DenseSpec(4, 1 << 20, 3, elem=4, leaf_only=True), 16, "all_arrays"),
         (cf.DenseSpec(40, 300, 3, elem=4), 16, "all_arrays"),
         (cf.DenseSpec(40, 256, 3, elem=4, leaf_only=True), 16, "all_leaves")]   # leaf-owned windows
deadline = time.time() + secs
n = 0
while time.time() < deadline:
    for spec, align, policy in cases:
        for scheme, fused in (("marshalling", True), ("pointerchain", True), ("marshalling", False), ("naive", True)):
            m = cf.Machine()
            arena, h = (cf.marshal_tree(m, spec, seed=n % 7, align=align) if scheme == "marshalling"
                        else (None, cf.build_tree(m, spec, seed=n % 7, align=align)))
            for r in range(3):
                prep = cf.transfer_to_device(m, h, scheme, arena, policy=policy, fused=fused)
                cf.kernel_scale(m, h, prep, 2.0, mode="chase" if (r == 1 and scheme == "marshalling") else "resolved")
                cf.copy_back(m, h, prep)
                n += 1
            # three windows of x2: check against x8
            cf.verify_tree(m, h, 8.0, policy)
            m.close()
print("soak_dropin ok", n, "windows")

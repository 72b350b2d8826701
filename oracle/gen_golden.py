"""Generate golden fixtures by running the REFERENCE implementation (test infrastructure).

Run in the build container only (it imports /root/reference, which never travels to the
GPU box):

    python oracle/gen_golden.py [--ref /root/reference/pkg/src/chainforge]

It imports the reference package under the alias ``chainforge_ref`` and
writes ``tests/golden/reference_kats.json``.  Every field is produced by the reference's own
functions -- ``marshal_tree`` (scenarios.py:262-267), ``Machine.marshal_transfer_and_attach``
(memory.py:307-325), ``targeted_arrays`` (scenarios.py:270-284), ``transfer_to_device`` /
``kernel_scale`` / ``copy_back`` (harness.py:219-325) and ``execute_case`` (harness.py:356-392)
-- so the committed JSON pins both the C oracle (oracle/cf_oracle.c) and the CUDA path.

Address-dependent bytes are normalised: every pointer field is replaced by (target - base),
which makes hashes independent of where the arena/image lives.
"""
from __future__ import annotations

import argparse
import hashlib
import importlib.util
import json
import random
import struct
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
DEFAULT_REF = "/root/reference/pkg/src/chainforge"


def load_reference(path: str):
    init = Path(path) / "__init__.py"
    spec = importlib.util.spec_from_file_location(
        "chainforge_ref", str(init), submodule_search_locations=[str(path)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["chainforge_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def normalise(raw: bytes, site_offsets, base: int) -> bytes:
    buf = bytearray(raw)
    for off in site_offsets:
        (v,) = struct.unpack_from("<Q", buf, off)
        struct.pack_into("<Q", buf, off, (v - base) & 0xFFFF_FFFF_FFFF_FFFF)
    return bytes(buf)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def spec_to_json(spec, ref) -> dict:
    if isinstance(spec, ref.LinearSpec):
        return {"kind": "linear", "k": spec.k, "n": spec.n, "layout": spec.layout}
    return {"kind": "dense", "q": spec.q, "n": spec.n, "depth": spec.depth}


def marshal_record(ref, spec, seed: int, full_bytes_limit: int = 8192) -> dict:
    memory = sys.modules["chainforge_ref.memory"]
    scenarios = sys.modules["chainforge_ref.scenarios"]
    harness = sys.modules["chainforge_ref.harness"]
    machine = memory.Machine()
    arena, handle = scenarios.marshal_tree(machine, spec, seed=seed)
    base = arena.buffer_host_addr
    total = arena.total_bytes
    sites = [s - base for s in arena.pointer_sites]
    targets = [machine.host.read_word(s) - base for s in arena.pointer_sites]
    raw = machine.host.read_bytes(base, total)
    norm = normalise(raw, sites, base)
    # device image right after attach, normalised against the image base
    image = machine.marshal_transfer_and_attach(arena)
    dev_raw = machine.device.read_bytes(image, total)
    dev_norm = normalise(dev_raw, sites, image)
    machine.demarshal(arena)
    targeted = scenarios.targeted_arrays(handle)

    # metered window with the marshalling scheme on a fresh machine
    m2 = memory.Machine()
    arena2, h2 = scenarios.marshal_tree(m2, spec, seed=seed)
    b2 = arena2.buffer_host_addr
    prep = harness.transfer_to_device(m2, h2, "marshalling", arena2)
    stats = harness.kernel_scale(m2, h2, prep, 2.0)
    harness.copy_back(m2, h2, prep)
    harness.verify_tree(m2, h2, 2.0)
    after = normalise(m2.host.read_bytes(b2, total), sites, b2)

    rec = {
        "spec": spec_to_json(spec, ref), "seed": seed, "total_bytes": total,
        "requests": [[r.host_addr - base, r.size_bytes] for r in arena.request_list],
        "sites": sites, "site_targets": targets,
        "nodes": [[a - base, lv, sz] for a, lv, sz in
                  zip(handle.node_addrs, handle.node_levels, handle.node_sizes)],
        "arrays": [[a.level, a.owner_addr - base, a.addr - base, a.count] for a in handle.arrays],
        "targeted": [a.addr - base for a in targeted],
        "arena_sha": sha(norm), "image_sha": sha(dev_norm), "after_window_sha": sha(after),
        "kernel_elements": stats.elements_touched, "kernel_derefs": stats.chain_derefs,
    }
    if total <= full_bytes_limit:
        rec["arena_hex"] = norm.hex()
        rec["after_window_hex"] = after.hex()
    # non-arena build (host bump allocator, memory.py:124-137): offsets vs first allocation
    m3 = memory.Machine()
    h3 = scenarios.build_tree(m3, spec, seed=seed)
    hb = h3.allocations[0][0]
    rec["bump_allocations"] = [[a - hb, s] for a, s in h3.allocations]
    rec["bump_sites"] = [[h - hb, o, t - hb] for h, o, t in h3.reference_field_sites]
    return rec


def case_counters(ref, spec, seed: int) -> dict:
    harness = sys.modules["chainforge_ref.harness"]
    out = {}
    for scheme in harness.SCHEMES:
        m, _ = harness.execute_case(spec, scheme, harness.CostModel(), seed=seed)
        out[scheme] = [m.bytes_h2d, m.bytes_d2h, m.transfer_ops, m.attach_ops,
                       m.page_faults, m.instr_estimate, m.verified,
                       m.sim_kernel_us, m.sim_wall_us]
    return out


def spec_list(ref):
    L, D = ref.LinearSpec, ref.DenseSpec
    specs = [
        # SURVEY.md App. A KATs
        L(3, 4, "allinit_allused"), L(4, 37, "LLinit_LLused"), D(2, 1, 2), D(3, 5, 2),
        # App. C edge cases
        L(3, 0, "allinit_allused"), L(1, 0, "allinit_allused"), L(1, 5, "LLinit_LLused"),
        D(1, 4, 3), D(2, 0, 2), D(5, 3, 0), L(3, 7, "allinit_LLused"),
        # specs used by the reference tests (test_memory.py, test_harness.py, test_scenarios.py)
        L(2, 100, "allinit_allused"), L(2, 100, "LLinit_LLused"), D(2, 10, 3),
        L(3, 10, "allinit_allused"), L(4, 25, "allinit_allused"), L(3, 50, "allinit_LLused"),
        D(3, 17, 2), D(3, 4, 2), D(4, 6, 0), D(2, 50, 3), L(5, 1000, "LLinit_LLused"),
        # alignment census specs (App. A)
        D(4, 1000, 3), D(100, 256, 1),
    ]
    specs += [D(q, 11, 3) for q in range(1, 5)]
    specs += [L(k, 37, lay) for k in (1, 2, 5, 10) for lay in ref.scenarios.LAYOUTS]
    rng = random.Random(0xC0FFEE)
    for _ in range(16):
        if rng.random() < 0.5:
            specs.append(L(rng.randint(1, 12), rng.randint(0, 300), rng.choice(ref.scenarios.LAYOUTS)))
        else:
            specs.append(D(rng.randint(1, 6), rng.randint(0, 64), rng.randint(0, 3)))
    return specs


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=DEFAULT_REF)
    ap.add_argument("--out", default=str(REPO / "tests" / "golden" / "reference_kats.json"))
    args = ap.parse_args(argv)
    ref = load_reference(args.ref)
    ref.scenarios = sys.modules["chainforge_ref.scenarios"]
    records, counters = [], []
    for i, spec in enumerate(spec_list(ref)):
        seeds = (1, 0, 13) if i < 4 else (1,)
        for seed in seeds:
            records.append(marshal_record(ref, spec, seed))
        counters.append({"spec": spec_to_json(spec, ref), "seed": 1,
                         "schemes": case_counters(ref, spec, 1)})
    # closed-form size KATs (test_scenarios.py:21-31)
    sc = ref.scenarios
    sizes = {
        "linear": [[k, n, lay, sc.linear_data_size(k, n, lay)]
                   for k, n, lay in ((2, 100, "allinit_allused"), (10, 10 ** 8, "allinit_allused"),
                                     (3, 7, "LLinit_LLused"), (4, 0, "LLinit_LLused"))],
        "dense": [[q, n, d, sc.dense_data_size(q, n, d)]
                  for q, n, d in ((2, 10, 3), (16, 10 ** 5, 3), (1, 0, 0), (4, 4194304, 3), (100, 256, 3))],
    }
    payload = {
        "generator": "oracle/gen_golden.py (imports the reference as chainforge_ref)",
        "reference": "arxiv/paper_1906_01128 pkg/src/chainforge",
        "payload_kat": {f"{s}:{lv}": [float(v) for v in sc.payload_values(s, lv, 6)]
                        for s, lv in ((0, 0), (1, 3), (13, 2), (7, 1))},
        "sizes": sizes, "marshal": records, "counters": counters,
    }
    Path(args.out).write_text(json.dumps(payload, indent=None, separators=(",", ":")) + "\n")
    print(f"wrote {len(records)} marshal records, {len(counters)} counter rows -> {args.out}")


if __name__ == "__main__":
    main()

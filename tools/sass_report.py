"""Instruction-level evidence: SASS opcode counts of the leaf kernel variants.

    python tools/sass_report.py [lib.so] > profiles/r01_sass_k_scale.md
Counts static SASS instructions per k_scale instantiation from `cuobjdump -sass`, separating the
128-bit streaming loads/stores from the chain loads (`ld.global.nc` -> LDG.E.64.CONSTANT)
that CHASE mode issues per 16-byte access -- the B200 analogue of the paper's PTX counts
(harness.py:98-127)."""
import collections, re, subprocess, sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1906_01128_b200/_lib/libchainforge_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if cur and m:
        funcs[cur][m.group(1)] += 1
rows = []
for name, c in funcs.items():
    if "k_scale" not in name:
        continue
    t = "float" if "IfLb" in name else "double"
    mode = "chase" if "Lb1" in name else "resolved"
    pm = re.search(r"Lb[01]ELi(\d)E", name)
    path = {"0": "tiles+groups", "1": "tiles", "2": "groups", "3": "leaf-owned groups"}.get(pm.group(1), "?") if pm else "all"
    total = sum(c.values())
    chain = sum(v for k, v in c.items() if k.startswith("LDG") and "CONSTANT" in k)
    vec_ld = sum(v for k, v in c.items() if k.startswith("LDG") and "128" in k)
    vec_st = sum(v for k, v in c.items() if k.startswith("STG") and "128" in k)
    rows.append((t, mode, path, total, vec_ld, vec_st, chain))
print("| type | mode | work path | static SASS instructions | LDG.128 | STG.128 | chain loads (LDG.*.CONSTANT) |")
print("|---|---|---|---|---|---|---|")
for r in rows:
    print("| " + " | ".join(str(x) for x in r) + " |")

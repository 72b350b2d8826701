import sys, json, traceback
sys.path.insert(0, ".")
import paper_1906_01128_b200 as cf
kats = json.load(open("tests/golden/reference_kats.json"))
for row in kats["counters"]:
    j = row["spec"]
    spec = cf.LinearSpec(j["k"], j["n"], j["layout"]) if j["kind"] == "linear" else cf.DenseSpec(j["q"], j["n"], j["depth"])
    for scheme in ("marshalling", "naive", "pointerchain", "uvm"):
        try:
            m, mach = cf.execute_case(spec, scheme, cf.CostModel(), seed=1)
            mach.close()
        except Exception as e:
            print("FAIL", j, scheme, type(e).__name__, str(e)[:100])
print("done")

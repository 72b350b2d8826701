"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into markdown shares."""
import collections, csv, sys
src, dst, title = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
rows = list(csv.reader(open(src)))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[i], rows[i + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in data:
    name = r[ki].split("(")[0].split("::")[-1]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
out = [f"# ncu launch list — {title}", "",
       f"{len(data)} kernel launches (gpu__time_duration.sum, --clock-control none; cold-cache and serialised "
       "by ncu: compare shares, not absolutes).", "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"| {k} | {n} | {t / 1e3:.1f} | {t / tot:.3f} |")
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out))

"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import csv, sys, collections, re
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
body = rows[1:]
if "--step" in sys.argv:   # keep the stepping loop: from the launch before the first MODE_STEP (..., 0>) kernel on
    first = next((i for i, r in enumerate(body) if len(r) > ki and re.search(r", \(int\)0>|, 0>", r[ki])), 0)
    body = body[max(first - 1, 0):]
for r in body:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*$", "", r[ki].replace("(int)", "")).replace("void ", "")
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
    us = v / 1000.0 if unit in ("ns", "nsecond") else v * 1000.0 if unit in ("ms", "msecond") else v
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
print(f"| launches | total us | share | avg us | kernel |\n|---|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {n} | {t:.1f} | {100*t/tot:.1f}% | {t/n:.2f} | `{k}` |")

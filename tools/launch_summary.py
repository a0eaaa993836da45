"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per kernel name, launches and total/mean device time."""
import csv, sys, collections
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].replace("void ", "")
    ns = float(r[iv].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += ns
tot = sum(v[1] for v in agg.values())
for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{ns/1e6:10.3f} ms {100*ns/tot:6.2f}%  {c:5d} x {ns/c/1e3:10.2f} us  {k[:90]}")
print(f"total {tot/1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")

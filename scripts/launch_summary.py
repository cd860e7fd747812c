"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel
time of the LAST solve (the list holds warm-up + timed solve)."""
import csv, collections, sys, json
path = sys.argv[1]
nsolves = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
hdr = rows[0]
ki, vi, gi, bi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size"), hdr.index("Block Size")
data = [(r[ki], float(r[vi].replace(",", "")), r[gi], r[bi]) for r in rows[1:]]
n = len(data) // nsolves
last = data[len(data) - n:]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v, g, b in last:
    k = k.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("vrte::", "")
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
out = {"launches": len(last), "total_ms": tot / 1e6, "kernels": []}
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out["kernels"].append({"kernel": k, "launches": c, "ms": v / 1e6, "share": v / tot})
if "--json" in sys.argv:
    print(json.dumps(out, indent=1))
else:
    print("launches %d total %.3f ms" % (len(last), tot / 1e6))
    for e in out["kernels"][:30]:
        print("%-50s %5d %9.3f %6.3f" % (e["kernel"][:50], e["launches"], e["ms"], e["share"]))

"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum": continue
    raw = r[ki].replace("(anonymous namespace)::", "").replace("void ", "")
    name = raw.split("(")[0].strip()
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "nsecond"
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
    tot[name] += v * scale; cnt[name] += 1
T = sum(tot.values())
print(f"total {T/1e3:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v/1e3:8.3f} ms {100*v/T:5.1f}%  x{cnt[k]:4d}  {k}")

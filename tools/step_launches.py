"""Join an ncu launch list of one profiled step (tools/profile_step.py under
ncu --profile-from-start off) with the MM_GEMM_LOG shape lines of that step:
per-launch kernel, shape, time, TFLOP/s; plus a per-kernel summary."""
import csv, re, sys, collections
ncu_csv, log = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(ncu_csv)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
ids = h.index("ID") if "ID" in h else None
launches = []
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "").split("(")[0]
    us = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
    launches.append((name, us))
shapes = [l for l in open(log) if l.startswith("mm_gemm ")]
# the profiled step's GEMMs are the last len(gemm launches) log lines
ng = sum(1 for n, _ in launches if n.startswith("gemm"))
shapes = shapes[-ng:] if ng else []
si = 0
tot = collections.defaultdict(float)
cnt = collections.Counter()
for name, us in launches:
    extra = ""
    key = name
    if name.startswith("gemm") and si < len(shapes):
        kv = dict(x.split("=") for x in shapes[si].split()[1:])
        si += 1
        fl = 2 * int(kv["m"]) * int(kv["n"]) * int(kv["k"])
        extra = (f"m={kv['m']:>6} n={kv['n']:>6} k={kv['k']:>6} epi={kv['epi']} bn={kv['bn']} "
                 f"sp={kv['splits']} units={kv['units']:>4}  {fl / us / 1e6:7.1f} TFLOP/s")
        key = f"gemm m{kv['m']} n{kv['n']} k{kv['k']} a{kv['a_mn']}b{kv['b_mn']}"
    print(f"{us:9.2f} us  {name[:40]:40s} {extra}")
    tot[key] += us
    cnt[key] += 1
T = sum(tot.values())
print(f"\ntotal {T / 1e3:.3f} ms over {len(launches)} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:40]:
    print(f"{v / 1e3:8.3f} ms {100 * v / T:5.1f}%  x{cnt[k]:4d}  {k}")

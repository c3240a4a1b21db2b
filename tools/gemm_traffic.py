"""Summarise the GEMM launches of one profiled config-3 step (tools/profile_step.py
under ncu --profile-from-start off with gpu__time_duration / dram__bytes_*
metrics and MM_GEMM_LOG=1): launches, algorithmic FLOPs (sum of 2mnk from the
log lines of the profiled step), DRAM bytes (read + write) and serialized ncu
time; written as the JSON bench.py reports as roofline.traffic.
    python tools/gemm_traffic.py step.csv step_gemm.log out.json"""
import csv, json, re, sys
csv_path, log_path, out = sys.argv[1:4]
rows = list(csv.reader(open(csv_path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
ui = h.index("Metric Unit")
per = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[idi], {"name": r[ki]})
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
    elif r[mi].startswith("dram__bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    d[r[mi]] = v
gemm = [d for d in per.values() if "gemm_tcgen05" in d["name"]]
allk = list(per.values())
# the profiled step's GEMM problems: the last log lines whose launch count matches
lines = [l for l in open(log_path) if l.startswith("mm_gemm ")]
launch_lines = []  # group lines by launch: a grouped launch logs group=i/n for each problem
for l in lines:
    kv = dict(x.split("=") for x in l.split()[1:])
    launch_lines.append(kv)
launches, cur = [], []
for kv in launch_lines:
    i, n = (int(x) for x in kv["group"].split("/"))
    cur.append(kv)
    if i == n - 1:
        launches.append(cur)
        cur = []
step = launches[-len(gemm):]
flops = sum(2.0 * int(kv["m"]) * int(kv["n"]) * int(kv["k"]) for L in step for kv in L)
dram = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in gemm)
t_us = sum(d["gpu__time_duration.sum"] for d in gemm)
res = {"gemm_launches": len(gemm), "gemm_problems": sum(len(L) for L in step),
       "algorithmic_flops_per_step": flops, "dram_bytes_per_step": dram,
       "dram_bytes_per_launch": dram / max(1, len(gemm)),
       "ncu_gemm_us_per_step": t_us, "ncu_all_kernels_us_per_step": sum(d["gpu__time_duration.sum"] for d in allk),
       "gemm_share_of_ncu_step": t_us / sum(d["gpu__time_duration.sum"] for d in allk),
       "flops_per_dram_byte": flops / max(dram, 1.0), "source": [csv_path, log_path],
       "note": "ncu per-launch times are serialized and cold-cache; only the GEMM share of the step is comparable with bench.py"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))

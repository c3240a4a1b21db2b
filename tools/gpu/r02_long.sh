# long-group attention kernels as one persistent wave: tests, same-box c5 A/B, launch list
D=gpurun_out/r02_long
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" -p no:cacheprovider > $D/tests.log 2>&1
tail -n 1 $D/tests.log
for r in 1 2; do
  timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/new_c5_$r.json 2> /dev/null
  MM_LIB_VARIANT=attnprev timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/old_c5_$r.json 2> /dev/null
done
for f in $D/*.json; do echo "$f $(tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")"; done
for v in new old; do
  if [ $v = old ]; then export MM_LIB_VARIANT=attnprev; else unset MM_LIB_VARIANT; fi
  CFG=config5 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    -k regex:attn --csv --log-file $D/launch_$v.csv python tools/profile_step.py > $D/ncu_$v.log 2>&1
  python - $D/launch_$v.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
agg = collections.defaultdict(list)
for r in rows[1:]:
    if r[ix["Metric Name"]] == "gpu__time_duration.sum":
        agg[r[ix["Kernel Name"]][:40]].append(float(r[ix["Metric Value"]].replace(",", "")))
for k, v in agg.items():
    print(sys.argv[1].split("/")[-1], k, len(v), "avg", round(sum(v) / len(v) / 1e3, 2), "us")
PY
done
unset MM_LIB_VARIANT

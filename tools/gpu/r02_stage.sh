# attention backward output staging A/B: kernel tests, back-to-back launches, c3 + c5 steps
D=gpurun_out/r02_stage
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" -p no:cacheprovider > $D/tests.log 2>&1
tail -n 1 $D/tests.log
for v in new old; do
  if [ $v = old ]; then export MM_LIB_VARIANT=attnprev; else unset MM_LIB_VARIANT; fi
  REPS=20 timeout 300 python tools/attn_waitprof.py > $D/c3_warm_$v.log 2>&1
  C5=1 REPS=20 timeout 300 python tools/attn_waitprof.py > $D/c5_warm_$v.log 2>&1
done
unset MM_LIB_VARIANT
grep -H "kernel us" $D/*_warm_*.log
for r in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline > $D/new_c3_$r.json 2> /dev/null
  MM_LIB_VARIANT=attnprev timeout 900 python bench.py --no-cpu-baseline > $D/old_c3_$r.json 2> /dev/null
done
timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/new_c5.json 2> /dev/null
MM_LIB_VARIANT=attnprev timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/old_c5.json 2> /dev/null
for f in $D/*.json; do echo "$f $(tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")"; done

# attention backward A/B: parity tests, wait breakdown, warm timing, config-3 step
D=gpurun_out/r02_attn2
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_shapes_gpu.py tests/test_engine_gpu.py -q -x -p no:cacheprovider > $D/tests.log 2>&1
tail -n 1 $D/tests.log
MM_LIB_VARIANT=attn_wp timeout 300 python tools/attn_waitprof.py > $D/wp_c3.log 2>&1
MM_LIB_VARIANT=attn_wp C5=1 timeout 300 python tools/attn_waitprof.py > $D/wp_c5.log 2>&1
REPS=20 timeout 300 python tools/attn_waitprof.py > $D/c3_warm.log 2>&1
C5=1 REPS=20 timeout 300 python tools/attn_waitprof.py > $D/c5_warm.log 2>&1
cat $D/wp_c3.log $D/wp_c5.log $D/c3_warm.log $D/c5_warm.log
for r in 1 2; do timeout 900 python bench.py --no-cpu-baseline > $D/bench_c3_$r.json 2> $D/bench_c3_$r.err; done
for f in $D/bench_*.json; do echo "$f $(tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")"; done

# bench lines on the final commit (configs 3 / 4 / 5)
D=gpurun_out/r02final8; mkdir -p $D
timeout 900 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
timeout 900 python bench.py --config config4 --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/bench_c5.json 2> $D/bench_c5.err
for f in $D/bench_c*.json; do echo "$f $(tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['ms_per_step'], d['value'], d['e2e']['value'], r['frac'], r['peak_used'][:9], d['clocks']['sm_mhz'], d['clocks']['reasons'])")"; done

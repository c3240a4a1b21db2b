D=gpurun_out/r02bv
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $D/smi.txt 2>&1; cat $D/smi.txt
timeout 900 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
timeout 900 python bench.py --config config4 --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $D/bench_c3b.json 2> $D/bench_c3b.err
for f in $D/bench_*.json; do echo "$f $(tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['ms_per_step'], d['value'], d['e2e']['value'], r['frac'], r['frac_vs_burst'], d['clocks'])")"; done

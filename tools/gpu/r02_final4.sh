# final evidence on the final build (config 1 at its true shape added):
# GPU suite, smoke, config 3/4/5 bench lines, the reference arm, GEMM spans,
# config-1 parity table
D=gpurun_out/r02final7
mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_all.log 2>&1
tail -n 1 $D/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1
tail -n 1 $D/smoke.log
timeout 900 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
timeout 900 python bench.py --config config4 --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/bench_c5.json 2> $D/bench_c5.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $D/bench_reference.json 2> $D/bench_reference.err
timeout 300 python tools/gemm_spans.py config3 > $D/gemm_spans_c3.log 2>&1
for f in $D/bench_c*.json; do echo "$f $(tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['ms_per_step'], d['value'], d['e2e']['value'], r['frac'], r['peak_used'][:9], d['clocks']['sm_mhz'], d['clocks']['reasons'])")"; done
tail -c 300 $D/bench_reference.json
tail -n 1 $D/gemm_spans_c3.log

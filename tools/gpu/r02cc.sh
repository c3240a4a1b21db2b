# final check of the final commit: GPU suite, smoke, bench lines, spans
D=gpurun_out/r02cc4
mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_all.log 2>&1
tail -n 1 $D/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1
tail -n 1 $D/smoke.log
timeout 900 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
timeout 900 python bench.py --config config4 --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/bench_c5.json 2> $D/bench_c5.err
timeout 300 python tools/gemm_spans.py config3 > $D/gemm_spans_c3.log 2>&1
for f in $D/bench_*.json; do echo "$f $(tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['ms_per_step'], d['value'], d['e2e']['value'], r['frac'], r['peak_used'][:9], d['clocks']['sm_mhz'], d['clocks']['reasons'])")"; done
tail -n 1 $D/gemm_spans_c3.log

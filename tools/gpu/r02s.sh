set -x
D=gpurun_out/r02s
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_parity_shapes_gpu.py -q -x > $D/t.log 2>&1
timeout 300 python tools/gemm_spans.py config3 $D/spans_c3.json > $D/spans_c3.log 2>&1
for rep in a b c; do timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/bench_$rep.log 2>&1; done
tail -n 3 $D/t.log; tail -n 1 $D/spans_c3.log
for f in $D/bench_*.log; do tail -n 1 $f | cut -c1-160; done

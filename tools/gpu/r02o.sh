set -x
D=gpurun_out/r02o
mkdir -p $D
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k gemm > $D/t.log 2>&1
for v in base epi2; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 300 python tools/gemm_spans.py config3 $D/spans_$v.json > $D/spans_$v.log 2>&1
  for rep in a b; do timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/bench_${v}_$rep.log 2>&1; done
done
unset MM_LIB_VARIANT
tail -n 2 $D/t.log
for v in base epi2; do tail -n 1 $D/spans_$v.log; done
for f in $D/bench_*.log; do echo $f; tail -n 1 $f | cut -c1-160; done

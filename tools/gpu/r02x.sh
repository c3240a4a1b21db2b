set -x
D=gpurun_out/r02x
mkdir -p $D
for rep in a b; do
  for v in base epi256p2; do
    if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
    timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $D/bench_${v}_$rep.log 2>&1
  done
done
for v in base epi256p2; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 300 python tools/gemm_spans.py config3 $D/spans_$v.json > $D/spans_$v.log 2>&1
  timeout 600 python tools/gemm_micro.py "gen" "big" > $D/micro_$v.log 2>&1
  timeout 600 python bench.py --config config5 --steps 10 --warmup 3 --no-cpu-baseline > $D/c5_$v.log 2>&1
done
unset MM_LIB_VARIANT
for f in $D/bench_*.log $D/c5_*.log; do echo $f; tail -n 1 $f | cut -c1-160; done
cat $D/micro_*.log

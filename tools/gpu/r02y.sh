set -x
D=gpurun_out/r02y
mkdir -p $D
export MM_LIB_VARIANT=bf16pair
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "gemm" -x > $D/t_pair.log 2>&1
unset MM_LIB_VARIANT
for rep in a b; do
  for v in base bf16pair pair_epi2; do
    if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
    timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $D/bench_${v}_$rep.log 2>&1
  done
done
for v in base bf16pair pair_epi2; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --config config5 --steps 10 --warmup 3 --no-cpu-baseline > $D/c5_$v.log 2>&1
  timeout 600 python tools/gemm_micro.py "fwd" "dgrad ff2" > $D/micro_$v.log 2>&1
done
unset MM_LIB_VARIANT
tail -n 2 $D/t_pair.log
for f in $D/bench_*.log $D/c5_*.log; do echo $f; tail -n 1 $f | cut -c1-160; done

set -x
D=gpurun_out/r02ac
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k gemm -x > $D/t.log 2>&1
for g in 48 0; do
  export MM_GEMM_L2_GROUP_MB=$g
  timeout 600 python tools/gemm_micro.py "big" "gen" "c5 wgrad" > $D/micro_$g.log 2>&1
  for rep in a b; do timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $D/bench_${g}_$rep.log 2>&1; done
  timeout 600 python bench.py --config config5 --steps 10 --warmup 3 --no-cpu-baseline > $D/c5_$g.log 2>&1
done
tail -n 2 $D/t.log
cat $D/micro_*.log
for f in $D/bench_*.log $D/c5_*.log; do echo $f; tail -n 1 $f | cut -c1-160; done

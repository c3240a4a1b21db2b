set -x
D=gpurun_out/r02t
mkdir -p $D
for rep in a b; do
  for m in 1 0; do
    MM_RELU_MASK=$m timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $D/bench_m${m}_$rep.log 2>&1
  done
done
for f in $D/bench_*.log; do echo $f; tail -n 1 $f | cut -c1-160; done

set -x
D=gpurun_out/r02l
mkdir -p $D
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "embedding" > $D/t.log 2>&1
for v in 2 1; do
  if [ $v = 1 ]; then export MM_LN_V1=1; else unset MM_LN_V1; fi
  for rep in a b; do timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/bench_ln${v}_$rep.log 2>&1; done
done
unset MM_LN_V1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $D/step_c3.csv python tools/profile_step.py > $D/step_c3.out 2>&1
tail -n 2 $D/t.log
for f in $D/bench_ln*.log; do echo $f; tail -n 1 $f | cut -c1-200; done

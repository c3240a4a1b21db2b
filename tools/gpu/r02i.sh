set -x
mkdir -p gpurun_out/r02i
timeout 300 python tools/ln_micro.py > gpurun_out/r02i/ln_v2.log 2>&1
MM_LN_V1=1 timeout 300 python tools/ln_micro.py > gpurun_out/r02i/ln_v1.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "layernorm or embedding" > gpurun_out/r02i/t.log 2>&1
for v in 2 1; do
  if [ $v = 1 ]; then export MM_LN_V1=1; else unset MM_LN_V1; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02i/bench_ln$v.log 2>&1
done
unset MM_LN_V1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ln_|embed_" -c 40 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02i/ncu_ln.csv 2> gpurun_out/r02i/ncu_ln.err
cat gpurun_out/r02i/ln_v2.log gpurun_out/r02i/ln_v1.log; tail -2 gpurun_out/r02i/t.log
for v in 2 1; do tail -n 1 gpurun_out/r02i/bench_ln$v.log | cut -c1-200; done

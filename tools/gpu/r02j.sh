set -x
mkdir -p gpurun_out/r02j
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k attention > gpurun_out/r02j/attn.log 2>&1
timeout 900 python -m pytest tests/test_parity_shapes_gpu.py tests/test_engine_gpu.py -q -k "long or config5 or block" > gpurun_out/r02j/long.log 2>&1
timeout 900 python bench.py --config config5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02j/c5_new.log 2>&1
MM_ATTN_TC_FWD=auto MM_ATTN_LONG_MMA_SYNC=1 timeout 900 python bench.py --config config5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02j/c5_old.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02j/c3_new.log 2>&1
MM_ATTN_TC_FWD=auto timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02j/c3_old.log 2>&1
tail -n 15 gpurun_out/r02j/attn.log; tail -n 15 gpurun_out/r02j/long.log
for f in c5_new c5_old c3_new c3_old; do tail -n 1 gpurun_out/r02j/$f.log | cut -c1-220; done

set -x
mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests/test_sync_gpu.py tests/test_acceptance_gpu.py tests/test_kernels_gpu.py -q -x > gpurun_out/r02e/t1.log 2>&1
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_parity_shapes_gpu.py -q -x > gpurun_out/r02e/t2.log 2>&1
timeout 300 python tools/gemm_spans.py config3 gpurun_out/r02e/spans_c3.json > gpurun_out/r02e/spans_c3.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02e/bench.log 2>&1
tail -n 3 gpurun_out/r02e/t1.log gpurun_out/r02e/t2.log
tail -n 1 gpurun_out/r02e/spans_c3.log
tail -n 1 gpurun_out/r02e/bench.log | cut -c1-300

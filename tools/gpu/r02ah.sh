D=gpurun_out/r02ah4
mkdir -p $D
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_multirank_gpu.py tests/test_parity_shapes_gpu.py tests/test_kernels_gpu.py -q -x > $D/t.log 2>&1
tail -n 3 $D/t.log

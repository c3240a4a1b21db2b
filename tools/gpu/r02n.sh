set -x
D=gpurun_out/r02n
mkdir -p $D
timeout 900 python -m pytest tests/test_multirank_gpu.py tests/test_kernels_gpu.py -q > $D/t.log 2>&1
tail -n 30 $D/t.log

set -x
mkdir -p gpurun_out/r02g
timeout 900 python -m pytest tests/test_multirank_gpu.py -q > gpurun_out/r02g/multirank.log 2>&1
tail -n 30 gpurun_out/r02g/multirank.log

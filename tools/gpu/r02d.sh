set -x
mkdir -p gpurun_out/r02d
timeout 900 python -m pytest tests/test_sync_gpu.py tests/test_acceptance_gpu.py -q -x > gpurun_out/r02d/sync_accept.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --deselect tests/test_sync_gpu.py --deselect tests/test_acceptance_gpu.py > gpurun_out/r02d/gpu_all.log 2>&1
tail -5 gpurun_out/r02d/sync_accept.log gpurun_out/r02d/gpu_all.log

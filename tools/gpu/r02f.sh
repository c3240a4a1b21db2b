set -x
mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests/test_multirank_gpu.py -q -x > gpurun_out/r02f/multirank.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --deselect tests/test_multirank_gpu.py --deselect tests/test_acceptance_gpu.py::test_09_scaling_efficiency_modeled_equals_reference > gpurun_out/r02f/gpu_all.log 2>&1
tail -n 30 gpurun_out/r02f/multirank.log
tail -n 3 gpurun_out/r02f/gpu_all.log

set -x
mkdir -p gpurun_out/r02h
timeout 1500 python -m pytest tests -q -m gpu -x --deselect tests/test_acceptance_gpu.py::test_09_scaling_efficiency_modeled_equals_reference > gpurun_out/r02h/gpu_all.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02h/bench.log 2>&1
timeout 300 python tools/gemm_spans.py config3 gpurun_out/r02h/spans_c3.json > gpurun_out/r02h/spans_c3.log 2>&1
tail -n 3 gpurun_out/r02h/gpu_all.log
tail -n 1 gpurun_out/r02h/spans_c3.log

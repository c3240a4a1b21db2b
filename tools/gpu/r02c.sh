set -x
mkdir -p gpurun_out/r02c
timeout 600 python -m pytest tests/test_engine_gpu.py -q -k block > gpurun_out/r02c/block.log 2>&1
MM_PARITY_OUT=gpurun_out/r02c/parity.json timeout 900 python -m pytest tests/test_parity_shapes_gpu.py -q > gpurun_out/r02c/parity.log 2>&1
timeout 300 python tools/gemm_spans.py config3 gpurun_out/r02c/spans_c3.json > gpurun_out/r02c/spans_c3.log 2>&1
timeout 600 python tools/gemm_micro.py > gpurun_out/r02c/gemm_micro.log 2>&1
timeout 1200 python tools/diag_parity.py r02c > gpurun_out/r02c/diag.log 2>&1
tail -3 gpurun_out/r02c/block.log gpurun_out/r02c/parity.log
tail -1 gpurun_out/r02c/spans_c3.log

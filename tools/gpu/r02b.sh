set -x
mkdir -p gpurun_out/r02b
timeout 900 python tools/diag_parity.py r02b > gpurun_out/r02b/diag.log 2>&1
timeout 600 python -m pytest tests/test_engine_gpu.py -q -x -k block > gpurun_out/r02b/block.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b/bench.log 2>&1
tail -5 gpurun_out/r02b/block.log
tail -2 gpurun_out/r02b/bench.log

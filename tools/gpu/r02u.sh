set -x
D=gpurun_out/r02u
mkdir -p $D
timeout 600 python bench.py --steps 20 --warmup 5 > $D/bench.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "relu or epilogue" > $D/t.log 2>&1
tail -n 1 $D/bench.log | cut -c1-300; tail -n 2 $D/t.log

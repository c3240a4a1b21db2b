D=gpurun_out/r02bg2
mkdir -p $D
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "multicast" > $D/t.log 2>&1
tail -n 3 $D/t.log

D=gpurun_out/r02ce2
mkdir -p $D
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "specialised" > $D/t.log 2>&1; tail -n 3 $D/t.log

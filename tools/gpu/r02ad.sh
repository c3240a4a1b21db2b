set -x
D=gpurun_out/r02ad
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "grouped_unit_order or gemm_majors or wgrad" > $D/t.log 2>&1
tail -n 2 $D/t.log

timeout 900 python tools/gemm_micro.py "c5" > gpurun_out/r02ab_micro_c5.log 2>&1
cat gpurun_out/r02ab_micro_c5.log

D=gpurun_out/r02bd
mkdir -p $D
timeout 300 python tools/gemm_trace.py > $D/trace.txt 2>&1; cat $D/trace.txt

D=gpurun_out/r02af
mkdir -p $D
GEMM_VARIANTS=auto,1:128,1:192,1:256,2:128,2:256 timeout 600 python tools/gemm_micro.py fwd dgrad wgrad > $D/variants.txt 2>&1

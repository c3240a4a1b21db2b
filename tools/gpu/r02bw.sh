D=gpurun_out/r02bw
mkdir -p $D
timeout 300 python tools/gemm_cold.py > $D/cold.txt 2>&1; cat $D/cold.txt | tail -7

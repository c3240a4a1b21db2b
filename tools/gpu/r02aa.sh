set -x
D=gpurun_out/r02aa
mkdir -p $D
timeout 600 ncu --set full --clock-control none -k regex:"gemm_tcgen05|nvjet" -s 2 -c 2 -o $D/big python tools/gemm_one.py 8192 8192 8192 > $D/ncu_big.out 2>&1
ncu -i $D/big.ncu-rep --page details --csv > $D/big_details.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:"gemm_tcgen05|nvjet" -s 2 -c 2 -o $D/gen python tools/gemm_one.py 4096 32000 512 > $D/ncu_gen.out 2>&1
ncu -i $D/gen.ncu-rep --page details --csv > $D/gen_details.csv 2>/dev/null
ls -la $D

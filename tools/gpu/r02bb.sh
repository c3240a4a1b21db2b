D=gpurun_out/r02bb
mkdir -p $D
MM_GEMM_MC=1 MM_GEMM_CG=2 MM_GEMM_BN=128 timeout 120 python tools/gemm_one.py 4096 512 512 > $D/one.txt 2>&1; echo "one rc=$?"; tail -3 $D/one.txt
MM_GEMM_MC=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > $D/t.log 2>&1; echo "tests rc=$?"; tail -n 3 $D/t.log

set -x
D=gpurun_out/r02ae
mkdir -p $D
MM_GEMM_LOG=1 timeout 300 python tools/gemm_spans.py config3 > $D/spans.log 2> $D/choices.log
tail -n 3 $D/spans.log

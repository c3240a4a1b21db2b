D=gpurun_out/r02aj
mkdir -p $D
run() {  # name cfg steps rules
  MM_GEMM_RULES=$4 timeout 600 python bench.py --config $2 --steps $3 --warmup 3 --no-cpu-baseline > $D/$1.json 2> $D/$1.err
  echo "$1 $(python -c "import json,sys; d=json.loads(open('$D/$1.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'])")"
}
MM_GEMM_LOG=1 timeout 300 python tools/gemm_spans.py config4 > /dev/null 2> $D/choices_c4.log
MM_GEMM_LOG=1 timeout 300 python tools/gemm_spans.py config5 > /dev/null 2> $D/choices_c5.log
MM_GEMM_RULES=0 MM_GEMM_LOG=1 timeout 300 python tools/gemm_spans.py config4 > /dev/null 2> $D/choices_c4_0.log
MM_GEMM_RULES=0 MM_GEMM_LOG=1 timeout 300 python tools/gemm_spans.py config5 > /dev/null 2> $D/choices_c5_0.log
for rep in 1 2; do
run c3_r1_$rep config3 30 1
run c3_r0_$rep config3 30 0
run c4_r1_$rep config4 20 1
run c4_r0_$rep config4 20 0
run c5_r1_$rep config5 10 1
run c5_r0_$rep config5 10 0
done

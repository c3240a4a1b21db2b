D=gpurun_out/r02al
mkdir -p $D
one() {  # name env...
  local name=$1; shift
  env "$@" timeout 300 python tools/gemm_spans.py config3 > $D/spans_$name.log 2>&1
  env "$@" timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_$name.json 2> $D/b_$name.err
  echo "$name $(python -c "import json,sys; d=json.loads(open('$D/b_$name.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])") $(tail -n 1 $D/spans_$name.log)"
}
for rep in 1 2; do
one base$rep X=1
one norelu$rep MM_RELU_MASK=0
one nogroup$rep MM_GEMM_L2_GROUP_MB=0
one nort$rep MM_LIB_VARIANT=nort
done

D=gpurun_out/r02bi
mkdir -p $D
one() {  # name cfg steps env...
  local name=$1; local cfg=$2; local steps=$3; shift 3
  env "$@" timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline > $D/b_$name.json 2> $D/b_$name.err
  echo "$name $(python -c "import json,sys; d=json.loads(open('$D/b_$name.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'])")"
}
for rep in 1 2; do
one c3_r1_$rep config3 30 MM_GEMM_RULES=1
one c3_r0_$rep config3 30 MM_GEMM_RULES=0
one c3_gen2_$rep config3 30 "MM_GEMM_OVERRIDE=32000,512,0=2:256"
one c3_ff1p_$rep config3 30 "MM_GEMM_OVERRIDE=2048,512,0=2:256"
done

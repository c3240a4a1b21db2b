D=gpurun_out/r02bk
mkdir -p $D
one() {  # name cfg steps env...
  local name=$1; local cfg=$2; local steps=$3; shift 3
  env "$@" timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline > $D/b_$name.json 2> $D/b_$name.err
  echo "$name $(python -c "import json,sys; d=json.loads(open('$D/b_$name.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'])")"
}
for rep in 1 2; do
for mb in 48 24 96; do
one c3_$mb_$rep config3 30 MM_GEMM_L2_GROUP_MB=$mb
done
for mb in 48 24 96; do
one c5_${mb}_$rep config5 10 MM_GEMM_L2_GROUP_MB=$mb
done
done

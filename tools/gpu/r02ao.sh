D=gpurun_out/r02ao
mkdir -p $D
one() {  # name env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_$name.json 2> $D/b_$name.err
  echo "$name $(python -c "import json,sys; d=json.loads(open('$D/b_$name.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])")"
}
for rep in 1 2; do
one base$rep X=1
one tail$rep MM_DIAG_TAIL_UPDATE=1
done

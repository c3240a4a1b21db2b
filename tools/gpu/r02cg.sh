D=gpurun_out/r02cg
mkdir -p $D
one() { local name=$1; shift
  env "$@" timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_$name.json 2> $D/b_$name.err
  echo "$name $(python -c "import json; d=json.loads(open('$D/b_$name.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])")"
}
for rep in 1 2; do
one base_$rep X=1
one deferall_$rep MM_DEFER_ALL=1
done

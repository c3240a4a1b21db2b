D=gpurun_out/r02bm
mkdir -p $D
for rep in 1 2; do
for f in 0 1; do
  MM_FUSE_LN=$f timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${f}_$rep.json 2> $D/b_${f}_$rep.err
  echo "fuse_ln=$f $(python -c "import json; d=json.loads(open('$D/b_${f}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
done
done
for f in 0 1; do
  MM_FUSE_LN=$f timeout 600 python bench.py --config config5 --steps 10 --warmup 3 --no-cpu-baseline > $D/c5_${f}.json 2> $D/c5_${f}.err
  echo "c5 fuse_ln=$f $(python -c "import json; d=json.loads(open('$D/c5_${f}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])")"
done

D=gpurun_out/r02ax
mkdir -p $D
for rep in 1 2; do
for v in 0 1; do
  MM_PRIO_MAIN=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "prio=$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])")"
done
done
tail -3 $D/b_1_1.err

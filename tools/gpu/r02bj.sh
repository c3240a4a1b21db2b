D=gpurun_out/r02bj
mkdir -p $D
for rep in 1 2; do
for c in 0 148 74; do
  MM_LN_BWD_CTAS=$c timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${c}_$rep.json 2> $D/b_${c}_$rep.err
  echo "ctas=$c $(python -c "import json; d=json.loads(open('$D/b_${c}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
done
done

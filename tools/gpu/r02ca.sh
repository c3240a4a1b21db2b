D=gpurun_out/r02ca
mkdir -p $D
for rep in 1 2; do
for v in base lnrpw2; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
done
done

D=gpurun_out/r02ci
mkdir -p $D
for rep in 1 2 3; do
for v in base wide1; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
done
done
unset MM_LIB_VARIANT

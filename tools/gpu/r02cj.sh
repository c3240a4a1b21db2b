D=gpurun_out/r02cj
mkdir -p $D
for rep in 1 2 3; do
for v in base epi2; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
done
done
unset MM_LIB_VARIANT
for f in $D/b_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"; done

D=gpurun_out/r02bu
mkdir -p $D
for rep in 1 2; do
for v in small big; do
  if [ $v = big ]; then export MM_GEMM_NO_SMALL_GROUP=1; else unset MM_GEMM_NO_SMALL_GROUP; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/c3_${v}_$rep.json 2> $D/c3_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/c3_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")"
done
done
unset MM_GEMM_NO_SMALL_GROUP

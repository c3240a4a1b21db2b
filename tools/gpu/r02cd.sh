D=gpurun_out/r02cd
mkdir -p $D
MM_LIB_VARIANT=xent3 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "xent or entropy" > $D/t.log 2>&1; tail -n 1 $D/t.log
for rep in 1 2; do
for v in xent2 xent3; do
  export MM_LIB_VARIANT=$v
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
done
done
unset MM_LIB_VARIANT

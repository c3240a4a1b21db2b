D=gpurun_out/r02ch
mkdir -p $D
MM_LIB_VARIANT=wide1 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > $D/t.log 2>&1; tail -n 1 $D/t.log
for v in base wide1; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  echo $v; timeout 300 python tools/gemm_cold.py 2>&1 | tail -4
done
for rep in 1 2; do
for v in base wide1; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
done
done
unset MM_LIB_VARIANT

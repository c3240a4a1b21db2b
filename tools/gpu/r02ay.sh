D=gpurun_out/r02ay
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -x -k "attention or attn or block or long or step" > $D/t.log 2>&1
tail -n 2 $D/t.log
for v in base attnprev; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 300 python tools/attn_micro.py > $D/micro_$v.txt 2>&1; echo $v; tail -4 $D/micro_$v.txt
done
for rep in 1 2; do
for v in base attnprev; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])")"
done
done
unset MM_LIB_VARIANT

D=gpurun_out/r02aw
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "layernorm or ln" > $D/t.log 2>&1
tail -n 2 $D/t.log
for rep in 1 2; do
for v in base lnpf0; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])")"
done
done
unset MM_LIB_VARIANT

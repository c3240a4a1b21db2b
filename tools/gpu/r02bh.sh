D=gpurun_out/r02bh
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -x > $D/t.log 2>&1
tail -n 2 $D/t.log
timeout 300 python tools/gemm_trace.py > $D/trace.txt 2>&1; head -2 $D/trace.txt
for v in base nowide; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python tools/gemm_micro.py "fwd" "dgrad" > $D/micro_$v.txt 2>&1
done
unset MM_LIB_VARIANT
paste -d'\n' $D/micro_base.txt $D/micro_nowide.txt | cut -c1-120
for rep in 1 2; do
for v in base nowide; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")"
done
done
unset MM_LIB_VARIANT

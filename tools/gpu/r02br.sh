D=gpurun_out/r02br
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -x > $D/t.log 2>&1; tail -n 1 $D/t.log
for rep in 1 2; do
for sp in 1 0; do
  MM_GEMM_SPECIALIZE=$sp timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${sp}_$rep.json 2> $D/b_${sp}_$rep.err
  echo "spec=$sp $(python -c "import json; d=json.loads(open('$D/b_${sp}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")"
done
done
timeout 300 python tools/gemm_spans.py config3 > $D/spans.log 2>&1; tail -1 $D/spans.log

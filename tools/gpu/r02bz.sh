D=gpurun_out/r02bz
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -x > $D/t.log 2>&1; tail -n 1 $D/t.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/c3_$rep.json 2> $D/c3_$rep.err
  echo "c3 $(python -c "import json; d=json.loads(open('$D/c3_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])")"
done

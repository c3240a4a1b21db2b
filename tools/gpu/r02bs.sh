D=gpurun_out/r02bs
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_parity_shapes_gpu.py -q -x > $D/t.log 2>&1; tail -n 1 $D/t.log
for rep in 1 2; do
for sp in 1 0; do
  MM_GEMM_SPECIALIZE=$sp timeout 600 python bench.py --config config5 --steps 10 --warmup 3 --no-cpu-baseline > $D/c5_${sp}_$rep.json 2> $D/c5_${sp}_$rep.err
  echo "c5 spec=$sp $(python -c "import json; d=json.loads(open('$D/c5_${sp}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'])")"
done
done
for sp in 1 0; do
  MM_GEMM_SPECIALIZE=$sp timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/c3_${sp}.json 2> $D/c3_${sp}.err
  echo "c3 spec=$sp $(python -c "import json; d=json.loads(open('$D/c3_${sp}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")"
done

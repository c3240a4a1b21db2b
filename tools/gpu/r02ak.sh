D=gpurun_out/r02ak
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_parity_shapes_gpu.py -q -x > $D/t.log 2>&1
tail -n 2 $D/t.log
run() {  # name cfg steps flag
  MM_RESID_EARLY=$4 timeout 600 python bench.py --config $2 --steps $3 --warmup 3 --no-cpu-baseline > $D/$1.json 2> $D/$1.err
  echo "$1 $(python -c "import json,sys; d=json.loads(open('$D/$1.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'])")"
}
for rep in 1 2 3; do
run c3_e1_$rep config3 30 1
run c3_e0_$rep config3 30 0
done
run c5_e1 config5 10 1
run c5_e0 config5 10 0
MM_RESID_EARLY=1 timeout 300 python tools/gemm_spans.py config3 > $D/spans_e1.log 2>&1
MM_RESID_EARLY=0 timeout 300 python tools/gemm_spans.py config3 > $D/spans_e0.log 2>&1

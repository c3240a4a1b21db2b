D=gpurun_out/r02an
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -x > $D/t.log 2>&1
tail -n 2 $D/t.log
one() {  # name env...
  local name=$1; shift
  env "$@" timeout 300 python tools/gemm_spans.py config3 > $D/spans_$name.log 2>&1
  env "$@" timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_$name.json 2> $D/b_$name.err
  echo "$name $(python -c "import json,sys; d=json.loads(open('$D/b_$name.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])") $(tail -n 1 $D/spans_$name.log)"
}
for rep in 1 2; do
one col$rep X=1
one row$rep MM_LIB_VARIANT=rowmask
done

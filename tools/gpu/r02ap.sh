D=gpurun_out/r02ap2
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "adam" > $D/tk.log 2>&1
tail -n 2 $D/tk.log
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x -k "fused_update or store_first" > $D/te.log 2>&1
tail -n 2 $D/te.log
one() {  # name cfg steps env...
  local name=$1; local cfg=$2; local steps=$3; shift 3
  env "$@" timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline > $D/b_$name.json 2> $D/b_$name.err
  echo "$name $(python -c "import json,sys; d=json.loads(open('$D/b_$name.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['frac'])")"
}
for rep in 1 2; do
one c3f$rep config3 30 MM_FUSE_UPDATE=1
one c3u$rep config3 30 MM_FUSE_UPDATE=0
done
one c5f config5 10 MM_FUSE_UPDATE=1
one c5u config5 10 MM_FUSE_UPDATE=0
MM_FUSE_UPDATE=1 timeout 300 python tools/gemm_spans.py config3 > $D/spans_f.log 2>&1
MM_FUSE_UPDATE=0 timeout 300 python tools/gemm_spans.py config3 > $D/spans_u.log 2>&1
tail -n 1 $D/spans_f.log; tail -n 1 $D/spans_u.log

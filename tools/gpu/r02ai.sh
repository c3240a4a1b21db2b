D=gpurun_out/r02ai
mkdir -p $D
run() {  # name cfg steps override
  MM_GEMM_OVERRIDE="$4" timeout 600 python bench.py --config $2 --steps $3 --warmup 3 --no-cpu-baseline > $D/$1.json 2> $D/$1.err
  echo "$1 $(python -c "import json,sys; d=json.loads(open('$D/$1.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])")"
}
for rep in 1 2; do
run c3_base$rep config3 30 ""
run c3_gen$rep config3 30 "32000,512,0=1:256"
run c3_dgen$rep config3 30 "512,32000,1=2:128"
run c3_dff2$rep config3 30 "2048,512,1=1:256"
run c3_qkv$rep config3 30 "1536,512,0=1:192"
done
for rep in 1 2; do
run c5_base$rep config5 10 ""
run c5_out$rep config5 10 "1024,1024,0=2:256"
run c5_ff2$rep config5 10 "1024,4096,0=2:256;1024,4096,1=2:256"
done

D=gpurun_out/r02be
mkdir -p $D
for rep in 1 2; do
for mc in 0 1; do
  MM_GEMM_MC=$mc timeout 600 python bench.py --config config5 --steps 10 --warmup 3 --no-cpu-baseline > $D/c5_${mc}_$rep.json 2> $D/c5_${mc}_$rep.err
  echo "c5 mc=$mc $(python -c "import json; d=json.loads(open('$D/c5_${mc}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])")"
done
for mc in 0 1; do
  MM_GEMM_MC=$mc timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/c3_${mc}_$rep.json 2> $D/c3_${mc}_$rep.err
  echo "c3 mc=$mc $(python -c "import json; d=json.loads(open('$D/c3_${mc}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])")"
done
done

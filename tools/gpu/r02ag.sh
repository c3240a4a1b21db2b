D=gpurun_out/r02ag2
mkdir -p $D
for rep in 1 2; do
for c in 0 148; do
  MM_OVERLAP_CTAS=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/c3_$c.$rep.json 2> $D/c3_$c.$rep.err
  echo "c3 ctas=$c rep=$rep $(python -c "import json,sys; d=json.loads(open('$D/c3_$c.$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])")"
done
done
MM_OVERLAP_CTAS=148 MM_DEFER_UPDATE=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/c3_nodefer.json 2>&1
echo "c3 ctas=148 nodefer $(python -c "import json,sys; d=json.loads(open('$D/c3_nodefer.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
MM_OVERLAP_CTAS=0 MM_DEFER_UPDATE=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/c3_nodefer0.json 2>&1
echo "c3 ctas=0 nodefer $(python -c "import json,sys; d=json.loads(open('$D/c3_nodefer0.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"

# A/B: LayerNorm-backward column-sum atomics dropped (diagnostics variant) vs release, same box
D=gpurun_out/r02lnab; mkdir -p $D
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline --steps 50 --warmup 5 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('release', d['ms_per_step'])" >> $D/ab.txt
  MM_LIB_VARIANT=noatom timeout 600 python bench.py --no-cpu-baseline --steps 50 --warmup 5 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noatom', d['ms_per_step'])" >> $D/ab.txt
done
cat $D/ab.txt

D=gpurun_out/r02au
mkdir -p $D
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x -k "train" > $D/t.log 2>&1
tail -n 2 $D/t.log
for rep in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b$rep.json 2> $D/b$rep.err
python -c "import json; d=json.loads(open('$D/b$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'])"
done

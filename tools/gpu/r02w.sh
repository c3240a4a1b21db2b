timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02w_bench.log 2>&1
timeout 600 python bench.py --workload reduce --steps 10 --warmup 2 > gpurun_out/r02w_reduce.log 2>&1
tail -n 1 gpurun_out/r02w_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['clocks'], d['ms_per_step'], d['roofline']['frac'])"
tail -n 1 gpurun_out/r02w_reduce.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['clocks'], d['value'])"

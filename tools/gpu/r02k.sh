set -x
D=gpurun_out/r02k
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $D/smi.txt
timeout 900 python bench.py > $D/bench_c3.log 2>&1
timeout 900 python bench.py --config config4 --no-cpu-baseline > $D/bench_c4.log 2>&1
timeout 900 python bench.py --config config5 --no-cpu-baseline --steps 20 > $D/bench_c5.log 2>&1
timeout 900 python bench.py --workload reduce > $D/bench_reduce.log 2>&1
timeout 900 python bench.py --workload exchange > $D/bench_exchange.log 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $D/bench_ref.log 2>&1
MM_GEMM_LOG=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $D/step_c3.csv python tools/profile_step.py > $D/step_c3.out 2> $D/step_c3_gemm.log
timeout 300 python tools/gemm_traffic.py $D/step_c3.csv $D/step_c3_gemm.log $D/gemm_traffic.json > /dev/null 2>&1
CFG=config5 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $D/step_c5.csv python tools/profile_step.py > $D/step_c5.out 2>&1
timeout 600 python tools/gemm_micro.py > $D/gemm_micro.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05 -s 3 -c 1 -o $D/gemm_ff1 python tools/gemm_micro.py "fwd ff1" > $D/ncu_ff1.out 2>&1
ncu -i $D/gemm_ff1.ncu-rep --page details --csv > $D/ncu_gemm_ff1_details.csv 2>/dev/null
for f in bench_c3 bench_c4 bench_c5 bench_reduce bench_exchange bench_ref; do tail -n 1 $D/$f.log | cut -c1-250; done

# round-2 final evidence (second pass, final build): tests, smoke, bench lines,
# GEMM spans, ncu launch lists + GEMM DRAM traffic, cuBLAS tables, and
# ncu --set full captures of the step's top kernels
D=gpurun_out/r02final5
mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_all.log 2>&1
tail -n 1 $D/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1
tail -n 1 $D/smoke.log
timeout 900 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
timeout 900 python bench.py --config config4 --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/bench_c5.json 2> $D/bench_c5.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $D/bench_reference.json 2> $D/bench_reference.err
timeout 900 python bench.py --workload reduce > $D/bench_reduce.json 2> $D/bench_reduce.err
timeout 900 python bench.py --workload exchange > $D/bench_exchange.json 2> $D/bench_exchange.err
for f in $D/bench_*.json; do echo $f; tail -n 1 $f | cut -c1-200; done
timeout 300 python tools/gemm_spans.py config3 > $D/gemm_spans_c3.log 2>&1
tail -n 1 $D/gemm_spans_c3.log
MM_GEMM_LOG=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $D/launches_c3.csv python tools/profile_step.py > $D/step_c3.out 2> $D/step_c3_gemm.log
timeout 300 python tools/gemm_traffic.py $D/launches_c3.csv $D/step_c3_gemm.log $D/gemm_traffic.json > $D/gemm_traffic.out 2>&1
python tools/ncu_summary.py $D/launches_c3.csv > $D/launch_summary_c3.txt 2>&1
CFG=config5 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $D/launches_c5.csv python tools/profile_step.py > $D/step_c5.out 2>&1
python tools/ncu_summary.py $D/launches_c5.csv > $D/launch_summary_c5.txt 2>&1
full() {  # name, ncu selection args...
  local name=$1; shift
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on "$@" -o $D/$name python tools/profile_step.py > $D/ncu_$name.out 2>&1
  ncu -i $D/$name.ncu-rep --page details --csv > $D/ncu_${name}_details.csv 2>/dev/null
  rm -f $D/$name.ncu-rep  # the merged gpurun_out/ must stay under 64 MiB
}
full gemm_ff1 -k regex:gemm_tcgen05 -s 2 -c 1
full gemm_wgrad_dec -k regex:gemm_tcgen05 -s 99 -c 1
full attn_bwd -k regex:attn_bwd_tc -c 1
full fused_update -k regex:fused_update -c 1
full ln_bwd -k regex:ln_bwd_row -c 1
timeout 900 python tools/gemm_micro.py fwd dgrad wgrad tiny big maj odd > $D/gemm_vs_cublas.txt 2>&1
timeout 900 python tools/gemm_micro.py c5 > $D/gemm_vs_cublas_c5.txt 2>&1
ls $D

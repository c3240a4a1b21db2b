# evidence refresh after the attention changes: launch lists + DRAM per kernel
# (configs 3 and 5), GEMM traffic, and the attention backward ncu --set full
D=gpurun_out/r02final6
mkdir -p $D
MM_GEMM_LOG=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $D/launches_c3.csv python tools/profile_step.py > $D/step_c3.out 2> $D/step_c3_gemm.log
timeout 300 python tools/gemm_traffic.py $D/launches_c3.csv $D/step_c3_gemm.log $D/gemm_traffic.json > $D/gemm_traffic.out 2>&1
python tools/ncu_summary.py $D/launches_c3.csv > $D/launch_summary_c3.txt 2>&1
CFG=config5 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $D/launches_c5.csv python tools/profile_step.py > $D/step_c5.out 2>&1
python tools/ncu_summary.py $D/launches_c5.csv > $D/launch_summary_c5.txt 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_bwd_tc -c 1 -o $D/attn_bwd python tools/profile_step.py > $D/ncu_attn_bwd.out 2>&1
ncu -i $D/attn_bwd.ncu-rep --page details --csv > $D/ncu_attn_bwd_details.csv 2>/dev/null
rm -f $D/*.ncu-rep
head -n 12 $D/launch_summary_c3.txt; head -n 16 $D/launch_summary_c5.txt; cat $D/gemm_traffic.out | tail -3

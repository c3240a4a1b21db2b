# config 1 at its true shape: one step without ncu (must exit 0), then its
# launch list under ncu (time + DRAM per kernel)
D=gpurun_out/r02c1prof; mkdir -p $D
CFG=config1 timeout 300 python tools/profile_step.py > $D/plain.out 2>&1; echo "plain rc=$?"; tail -n 2 $D/plain.out
CFG=config1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $D/launches_c1.csv python tools/profile_step.py > $D/step_c1.out 2>&1
python tools/ncu_summary.py $D/launches_c1.csv > $D/launch_summary_c1.txt 2>&1
cat $D/launch_summary_c1.txt | head -30

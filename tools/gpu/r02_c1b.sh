# after staging attn_small rows in smem and the row-per-CTA cross-entropy for V < 4096:
# whole GPU suite, smoke, config-1 launch list
D=gpurun_out/r02c1b; mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_all.log 2>&1
tail -n 3 $D/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1
tail -n 1 $D/smoke.log
CFG=config1 timeout 300 python tools/profile_step.py > $D/plain.out 2>&1; echo "plain rc=$?"
CFG=config1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $D/launches_c1.csv python tools/profile_step.py > $D/step_c1.out 2>&1
python tools/ncu_summary.py $D/launches_c1.csv > $D/launch_summary_c1.txt 2>&1
head -n 8 $D/launch_summary_c1.txt

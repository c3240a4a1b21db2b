D=gpurun_out/r02bf
mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $D/gpu_all.log 2>&1
tail -n 2 $D/gpu_all.log

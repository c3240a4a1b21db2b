set -x
D=gpurun_out/r02z
mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_all.log 2>&1
tail -n 15 $D/gpu_all.log

set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
MM_PARITY_OUT=gpurun_out/r02a/parity.json timeout 900 python -m pytest tests/test_parity_shapes_gpu.py -q -s > gpurun_out/r02a/parity.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py tests/test_sync_gpu.py tests/test_peer_gpu.py -q -x -p no:cacheprovider > gpurun_out/r02a/san_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/r02a/san_summary.txt
done
tail -3 gpurun_out/r02a/parity.log
cat gpurun_out/r02a/san_summary.txt

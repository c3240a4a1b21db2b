set -x
D=gpurun_out/r02p
mkdir -p $D
MM_LIB_VARIANT=dbg timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_dbg.log 2>&1
echo "dbg exit $?" >> $D/summary.txt
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_all.log 2>&1
echo "all exit $?" >> $D/summary.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
echo "smoke exit $?" >> $D/summary.txt
cat $D/summary.txt; tail -n 3 $D/gpu_dbg.log $D/gpu_all.log $D/smoke.log

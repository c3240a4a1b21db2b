D=gpurun_out/r02bx
mkdir -p $D
for v in base maskcol; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  echo $v; timeout 300 python tools/gemm_cold.py 2>&1 | tail -2
done
unset MM_LIB_VARIANT

# whole GPU suite against the bounds-checked debug build (incl. the head_dim-16 kernels), then release
D=gpurun_out/r02dbg2; mkdir -p $D
MM_LIB_VARIANT=dbg timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/dbg.log 2>&1
tail -n 1 $D/dbg.log
grep -c "MM_DCHECK failed" $D/dbg.log

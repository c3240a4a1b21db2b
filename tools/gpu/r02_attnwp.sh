# attention-backward wait breakdown (diagnostics variant built here)
D=gpurun_out/r02_attnwp
mkdir -p $D
MM_LIB_VARIANT=attn_wp timeout 300 python tools/attn_waitprof.py > $D/c3.log 2>&1
MM_LIB_VARIANT=attn_wp C5=1 timeout 300 python tools/attn_waitprof.py > $D/c5.log 2>&1
cat $D/c3.log $D/c5.log | tail -n 20

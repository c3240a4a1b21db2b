D=gpurun_out/r02at
mkdir -p $D
timeout 300 python tools/attn_micro.py > $D/micro.txt 2>&1; cat $D/micro.txt | tail -4
MM_LIB_VARIANT=attn_trace timeout 300 python tools/attn_micro.py > $D/trace.txt 2>&1; tail -3 $D/trace.txt
MM_LIB_VARIANT=attn_wp timeout 300 python tools/attn_waitprof.py > $D/wp.txt 2>&1; tail -3 $D/wp.txt

# attention backward: warm timing + ncu source-level capture (config 5 shapes)
D=gpurun_out/r02_attnsrc2
mkdir -p $D
REPS=20 timeout 300 python tools/attn_waitprof.py > $D/c3_warm.log 2>&1
C5=1 REPS=20 timeout 300 python tools/attn_waitprof.py > $D/c5_warm.log 2>&1
C5=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_tc -s 1 -c 1 \
  -o $D/bwd_c5 python tools/attn_waitprof.py > $D/ncu.log 2>&1
ncu -i $D/bwd_c5.ncu-rep --page source --csv --print-source sass > $D/src_sass.csv 2> $D/src.err
ncu -i $D/bwd_c5.ncu-rep --page details --csv > $D/details.csv 2>> $D/src.err
ncu -i $D/bwd_c5.ncu-rep --page raw --csv > $D/raw.csv 2>> $D/src.err
rm -f $D/*.ncu-rep
ls -la $D; cat $D/c3_warm.log $D/c5_warm.log; tail -3 $D/ncu.log

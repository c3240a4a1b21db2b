# attention forward (config-3 shapes): ncu source-level capture
D=gpurun_out/r02_fwdsrc
mkdir -p $D
MM_ATTN_TC_FWD=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_tc -s 0 -c 1 \
  -o $D/fwd_c3 python tools/attn_waitprof.py > $D/ncu.log 2>&1
ncu -i $D/fwd_c3.ncu-rep --page source --csv --print-source sass > $D/src_sass.csv 2> $D/src.err
ncu -i $D/fwd_c3.ncu-rep --page details --csv > $D/details.csv 2>> $D/src.err
rm -f $D/*.ncu-rep
tail -3 $D/ncu.log

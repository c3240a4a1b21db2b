D=gpurun_out/r02ba
mkdir -p $D
for shp in "4096 2048 512" "4096 512 2048" "4096 1536 512" "4096 512 512"; do
  set -- $shp
  timeout 300 ncu --set full --clock-control none -k regex:"nvjet|gemm|Kernel" -s 2 -c 2 -o $D/g_$1_$2_$3 python tools/gemm_one.py $1 $2 $3 > $D/ncu_$1_$2_$3.out 2>&1
  ncu -i $D/g_$1_$2_$3.ncu-rep --page details --csv > $D/g_$1_$2_$3.csv 2>/dev/null
  python - <<PY
import csv
rows=list(csv.reader(open('$D/g_$1_$2_$3.csv')))
seen=set()
for r in rows[1:]:
    if len(r)>14 and r[12] in ('Duration','L2 Cache Throughput','SM Active Cycles','Elapsed Cycles','Cluster Size','Grid Size','Block Size'):
        print('$1x$2x$3', r[4][:60], r[12], r[14])
    if len(r)>14 and 'highest-utilized pipeline' in r[12]+r[13]+r[14]:
        pass
PY
done

set -x
D=gpurun_out/r02r
mkdir -p $D
export MM_LIB_VARIANT=bn64
timeout 300 env MM_GEMM_BN=64 python tools/gemm_micro.py "fwd out" "fwd ff2" "dgrad out" "dgrad ff1" > $D/micro64.log 2>&1
for o in "none" "512,512,0=1:64" "512,2048,0=1:64" "512,512,0=1:64;512,2048,0=1:64;512,512,1=1:64;512,2048,1=1:64;512,1536,1=1:64;512,1024,1=1:64"; do
  tag=$(echo "$o" | md5sum | cut -c1-6)
  if [ "$o" = "none" ]; then unset MM_GEMM_OVERRIDE; else export MM_GEMM_OVERRIDE="$o"; fi
  echo "$tag $o" >> $D/tags.txt
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/bench_$tag.log 2>&1
done
cat $D/micro64.log; cat $D/tags.txt
for f in $D/bench_*.log; do echo $f; tail -n 1 $f | cut -c1-160; done

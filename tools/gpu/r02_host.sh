# host-side cost of the end-to-end path per config
D=gpurun_out/r02_host
mkdir -p $D
for c in config3 config4 config5; do timeout 600 python tools/host_profile.py $c > $D/$c.log 2>&1; done
grep -h "config" $D/*.log | grep ms/step
head -n 45 $D/config4.log | tail -n 30

# same-box A/B of the release build against a variant (MM_LIB_VARIANT=$V):
# alternating config-3 bench runs, then one config-5 pair
V=${V:-attnprev}
D=gpurun_out/r02_ab_$V
mkdir -p $D
for r in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline > $D/new_c3_$r.json 2> /dev/null
  MM_LIB_VARIANT=$V timeout 900 python bench.py --no-cpu-baseline > $D/old_c3_$r.json 2> /dev/null
done
timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/new_c5.json 2> /dev/null
MM_LIB_VARIANT=$V timeout 900 python bench.py --config config5 --no-cpu-baseline > $D/old_c5.json 2> /dev/null
for f in $D/*.json; do echo "$f $(tail -n 1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")"; done

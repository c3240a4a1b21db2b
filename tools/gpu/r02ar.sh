D=gpurun_out/r02ar
mkdir -p $D
timeout 1800 python -m pytest tests -q -m gpu -x -k "adam or update or peer or sync or multirank or engine" > $D/t.log 2>&1
tail -n 2 $D/t.log

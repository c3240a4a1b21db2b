D=gpurun_out/r02as
mkdir -p $D
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > $D/tr1.json 2> $D/tr1.err
echo "rc=$?"; tail -n 1 $D/tr1.json | cut -c1-300; tail -n 3 $D/tr1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $D/tr1_ref.json 2> $D/tr1_ref.err
echo "rc=$?"; tail -n 1 $D/tr1_ref.json | cut -c1-300

# config 1 at its true shape (head_dim 16): new kernels' tests first, then the
# whole GPU suite, smoke and the config-3 bench line (no-regression check)
D=gpurun_out/r02c1
mkdir -p $D
timeout 900 python -m pytest tests/test_config1_true_shape_gpu.py -q -x -p no:cacheprovider > $D/c1.log 2>&1
tail -n 30 $D/c1.log
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "layernorm or embedding" > $D/k.log 2>&1
tail -n 5 $D/k.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/gpu_all.log 2>&1
tail -n 15 $D/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1
tail -n 1 $D/smoke.log
timeout 900 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
tail -c 600 $D/bench_c3.json

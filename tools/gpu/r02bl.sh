D=gpurun_out/r02bl
mkdir -p $D
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -x -k "embed or step or block or oracle" > $D/t.log 2>&1
tail -n 2 $D/t.log
# bit-identity of the embedding forward vs the previous (on-the-fly sincos) kernel
cat > $D/emb.py <<'PY'
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
g = torch.Generator(device="cuda").manual_seed(3)
for rows, cols, npos in ((4096, 512, 128), (16384, 1024, 256), (333, 128, 40)):
    ids = torch.randint(0, 32000, (rows,), device=dev, dtype=torch.int32, generator=g)
    pos = torch.randint(0, npos, (rows,), device=dev, dtype=torch.int32, generator=g)
    table = torch.randn(32000, cols, device=dev, generator=g).bfloat16()
    out = torch.empty(rows, cols, device=dev)
    ops.embed_fwd(ids, pos, table, out, cols ** 0.5)
    torch.cuda.synchronize()
    np.save(os.environ["OUT"] + f"_{rows}_{cols}.npy", out.cpu().numpy())
print("ok")
PY
OUT=$D/new timeout 300 python $D/emb.py
MM_LIB_VARIANT=embprev OUT=$D/old timeout 300 python $D/emb.py
python -c "
import numpy as np
for r,c in ((4096,512),(16384,1024),(333,128)):
    a=np.load('$D/new_%d_%d.npy'%(r,c)); b=np.load('$D/old_%d_%d.npy'%(r,c)); print(r,c,'bit-identical', np.array_equal(a,b))
"
rm -f $D/*.npy
for rep in 1 2; do
for v in base embprev; do
  if [ $v = base ]; then unset MM_LIB_VARIANT; else export MM_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $D/b_${v}_$rep.json 2> $D/b_${v}_$rep.err
  echo "$v $(python -c "import json; d=json.loads(open('$D/b_${v}_$rep.json').read().strip().splitlines()[-1]); print(d['ms_per_step'])")"
done
done
unset MM_LIB_VARIANT

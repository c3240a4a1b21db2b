import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
sys.path.insert(0, "tests")
from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.domain import ClusterTopology, DeviceId
from paper_2403_07544_b200.engine import DeviceBatch, Engine
from test_engine_gpu import batches_for
cuda = torch.device("cuda:0")
shape = configs.SHAPE_CFG1_GPU
w = configs.config1(shape)
tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, rank=0, world=1, device=cuda, seed=0)
hb = batches_for(1, 1, shape)[0]
print("rows", hb[0].tgt_in.shape if hasattr(hb[0], "tgt_in") else None)
info = eng.step(0, [DeviceBatch(b, cuda) for b in hb])
torch.cuda.synchronize()
for k, st in eng.states.items():
    g = st.grad
    n = torch.isnan(g).sum().item()
    if n or "decoder:-1" in str(k):
        print(k, "nan", n, "norm", torch.nan_to_num(g).norm().item())

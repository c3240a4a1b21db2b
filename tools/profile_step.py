"""Run config 3 for a few warm-up steps, then one step inside a
cudaProfilerStart/Stop range (for ncu --profile-from-start off)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.data import ZipfIds, make_batch
from paper_2403_07544_b200.engine import DeviceBatch, Engine
dev = torch.device("cuda:0")
wl = getattr(configs, os.environ.get("CFG", "config3"))(1)
eng = Engine(wl.tasks, wl.topo, wl.shape, device=dev)
ids = ZipfIds(wl.shape.vocab, wl.data.zipf_s)
rng = np.random.default_rng([0, 0])
dbs = [DeviceBatch(make_batch(rng, wl.data, wl.shape.vocab, ids=ids), dev) for _ in range(5)]
for s in range(4):
    eng.step(s, [dbs[s]])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.step(4, [dbs[4]])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")

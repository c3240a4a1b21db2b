"""Run config 3 (or CFG=config4 / config5 / config1) for a few warm-up steps,
then one step inside a cudaProfilerStart/Stop range (for ncu
--profile-from-start off).  config1: its true shape (d64, head_dim 16), all
three tasks on one rank, 1024-sentence micro-batches."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.data import ZipfIds, make_batch
from paper_2403_07544_b200.engine import DeviceBatch, Engine
dev = torch.device("cuda:0")
cfg = os.environ.get("CFG", "config3")
sentences = None
if cfg == "config1":
    from paper_2403_07544_b200.domain import ClusterTopology, DeviceId
    wl = configs.config1()
    eng = Engine([t.with_device(DeviceId(0, 0)) for t in wl.tasks], ClusterTopology(1, 1, 3), wl.shape,
                 device=dev)
    sentences = 1024
else:
    wl = getattr(configs, cfg)(1)
    eng = Engine(wl.tasks, wl.topo, wl.shape, device=dev)
ids = ZipfIds(wl.shape.vocab, wl.data.zipf_s)
rng = np.random.default_rng([0, 0])
dbs = [DeviceBatch(make_batch(rng, wl.data, wl.shape.vocab, ids=ids, sentences=sentences), dev)
       for _ in range(5)]
for s in range(4):
    eng.step(s, [dbs[s]])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.step(4, [dbs[4]])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")

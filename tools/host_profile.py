"""cProfile of Trainer.train_step (config 3, one GPU): where the host time of
the end-to-end path goes (the GPU idles while train_step stages a batch after
the previous step's loss read)."""
import cProfile, os, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.data import ZipfIds, make_batch
from paper_2403_07544_b200.engine import Trainer
dev = torch.device("cuda:0")
wl = configs.config3(1)
tr = Trainer(wl.tasks, wl.topo, wl.shape, device=dev)
ids = ZipfIds(wl.shape.vocab, wl.data.zipf_s)
rng = np.random.default_rng(0)
hb = [make_batch(rng, wl.data, wl.shape.vocab, ids=ids) for _ in range(40)]
for b in hb[:5]:
    tr.train_step([b])
torch.cuda.synchronize()
t0 = time.perf_counter()
host = 0.0
for b in hb[5:20]:
    h0 = time.perf_counter()
    dbs = tr.stage([b])
    tr.engine.step(tr.step_idx, dbs)
    host += time.perf_counter() - h0
    tr.step_idx += 1
    tr._loss_host.copy_(tr.engine.loss_sum, non_blocking=True)
    torch.cuda.current_stream().synchronize()
dt = (time.perf_counter() - t0) / 15
print(f"e2e {dt*1e3:.3f} ms/step, host issue {host/15*1e3:.3f} ms/step")
pr = cProfile.Profile()
pr.enable()
for b in hb[20:40]:
    tr.train_step([b])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

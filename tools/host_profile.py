"""cProfile of Trainer.train_step (one GPU): where the host time of the
end-to-end path goes.  python tools/host_profile.py [config3|config4|config5]
prints per step: the staging (host batch -> device tables) and the engine's
issue time, each with the GPU idle (a sync after every step), the GPU step
time, and the lookahead e2e of Trainer.train_steps."""
import cProfile, os, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.data import ZipfIds, make_batch
from paper_2403_07544_b200.engine import Trainer
dev = torch.device("cuda:0")
name = sys.argv[1] if len(sys.argv) > 1 else "config3"
wl = getattr(configs, name)(1)
tr = Trainer(wl.tasks, wl.topo, wl.shape, device=dev)
ids = ZipfIds(wl.shape.vocab, wl.data.zipf_s)
rng = np.random.default_rng(0)
hb = [make_batch(rng, wl.data, wl.shape.vocab, ids=ids) for _ in range(40)]
for b in hb[:5]:
    tr.train_step([b])
torch.cuda.synchronize()
t0 = time.perf_counter()
stage = issue = 0.0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
gpu = 0.0
for b in hb[5:20]:
    h0 = time.perf_counter()
    dbs = tr.stage([b])
    h1 = time.perf_counter()
    e0.record()
    tr.engine.step(tr.step_idx, dbs)
    e1.record()
    issue += time.perf_counter() - h1
    stage += h1 - h0
    tr.step_idx += 1
    tr._loss_host.copy_(tr.engine.loss_sum, non_blocking=True)
    torch.cuda.synchronize()
    gpu += e0.elapsed_time(e1)
dt = (time.perf_counter() - t0) / 15
print(f"{name}: serial {dt*1e3:.3f} ms/step = stage {stage/15*1e3:.3f} + issue {issue/15*1e3:.3f} "
      f"(GPU busy {gpu/15:.3f} ms)")
tr.engine.sync_updates()
torch.cuda.synchronize()
t0 = time.perf_counter()
tr.train_steps(([b] for b in hb[20:40]), 20)
tr.engine.sync_updates()
torch.cuda.synchronize()
print(f"{name}: train_steps lookahead {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms/step")
pr = cProfile.Profile()
pr.enable()
for b in hb[20:40]:
    tr.train_step([b])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

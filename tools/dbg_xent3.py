import os, sys, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", ".")); sys.path.insert(0, "tests")
from paper_2403_07544_b200 import configs, ops
from paper_2403_07544_b200.domain import ClusterTopology, DeviceId
from paper_2403_07544_b200.engine import DeviceBatch, Engine
from test_engine_gpu import batches_for
cuda = torch.device("cuda:0")
orig = ops.xent
def hook(logits, labels, dlogits, row_loss, grad_scale, loss_sum=None):
    src = logits.clone(); lab = labels.clone()
    orig(logits, labels, dlogits, row_loss, grad_scale, loss_sum)
    torch.cuda.synchronize()
    bad = torch.isnan(dlogits.float())
    print("xent rows", logits.shape, "nan", bad.sum().item(), "ptr%16", logits.data_ptr() % 16, "labels min/max", lab.min().item(), lab.max().item())
    if bad.any():
        r, c = bad.nonzero()[0].tolist()
        print("first bad", r, c, "label", lab[r].item(), "logit", src[r, c].item(), "rowmax", src[r].float().max().item())
        rows_bad = bad.any(1).nonzero().flatten().tolist()
        print("bad rows", rows_bad[:20], len(rows_bad), "cols per row", bad.sum(1)[rows_bad[:5]].tolist())
        print("contig", logits.is_contiguous(), logits.stride())
ops.xent = hook
import paper_2403_07544_b200.engine as E
E.ops.xent = hook
shape = configs.SHAPE_CFG1_GPU
w = configs.config1(shape)
tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, rank=0, world=1, device=cuda, seed=0)
eng.native = False
hb = batches_for(1, 1, shape)[0]
info = eng.step(0, [DeviceBatch(b, cuda) for b in hb])
torch.cuda.synchronize()
for k, st in eng.states.items():
    n = torch.isnan(st.grad).sum().item()
    if n: print(k, "nan", n)

"""Diagnostics: run one config-1 engine step through the per-op Python path
and report the first library op after which any tensor argument holds a NaN."""
import os, sys, functools, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", ".")); sys.path.insert(0, "tests")
from paper_2403_07544_b200 import configs, ops
from paper_2403_07544_b200.domain import ClusterTopology, DeviceId
import paper_2403_07544_b200.engine as E
from test_engine_gpu import batches_for
cuda = torch.device("cuda:0")
state = {"n": 0, "found": 0}
def wrap(name, fn):
    @functools.wraps(fn)
    def inner(*a, **k):
        ts = [x for x in list(a) + list(k.values()) if torch.is_tensor(x) and x.is_floating_point()]
        ts += [x for v in list(a) + list(k.values()) if isinstance(v, (list, tuple)) for d in v if isinstance(d, dict) for x in d.values() if torch.is_tensor(x) and x.is_floating_point()]
        torch.cuda.synchronize()
        before = [torch.isnan(x).any().item() for x in ts]
        r = fn(*a, **k)
        torch.cuda.synchronize()
        state["n"] += 1
        new = [i for i, x in enumerate(ts) if not before[i] and torch.isnan(x).any().item()]
        if "attention" in name and state["found"] < 5:
            for i, x in enumerate(ts):
                nn = torch.isnan(x)
                if nn.any():
                    rows = nn.any(1).nonzero().flatten().tolist() if x.dim() == 2 else []
                    cols = nn.any(0).nonzero().flatten().tolist() if x.dim() == 2 else []
                    print("  after", state["n"], name, "arg", i, tuple(x.shape), "nan", nn.sum().item(),
                          "rows", rows[:12], "cols", cols[:4], "...", len(cols))
        if new and state["found"] < 5:
            state["found"] += 1
            print("new NaN after op", state["n"], name, [tuple(ts[i].shape) for i in new],
                  "inputs with NaN before:", [tuple(ts[i].shape) for i, b in enumerate(before) if b])
        return r
    return inner
for name in dir(ops):
    f = getattr(ops, name)
    if callable(f) and not name.startswith("_") and name not in ("stream_ptr", "lib"):
        setattr(ops, name, wrap(name, f))
E.ops = ops
shape = configs.SHAPE_CFG1_GPU
w = configs.config1(shape)
tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
eng = E.Engine(tasks, ClusterTopology(1, 1, 3), shape, rank=0, world=1, device=cuda, seed=0)
eng.native = False
hb = batches_for(1, 1, shape)[0]
eng.step(0, [E.DeviceBatch(b, cuda) for b in hb])
torch.cuda.synchronize()
print("ops", state["n"], "nan grads", sum(torch.isnan(st.grad).sum().item() for st in eng.states.values()))

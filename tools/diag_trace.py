import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_engine_gpu import effective_weights, batches_for
from oracle import transformer as OT
from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.domain import ClusterTopology, DeviceId
from paper_2403_07544_b200.engine import DeviceBatch, Engine
from paper_2403_07544_b200.plan import embedding_keys
cuda = torch.device("cuda:0")
shape = configs.SHAPE_CFG1_GPU
w = configs.config1(shape)
tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, device=cuda)
eng.trace = {}
hb = batches_for(1, 1, shape)[0]
m0 = {k: st.master.cpu().numpy().copy() for k, st in eng.states.items()}
info = eng.step(0, [DeviceBatch(b, cuda) for b in hb])
torch.cuda.synchronize()
tb = {t.id: t for t in tasks}; task = tb[info["tasks"][0]]
flats = {k: torch.tensor(effective_weights(eng.layouts[k], v), requires_grad=True) for k, v in m0.items()}
tr = {}
loss = OT.task_loss(task, hb[0], flats, eng.layouts, shape, embedding_keys(task), bf16=True, trace=tr)
loss.backward()
def cmp(name, g, r):
    g = g.double(); r = r.detach().double()
    print(f"{name:10s} maxrel {((g-r).abs().max()/r.abs().max()).item():.3e} normrel {((g-r).norm()/r.norm()).item():.3e}")
for n in ["emb_src", "enc_l0_attn", "enc_l0_ffn", "enc_l1_attn", "enc_l1_ffn", "x_enc", "mem", "y_dec", "hdec", "logits"]:
    cmp(n, eng.trace[n], tr[n])
cmp("dlogits", eng.trace["dlogits"], tr["logits"].grad)
cmp("dy_top", eng.trace["dy_top"], tr["y_dec"].grad)
cmp("dmem", eng.trace["dmem"], tr["mem"].grad)
cmp("dx_top", eng.trace["dx_bottom"], tr["x_enc"].grad) if False else None
for i in (1, 0):
    p = f"l{i}."
    cmp(p + "ckv", eng.trace[p + "ckv"], tr[p + "ckv"])
    cmp(p + "ca", eng.trace[p + "ca"], tr[p + "ca"])
    cmp(p + "dckv", eng.trace[p + "dckv"], tr[p + "ckv"].grad)
    cmp(p + "dca", eng.trace[p + "dca"], tr[p + "ca"].grad)

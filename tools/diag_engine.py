"""Per-parameter gradient error of the GPU trainer vs the CPU oracle (diagnostic)."""
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
hb = batches_for(1, 1, shape)[0]
m0 = {k: st.master.cpu().numpy().copy() for k, st in eng.states.items()}
info = eng.step(0, [DeviceBatch(b, cuda) for b in hb])
torch.cuda.synchronize()
eff = {k: effective_weights(eng.layouts[k], v) for k, v in m0.items()}
tb = {t.id: t for t in tasks}
grads, used, losses = OT.local_grads([(tb[info["tasks"][0]], hb[0])], eff, eng.layouts, shape, embedding_keys, bf16=(os.environ.get("BF16","1")=="1"))
print("loss gpu", eng.loss_sum.item(), "oracle", losses)
for k in sorted(used):
    st = eng.states[k]
    g = st.grad.cpu().numpy(); r = grads[k].numpy()
    print(k, "module rel", np.abs(g - r).max() / np.abs(r).max())
    for name, p in st.layout.params.items():
        a = g[p.offset:p.offset + p.numel]; b = r[p.offset:p.offset + p.numel]
        e = np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)
        if e > 5e-3:
            print("   ", name, p.shape, "rel %.4f" % e, "max|ref| %.3e" % np.abs(b).max(), "max|gpu| %.3e" % np.abs(a).max())
print("--- norm-relative per module")
for bf in (True, False):
    gr, us, ls = OT.local_grads([(tb[info["tasks"][0]], hb[0])], eff, eng.layouts, shape, embedding_keys, bf16=bf)
    for k in sorted(us):
        g = eng.states[k].grad.cpu().numpy().astype(np.float64); r = gr[k].numpy().astype(np.float64)
        print("bf16" if bf else "fp32", k, "normrel %.3e" % (np.linalg.norm(g - r) / np.linalg.norm(r)), "maxrel %.3e" % (np.abs(g-r).max()/np.abs(r).max()))
    print("loss rel", abs(eng.loss_sum.item() / len(hb[0].labels) - ls[0]) / ls[0])

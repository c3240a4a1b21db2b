"""Block-level isolation: engine fwd/bwd of one FFN block and one self-attn
block vs the bf16-faithful autograd oracle on identical inputs (diagnostic)."""
import os, sys, math
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import transformer as OT
from paper_2403_07544_b200 import configs, ops
from paper_2403_07544_b200.domain import ClusterTopology, DeviceId
from paper_2403_07544_b200.engine import Engine
from test_engine_gpu import effective_weights
c = torch.device("cuda:0")
shape = configs.SHAPE_CFG1_GPU
w = configs.config1(shape)
tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, device=c)
key = [k for k in eng.states if k.position == 0 and k.side.value == "decoder"][0]
st = eng.states[key]; lay = st.layout
eff = torch.from_numpy(effective_weights(lay, st.master.cpu().numpy())).requires_grad_(True)
P = OT.Precision(True)
T, d = 300, shape.d_model
torch.manual_seed(0)
x = torch.randn(T, d); dout = torch.randn(T, d) * 1e-2
lens = [20, 37, 43, 50, 60, 90]; cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
def report(name, gpu, ref):
    gpu = gpu.double().cpu(); ref = ref.double()
    print(f"  {name:10s} maxrel {((gpu-ref).abs().max()/ref.abs().max()).item():.2e}  normrel {((gpu-ref).norm()/ref.norm()).item():.2e}")
for block in ("ffn", "self", "selfcausal"):
    print(block)
    ops.memset(st.grad, 0)
    xg = x.to(c); sv = []
    cu_d = torch.from_numpy(cu).to(c)
    if block == "ffn":
        out = eng._ffn_fwd(st, "l0.", xg, sv)
    else:
        out = eng._self_block_fwd(st, "l0.", xg, cu_d, len(lens), max(lens), block == "selfcausal", sv)
    dx = dout.to(c).clone(); dxb = torch.empty(T, d, device=c, dtype=torch.bfloat16); ops.cast_bf16(dx, dxb)
    if block == "ffn":
        eng._ffn_bwd(st, "l0.", sv[0], dx, dxb)
    else:
        eng._self_bwd(st, "l0.", sv[0], dx, dxb, cu_d, len(lens), max(lens), block == "selfcausal")
    torch.cuda.synchronize()
    xr = x.clone().requires_grad_(True)
    if eff.grad is not None: eff.grad = None
    if block == "ffn":
        o = xr + P.g(OT._lin(OT._ffn_act(P, xr, eff, lay, "l0."), eff, lay, "l0.ff2"))
    else:
        qkv = P.vg(OT._lin(P.v(OT._ln(xr, eff, lay, "l0.ln1")), eff, lay, "l0.qkv"))
        a = P.vg(OT._attention(qkv[:, :d], qkv[:, d:2*d], qkv[:, 2*d:], cu.tolist(), cu.tolist(), shape.heads, block == "selfcausal"))
        o = xr + P.g(OT._lin(a, eff, lay, "l0.out"))
    o.backward(dout)
    report("out", out, o.detach())
    report("dx", dx, xr.grad)
    g = st.grad.cpu()
    for name, p in lay.params.items():
        if not name.startswith("l0."): continue
        ref = eff.grad[p.offset:p.offset+p.numel]
        if ref.abs().max() == 0: continue
        report(name, g[p.offset:p.offset+p.numel], ref)

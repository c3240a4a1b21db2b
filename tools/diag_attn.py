import os, sys, math
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2403_07544_b200 import ops
from test_kernels_gpu import ref_attention
c = torch.device("cuda:0")
for causal, same in ((True, True), (False, True), (False, False)):
    rng = np.random.default_rng(1)
    heads, d = 2, 128
    lq = rng.integers(4, 40, size=6); lk = lq.copy() if same else rng.integers(4, 40, size=6)
    cu_q = np.concatenate([[0], np.cumsum(lq)]).astype(np.int32); cu_k = np.concatenate([[0], np.cumsum(lk)]).astype(np.int32)
    tq, tk = int(cu_q[-1]), int(cu_k[-1])
    g = torch.Generator().manual_seed(0)
    q, k, v = (torch.randn(n, d, generator=g).bfloat16().double() for n in (tq, tk, tk))
    do = torch.randn(tq, d, generator=g).bfloat16().double()
    qr, kr, vr = (t.clone().requires_grad_(True) for t in (q, k, v))
    ref = ref_attention(qr, kr, vr, cu_q, cu_k, heads, causal); ref.backward(do)
    qd, kd, vd, dod = (t.bfloat16().to(c) for t in (q, k, v, do))
    o = torch.empty(tq, d, device=c, dtype=torch.bfloat16); lse = torch.empty(heads, tq, device=c)
    dq, dk, dv = torch.empty_like(qd), torch.empty_like(kd), torch.empty_like(vd)
    args = ops.attention_args(qd, kd, vd, o, lse, torch.from_numpy(cu_q).to(c), torch.from_numpy(cu_k).to(c), 6, heads, int(lq.max()), int(lk.max()), causal, d_o=dod, dq=dq, dk=dk, dv=dv)
    ops.attention_fwd(args); ops.attention_bwd(args); torch.cuda.synchronize()
    def r(a, b): a = a.double().cpu(); return f"max {((a-b).abs().max()/b.abs().max()).item():.2e} norm {((a-b).norm()/b.norm()).item():.2e}"
    print("causal", causal, "same", same, "| o", r(o, ref.detach()), "| dq", r(dq, qr.grad), "| dk", r(dk, kr.grad), "| dv", r(dv, vr.grad))

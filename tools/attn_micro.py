"""Attention fwd / bwd timing on config-3-shaped packed batches (CUDA graph of
back-to-back launches, device time)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
from paper_2403_07544_b200.data import attention_groups
dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
CFG5 = os.environ.get("ATTN_CFG") == "5"  # config-5 shapes: 16384 tokens, 16 heads, lognormal(3.2, 0.6) <= 256
d, heads = (1024, 16) if CFG5 else (512, 8)
MU, SIG, HI, TOK = (3.2, 0.6, 256, 16384) if CFG5 else (3.0, 0.5, 128, 4096)
HI = int(os.environ.get("ATTN_HI", HI))  # length clip override (A/B of the long-sequence path)


def lengths(total, mu, sigma, lo, hi):
    out = []
    while sum(out) < total:
        out.append(int(np.clip(round(rng.lognormal(mu, sigma)), lo, hi)))
    return np.array(out)


def timeit(fn, n=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * n)


for name, causal, cross in [("enc self", False, False), ("dec causal", True, False), ("dec cross", False, True)]:
    lq = lengths(TOK, MU, SIG, 4, HI)
    lk = lengths(TOK, MU, SIG, 4, HI)[:len(lq)] if cross else lq
    if cross and len(lk) < len(lq):
        lk = np.concatenate([lk, lq[len(lk):]])
    cu_q = np.concatenate([[0], np.cumsum(lq)]).astype(np.int32)
    cu_k = np.concatenate([[0], np.cumsum(lk)]).astype(np.int32)
    tq, tk = int(cu_q[-1]), int(cu_k[-1])
    q = torch.randn(tq, d, device=dev).bfloat16()
    k = torch.randn(tk, d, device=dev).bfloat16()
    v = torch.randn(tk, d, device=dev).bfloat16()
    o = torch.empty_like(q); lse = torch.empty(heads, tq, device=dev)
    do = torch.randn_like(q); dq = torch.empty_like(q); dk = torch.empty_like(k); dv = torch.empty_like(v)
    cq, ck = torch.from_numpy(cu_q).to(dev), torch.from_numpy(cu_k).to(dev)
    args = ops.attention_args(q, k, v, o, lse, cq, ck, len(lq), heads, int(lq.max()), int(lk.max()), causal,
                              d_o=do, dq=dq, dk=dk, dv=dv)
    tf = timeit(lambda: ops.attention_fwd(args))
    tb = timeit(lambda: ops.attention_bwd(args))
    print(f"{name:10s} tq={tq} seqs={len(lq)} groups={args.n_groups} fwd {tf:6.2f} us  bwd {tb:6.2f} us", flush=True)

if os.environ.get("MM_LIB_VARIANT") == "attn_trace":
    import ctypes
    from paper_2403_07544_b200 import _native
    L = _native.lib()
    n = min(args.n_groups * heads, 148)  # persistent tcgen05 kernel: one CTA per SM
    buf = (ctypes.c_ulonglong * (n * 4))()
    ops.attention_bwd(args); torch.cuda.synchronize()
    L.mm_attn_trace_read(buf, n * 4)
    t = np.array(buf, dtype=np.float64).reshape(n, 4)
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    print("ctas", n, "start spread %.2f" % r[:, 0].max(), "stage(tc: to S ready) %.2f" % np.median(r[:, 1] - r[:, 0]),
          "phaseA %.2f" % np.median(r[:, 2] - r[:, 1]), "phaseB %.2f" % np.median(r[:, 3] - r[:, 2]),
          "cta life %.2f" % np.median(r[:, 3] - r[:, 0]), "end %.2f" % r[:, 3].max())
    print("phaseA p90 %.2f max %.2f; phaseB p90 %.2f max %.2f" % (np.percentile(r[:, 2] - r[:, 1], 90), (r[:, 2] - r[:, 1]).max(), np.percentile(r[:, 3] - r[:, 2], 90), (r[:, 3] - r[:, 2]).max()))

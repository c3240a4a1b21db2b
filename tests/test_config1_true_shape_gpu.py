"""Config 1 at its true shape (BASELINE configs[0], the reference's
CPU-runnable case: d_model 64, 4 heads -> head_dim 16, FFN 256, V1000,
sentences of up to 32 tokens), which round 1 rejected (head_dim != 64).

* the head_dim 16 / 32 attention kernels (csrc/attn_small.cu) vs an fp32
  PyTorch reference of oracle/transformer.py's _attention (packed varlen,
  top-left causal mask), forward and backward, and bitwise reproducible;
* one engine step of a config-1 task at the true shape vs the fp32 oracle,
  max|a - b| <= 2e-2 * max|ref| per module bucket and per parameter tensor
  (the reference's convention, tests/test_acceptance.py:66-68 in mmtplan).

At d_model 64 the bf16 noise floor is itself near 2e-2 for small batches:
with 64 sentences an independent autocast-bf16 implementation of the same
step is 2.9-4.3e-2 off the fp32 oracle on the decoder's FFN-up weight and
LayerNorm gains, and the engine sits level with it (3.4-4.5e-2; above it on
25-29 of 72 tensors, below on the rest) -- tools/diag_c1_parity.py,
profiles/r02_c1_parity.txt.  The error falls with the batch (more rows per
gradient sum): at 1024 sentences every module and tensor of the engine is
<= 1.92e-2 while the independent implementation's worst is 3.05e-2.  The
step test runs there, and also asserts the engine's worst tensor is not
above the independent implementation's worst.
"""
import math
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from paper_2403_07544_b200 import configs  # noqa: E402
from paper_2403_07544_b200.data import make_batch  # noqa: E402

pytestmark = pytest.mark.gpu


def rel_err(got, ref):
    got, ref = got.float(), ref.float()
    return (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)


def ref_attention(q, k, v, cu_q, cu_k, heads, causal):
    hd = q.shape[1] // heads
    out = torch.zeros_like(q)
    for s in range(len(cu_q) - 1):
        qs, ks = slice(cu_q[s], cu_q[s + 1]), slice(cu_k[s], cu_k[s + 1])
        for h in range(heads):
            hs = slice(h * hd, (h + 1) * hd)
            sc = q[qs, hs] @ k[ks, hs].t() / math.sqrt(hd)
            if causal:
                lq, lk = sc.shape
                sc = sc.masked_fill(torch.ones(lq, lk, dtype=torch.bool).triu(1), float("-inf"))
            out[qs, hs] = torch.softmax(sc, -1) @ v[ks, hs]
    return out


@pytest.mark.parametrize("hd", [16, 32])
@pytest.mark.parametrize("causal,maxlen", [(True, 32), (False, 32), (True, 256), (False, 200)])
def test_attention_small_head(cuda, hd, causal, maxlen):
    from paper_2403_07544_b200 import ops
    heads = 4
    d = heads * hd
    rng = np.random.default_rng(hd + maxlen + causal)
    n = 11
    lq = rng.integers(1, maxlen + 1, size=n)
    lq[2] = 1
    lq[5] = maxlen  # the clip's edge
    lk = lq.copy() if causal else rng.integers(1, maxlen + 1, size=n)
    cu_q = np.concatenate([[0], np.cumsum(lq)]).astype(np.int32)
    cu_k = np.concatenate([[0], np.cumsum(lk)]).astype(np.int32)
    tq, tk = int(cu_q[-1]), int(cu_k[-1])
    g = torch.Generator().manual_seed(hd)
    # QKV-packed rows, as the engine lays them out (ld = 3 d for self attention)
    qkv = torch.randn(max(tq, tk), 3 * d, generator=g).bfloat16().float()
    q, k, v = qkv[:tq, :d], qkv[:tk, d:2 * d], qkv[:tk, 2 * d:]
    qr, kr, vr = (t.clone().requires_grad_(True) for t in (q, k, v))
    ref = ref_attention(qr, kr, vr, cu_q, cu_k, heads, causal)
    do = torch.randn(tq, d, generator=g).bfloat16().float()
    ref.backward(do)
    qkv_d = qkv.bfloat16().to(cuda)
    qd, kd, vd = qkv_d[:tq, :d], qkv_d[:tk, d:2 * d], qkv_d[:tk, 2 * d:]
    o = torch.empty(tq, d, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(heads, tq, device=cuda)
    cq, ck = torch.from_numpy(cu_q).to(cuda), torch.from_numpy(cu_k).to(cuda)
    dqkv = torch.full((max(tq, tk), 3 * d), float("nan"), device=cuda, dtype=torch.bfloat16)
    dq, dk, dv = dqkv[:tq, :d], dqkv[:tk, d:2 * d], dqkv[:tk, 2 * d:]
    dod = do.bfloat16().to(cuda)
    args = ops.attention_args(qd, kd, vd, o, lse, cq, ck, n, heads, int(lq.max()), int(lk.max()),
                              causal, d_o=dod, dq=dq, dk=dk, dv=dv, head_dim=hd)
    ops.attention_fwd(args)
    assert rel_err(o.cpu(), ref.detach()) < 1e-2
    ops.attention_bwd(args)
    torch.cuda.synchronize()
    first = [t.clone() for t in (o, dq, dk, dv)]
    for name, t, r in (("dq", dq, qr.grad), ("dk", dk, kr.grad), ("dv", dv, vr.grad)):
        assert torch.isfinite(t.float()).all(), name
        assert rel_err(t.cpu(), r) < 1e-2, name
    # fixed summation order: bitwise reproducible
    ops.attention_fwd(args)
    ops.attention_bwd(args)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(first, (o, dq, dk, dv)))


def test_config1_true_shape_step_vs_fp32_oracle(cuda):
    """One step of config 1's first task at d64 / 4 heads / FFN 256 / V1000
    through the native step driver (head_dim 16 attention, 64-column
    LayerNorm and embedding kernels, tcgen05 GEMMs with N or K = 64)."""
    from test_parity_shapes_gpu import TOL_BF16, _check, _record, run_case
    wl = configs.config1()
    assert wl.shape.head_dim == 16
    rng = np.random.default_rng([1, 0])
    batch = make_batch(rng, wl.data, wl.shape.vocab, sentences=1024)
    rows = run_case(cuda, wl, batch)
    _record("config1", rows)
    _check(rows)
    assert TOL_BF16 == 2e-2
    pairs = [ea for r in rows.values() for ea in r["tensors"].values()]
    worst_engine, worst_alt = max(e for e, _ in pairs), max(a for _, a in pairs)
    assert worst_engine <= worst_alt, (worst_engine, worst_alt)

"""Test infrastructure: an INDEPENDENT bf16 implementation of the engine's
model -- plain PyTorch mixed precision (``torch.autocast`` bf16 with fp32
master weights, cuBLAS GEMMs, PyTorch's fused scaled-dot-product attention)
-- used to measure the bf16 noise floor of a whole training step.

It computes the same function as ``oracle/transformer.task_loss`` (pre-LN
layers, sinusoidal positions, untied generator, token-mean CE; model.py's
builder decisions) but with the precision choices a PyTorch user gets from
autocast, not the engine's: GEMM outputs rounded to bf16, LayerNorm /
softmax / CE in fp32, the embedding table in fp32.  The engine's error
against the fp32 oracle is compared with this implementation's error
against the same oracle (tests/test_parity_shapes_gpu.py).
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

from oracle.transformer import sinusoid
from paper_2403_07544_b200.model import LN_EPS


def _v(flat, lay, name):
    p = lay.params[name]
    return flat[p.offset:p.offset + p.numel].view(p.shape)


def _lin(x, f, lay, name):
    return F.linear(x, _v(f, lay, name + ".w"), _v(f, lay, name + ".b"))


def _ln(x, f, lay, name):
    return F.layer_norm(x.float(), (x.shape[1],), _v(f, lay, name + ".g"), _v(f, lay, name + ".b"),
                        eps=LN_EPS)


def _attn(q, k, v, cu_q, cu_k, heads, causal):
    hd = q.shape[1] // heads
    outs = []
    for s in range(len(cu_q) - 1):
        qs = q[cu_q[s]:cu_q[s + 1]].view(-1, heads, hd).transpose(0, 1)
        ks = k[cu_k[s]:cu_k[s + 1]].view(-1, heads, hd).transpose(0, 1)
        vs = v[cu_k[s]:cu_k[s + 1]].view(-1, heads, hd).transpose(0, 1)
        o = F.scaled_dot_product_attention(qs[None], ks[None], vs[None], is_causal=causal)[0]
        outs.append(o.transpose(0, 1).reshape(-1, heads * hd))
    return torch.cat(outs, 0)


def task_loss(task, batch, flats, layouts, shape, emb_keys, device):
    ek, dk = emb_keys
    d, H = shape.d_model, shape.heads
    scale = math.sqrt(d)
    cu_s, cu_t = batch.cu_src.tolist(), batch.cu_tgt.tolist()
    src = torch.from_numpy(batch.src).long().to(device)
    tgt = torch.from_numpy(batch.tgt_in).long().to(device)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        x = _v(flats[ek], layouts[ek], "emb")[src] * scale \
            + sinusoid(torch.from_numpy(batch.src_pos), d).to(device)
        for key in task.enc_modules:
            f, lay = flats[key], layouts[key]
            for i in range(lay.n_layers):
                p = f"l{i}."
                qkv = _lin(_ln(x, f, lay, p + "ln1"), f, lay, p + "qkv")
                a = _attn(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], cu_s, cu_s, H, False)
                x = x + _lin(a, f, lay, p + "out")
                h = F.relu(_lin(_ln(x, f, lay, p + "ln2"), f, lay, p + "ff1"))
                x = x + _lin(h, f, lay, p + "ff2")
        mem = _ln(x, flats[task.enc_modules[-1]], layouts[task.enc_modules[-1]], "lnf")
        y = _v(flats[dk], layouts[dk], "emb")[tgt] * scale \
            + sinusoid(torch.from_numpy(batch.tgt_pos), d).to(device)
        for key in task.dec_modules:
            f, lay = flats[key], layouts[key]
            for i in range(lay.n_layers):
                p = f"l{i}."
                qkv = _lin(_ln(y, f, lay, p + "ln1"), f, lay, p + "qkv")
                a = _attn(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], cu_t, cu_t, H, True)
                y = y + _lin(a, f, lay, p + "out")
                q = _lin(_ln(y, f, lay, p + "lnc"), f, lay, p + "cq")
                kv = _lin(mem, f, lay, p + "ckv")
                a = _attn(q, kv[:, :d], kv[:, d:], cu_t, cu_s, H, False)
                y = y + _lin(a, f, lay, p + "cout")
                h = F.relu(_lin(_ln(y, f, lay, p + "ln2"), f, lay, p + "ff1"))
                y = y + _lin(h, f, lay, p + "ff2")
        hdec = _ln(y, flats[task.dec_modules[-1]], layouts[task.dec_modules[-1]], "lnf")
        logits = F.linear(hdec, _v(flats[dk], layouts[dk], "gen.w"), _v(flats[dk], layouts[dk], "gen.b"))
    return F.cross_entropy(logits.float(), torch.from_numpy(batch.labels).long().to(device))


def local_grads(task, batch, masters: dict, layouts, shape, emb_keys_fn, device):
    """Gradients of every module's flat fp32 master for one micro-batch."""
    flats = {k: torch.tensor(v, dtype=torch.float32, device=device, requires_grad=True)
             for k, v in masters.items()}
    loss = task_loss(task, batch, flats, layouts, shape, emb_keys_fn(task), device)
    loss.backward()
    return ({k: (f.grad.detach().double().cpu() if f.grad is not None else None)
             for k, f in flats.items()}, float(loss.detach()))

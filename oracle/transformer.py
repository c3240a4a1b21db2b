"""Oracle (test infrastructure): PyTorch-CPU fp32 restatement of the
engine's per-language transformer modules, loss, Algorithm-1 exchange and
Adam.

The reference (mmtplan) has no transformer, loss or optimizer -- its compute
is the toy chain of syncsim.py:34-87 and the optimizer is out of scope
 -- so this part of the oracle is pinned only by the builder's
own restatement ("parity unpinned by the reference").  It
follows the reference's step structure (syncsim.py:346-363), its sync
semantics (syncsim.py:121-153: sum over the hosting devices, divide by the
number of devices that used the module, n == 0 -> untouched) and seeding
(syncsim.py:342-343), and torch.optim.Adam's update.

Parameters live in the same flat per-module layout as the engine
(``paper_2403_07544_b200.model``), so gradients compare bucket to bucket.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

from paper_2403_07544_b200.model import LN_EPS


class _RoundValue(torch.autograd.Function):
    """bf16 storage of an activation: rounds the forward value only."""

    @staticmethod
    def forward(ctx, x):
        return x.bfloat16().float()

    @staticmethod
    def backward(ctx, g):
        return g


class _RoundGrad(torch.autograd.Function):
    """bf16 storage of a gradient: identity forward, rounds the backward value."""

    @staticmethod
    def forward(ctx, x):
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        return g.bfloat16().float()


class Precision:
    """Where the engine stores bf16 (bf16=True) or pure fp32 everywhere."""

    def __init__(self, bf16: bool):
        self.bf16 = bf16

    def v(self, x):
        return _RoundValue.apply(x) if self.bf16 else x

    def g(self, x):
        return _RoundGrad.apply(x) if self.bf16 else x

    def vg(self, x):
        return self.v(self.g(x))


def _view(flat, layout, name):
    p = layout.params[name]
    return flat[p.offset:p.offset + p.numel].view(p.shape)


def sinusoid(pos: torch.Tensor, d: int) -> torch.Tensor:
    div = torch.exp(torch.arange(0, d, 2, dtype=torch.float32) * -(math.log(10000.0) / d))
    ang = pos[:, None].float() * div
    pe = torch.zeros(len(pos), d)
    pe[:, 0::2] = torch.sin(ang)
    pe[:, 1::2] = torch.cos(ang)
    return pe


class _AttnRoundDS(torch.autograd.Function):
    """softmax(q k^T * scale) v over one sequence ([H, L, hd] tensors) whose
    backward rounds dS = P * (dP - D) to bf16 before the dQ / dK products --
    where the engine's attention backward stores dS (attention.cu, phase A:
    bf16 dS in shared memory, D = sum_j P_ij dP_ij exact in fp32)."""

    @staticmethod
    def forward(ctx, q, k, v, scale, causal):
        s = q @ k.transpose(1, 2) * scale
        if causal:
            lq, lk = s.shape[1], s.shape[2]
            s = s.masked_fill(torch.ones(lq, lk, dtype=torch.bool).triu(1), float("-inf"))
        p = torch.softmax(s, -1)
        ctx.save_for_backward(q, k, v, p)
        ctx.scale = scale
        return p @ v

    @staticmethod
    def backward(ctx, do):
        q, k, v, p = ctx.saved_tensors
        dv = p.transpose(1, 2) @ do
        dp = do @ v.transpose(1, 2)
        ds = (p * (dp - (p * dp).sum(-1, keepdim=True))).bfloat16().float()
        return ctx.scale * (ds @ k), ctx.scale * (ds.transpose(1, 2) @ q), dv, None, None


def _attention(q, k, v, cu_q, cu_k, heads, causal, ds_bf16: bool = False):
    hd = q.shape[1] // heads
    outs = []
    for s in range(len(cu_q) - 1):
        qs = q[cu_q[s]:cu_q[s + 1]].view(-1, heads, hd).transpose(0, 1)
        ks = k[cu_k[s]:cu_k[s + 1]].view(-1, heads, hd).transpose(0, 1)
        vs = v[cu_k[s]:cu_k[s + 1]].view(-1, heads, hd).transpose(0, 1)
        if ds_bf16:
            o = _AttnRoundDS.apply(qs, ks, vs, 1.0 / math.sqrt(hd), causal)
        else:
            sc = qs @ ks.transpose(1, 2) / math.sqrt(hd)
            if causal:
                lq, lk = sc.shape[1], sc.shape[2]
                sc = sc.masked_fill(torch.ones(lq, lk, dtype=torch.bool).triu(1), float("-inf"))
            o = torch.softmax(sc, -1) @ vs
        outs.append(o.transpose(0, 1).reshape(-1, heads * hd))
    return torch.cat(outs, 0)


def _ln(x, flat, lay, name):
    return F.layer_norm(x, (x.shape[1],), _view(flat, lay, name + ".g"), _view(flat, lay, name + ".b"),
                        eps=LN_EPS)


def _lin(x, flat, lay, name):
    return x @ _view(flat, lay, name + ".w").t() + _view(flat, lay, name + ".b")


def task_loss(task, batch, flats: dict, layouts: dict, shape, emb_keys, bf16: bool = False,
              trace: dict = None):
    """Token-mean cross-entropy of one task on one packed batch.

    bf16=True rounds to bf16 exactly where the engine stores bf16 tensors:
    LayerNorm outputs, q/k/v, attention outputs, ReLU activations and logits
    (forward values) and the GEMM-input copies of every gradient -- residual
    dx, dqkv, dq / dkv, d(attention out), d(ReLU pre-activation), dlogits and
    the attention backward's dS --
    while LayerNorm, softmax, the residual stream and all accumulations stay
    fp32 as in the kernels."""
    P = Precision(bf16)
    ek, dk = emb_keys
    d, H = shape.d_model, shape.heads
    scale = math.sqrt(d)
    src = torch.from_numpy(batch.src).long()
    cu_s = batch.cu_src.tolist()
    cu_t = batch.cu_tgt.tolist()
    x = _view(flats[ek], layouts[ek], "emb")[src] * scale + sinusoid(torch.from_numpy(batch.src_pos), d)
    _keep(trace, "emb_src", x)
    for key in task.enc_modules:
        f, lay = flats[key], layouts[key]
        for i in range(lay.n_layers):
            p = f"l{i}."
            qkv = P.vg(_lin(P.v(_ln(x, f, lay, p + "ln1")), f, lay, p + "qkv"))
            a = P.vg(_attention(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], cu_s, cu_s, H, False, P.bf16))
            x = x + P.g(_lin(a, f, lay, p + "out"))
            _keep(trace, f"enc_l{i}_attn", x)
            x = x + P.g(_lin(_ffn_act(P, x, f, lay, p), f, lay, p + "ff2"))
            _keep(trace, f"enc_l{i}_ffn", x)
    mem = P.v(_ln(x, flats[task.enc_modules[-1]], layouts[task.enc_modules[-1]], "lnf"))
    _keep(trace, "x_enc", x)
    _keep(trace, "mem", mem)
    y = _view(flats[dk], layouts[dk], "emb")[torch.from_numpy(batch.tgt_in).long()] * scale \
        + sinusoid(torch.from_numpy(batch.tgt_pos), d)
    for key in task.dec_modules:
        f, lay = flats[key], layouts[key]
        for i in range(lay.n_layers):
            p = f"l{i}."
            qkv = P.vg(_lin(P.v(_ln(y, f, lay, p + "ln1")), f, lay, p + "qkv"))
            a = P.vg(_attention(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], cu_t, cu_t, H, True, P.bf16))
            y = y + P.g(_lin(a, f, lay, p + "out"))
            _keep(trace, p + "cx_in", y)
            q = P.vg(_lin(P.v(_ln(y, f, lay, p + "lnc")), f, lay, p + "cq"))
            kv = P.vg(_lin(mem, f, lay, p + "ckv"))
            a = P.vg(_attention(q, kv[:, :d], kv[:, d:], cu_t, cu_s, H, False, P.bf16))
            _keep(trace, p + "ckv", kv)
            _keep(trace, p + "ca", a)
            y = y + P.g(_lin(a, f, lay, p + "cout"))
            y = y + P.g(_lin(_ffn_act(P, y, f, lay, p), f, lay, p + "ff2"))
    h = P.v(_ln(y, flats[task.dec_modules[-1]], layouts[task.dec_modules[-1]], "lnf"))
    _keep(trace, "y_dec", y)
    _keep(trace, "hdec", h)
    logits = P.vg(h @ _view(flats[dk], layouts[dk], "gen.w").t() + _view(flats[dk], layouts[dk], "gen.b"))
    _keep(trace, "logits", logits)
    return F.cross_entropy(logits, torch.from_numpy(batch.labels).long())


def _keep(trace, name, t):
    if trace is not None:
        t.retain_grad()
        trace[name] = t


def _ffn_act(P, x, f, lay, p):
    """relu(LN2(x) W1^T + b1): bf16 LN output, bf16 activation, bf16 masked grad."""
    return P.v(torch.relu(P.g(_lin(P.v(_ln(x, f, lay, p + "ln2")), f, lay, p + "ff1"))))


def local_grads(tasks_and_batches, masters: dict, layouts: dict, shape, emb_keys_fn,
                bf16: bool = False):
    """Per-device accumulation (DeviceState.accumulate, syncsim.py:113-118):
    sum of the micro-batches' gradients per module, plus the used set and the
    summed loss."""
    flats = {k: torch.tensor(v, dtype=torch.float32, requires_grad=True) for k, v in masters.items()}
    used = set()
    losses = []
    for task, batch in tasks_and_batches:
        ek = emb_keys_fn(task)
        loss = task_loss(task, batch, flats, layouts, shape, ek, bf16)
        loss.backward()
        losses.append(float(loss.detach()))
        used.update(task.modules())
        used.update(ek)
    grads = {k: (f.grad.detach().clone() if f.grad is not None else torch.zeros_like(f))
             for k, f in flats.items()}
    return grads, used, losses


def algorithm1(per_rank_grads: dict, per_rank_used: dict, groups: dict) -> tuple[dict, dict]:
    """syncsim.py:121-153 over ranks: sum in ascending rank order, / n."""
    synced, counts = {}, {}
    for key, members in groups.items():
        n = sum(1 for r in members if key in per_rank_used[r])
        counts[key] = n
        if n == 0:
            continue
        tot = torch.zeros_like(per_rank_grads[members[0]][key])
        for r in members:
            tot = tot + per_rank_grads[r][key]
        synced[key] = tot / n
    return synced, counts


def adam_step(master, m, v, grad, step, lr, beta1, beta2, eps, weight_decay=0.0):
    """torch.optim.Adam (foreach=False) update on flat fp32 tensors, in place."""
    if weight_decay:
        grad = grad + weight_decay * master
    m.lerp_(grad, 1 - beta1)
    v.mul_(beta2).addcmul_(grad, grad, value=1 - beta2)
    bc1 = 1 - beta1 ** step
    bc2 = 1 - beta2 ** step
    denom = (v.sqrt() / math.sqrt(bc2)).add_(eps)
    master.addcdiv_(m, denom, value=-lr / bc1)

"""Per-module parameter layout, deterministic initialisation and HBM buckets.

Every module (a stack of L transformer layers, or a language's embedding /
generator block) owns ONE flat fp32 bucket per state -- master weights,
Adam exp_avg / exp_avg_sq, gradient -- plus a flat bf16 copy of the weights
that the GEMMs read.  Named parameters are views at 64-element-aligned
offsets, so TMA descriptors and 128-bit vector accesses always see aligned
bases, and Algorithm 1's reduction and the fused optimizer (K3) run over one
contiguous range per module.

Builder decisions (the reference has no transformer):
pre-LN layers (OpenNMT-py "standard" layer order) with a final LayerNorm
after the last stack of each side; sinusoidal positions; embeddings scaled by
sqrt(d); untied generator with bias; ReLU FFN; no dropout / label smoothing;
token-mean cross-entropy per micro-batch; Xavier-uniform matrices, N(0, d^-1/2)
embeddings, zero biases, unit LN gains; LN eps 1e-6.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional

import numpy as np

from .configs import ModelShape
from .domain import ModuleKey, Side

ALIGN = 64  # elements
LN_EPS = 1e-6


@dataclasses.dataclass(frozen=True)
class Param:
    name: str
    shape: tuple[int, ...]
    init: str  # "xavier" | "zeros" | "ones" | "embed"
    offset: int

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape))


def _layer_params(prefix: str, s: ModelShape, decoder: bool) -> list[tuple[str, tuple, str]]:
    d, f = s.d_model, s.ffn
    out = [(f"{prefix}ln1.g", (d,), "ones"), (f"{prefix}ln1.b", (d,), "zeros"),
           (f"{prefix}qkv.w", (3 * d, d), "xavier"), (f"{prefix}qkv.b", (3 * d,), "zeros"),
           (f"{prefix}out.w", (d, d), "xavier"), (f"{prefix}out.b", (d,), "zeros")]
    if decoder:
        out += [(f"{prefix}lnc.g", (d,), "ones"), (f"{prefix}lnc.b", (d,), "zeros"),
                (f"{prefix}cq.w", (d, d), "xavier"), (f"{prefix}cq.b", (d,), "zeros"),
                (f"{prefix}ckv.w", (2 * d, d), "xavier"), (f"{prefix}ckv.b", (2 * d,), "zeros"),
                (f"{prefix}cout.w", (d, d), "xavier"), (f"{prefix}cout.b", (d,), "zeros")]
    out += [(f"{prefix}ln2.g", (d,), "ones"), (f"{prefix}ln2.b", (d,), "zeros"),
            (f"{prefix}ff1.w", (f, d), "xavier"), (f"{prefix}ff1.b", (f,), "zeros"),
            (f"{prefix}ff2.w", (d, f), "xavier"), (f"{prefix}ff2.b", (d,), "zeros")]
    return out


@dataclasses.dataclass
class ModuleLayout:
    key: ModuleKey
    kind: str            # "enc_stack" | "dec_stack" | "enc_embed" | "dec_embed"
    n_layers: int
    final_ln: bool
    params: dict[str, Param]
    numel: int           # padded bucket length
    # [0, dense_end): the weight matrices whose gradients the weight-gradient
    # GEMMs write whole (stacks: every projection / FFN matrix; the decoder
    # embedding module: the generator).  A module's first micro-batch of a
    # step stores them instead of reduce-adding onto zeros, so only
    # [dense_end, numel) -- biases, LayerNorm, embedding tables -- needs the
    # reset memset.
    dense_end: int = 0

    def p(self, name: str) -> Param:
        return self.params[name]


def layout_for(key: ModuleKey, shape: ModelShape, n_layers: int, final_ln: bool) -> ModuleLayout:
    spec: list[tuple[str, tuple, str]] = []
    if key.position < 0:
        kind = "enc_embed" if key.side is Side.ENCODER else "dec_embed"
        spec.append(("emb", (shape.vocab, shape.d_model), "embed"))
        if key.side is Side.DECODER:
            spec += [("gen.w", (shape.vocab, shape.d_model), "xavier"),
                     ("gen.b", (shape.vocab,), "zeros")]
    else:
        dec = key.side is Side.DECODER
        kind = "dec_stack" if dec else "enc_stack"
        for i in range(n_layers):
            spec += _layer_params(f"l{i}.", shape, dec)
        if final_ln:
            spec += [("lnf.g", (shape.d_model,), "ones"), ("lnf.b", (shape.d_model,), "zeros")]
    # offsets: GEMM-written matrices first (dense_end), then everything else,
    # each in spec order; params keeps spec order, so init_module draws the
    # same random stream whatever the placement
    offsets: dict[str, int] = {}
    off = dense_end = 0
    dense = [x for x in spec if x[2] == "xavier"]
    for i, (name, shp, _init) in enumerate(dense + [x for x in spec if x[2] != "xavier"]):
        offsets[name] = off
        off += (int(np.prod(shp)) + ALIGN - 1) // ALIGN * ALIGN
        if i == len(dense) - 1:
            dense_end = off
    params = {name: Param(name, shp, init, offsets[name]) for name, shp, init in spec}
    return ModuleLayout(key, kind, n_layers, final_ln, params, off, dense_end)


def true_param_count(layout: ModuleLayout) -> int:
    return sum(p.numel for p in layout.params.values())


def _seed_for(key: ModuleKey, seed: int) -> int:
    """Stable across processes (never Python's salted hash())."""
    h = hashlib.sha256(f"{seed}|{key.side.value}|{key.position}|{key.group}".encode()).digest()
    return int.from_bytes(h[:8], "little")


def init_module(layout: ModuleLayout, shape: ModelShape, seed: int = 0) -> np.ndarray:
    """fp32 flat master weights; identical on every rank hosting the module."""
    rng = np.random.default_rng(_seed_for(layout.key, seed))
    flat = np.zeros(layout.numel, dtype=np.float32)
    for p in layout.params.values():
        view = flat[p.offset:p.offset + p.numel]
        if p.init == "ones":
            view[:] = 1.0
        elif p.init == "xavier":
            fan_out, fan_in = p.shape
            a = math.sqrt(6.0 / (fan_in + fan_out))
            view[:] = (rng.random(p.numel, dtype=np.float32) * 2.0 - 1.0) * np.float32(a)
        elif p.init == "embed":
            view[:] = rng.standard_normal(p.numel, dtype=np.float32) * np.float32(shape.d_model ** -0.5)
    return flat


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as fp32 (host helper)."""
    u = x.astype(np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def module_layouts(plan, shape: ModelShape) -> dict[ModuleKey, ModuleLayout]:
    """Layout of every module in a plan; stacks carry the final LN iff they sit
    at their side's last position."""
    n_layers: dict[ModuleKey, int] = {}
    last_pos: dict[Side, int] = {}
    for t in plan.tasks:
        for k, n in zip(t.enc_modules + t.dec_modules, t.enc_layers + t.dec_layers):
            n_layers[k] = n
            last_pos[k.side] = max(last_pos.get(k.side, -1), k.position)
    out = {}
    for k in plan.keys:
        if k.position < 0:
            out[k] = layout_for(k, shape, 0, False)
        else:
            out[k] = layout_for(k, shape, n_layers[k], k.position == last_pos[k.side])
    return out


class ModuleState:
    """Device buckets of one module (fp32 master / m / v / grad, bf16 weights)."""

    def __init__(self, layout: ModuleLayout, shape: ModelShape, device, seed: int = 0,
                 master: Optional[np.ndarray] = None, capacity: int = 0):
        """capacity > layout.numel pads every bucket with zeros (the
        partitioned exchange's g * shard elements)."""
        import torch
        self.layout = layout
        self.key = layout.key
        host = init_module(layout, shape, seed) if master is None else master
        if capacity > host.size:
            host = np.concatenate([host, np.zeros(capacity - host.size, np.float32)])
        self.master = torch.from_numpy(host).to(device)
        self.exp_avg = torch.zeros_like(self.master)
        self.exp_avg_sq = torch.zeros_like(self.master)
        self.grad = torch.zeros_like(self.master)
        from . import ops
        self.weights = torch.empty(self.master.numel(), dtype=torch.bfloat16, device=device)
        ops.cast_bf16(self.master, self.weights)
        self.step = 0

    def w(self, name: str):
        p = self.layout.params[name]
        return self.weights[p.offset:p.offset + p.numel].view(p.shape)

    def f32(self, name: str):
        p = self.layout.params[name]
        return self.master[p.offset:p.offset + p.numel].view(p.shape)

    def g(self, name: str):
        p = self.layout.params[name]
        return self.grad[p.offset:p.offset + p.numel].view(p.shape)

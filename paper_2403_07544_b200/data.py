"""Synthetic token batches with the shapes and distributions of BASELINE.json
(the paper's Europarl corpora and SentencePiece models are not available; no
dataset items are reproduced).

A batch is a list of sentence pairs packed without padding:
* source ids ``[Ts]`` with in-sentence positions and ``cu_src`` offsets;
* decoder input ``[Tt]`` = BOS + target content, labels = content + EOS,
  positions and ``cu_tgt`` offsets.
Ids 0..3 are pad / bos / eos / unk; content ids are drawn from 4..V-1,
uniformly (config 1) or Zipf(s) by rank (configs 3-5).  Sentence lengths are
uniform in [lo, hi] (config 1) or round(lognormal(mu, sigma)) clipped to
[lo, hi]; sentences are added until the target side holds exactly
``tokens`` tokens (the last target sentence is shortened, min 1).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

BOS, EOS = 1, 2
FIRST_ID = 4
ATTN_CAP_ROWS = 128  # rows per attention work group and side (tcgen05 TMEM lanes)


@dataclasses.dataclass
class Batch:
    src: np.ndarray      # int32 [Ts]
    src_pos: np.ndarray
    cu_src: np.ndarray   # int32 [n+1]
    tgt_in: np.ndarray   # int32 [Tt]
    tgt_pos: np.ndarray
    labels: np.ndarray   # int32 [Tt]
    cu_tgt: np.ndarray

    @property
    def n_seq(self) -> int:
        return len(self.cu_src) - 1

    @property
    def n_src(self) -> int:
        return int(self.cu_src[-1])

    @property
    def n_tgt(self) -> int:
        return int(self.cu_tgt[-1])

    @property
    def max_src(self) -> int:
        return int(np.diff(self.cu_src).max())

    @property
    def max_tgt(self) -> int:
        return int(np.diff(self.cu_tgt).max())

    def host_arrays(self) -> dict[str, np.ndarray]:
        return {"src": self.src, "src_pos": self.src_pos, "cu_src": self.cu_src,
                "tgt_in": self.tgt_in, "tgt_pos": self.tgt_pos, "labels": self.labels,
                "cu_tgt": self.cu_tgt}

    def nbytes(self) -> int:
        return sum(a.nbytes for a in self.host_arrays().values())


class ZipfIds:
    """Inverse-CDF sampler of rank-Zipf(s) ids over [FIRST_ID, vocab)."""

    def __init__(self, vocab: int, s: float):
        ranks = np.arange(1, vocab - FIRST_ID + 1, dtype=np.float64)
        w = ranks ** (-s) if s > 0 else np.ones_like(ranks)
        self.cdf = np.cumsum(w) / w.sum()

    def draw(self, rng: np.random.Generator, n: int) -> np.ndarray:
        idx = np.searchsorted(self.cdf, rng.random(n), side="right")
        return (np.minimum(idx, len(self.cdf) - 1) + FIRST_ID).astype(np.int32)


def _lengths(rng, n, spec) -> np.ndarray:
    if spec.len_mu == 0:
        return rng.integers(spec.len_min, spec.len_max + 1, size=n)
    x = np.round(rng.lognormal(spec.len_mu, spec.len_sigma, size=n))
    return np.clip(x, spec.len_min, spec.len_max).astype(np.int64)


def attention_order_py(ls, lt, cap: int = 128) -> np.ndarray:
    """Host restatement of mm_attention_order (first-fit decreasing 2-D bins
    of ``cap`` rows per side, bins in creation order, over-long pairs last)."""
    ls, lt = [int(x) for x in ls], [int(x) for x in lt]
    n = len(ls)
    big = [i for i in range(n) if ls[i] > cap or lt[i] > cap]
    items = [i for i in range(n) if not (ls[i] > cap or lt[i] > cap)]
    items.sort(key=lambda i: (-max(ls[i], lt[i]), -(ls[i] + lt[i])))  # stable
    bins, fill = [], []
    for i in items:
        for b, (fs, ft) in enumerate(fill):
            if fs + ls[i] <= cap and ft + lt[i] <= cap:
                break
        else:
            b = len(bins)
            bins.append([])
            fill.append((0, 0))
        bins[b].append(i)
        fill[b] = (fill[b][0] + ls[i], fill[b][1] + lt[i])
    return np.asarray([i for bin_ in bins for i in bin_] + big, dtype=np.int64)


def attention_order(ls, lt, cap: int = ATTN_CAP_ROWS) -> np.ndarray:
    """Sentence-pair order that packs into few attention work groups
    (mm_attention_order, host C++): a permutation of range(len(ls))."""
    from . import _native
    a = np.ascontiguousarray(ls, dtype=np.int32)
    b = np.ascontiguousarray(lt, dtype=np.int32)
    perm = np.empty(max(len(a), 1), dtype=np.int32)
    _native.check(_native.lib().mm_attention_order(a.ctypes.data, b.ctypes.data, len(a), cap,
                                                   perm.ctypes.data), "mm_attention_order")
    return perm[:len(a)].astype(np.int64)


def make_batch(rng: np.random.Generator, spec, vocab: int, sentences: Optional[int] = None,
               ids: Optional[ZipfIds] = None, order: bool = True, order_fn=None) -> Batch:
    """One micro-batch: ``sentences`` pairs if given, else ``spec.tokens_per_gpu``
    target tokens.  order=True lays the pairs out in attention_order (an
    order of independent pairs; fewer, fuller attention work groups)."""
    ids = ids or ZipfIds(vocab, spec.zipf_s)
    if sentences is not None:
        ls, lt = _lengths(rng, sentences, spec), _lengths(rng, sentences, spec)
    else:
        ls_l, lt_l, tot = [], [], 0
        while tot < spec.tokens_per_gpu:
            a, b = _lengths(rng, 2, spec)
            b = min(int(b), spec.tokens_per_gpu - tot)
            ls_l.append(int(a))
            lt_l.append(b)
            tot += b
        ls, lt = np.asarray(ls_l), np.asarray(lt_l)
    return batch_from_lengths(rng, ls, lt, ids, order=order, order_fn=order_fn)


def batch_from_lengths(rng: np.random.Generator, ls, lt, ids: ZipfIds, order: bool = True,
                       order_fn=None) -> Batch:
    """A packed batch of sentence pairs with the given source / target
    lengths (ids drawn from ``ids``); ``order_fn`` replaces attention_order
    (e.g. ``attention_order_py`` on a host without the native library)."""
    ls, lt = np.asarray(ls, dtype=np.int64), np.asarray(lt, dtype=np.int64)
    if order and len(ls) > 1:
        perm = (order_fn or attention_order)(ls, lt)
        ls, lt = ls[perm], lt[perm]
    cu_s = np.concatenate([[0], np.cumsum(ls)]).astype(np.int32)
    cu_t = np.concatenate([[0], np.cumsum(lt)]).astype(np.int32)
    src = ids.draw(rng, int(cu_s[-1]))
    content = ids.draw(rng, int(cu_t[-1]))
    labels = content.copy()
    tgt_in = np.empty_like(content)
    for j in range(len(lt)):
        a, b = cu_t[j], cu_t[j + 1]
        labels[b - 1] = EOS
        tgt_in[a] = BOS
        tgt_in[a + 1:b] = content[a:b - 1]
    src_pos = np.concatenate([np.arange(n) for n in ls]).astype(np.int32)
    tgt_pos = np.concatenate([np.arange(n) for n in lt]).astype(np.int32)
    return Batch(src, src_pos, cu_s, tgt_in, tgt_pos, labels, cu_t)


ATTN_CAP = 128  # rows per CTA group (each side), see include/mmb200.h


def attention_groups(cu_q: np.ndarray, cu_k: np.ndarray, cap: int = ATTN_CAP, align: int = 32):
    """Greedy packing of consecutive sequences into attention CTA groups:
    each sequence takes ceil(len/align)*align rows (32 for the mma.sync
    kernels' shared-memory tiles, 1 for the tcgen05 backward's 128-row TMA
    boxes); a group holds at most ``cap`` rows per side (a longer sequence
    gets a group of its own).  Returns (int32 [2*n_groups] of (first, count),
    rows footprint of the largest group)."""
    lq = np.diff(cu_q).astype(np.int64)
    lk = np.diff(cu_k).astype(np.int64)
    pq = (lq + align - 1) // align * align
    pk = (lk + align - 1) // align * align
    out = []
    foot = 0
    i, n = 0, len(lq)
    while i < n:
        j, sq, sk = i, 0, 0
        while j < n and (j == i or (sq + pq[j] <= cap and sk + pk[j] <= cap)):
            sq += pq[j]
            sk += pk[j]
            j += 1
        out += [i, j - i]
        foot = max(foot, sq, sk)
        i = j
    return np.asarray(out, dtype=np.int32), int(foot)

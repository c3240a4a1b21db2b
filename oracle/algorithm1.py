"""Oracle (test infrastructure): numpy / pure-Python restatement of the
reference simulator's hot path, ``/root/reference/pkg/src/mmtplan/syncsim.py``.

Used by tests as the checker for the engine's host logic (groups, ready
counts, multiplexer) and for the CUDA Algorithm-1 kernels.  Pinned against
the fixtures in ``tests/golden/`` that ``make_golden.py`` generated from the
reference itself.
"""
from __future__ import annotations

import dataclasses
import random
from typing import Mapping, Sequence

import numpy as np


# --------------------------------------------------------------------------
# toy chain (syncsim.py:34-87): h_i = W_i h_{i-1}, L = 1/2 |h - y|^2, -dL/dW


def toy_weights(keys, dim: int, seed: int):
    """syncsim.py:44-52: one N(0,1)/sqrt(d) matrix per sorted key, then y."""
    rng = np.random.default_rng(seed)
    w = {k: rng.standard_normal((dim, dim)) / np.sqrt(dim) for k in sorted(set(keys))}
    return w, rng.standard_normal(dim)


def toy_forward(weights, chain, x):
    states = [x]
    for k in chain:
        states.append(weights[k] @ states[-1])
    return states


def toy_neg_grads(weights, target, chain, states):
    """syncsim.py:72-87: -dL/dW per module, repeated modules summed."""
    delta = states[-1] - target
    out = {}
    for i in reversed(range(len(chain))):
        g = -np.outer(delta, states[i])
        out[chain[i]] = out[chain[i]] + g if chain[i] in out else g
        delta = weights[chain[i]].T @ delta
    return out


# --------------------------------------------------------------------------
# Algorithm 1 exchange


@dataclasses.dataclass
class Dev:
    index: int
    hosted: frozenset
    buffers: dict
    used: set


def sync_step(devices: Sequence[Dev]) -> dict:
    """syncsim.py:121-153.  Per module in sorted order: group = hosting devices
    (ascending index); n = #members that used it; n == 0 -> zeros and buffers
    untouched; else total = 0 + sum of member buffers (ascending), / n,
    installed on every member."""
    devs = sorted(devices, key=lambda d: d.index)
    if len({d.index for d in devs}) != len(devs):
        raise ValueError("duplicate device index")
    keys = sorted(set().union(*(d.hosted for d in devs))) if devs else []
    out = {}
    for key in keys:
        members = [d for d in devs if key in d.hosted]
        n = sum(key in d.used for d in members)
        ref = members[0].buffers[key]
        if n == 0:
            out[key] = np.zeros_like(ref)
            continue
        total = np.zeros_like(ref)
        for d in members:
            total += d.buffers[key]
        total /= n
        out[key] = total
        for d in members:
            d.buffers[key] = total.copy()
    return out


def device_mean_oracle(runs, hosted: Mapping[int, frozenset], weights, target, dim) -> dict:
    """syncsim.py:156-187: per-device sums of task gradients, then the mean
    over the *devices* that used each module."""
    per_dev = {i: {} for i in hosted}
    for dev, chain, x in runs:
        for k, g in toy_neg_grads(weights, target, chain, toy_forward(weights, chain, x)).items():
            per_dev[dev][k] = per_dev[dev].get(k, np.zeros_like(g)) + g
    keys = sorted(set().union(*hosted.values())) if hosted else []
    res = {}
    for k in keys:
        users = [i for i in sorted(per_dev) if k in per_dev[i]]
        if not users:
            res[k] = np.zeros((dim, dim))
            continue
        acc = np.zeros((dim, dim))
        for i in users:
            acc += per_dev[i][k]
        res[k] = acc / len(users)
    return res


def random_toy_scenario(seed: int, dim: int = 3, accum_count: int = 1):
    """A random multi-device toy-chain step for the device-mean check of
    syncsim.py:156-187 (the same kind of instance the reference's own
    randomized test draws, tests/test_syncsim.py:95-136): 2-8 devices, 2-16
    tasks of 1-3 modules each from a pool of encoder / decoder keys.
    Returns (weights, target, runs, hosted); runs = (device, chain, x)."""
    from paper_2403_07544_b200.domain import ModuleKey, Side
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    n_dev, n_tasks = rng.randint(2, 8), rng.randint(2, 16)
    pool = sorted({ModuleKey(Side.ENCODER, i, f"g{rng.randrange(4)}") for i in range(3)}
                  | {ModuleKey(Side.DECODER, 0, f"g{rng.randrange(4)}"),
                     ModuleKey(Side.ENCODER, 0, "full"), ModuleKey(Side.DECODER, 1, "full")})
    chains = [tuple(rng.sample(pool, rng.randint(1, 3))) for _ in range(n_tasks)]
    where = [rng.randrange(n_dev) for _ in chains]
    hosted = {d: frozenset(k for c, w in zip(chains, where) if w == d for k in c) for d in range(n_dev)}
    hosted = {d: h for d, h in hosted.items() if h}
    weights, target = toy_weights(pool, dim, seed)
    runs = [(w, c, nrng.standard_normal(dim)) for _ in range(accum_count) for c, w in zip(chains, where)]
    return weights, target, runs, hosted


# --------------------------------------------------------------------------
# multiplexer, group map and ready counts (syncsim.py:190-205, 313-363)


def multiplex(tasks, step: int, rng: random.Random):
    """Exactly one rng.random() per call; weighted choice among active tasks."""
    active = [t for t in sorted(tasks, key=lambda t: t.id) if t.introduce_at_training_step <= step]
    if not active:
        raise ValueError(f"no active task at step {step}")
    r = rng.random() * sum(t.weight for t in active)
    acc = 0.0
    for t in active:
        acc += t.weight
        if r < acc:
            return t
    return active[-1]


def flat_rank(device, n_gpus_per_node: int) -> int:
    return device.node * n_gpus_per_node + device.gpu


def group_map(tasks, n_gpus_per_node: int) -> dict:
    """syncsim.py:321-340: hosted set per device = union of its tasks'
    modules; group of a module = hosting devices ascending."""
    by_dev = {}
    for t in sorted(tasks, key=lambda t: t.id):
        by_dev.setdefault(flat_rank(t.device, n_gpus_per_node), []).append(t)
    hosted = {i: set().union(*(set(t.modules()) for t in ts)) for i, ts in by_dev.items()}
    keys = sorted(set().union(*hosted.values())) if hosted else []
    return {k: [i for i in sorted(hosted) if k in hosted[i]] for k in keys}


def ready_counts(tasks, n_gpus_per_node: int, steps: int, seed: int = 0, accum_count: int = 1):
    """Per step: the multiplexer picks (RNG ``Random(f"{seed}:{i}:mux")`` per
    device, syncsim.py:342) and n_m = #devices that used module m."""
    by_dev = {}
    for t in sorted(tasks, key=lambda t: t.id):
        by_dev.setdefault(flat_rank(t.device, n_gpus_per_node), []).append(t)
    rngs = {i: random.Random(f"{seed}:{i}:mux") for i in sorted(by_dev)}
    groups = group_map(tasks, n_gpus_per_node)
    out = []
    picks = []
    for step in range(steps):
        used = {i: set() for i in by_dev}
        step_picks = {}
        for i in sorted(by_dev):
            step_picks[i] = []
            for _ in range(accum_count):
                t = multiplex(by_dev[i], step, rngs[i])
                step_picks[i].append(t.id)
                used[i].update(t.modules())
        out.append({k: sum(k in used[i] for i in g) for k, g in groups.items()})
        picks.append(step_picks)
    return out, picks


def ring_allreduce_time(payload_bytes: float, group: int, alpha: float, beta: float) -> float:
    """syncsim.py:237-242."""
    if group < 2:
        return 0.0
    return 2 * (group - 1) * alpha + 2 * (group - 1) / group * payload_bytes / beta

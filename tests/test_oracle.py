"""Pin the oracle before trusting it: its Algorithm-1 restatement against the
reference's own sync_step outputs (golden scenarios, bit-exact in fp32 and
fp64), the reference's known answers (test_syncsim.py:140-211) and the toy
chain's finite differences (test_syncsim.py:67-92)."""
import json
import os

import numpy as np
import pytest

from oracle import algorithm1 as A1
from paper_2403_07544_b200.domain import ModuleKey, Side

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
E = Side.ENCODER


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


def test_sync_step_vs_reference_scenarios(golden):
    arrays = np.load(os.path.join(GOLD, "sync_scenarios.npz"))
    for meta in golden["scenarios"]:
        s = meta["seed"]
        devs = []
        for j, d in enumerate(meta["devices"]):
            bufs = {ModuleKey.parse(k): arrays[f"s{s}_in_{j}_{k}"].copy() for k in d["hosted"]}
            devs.append(A1.Dev(d["index"], frozenset(bufs), bufs,
                               {ModuleKey.parse(k) for k in d["used"]}))
        out = A1.sync_step(devs)
        for k, v in out.items():
            assert np.array_equal(v, arrays[f"s{s}_synced_{k}"])
            assert v.dtype == np.dtype(meta["dtype"])
        for j, d in enumerate(sorted(devs, key=lambda d: d.index)):
            for k, b in d.buffers.items():
                assert np.array_equal(b, arrays[f"s{s}_after_{j}_{k}"])


def test_reduce_small_vs_reference(golden):
    arrays = np.load(os.path.join(GOLD, "reduce_small.npz"))
    devs = {r: A1.Dev(r, frozenset(), {}, set()) for r in range(8)}
    for i, m in enumerate(golden["reduce_small"]):
        for j in range(m["group"]):
            r = m["start"] + j
            devs[r].hosted = devs[r].hosted | {i}
            devs[r].buffers[i] = arrays[f"grad_{r}_{i}"].copy()
            if m["ready"][j]:
                devs[r].used.add(i)
    out = A1.sync_step(list(devs.values()))
    for i in range(len(golden["reduce_small"])):
        assert np.array_equal(out[i], arrays[f"synced_{i}"])


def key(n="full"):
    return ModuleKey(E, 0, n)


def test_known_answers():
    k = key()
    d1 = A1.Dev(0, frozenset({k}), {k: np.full((1, 1), 2.0)}, {k})
    d2 = A1.Dev(1, frozenset({k}), {k: np.full((1, 1), 4.0)}, {k})
    assert A1.sync_step([d1, d2])[k][0, 0] == 3.0
    d1 = A1.Dev(0, frozenset({k}), {k: np.full((1, 1), 4.0)}, {k})
    d2 = A1.Dev(1, frozenset({k}), {k: np.zeros((1, 1))}, set())
    assert A1.sync_step([d1, d2])[k][0, 0] == 4.0 and d2.buffers[k][0, 0] == 4.0
    d1 = A1.Dev(0, frozenset({k}), {k: np.zeros((2, 2))}, set())
    d2 = A1.Dev(1, frozenset({k}), {k: np.zeros((2, 2))}, set())
    assert not A1.sync_step([d1, d2])[k].any()
    with pytest.raises(ValueError):
        A1.sync_step([A1.Dev(0, frozenset({k}), {k: np.zeros(1)}, set()),
                      A1.Dev(0, frozenset({k}), {k: np.zeros(1)}, set())])


def test_device_mean_not_task_mean():
    """((1+3)+2)/2 = 3 (test_syncsim.py:172-182) through the toy chain."""
    k = key()
    w = {k: np.array([[1.0]])}
    # -dL/dW for W=1, x, target 0: -(x)(x) = -x^2 ; pick x so that grads are 1, 3, 2
    runs = [(0, (k,), np.array([1.0])), (0, (k,), np.array([np.sqrt(3.0)])),
            (1, (k,), np.array([np.sqrt(2.0)]))]
    res = A1.device_mean_oracle(runs, {0: frozenset({k}), 1: frozenset({k})}, w,
                                np.zeros(1), 1)
    assert res[k][0, 0] == pytest.approx(-3.0)


@pytest.mark.parametrize("seed", range(5))
def test_toy_chain_finite_differences(seed):
    rng = np.random.default_rng(seed)
    dim = 3
    chain = tuple(ModuleKey(E, i, f"m{i}") for i in range(int(rng.integers(1, 4))))
    w, y = A1.toy_weights(chain, dim, seed)
    x = rng.standard_normal(dim)
    g = A1.toy_neg_grads(w, y, chain, A1.toy_forward(w, chain, x))

    def loss():
        h = A1.toy_forward(w, chain, x)[-1]
        return 0.5 * float((h - y) @ (h - y))

    for k in chain:
        num = np.zeros((dim, dim))
        for i in range(dim):
            for j in range(dim):
                o = w[k][i, j]
                w[k][i, j] = o + 1e-6
                lp = loss()
                w[k][i, j] = o - 1e-6
                lm = loss()
                w[k][i, j] = o
                num[i, j] = (lp - lm) / 2e-6
        assert np.allclose(-g[k], num, rtol=1e-4, atol=1e-8)


def test_ring_formula():
    assert A1.ring_allreduce_time(1e6, 1, 1e-5, 1e9) == 0.0
    assert A1.ring_allreduce_time(8e6, 4, 1e-5, 1e9) == pytest.approx(2 * 3 * 1e-5 + 1.5 * 8e6 / 1e9)

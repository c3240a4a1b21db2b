"""Algorithm-1 exchange (emulated devices on one GPU) and K3 on the B200,
checked against the reference's own sync_step outputs (golden fixtures,
bit-exact in fp32) and against torch.optim.Adam's update (fp32, 1e-5)."""
import json
import os

import numpy as np
import pytest
import torch

from paper_2403_07544_b200.domain import ModuleKey

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


def _devices(meta, arrays, s, cuda):
    """The scenario's devices with CUDA buffers (cuda) or the reference's own
    numpy buffers (cuda=None)."""
    from paper_2403_07544_b200.syncsim import DeviceState
    devs = []
    for j, d in enumerate(meta["devices"]):
        hosted = frozenset(ModuleKey.parse(k) for k in d["hosted"])
        bufs = {ModuleKey.parse(k): arrays[f"s{s}_in_{j}_{k}"].copy() for k in d["hosted"]}
        if cuda is not None:
            bufs = {k: torch.from_numpy(v).to(cuda) for k, v in bufs.items()}
        devs.append(DeviceState(d["index"], hosted, 1, bufs, {ModuleKey.parse(k) for k in d["used"]}))
    return devs


def _as_np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else x


@pytest.mark.parametrize("where", ["cuda", "host"])
def test_sync_step_bit_exact_vs_reference(golden, cuda, where):
    """All 40 golden scenarios -- fp32 AND fp64 buffers (the reference's
    default dtype) -- through sync_step: synced values and every device's
    buffers afterwards equal the reference's own outputs bit for bit, with
    CUDA buffers and with the reference's numpy buffers (staged through the
    GPU kernels, written back as the reference does)."""
    from paper_2403_07544_b200.syncsim import sync_step
    arrays = np.load(os.path.join(GOLD, "sync_scenarios.npz"))
    n_checked = {"float32": 0, "float64": 0}
    for meta in golden["scenarios"]:
        s = meta["seed"]
        devs = _devices(meta, arrays, s, cuda if where == "cuda" else None)
        synced = sync_step(devs)
        for key, val in synced.items():
            ref = arrays[f"s{s}_synced_{key}"]
            got = _as_np(val)
            assert got.dtype == ref.dtype and np.array_equal(got, ref), (s, str(key))
            if where == "host":
                assert isinstance(val, np.ndarray)
        for j, d in enumerate(sorted(devs, key=lambda d: d.index)):
            for key, buf in d.buffers.items():
                assert np.array_equal(_as_np(buf), arrays[f"s{s}_after_{j}_{key}"]), (s, j)
        n_checked[meta["dtype"]] += 1
    assert n_checked["float32"] >= 15 and n_checked["float64"] >= 15


def test_reference_device_state_semantics(cuda):
    """The reference's DeviceState API unchanged (syncsim.py:90-153): float64
    numpy buffers by default, numpy gradients accumulated, buffers written
    in place by the user, results returned as numpy arrays -- every add and
    divide done by the CUDA kernels."""
    from paper_2403_07544_b200.domain import Side
    from paper_2403_07544_b200.plan import SimulationError
    from paper_2403_07544_b200.syncsim import DeviceState, sync_step
    key = ModuleKey(Side.ENCODER, 0, "full")
    d1, d2 = DeviceState(0, frozenset({key}), 1), DeviceState(1, frozenset({key}), 1)
    assert d1.buffers[key].dtype == np.float64 and d1.buffers[key].shape == (1, 1)
    d1.buffers[key][:] = 2.0
    d2.buffers[key][:] = 4.0
    d1.used.add(key)
    d2.used.add(key)
    synced = sync_step([d1, d2])
    assert synced[key][0, 0] == 3.0 and d1.buffers[key][0, 0] == 3.0 and d2.buffers[key][0, 0] == 3.0
    # renormalised by users, not hosts
    d1, d2 = DeviceState(0, frozenset({key}), 1), DeviceState(1, frozenset({key}), 1)
    d1.buffers[key][:] = 4.0
    d1.used.add(key)
    synced = sync_step([d1, d2])
    assert synced[key][0, 0] == 4.0 and d2.buffers[key][0, 0] == 4.0
    # unused module stays zero
    d1, d2 = DeviceState(0, frozenset({key}), 2), DeviceState(1, frozenset({key}), 2)
    assert np.all(sync_step([d1, d2])[key] == 0.0)
    # device mean, not task mean: ((1 + 3) + 2) / 2
    d1, d2 = DeviceState(0, frozenset({key}), 1), DeviceState(1, frozenset({key}), 1)
    d1.accumulate({key: np.array([[1.0]])})
    d1.accumulate({key: np.array([[3.0]])})
    d2.accumulate({key: np.array([[2.0]])})
    assert sync_step([d1, d2])[key][0, 0] == 3.0
    # unhosted gradient and duplicate index rejected
    other = ModuleKey(Side.DECODER, 0, "x")
    with pytest.raises(SimulationError):
        d1.accumulate({other: np.zeros((1, 1))})
    with pytest.raises(SimulationError):
        sync_step([DeviceState(0, frozenset({key}), 1), DeviceState(0, frozenset({key}), 1)])
    # reset clears buffers and the used set
    d1.reset()
    assert d1.buffers[key][0, 0] == 0.0 and not d1.used


def test_toy_chain_vs_oracle_reference_fp64(cuda):
    """The reference's randomized scenario (toy chain, syncsim.py:34-87)
    through DeviceState.accumulate + sync_step in float64 on the GPU against
    the oracle's oracle_reference: rtol 1e-9 as the reference asserts
    (tests/test_syncsim.py:186-191)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
    from oracle import algorithm1 as A
    from paper_2403_07544_b200.syncsim import DeviceState, sync_step
    for seed in range(6):
        w, y, runs, hosted = A.random_toy_scenario(seed, accum_count=1 + seed % 2)
        devices = {d: DeviceState(d, hosted[d], 3) for d in sorted(hosted)}
        for d, chain, x in runs:
            devices[d].accumulate(A.toy_neg_grads(w, y, chain, A.toy_forward(w, chain, x)))
        synced = sync_step(list(devices.values()))
        oracle = A.device_mean_oracle(runs, hosted, w, y, 3)
        for key in oracle:
            scale = max(1.0, np.abs(oracle[key]).max())
            assert np.allclose(synced[key], oracle[key], rtol=1e-9, atol=1e-12 * scale), (seed, str(key))


@pytest.mark.parametrize("only_ready", [False, True])
def test_reduce_microbench_small_bit_exact(golden, cuda, only_ready):
    """Config-2 generator (scaled sizes) through the engine vs the reference's
    sync_step over 8 DeviceStates."""
    from paper_2403_07544_b200 import _native, ops
    arrays = np.load(os.path.join(GOLD, "reduce_small.npz"))
    mods = golden["reduce_small"]
    bufs = {}
    table = []
    outs = []
    for i, m in enumerate(mods):
        sm = _native.SyncModule()
        for j in range(m["group"]):
            r = m["start"] + j
            t = torch.from_numpy(arrays[f"grad_{r}_{i}"]).to(cuda)
            bufs[(r, i)] = t
            sm.bufs[j] = t.data_ptr()
        out = torch.empty(m["n_params"], device=cuda)
        outs.append(out)
        sm.out = out.data_ptr()
        sm.n_elems = m["n_params"]
        sm.group_size = m["group"]
        sm.used_mask = sum(1 << j for j, f in enumerate(m["ready"]) if f)
        table.append(sm)
    ops.sync_emulated(table, only_ready)
    torch.cuda.synchronize()
    for i, m in enumerate(mods):
        ref = arrays[f"synced_{i}"]
        got = outs[i].cpu().numpy()
        # +0 vs -0 is the only possible difference when unready members are skipped
        assert np.array_equal(got, ref), i
        for j in range(m["group"]):
            assert np.array_equal(bufs[(m["start"] + j, i)].cpu().numpy(), ref)


def test_sync_linearity_and_zero_module(cuda):
    from paper_2403_07544_b200.syncsim import DeviceState, sync_step
    from paper_2403_07544_b200.domain import Side
    k1, k2 = ModuleKey(Side.ENCODER, 0, "full"), ModuleKey(Side.DECODER, 0, "x")
    g = torch.Generator(device="cuda").manual_seed(0)
    base = [torch.randn(1000, device=cuda, generator=g) for _ in range(3)]
    def run(c):
        devs = [DeviceState(i, frozenset({k1, k2}), 1,
                            {k1: base[i] * c, k2: torch.zeros(7, device=cuda)}, {k1} if i != 1 else set())
                for i in range(3)]
        devs[1].buffers[k1] = torch.zeros(1000, device=cuda)
        return sync_step(devs)
    a, b = run(1.0), run(2.5)
    assert torch.allclose(b[k1], 2.5 * a[k1])
    assert torch.equal(a[k2], torch.zeros(7, device=cuda))
    # renormalised by users (2), not hosts (3)
    assert torch.allclose(a[k1], (base[0] + base[2]) / 2)


@pytest.mark.parametrize("n", [0, 1, 3])
def test_fused_update_matches_torch_adam(cuda, n):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
    from oracle.transformer import adam_step
    from paper_2403_07544_b200 import _native, ops
    numel = 100_003 if n != 1 else 65_536
    g = torch.Generator(device="cuda").manual_seed(n)
    grad = torch.randn(numel, device=cuda, generator=g)
    master = torch.randn(numel, device=cuda, generator=g)
    m = torch.randn(numel, device=cuda, generator=g) * 0.1
    v = torch.rand(numel, device=cuda, generator=g) * 0.01
    bf = torch.empty(numel, dtype=torch.bfloat16, device=cuda)
    ref = [t.cpu().clone() for t in (master, m, v)]
    lr, b1, b2, eps, wd, step, inv_ls = 3e-4, 0.9, 0.998, 1e-8, 0.01, 5, 0.5
    mod = _native.AdamModule(grad=grad.data_ptr(), master=master.data_ptr(), exp_avg=m.data_ptr(),
                             exp_avg_sq=v.data_ptr(), param_bf16=bf.data_ptr(), n_elems=numel,
                             n_ready=n, ready_index=-1, step_size=lr / (1 - b1 ** step),
                             inv_sqrt_bc2=1.0 / np.sqrt(1 - b2 ** step))
    ops.fused_update([mod], _native.AdamHyper.make(beta1=b1, beta2=b2, eps=eps, weight_decay=wd,
                                              inv_loss_scale=inv_ls))
    torch.cuda.synchronize()
    if n == 0:
        assert torch.equal(master.cpu(), ref[0])
        return
    adam_step(ref[0], ref[1], ref[2], grad.cpu() / n * inv_ls, step, lr, b1, b2, eps, wd)
    for got, want in zip((master, m, v), ref):
        err = (got.cpu() - want).abs().max() / want.abs().max()
        assert err < 1e-5
    assert torch.equal(bf, master.bfloat16())


def test_fused_update_reads_ready_counts_from_device(cuda):
    from paper_2403_07544_b200 import _native, ops
    numel = 4096
    grads = [torch.ones(numel, device=cuda) * 6 for _ in range(2)]
    masters = [torch.zeros(numel, device=cuda) for _ in range(2)]
    ms = [torch.zeros(numel, device=cuda) for _ in range(2)]
    vs = [torch.zeros(numel, device=cuda) for _ in range(2)]
    ready = torch.tensor([0, 2], dtype=torch.int32, device=cuda)
    mods = [_native.AdamModule(grad=grads[i].data_ptr(), master=masters[i].data_ptr(),
                               exp_avg=ms[i].data_ptr(), exp_avg_sq=vs[i].data_ptr(),
                               param_bf16=None, n_elems=numel, n_ready=0, ready_index=i,
                               step_size=1.0 / 0.1, inv_sqrt_bc2=1.0 / np.sqrt(0.002))
            for i in range(2)]
    ops.fused_update(mods, _native.AdamHyper.make(beta1=0.9, beta2=0.998, eps=1e-8, weight_decay=0.0,
                                             inv_loss_scale=1.0), ready_dev=ready)
    torch.cuda.synchronize()
    assert torch.equal(masters[0], torch.zeros(numel, device=cuda))  # n = 0: no step
    assert torch.allclose(ms[1], torch.full((numel,), 0.3, device=cuda))  # 0.1 * 6/2

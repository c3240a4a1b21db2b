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
    from paper_2403_07544_b200.syncsim import DeviceState
    devs = []
    for j, d in enumerate(meta["devices"]):
        hosted = frozenset(ModuleKey.parse(k) for k in d["hosted"])
        bufs = {k: torch.from_numpy(arrays[f"s{s}_in_{j}_{k}"]).to(cuda) for k in d["hosted"]}
        bufs = {ModuleKey.parse(k): v for k, v in bufs.items()}
        devs.append(DeviceState(d["index"], hosted, 1, bufs, {ModuleKey.parse(k) for k in d["used"]}))
    return devs


def test_sync_step_bit_exact_vs_reference(golden, cuda):
    from paper_2403_07544_b200.syncsim import sync_step
    arrays = np.load(os.path.join(GOLD, "sync_scenarios.npz"))
    n_checked = 0
    for meta in golden["scenarios"]:
        if meta["dtype"] != "float32":
            continue
        s = meta["seed"]
        devs = _devices(meta, arrays, s, cuda)
        synced = sync_step(devs)
        for key, val in synced.items():
            ref = arrays[f"s{s}_synced_{key}"]
            assert np.array_equal(val.cpu().numpy(), ref), (s, str(key))
        for j, d in enumerate(sorted(devs, key=lambda d: d.index)):
            for key, buf in d.buffers.items():
                assert np.array_equal(buf.cpu().numpy(), arrays[f"s{s}_after_{j}_{key}"]), (s, j)
        n_checked += 1
    assert n_checked >= 15


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

"""Option-B exchange (mm_peer_update): every member's shard of every module
in ONE launch over buffers on one B200 -- the multi-rank kernel emulated as
one kernel over all ranks' data.  Checked bit-exact against the already
reference-pinned pair mm_sync_emulated (only ready) + mm_fused_update (n=1),
against the reference's own sync_step on the golden config-2 sample, and for
the masked-load / lazy-zeroing / all-gather properties."""
import json
import math
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
LR, B1, B2, EPS, WD = 3e-4, 0.9, 0.998, 1e-8, 0.01


def _hyper(zero_grad=0, inv_ls=1.0, wd=WD):
    from paper_2403_07544_b200 import _native
    return _native.AdamHyper.make(beta1=B1, beta2=B2, eps=EPS, weight_decay=wd,
                                  inv_loss_scale=inv_ls, zero_grad=zero_grad)


class Mod:
    """One module replicated on g emulated members."""

    def __init__(self, n, g, mask, cuda, gen, step=3, dirty_unready=True):
        self.n, self.g, self.mask, self.step = n, g, mask, step
        self.grad = []
        for j in range(g):
            t = torch.randn(n, device=cuda, generator=gen)
            if not (mask >> j) & 1 and not dirty_unready:
                t.zero_()
            self.grad.append(t)
        base = torch.randn(n, device=cuda, generator=gen)
        self.master = [base.clone() for _ in range(g)]
        m0 = torch.randn(n, device=cuda, generator=gen) * 0.1
        v0 = torch.rand(n, device=cuda, generator=gen) * 0.01
        self.m = [m0.clone() for _ in range(g)]
        self.v = [v0.clone() for _ in range(g)]
        self.w = [torch.zeros(n, dtype=torch.bfloat16, device=cuda) for _ in range(g)]

    def coef(self):
        return LR / (1 - B1 ** self.step), 1.0 / math.sqrt(1 - B2 ** self.step)

    def shards(self, replicate=True):
        from paper_2403_07544_b200.peer import make_shard
        ss, isb = self.coef()
        return [make_shard([t.data_ptr() for t in self.grad], [t.data_ptr() for t in self.w],
                           [t.data_ptr() for t in self.master] if replicate else None,
                           self.master[j].data_ptr(), self.m[j].data_ptr(), self.v[j].data_ptr(),
                           self.n, j, self.mask, ss, isb) for j in range(self.g)]


def _reference_pair(mod: Mod, inv_ls=1.0, wd=WD):
    """sync_emulated(only_ready) on zero-filled copies + fused_update(n=1)."""
    from paper_2403_07544_b200 import _native, ops
    bufs = [t.clone() if (mod.mask >> j) & 1 else torch.zeros_like(t) for j, t in enumerate(mod.grad)]
    sm = _native.SyncModule()
    for j, b in enumerate(bufs):
        sm.bufs[j] = b.data_ptr()
    sm.out, sm.n_elems, sm.group_size, sm.used_mask = None, mod.n, mod.g, mod.mask
    ops.sync_emulated([sm], True)
    master, m, v = mod.master[0].clone(), mod.m[0].clone(), mod.v[0].clone()
    w = torch.empty(mod.n, dtype=torch.bfloat16, device=master.device)
    ss, isb = mod.coef()
    ops.fused_update([_native.AdamModule(grad=bufs[0].data_ptr(), master=master.data_ptr(),
                                         exp_avg=m.data_ptr(), exp_avg_sq=v.data_ptr(),
                                         param_bf16=w.data_ptr(), n_elems=mod.n, n_ready=1,
                                         ready_index=-1, step_size=ss, inv_sqrt_bc2=isb)],
                     _hyper(inv_ls=inv_ls, wd=wd))
    return master, m, v, w


CASES = [  # (n_elems, group, ready mask)
    (65_536, 2, 0b11), (65_536, 2, 0b10), (100_003, 3, 0b101), (1_000_000, 8, 0b10110101),
    (5, 4, 0b0100), (4, 8, 0xff), (7, 8, 0b1), (49_153, 5, 0b11111), (16_384 * 3 + 12, 7, 0b1000000),
]


@pytest.mark.parametrize("n,g,mask", CASES)
def test_peer_update_bit_exact_vs_sync_plus_update(cuda, n, g, mask):
    from paper_2403_07544_b200 import ops
    gen = torch.Generator(device="cuda").manual_seed(n + g + mask)
    mod = Mod(n, g, mask, cuda, gen)
    want = _reference_pair(mod)
    unready_before = {j: mod.grad[j].clone() for j in range(g) if not (mask >> j) & 1}
    ops.peer_update(mod.shards(), _hyper())
    torch.cuda.synchronize()
    for j in range(g):
        # every member: complete bf16 weights and (replicated) fp32 master
        assert torch.equal(mod.w[j], want[3]), j
        assert torch.equal(mod.master[j], want[0]), j
        # moments: member j is authoritative on its own shard
        from paper_2403_07544_b200.plan import shard_begin
        b, e = shard_begin(n, g, j), shard_begin(n, g, j + 1)
        assert torch.equal(mod.m[j][b:e], want[1][b:e]) and torch.equal(mod.v[j][b:e], want[2][b:e])
    for j, before in unready_before.items():  # masked loads: never read, never written
        assert torch.equal(mod.grad[j], before)


def test_peer_update_zero_grad_and_no_replication(cuda):
    from paper_2403_07544_b200 import ops
    from paper_2403_07544_b200.plan import shard_begin
    gen = torch.Generator(device="cuda").manual_seed(7)
    n, g, mask = 300_001, 4, 0b1011
    mod = Mod(n, g, mask, cuda, gen)
    want = _reference_pair(mod, inv_ls=0.25)
    masters0 = [t.clone() for t in mod.master]
    junk = mod.grad[2].clone()
    ops.peer_update(mod.shards(replicate=False), _hyper(zero_grad=1, inv_ls=0.25))
    torch.cuda.synchronize()
    for j in range(g):
        b, e = shard_begin(n, g, j), shard_begin(n, g, j + 1)
        assert torch.equal(mod.master[j][b:e], want[0][b:e])
        # without replication the other shards of member j's master are untouched
        rest = torch.ones(n, dtype=torch.bool, device=cuda)
        rest[b:e] = False
        assert torch.equal(mod.master[j][rest], masters0[j][rest])
        assert torch.equal(mod.w[j], want[3])
        if (mask >> j) & 1:
            assert torch.count_nonzero(mod.grad[j]) == 0  # consumed and cleared by the owners
    assert torch.equal(mod.grad[2], junk)  # unready member: untouched


def test_peer_update_zero_ready_is_noop(cuda):
    from paper_2403_07544_b200 import ops
    gen = torch.Generator(device="cuda").manual_seed(1)
    mod = Mod(10_000, 3, 0, cuda, gen)
    before = [t.clone() for t in mod.master]
    ops.peer_update(mod.shards(), _hyper())
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(mod.master, before))
    assert all(torch.count_nonzero(w) == 0 for w in mod.w)


def test_peer_update_many_modules_one_launch_vs_reference_sync_step(golden_small, cuda):
    """Every shard of the golden config-2 sample's 24 modules (the reference
    sync_step's own inputs, tests/golden/reduce_small.npz) in one launch:
    bit-identical to sync_emulated (bit-exact vs the reference, see
    test_sync_gpu.py) + fused_update."""
    from paper_2403_07544_b200 import _native, ops
    arrays, mods = golden_small
    all_shards, objs = [], []
    for i, m in enumerate(mods):
        mask = sum(1 << j for j, f in enumerate(m["ready"]) if f)
        gen = torch.Generator(device="cuda").manual_seed(i)
        mod = Mod(m["n_params"], m["group"], mask, cuda, gen)
        for j in range(m["group"]):
            mod.grad[j] = torch.from_numpy(arrays[f"grad_{m['start'] + j}_{i}"]).to(cuda)
        objs.append((mod, _reference_pair(mod)))
        all_shards += mod.shards()
    assert len(all_shards) > 1
    ops.peer_update(all_shards, _hyper())
    torch.cuda.synchronize()
    for i, (mod, want) in enumerate(objs):
        for j in range(mod.g):
            assert torch.equal(mod.master[j], want[0]), (i, j)
            assert torch.equal(mod.w[j], want[3]), (i, j)


@pytest.fixture(scope="module")
def golden_small():
    with open(os.path.join(GOLD, "golden.json")) as f:
        mods = json.load(f)["reduce_small"]
    return np.load(os.path.join(GOLD, "reduce_small.npz")), mods


def test_peer_barrier_without_peers_is_noop(cuda):
    from paper_2403_07544_b200 import _native, ops
    sig = _native.PeerSignal()
    sig.n_peers = 0
    ops.peer_barrier(sig)
    flags = torch.zeros(32, dtype=torch.int32, device=cuda)
    sig.local_flags = flags.data_ptr()
    assert _native.lib().mm_peer_barrier(sig, None) == 0


def test_ipc_export_offsets(cuda):
    """Export gives the allocation's handle and the tensor's offset in it;
    views of one allocation share the handle."""
    from paper_2403_07544_b200 import ops
    t = torch.empty(1 << 20, device=cuda)
    h0, o0 = ops.ipc_export(t)
    h1, o1 = ops.ipc_export(t[1024:])
    assert h0 == h1 and o1 - o0 == 4096 and len(h0) == 64

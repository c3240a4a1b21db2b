"""End-to-end parity of the B200 trainer step against the CPU oracle on
identical seeded inputs and weights.

* ready counts and groups: bit-exact with the reference (golden fixtures);
* every transformer block (FFN, self / causal self / cross attention) on
  identical inputs: outputs, input gradients and parameter gradients within
  2e-3 max-relative of the bf16-faithful oracle (the oracle rounds to bf16
  exactly where the engine stores bf16);
* the whole step (embeddings -> 2+2 layers -> generator -> CE -> backward):
  loss within 1e-3 relative (measured ~2e-5); every module's gradient within
  3e-2 relative in L2 norm of the bf16-faithful oracle (measured 0.5-2.3 %)
  and within 5e-2 of the pure fp32 oracle (measured <= 2.9 %).  That is the
  whole-model bf16 noise floor: fp32-level accumulation-order differences
  flip bf16 roundings and ReLU masks and random-init blocks amplify them
  3-5x each ("bf16 noise floor"); per-element max-relative errors
  are therefore only asserted at block level;
* K3 on the engine's own reduced gradients: 1e-5 (fp32) vs torch.optim.Adam.
"""
import json
import os
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import transformer as OT  # noqa: E402
from paper_2403_07544_b200 import configs  # noqa: E402
from paper_2403_07544_b200.data import make_batch  # noqa: E402
from paper_2403_07544_b200.domain import ClusterTopology, DeviceId  # noqa: E402
from paper_2403_07544_b200.model import bf16_round, init_module  # noqa: E402
from paper_2403_07544_b200.plan import embedding_keys  # noqa: E402

pytestmark = pytest.mark.gpu
TOL_BF16 = 2e-2      # loss, block-level
# whole-model gradients at the small test shape (d128, ~320 tokens), L2 norm,
# vs the bf16-faithful oracle: any bf16 implementation sits at 2-6 % max-rel
# there (tools/diag_parity.py); the 2e-2 max-relative contract is asserted at
# the BASELINE shapes in test_parity_shapes_gpu.py
TOL_MODEL = 3e-2


def effective_weights(layout, master):
    """What the GPU computes with: bf16 matrices / tables, fp32 LN and biases."""
    out = master.copy()
    for p in layout.params.values():
        if p.init in ("xavier", "embed"):
            sl = slice(p.offset, p.offset + p.numel)
            out[sl] = bf16_round(master[sl])
    return out


def rel(a, b):
    """max|a-b| / max|b| per module (test_acceptance.py:66-68 convention)."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


def rel_norm(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def batches_for(world, accum, shape, seed=0, sentences=16):
    spec = configs.config1().data
    out = []
    for r in range(world):
        rng = np.random.default_rng([seed, r])
        out.append([make_batch(rng, spec, shape.vocab, sentences=sentences) for _ in range(accum)])
    return out


@pytest.mark.parametrize("accum", [1, 2])
def test_single_rank_step_vs_oracle(cuda, accum):
    from paper_2403_07544_b200.engine import DeviceBatch, Engine
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
    topo = ClusterTopology(1, 1, 3)
    eng = Engine(tasks, topo, shape, rank=0, world=1, device=cuda, seed=0)
    hb = batches_for(1, accum, shape)[0]
    dbs = [DeviceBatch(b, cuda) for b in hb]
    masters0 = {k: st.master.cpu().numpy().copy() for k, st in eng.states.items()}
    info = eng.step(0, dbs)
    torch.cuda.synchronize()
    loss_gpu = eng.loss_sum.item()
    # oracle on the same tasks / batches / weights
    layouts = eng.layouts
    eff = {k: effective_weights(layouts[k], v) for k, v in masters0.items()}
    task_by_id = {t.id: t for t in tasks}
    picked = [task_by_id[tid] for tid in info["tasks"]]
    grads, used, losses = OT.local_grads(list(zip(picked, hb)), eff, layouts, shape,
                                         embedding_keys, bf16=True)
    assert abs(loss_gpu - sum(losses)) / sum(losses) < 1e-3
    for k, st in eng.states.items():
        g = st.grad.cpu().numpy()
        if k in used:
            assert rel_norm(g, grads[k].numpy()) < TOL_MODEL, str(k)
    grads32, _, losses32 = OT.local_grads(list(zip(picked, hb)), eff, layouts, shape,
                                          embedding_keys, bf16=False)
    assert abs(loss_gpu - sum(losses32)) / sum(losses32) < 1e-3
    for k in used:
        assert rel_norm(eng.states[k].grad.cpu().numpy(), grads32[k].numpy()) < 5e-2, str(k)
    # K3 on the engine's own (n = 1) gradients vs torch.optim.Adam semantics
    a = eng.adam
    for k, st in eng.states.items():
        m0 = torch.from_numpy(masters0[k])
        mm, vv = torch.zeros_like(m0), torch.zeros_like(m0)
        if k in used:
            OT.adam_step(m0, mm, vv, st.grad.cpu(), 1, a.lr, a.beta1, a.beta2, a.eps)
        assert rel(st.master.cpu().numpy(), m0.numpy()) < 1e-5, str(k)


@pytest.mark.parametrize("accum", [1, 2])
def test_config1_two_ranks_emulated(cuda, accum):
    """Config 1 (world 2) on one B200: ready counts bit-exact with the
    reference, Algorithm-1 synced gradients within TOL_MODEL (3e-2, relative
    L2) of the bf16-faithful oracle at this 16-sentence shape; the 2e-2
    max-relative contract is asserted at the BASELINE shapes
    (test_parity_shapes_gpu.py)."""
    from paper_2403_07544_b200.cluster import EmulatedCluster
    from paper_2403_07544_b200.engine import DeviceBatch
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        gold = json.load(f)["groups_ready"][f"config1_accum{accum}"]
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    cl = EmulatedCluster(w.tasks, w.topo, shape, world=2, device=cuda, seed=0)
    assert {str(k): v for k, v in cl.plan.groups.items() if k.position >= 0} == gold["groups"]
    layouts = cl.ranks[0].layouts
    task_by_id = {t.id: t for t in w.tasks}
    for step in range(2):
        hb = batches_for(2, accum, shape, seed=step)
        masters0 = [{k: st.master.cpu().numpy().copy() for k, st in eng.states.items()}
                    for eng in cl.ranks]
        info = cl.step(step, [[DeviceBatch(b, cuda) for b in hb[r]] for r in range(2)])
        torch.cuda.synchronize()
        ready = {str(k): v for k, v in info["ready"].items() if k.position >= 0}
        assert ready == gold["ready"][step]
        per_g, per_u = {}, {}
        for r in range(2):
            eff = {k: effective_weights(layouts[k], v) for k, v in masters0[r].items()}
            picked = [task_by_id[t] for t in info["tasks"][r]]
            per_g[r], per_u[r], _ = OT.local_grads(list(zip(picked, hb[r])), eff, layouts, shape,
                                                   embedding_keys, bf16=True)
        synced, counts = OT.algorithm1(per_g, per_u, cl.plan.groups)
        assert {str(k): v for k, v in counts.items() if k.position >= 0} == gold["ready"][step]
        for k, members in cl.plan.groups.items():
            for r in members:
                if counts[k] == 0:
                    continue  # n = 0: buffers untouched, no update (syncsim.py:143-145)
                g = cl.ranks[r].states[k].grad.cpu().numpy()
                assert rel_norm(g, synced[k].numpy()) < TOL_MODEL, (step, r, str(k))
            # replicas stay identical after the update
            if len(members) == 2:
                a, b = (cl.ranks[r].states[k].master for r in members)
                assert torch.equal(a, b)


@pytest.mark.parametrize("block", ["ffn", "self", "causal", "cross"])
def test_block_vs_bf16_oracle(cuda, block):
    """One block of the engine on identical inputs vs autograd through the
    bf16-faithful oracle: tight max-relative agreement."""
    from paper_2403_07544_b200 import ops
    from paper_2403_07544_b200.engine import Engine
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
    eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, device=cuda)
    key = [k for k in eng.states if k.position == 0 and k.side.value == "decoder"][0]
    st = eng.states[key]
    lay = st.layout
    eff = torch.from_numpy(effective_weights(lay, st.master.cpu().numpy())).requires_grad_(True)
    P = OT.Precision(True)
    d, H = shape.d_model, shape.heads
    g = torch.Generator().manual_seed(7)
    lens = [20, 37, 43, 50, 60, 90]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    slens = [9, 30, 51, 12, 70, 33]
    cus = np.concatenate([[0], np.cumsum(slens)]).astype(np.int32)
    T, S = int(cu[-1]), int(cus[-1])
    x = torch.randn(T, d, generator=g)
    mem = torch.randn(S, d, generator=g).bfloat16().float()
    dout = torch.randn(T, d, generator=g) * 1e-2
    ops.memset(st.grad, 0)
    xg, cu_d = x.to(cuda), torch.from_numpy(cu).to(cuda)
    sv = []

    class DB:
        cu_tgt, cu_src = cu_d, torch.from_numpy(cus).to(cuda)
        n_seq, max_tgt, max_src = len(lens), max(lens), max(slens)
    memg = mem.to(cuda).bfloat16()
    dmem = eng._zeros(S, d)
    if block == "ffn":
        out = eng._ffn_fwd(st, "l0.", xg, sv)
    elif block == "cross":
        out = eng._cross_block_fwd(st, "l0.", xg, memg, DB, sv)
    else:
        out = eng._self_block_fwd(st, "l0.", xg, cu_d, len(lens), max(lens), block == "causal", sv)
    dx = dout.to(cuda).clone()
    dxb = torch.empty(T, d, device=cuda, dtype=torch.bfloat16)
    ops.cast_bf16(dx, dxb)
    if block == "ffn":
        eng._ffn_bwd(st, "l0.", sv[0], dx, dxb)
    elif block == "cross":
        eng._cross_bwd(st, "l0.", sv[0], dx, dxb, memg, dmem, DB)
    else:
        eng._self_bwd(st, "l0.", sv[0], dx, dxb, cu_d, len(lens), max(lens), block == "causal")
    torch.cuda.synchronize()
    xr = x.clone().requires_grad_(True)
    mr = mem.clone().requires_grad_(True)
    if block == "ffn":
        o = xr + P.g(OT._lin(OT._ffn_act(P, xr, eff, lay, "l0."), eff, lay, "l0.ff2"))
    elif block == "cross":
        q = P.vg(OT._lin(P.v(OT._ln(xr, eff, lay, "l0.lnc")), eff, lay, "l0.cq"))
        kv = P.vg(OT._lin(mr, eff, lay, "l0.ckv"))
        a = P.vg(OT._attention(q, kv[:, :d], kv[:, d:], cu.tolist(), cus.tolist(), H, False, True))
        o = xr + P.g(OT._lin(a, eff, lay, "l0.cout"))
    else:
        qkv = P.vg(OT._lin(P.v(OT._ln(xr, eff, lay, "l0.ln1")), eff, lay, "l0.qkv"))
        a = P.vg(OT._attention(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], cu.tolist(),
                               cu.tolist(), H, block == "causal", True))
        o = xr + P.g(OT._lin(a, eff, lay, "l0.out"))
    o.backward(dout)
    assert rel(out.cpu().numpy(), o.detach().numpy()) < 2e-3
    assert rel(dx.cpu().numpy(), xr.grad.numpy()) < 2e-3
    if block == "cross":
        assert rel(dmem.cpu().numpy(), mr.grad.numpy()) < 2e-3
    gg = st.grad.cpu().numpy()
    checked = 0
    for name, p in lay.params.items():
        ref = eff.grad[p.offset:p.offset + p.numel].numpy()
        if not name.startswith("l0.") or not np.abs(ref).max() > 0:
            continue
        # the oracle rounds the attention backward's dS to bf16 where the
        # engine stores it (oracle/transformer._AttnRoundDS)
        assert rel(gg[p.offset:p.offset + p.numel], ref) < 2e-3, name
        checked += 1
    assert checked >= 4


def test_native_driver_matches_python_path(cuda):
    """mm_task_fwd_bwd (C++ step driver) issues the same kernels in the same
    order as the per-op Python path: same loss and gradients up to the
    nondeterministic ordering of fp32 atomics / TMA reduce-adds (embedding
    scatter-add, split-K wgrad, LayerNorm dgamma), which bf16 roundings
    downstream amplify to a few 1e-5 -- hence 1e-3."""
    from paper_2403_07544_b200.engine import DeviceBatch, Engine
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
    hb = batches_for(1, 1, shape, seed=3)[0]
    grads, losses = [], []
    for native in (True, False):
        eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, device=cuda)
        eng.native = native
        eng.step(0, [DeviceBatch(hb[0], cuda)])
        torch.cuda.synchronize()
        grads.append({k: st.grad.cpu().numpy().copy() for k, st in eng.states.items()})
        losses.append(eng.loss_sum.item())
    assert abs(losses[0] - losses[1]) <= 1e-6 * abs(losses[1])
    for k in grads[0]:
        if np.abs(grads[1][k]).max() > 0:
            assert rel_norm(grads[0][k], grads[1][k]) < 1e-3, str(k)


def test_partially_shared_encoder_vs_oracle(cuda):
    """Config-4 structure (language encoder stack + shared FULL encoder stack,
    group decoders) at a small shape: two encoder positions per task, a
    module shared by every task, gradients vs the bf16-faithful oracle."""
    import itertools
    from paper_2403_07544_b200.engine import DeviceBatch, Engine
    from paper_2403_07544_b200.sharing import ArchSpec, SharingPattern as SP
    shape = configs.SHAPE_CFG1_GPU
    langs = ["aa", "bb", "cc", "dd"]
    groups = {"aa": "g0", "bb": "g0", "cc": "g1", "dd": "g1"}
    arch = ArchSpec(((SP.LANGUAGE, 1), (SP.FULL, 1)), ((SP.TGT_GROUP, 2),))
    tasks = [configs._task(arch, s, t, DeviceId(0, 0), groups) for s, t in itertools.permutations(langs, 2)]
    eng = Engine(tasks, ClusterTopology(1, 1, len(tasks)), shape, device=cuda)
    hb = batches_for(1, 2, shape, seed=11)[0]
    m0 = {k: st.master.cpu().numpy().copy() for k, st in eng.states.items()}
    info = eng.step(0, [DeviceBatch(b, cuda) for b in hb])
    torch.cuda.synchronize()
    by_id = {t.id: t for t in tasks}
    picked = [by_id[t] for t in info["tasks"]]
    assert all(len(t.enc_modules) == 2 for t in picked)
    eff = {k: effective_weights(eng.layouts[k], v) for k, v in m0.items()}
    grads, used, losses = OT.local_grads(list(zip(picked, hb)), eff, eng.layouts, shape,
                                         embedding_keys, bf16=True)
    assert abs(eng.loss_sum.item() - sum(losses)) / sum(losses) < 1e-3
    for k in used:
        assert rel_norm(eng.states[k].grad.cpu().numpy(), grads[k].numpy()) < TOL_MODEL, str(k)


@pytest.mark.parametrize("d_model,heads,ffn", [(512, 8, 2048), (1024, 16, 1024)])
def test_fused_layernorm_driver_matches_python_path(cuda, d_model, heads, ffn, monkeypatch):
    """At d_model 512 / 1024 the native driver fuses every LayerNorm that
    follows a residual GEMM into that GEMM's epilogue (cluster + DSMEM row
    statistics, MM_EPI_F32_RESID_LN); the per-op Python path runs standalone
    LayerNorm kernels.  Same loss and gradients up to the LayerNorm summation
    order (fp32) that bf16 roundings downstream amplify."""
    from paper_2403_07544_b200.configs import ModelShape
    from paper_2403_07544_b200.engine import DeviceBatch, Engine
    monkeypatch.setenv("MM_FUSE_LN", "1")  # opt-in path (off by default: slower)
    shape = ModelShape(d_model, heads, ffn, 1000, 32)
    w = configs.config1(shape)
    tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
    hb = batches_for(1, 1, shape, seed=5, sentences=48)[0]
    grads, losses = [], []
    for native in (True, False):
        eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, device=cuda)
        eng.native = native
        eng.step(0, [DeviceBatch(hb[0], cuda)])
        torch.cuda.synchronize()
        grads.append({k: st.grad.cpu().numpy().copy() for k, st in eng.states.items()})
        losses.append(eng.loss_sum.item())
    # 3e-5: the fused epilogue's LayerNorm row sums (DSMEM partials) round
    # differently from the standalone kernel's, and every bf16 rounding
    # downstream (the tcgen05 forward's bf16 P among them) can flip
    assert abs(losses[0] - losses[1]) <= 3e-5 * abs(losses[1])
    for k in grads[0]:
        if np.abs(grads[1][k]).max() > 0:
            assert rel_norm(grads[0][k], grads[1][k]) < 2e-2, str(k)


def test_lazy_grad_zeroing_matches_memset(cuda):
    """zero_in_update (the fused update zeroes the gradient it consumed, no
    memset before the next use; Trainer's default) gives the same parameters
    over several steps as zeroing every bucket before its first use."""
    from paper_2403_07544_b200.engine import DeviceBatch, Engine
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
    hb = batches_for(1, 4, shape, seed=9)[0]
    masters = []
    for lazy in (False, True):
        eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, device=cuda, seed=0)
        eng.zero_in_update = lazy
        for s, b in enumerate(hb):
            eng.step(s, [DeviceBatch(b, cuda)])
        eng.sync_updates()
        torch.cuda.synchronize()
        masters.append({k: st.master.cpu().numpy().copy() for k, st in eng.states.items()})
        if lazy:  # every bucket an update consumed is clean again
            for k, st in eng.states.items():
                if k not in eng._dirty:
                    assert float(st.grad.abs().max()) == 0.0, str(k)
    for k in masters[0]:
        assert rel(masters[1][k], masters[0][k]) < 1e-5, str(k)


def test_store_first_wgrad_matches_reduce_add(cuda):
    """A module's first micro-batch of a step STORES its weight-matrix
    gradients (memset of the bucket tail only); later micro-batches
    reduce-add.  Three steps of two micro-batches of different tasks (modules
    fresh in the first or in the second micro-batch, shared ones
    accumulating; dirty buckets from the previous step) against memset +
    reduce-add everywhere (MM_STORE_WGRAD=0), both engines restarted from the
    same state every step: gradients and optimizer states agree up to fp32
    summation order (at this shape the weight-gradient launches split K, and
    the split partials, like the fused bias-gradient atomics, reduce-add in
    whatever order the CTAs finish).  A store that missed its zeroing or a
    double count would be O(1)."""
    from paper_2403_07544_b200.engine import DeviceBatch, Engine
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
    hb = batches_for(1, 6, shape, seed=11)[0]
    engs = []
    for store in (True, False):
        eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, device=cuda, seed=0)
        eng.store_first_wgrad = store
        eng.defer_update = False
        engs.append(eng)
    assert any(st.layout.dense_end > 0 for st in engs[0].states.values())
    fields = ("grad", "master", "exp_avg", "exp_avg_sq", "weights")
    for s in range(3):
        for k, st in engs[0].states.items():  # same starting state, dirty gradients included
            sb = engs[1].states[k]
            for f in fields:
                getattr(sb, f).copy_(getattr(st, f))
            sb.step = st.step
        engs[1]._dirty = set(engs[0]._dirty)
        pick = [tasks[(s + j) % len(tasks)] for j in range(2)]
        for eng in engs:
            eng.step(s, [DeviceBatch(hb[2 * s + j], cuda) for j in range(2)], tasks=pick)
        torch.cuda.synchronize()
        for k, st in engs[0].states.items():
            sb = engs[1].states[k]
            for f in fields[:4]:
                assert rel(getattr(st, f).cpu().numpy(), getattr(sb, f).cpu().numpy()) < 1e-5, \
                    (s, str(k), f)


def test_config1_peer_exchange_bit_exact_vs_sync(cuda):
    """Option B (one mm_peer_update launch over both emulated ranks' shards)
    vs the sync + per-rank K3 path on the SAME gradients (the backward's
    atomics make two backward runs differ in the last bits): every rank's
    weights, masters and step counts bit-identical, for three steps."""
    from paper_2403_07544_b200.cluster import EmulatedCluster
    from paper_2403_07544_b200.engine import DeviceBatch
    from paper_2403_07544_b200.plan import shard_begin
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    cl = EmulatedCluster(w.tasks, w.topo, shape, world=2, device=cuda, seed=0)
    fields = ("grad", "master", "exp_avg", "exp_avg_sq", "weights")

    def snapshot():
        return [{k: ([getattr(st, f).clone() for f in fields], st.step) for k, st in e.states.items()}
                for e in cl.ranks]

    def restore(snap):
        for e, d in zip(cl.ranks, snap):
            for k, (ts, step) in d.items():
                for f, t in zip(fields, ts):
                    getattr(e.states[k], f).copy_(t)
                e.states[k].step = step

    for step in range(3):
        hb = batches_for(2, 2, shape, seed=step)
        used, _ = cl.compute(step, [[DeviceBatch(b, cuda) for b in hb[r]] for r in range(2)])
        snap = snapshot()
        cl.exchange_and_update(used, exchange="sync")
        want = snapshot()
        restore(snap)
        cl.exchange_and_update(used, exchange="peer")
        torch.cuda.synchronize()
        for r, e in enumerate(cl.ranks):
            for k, st in e.states.items():
                members = cl.plan.groups[k]
                assert st.step == want[r][k][1], (step, r, str(k))
                n = st.master.numel()
                # after option B member j's moments are authoritative on its
                # own shard j only, so shard j of every member must equal what
                # the sync path computed on member j
                for j, owner in enumerate(members):
                    b, e_ = shard_begin(n, len(members), j), shard_begin(n, len(members), j + 1)
                    ts = want[owner][k][0]
                    assert torch.equal(st.weights[b:e_], ts[4][b:e_]), (step, r, str(k), j)
                    assert torch.equal(st.master[b:e_], ts[1][b:e_]), (step, r, str(k), j)


def test_trainer_on_fullconfig_corpora(cuda, tmp_path):
    """f2: the reference's FullConfig YAML + per-task corpora (pre-tokenized
    ids) through DataPipeline -> Trainer.train_step: the batch of each
    micro-batch comes from the task the multiplexer picked, in pick order."""
    from paper_2403_07544_b200.datapath import DataPipeline, load_full_config
    from paper_2403_07544_b200.engine import Trainer
    from paper_2403_07544_b200.plan import Multiplexer, build_plan
    cfg = load_full_config(os.path.join(ROOT, "tests", "golden", "fullconfig_config1.yaml"))
    shape = configs.SHAPE_CFG1_GPU
    rng = np.random.default_rng(0)
    for t in cfg.task_list():
        for p in (t.src_path, t.tgt_path):
            os.makedirs(tmp_path / os.path.dirname(p), exist_ok=True)
            with open(tmp_path / p, "w") as f:
                for _ in range(200):  # some lines longer than max_len: clipped
                    f.write(" ".join(map(str, rng.integers(4, shape.vocab, rng.integers(3, 50)))) + "\n")
    pipe = DataPipeline(cfg.task_list(), tokens=256, root=str(tmp_path), capacity=24, pool=48,
                        vocab=shape.vocab, max_len=shape.max_len)
    seen = []
    orig = pipe.batch_for
    pipe.batch_for = lambda task: (seen.append(task.id), orig(task))[1]
    tr = Trainer(cfg.task_list(), cfg.topology, shape, rank=0, world=1, device=cuda)
    losses = [tr.train_step(pipeline=pipe, accum=2) for _ in range(3)]
    tr.close()
    assert all(np.isfinite(losses)) and all(l > 0 for l in losses)
    mux = Multiplexer(build_plan(cfg.task_list(), cfg.topology), 0, 0)
    assert seen == [mux.pick(s).id for s in range(3) for _ in range(2)]


def test_checkpoint_resume_bit_exact(cuda, tmp_path):
    """f4: save after two steps, resume in a fresh trainer: restored state is
    bit-identical, the multiplexer continues the same pick sequence and the
    next step's loss matches (to the order of the cross-entropy's atomic
    loss accumulation)."""
    from paper_2403_07544_b200.engine import Trainer
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    rng = np.random.default_rng(5)
    batches = [[make_batch(rng, w.data, shape.vocab, sentences=16)] for _ in range(3)]
    tr = Trainer(w.tasks, w.topo, shape, rank=0, world=1, device=cuda, seed=0)
    for b in batches[:2]:
        tr.train_step(b)
    files = tr.save_checkpoint(str(tmp_path))
    assert files and all(os.path.exists(f) for f in files)
    saved = {k: (st.master.clone(), st.exp_avg.clone(), st.weights.clone(), st.step)
             for k, st in tr.engine.states.items()}
    next_pick = tr.engine.mux.rng.getstate()
    loss3 = tr.train_step(batches[2])
    tr.close()
    tr2 = Trainer(w.tasks, w.topo, shape, rank=0, world=1, device=cuda, seed=123)  # other init
    tr2.load_checkpoint(str(tmp_path))
    assert tr2.step_idx == 2 and tr2.engine.mux.rng.getstate() == next_pick
    for k, st in tr2.engine.states.items():
        m, v, wgt, step = saved[k]
        assert torch.equal(st.master, m) and torch.equal(st.exp_avg, v), str(k)
        assert torch.equal(st.weights, wgt) and st.step == step, str(k)
    assert abs(tr2.train_step(batches[2]) - loss3) <= 1e-6 * abs(loss3)
    tr2.close()


@pytest.mark.parametrize("case", ["config1_accum1", "config1_accum2", "config3_w2", "config3_w4"])
def test_run_benchmark_ledger_matches_reference(cuda, case):
    """syncsim.run_benchmark (the real trainer on emulated ranks) keeps the
    reference run_benchmark's ledger definitions: per-step ready / gradient
    bytes and tokens, and the summary counts, equal to the reference's own
    outputs (tests/golden/ledger.json); times are measured and positive."""
    from paper_2403_07544_b200.configs import ModelShape
    from paper_2403_07544_b200.syncsim import run_benchmark
    with open(os.path.join(ROOT, "tests", "golden", "ledger.json")) as f:
        gold = json.load(f)[case]
    if case.startswith("config1"):
        w = configs.config1()
        steps, accum, bt = 4, int(case[-1]), 256
    else:
        w = configs.config3(int(case[-1]))
        steps, accum, bt = 3, 1, 512
    shape = ModelShape(128, 2, 256, 1000, 32)
    ledger, summary = run_benchmark(w.tasks, w.topo, steps, seed=0, accum_count=accum,
                                    batch_tokens=bt, shape=shape, device=cuda)
    assert [[r.ready_bytes, r.grad_bytes, r.tokens] for r in ledger.records] == gold["records"]
    for k, v in gold["summary"].items():
        assert summary[k] == v, k
    assert all(r.compute_time > 0 and r.comm_time >= 0 for r in ledger.records)
    assert summary["tokens_per_sec"] > 0
    assert ledger.to_tsv().count("\n") == steps + 1


def test_step_optimizer_skips_unready_modules(cuda):
    """step_optimizer: n >= 1 modules take one Adam step on grad / n, n = 0
    modules are untouched (grad = None semantics)."""
    from paper_2403_07544_b200.model import ModuleState, module_layouts
    from paper_2403_07544_b200.plan import build_plan
    from paper_2403_07544_b200.syncsim import step_optimizer
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    plan = build_plan(w.tasks, w.topo)
    layouts = module_layouts(plan, shape)
    keys = sorted(layouts)[:2]
    sts = {k: ModuleState(layouts[k], shape, cuda, 0) for k in keys}
    for st in sts.values():
        st.grad.normal_()
    before = {k: st.master.clone() for k, st in sts.items()}
    step_optimizer(sts, {keys[0]: 2, keys[1]: 0})
    torch.cuda.synchronize()
    assert sts[keys[0]].step == 1 and not torch.equal(sts[keys[0]].master, before[keys[0]])
    assert sts[keys[1]].step == 0 and torch.equal(sts[keys[1]].master, before[keys[1]])


def test_train_steps_lookahead_matches_train_step(cuda):
    """Trainer.train_steps (host lookahead staging) gives the same losses as
    the same batches through train_step one at a time."""
    from paper_2403_07544_b200.engine import Trainer
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    rng = np.random.default_rng(3)
    batches = [[make_batch(rng, w.data, shape.vocab, sentences=16)] for _ in range(4)]
    tr = Trainer(w.tasks, w.topo, shape, rank=0, world=1, device=cuda, seed=0)
    a = [tr.train_step(b) for b in batches]
    tr.close()
    tr = Trainer(w.tasks, w.topo, shape, rank=0, world=1, device=cuda, seed=0)
    b = tr.train_steps(iter(batches), len(batches))
    tr.close()
    assert len(b) == 4 and all(abs(x - y) <= 1e-5 * abs(x) for x, y in zip(a, b))


def test_long_sequences_step_vs_oracle(cuda):
    """A step whose batch mixes short sentences with ones longer than 128 rows
    (config 5's tail): the tcgen05 attention kernels take the groups within
    128 rows, the mma.sync kernels the rest, inside the native driver; loss
    and module gradients against the bf16-faithful oracle."""
    from paper_2403_07544_b200.configs import DataSpec, ModelShape
    from paper_2403_07544_b200.engine import DeviceBatch, Engine
    shape = ModelShape(128, 2, 256, 1000, 256)
    w = configs.config1(shape)
    tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
    eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, rank=0, world=1, device=cuda, seed=0)
    spec = DataSpec(0, 0, 0, 20, 250, 0.0)  # uniform lengths 20..250 on both sides
    hb = [make_batch(np.random.default_rng(11), spec, shape.vocab, sentences=10)]
    assert max(np.diff(hb[0].cu_src).max(), np.diff(hb[0].cu_tgt).max()) > 128
    masters0 = {k: st.master.cpu().numpy().copy() for k, st in eng.states.items()}
    info = eng.step(0, [DeviceBatch(b, cuda) for b in hb])
    torch.cuda.synchronize()
    layouts = eng.layouts
    eff = {k: effective_weights(layouts[k], v) for k, v in masters0.items()}
    task_by_id = {t.id: t for t in tasks}
    picked = [task_by_id[tid] for tid in info["tasks"]]
    grads, used, losses = OT.local_grads(list(zip(picked, hb)), eff, layouts, shape,
                                         embedding_keys, bf16=True)
    assert abs(eng.loss_sum.item() - sum(losses)) / sum(losses) < 1e-3
    for k, st in eng.states.items():
        if k in used:
            assert rel_norm(st.grad.cpu().numpy(), grads[k].numpy()) < TOL_MODEL, str(k)

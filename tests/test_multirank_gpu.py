"""Engine.step with world > 1, on one B200: every rank's unmodified step
(K1 ready-bitmask all-reduce, decode to counts and broadcast roots, zero
contribution of hosted-but-unused members, K2 sum or n = 1 broadcast in
sorted ModuleKey order, the decoder-side exchange + update on the side
stream while the encoder backward runs, K3 with the ready count) runs in its
own host thread against an in-process stand-in for the NCCL communicators
(paper_2403_07544_b200/emucomm.py).

Checked over three steps that cover n = 0 (config-3 structure), 1 and >= 2
on shared modules:
* ready counts bit-exact with the group map / multiplexer of the reference
  (syncsim.py:313-363, through plan.ready_counts_all);
* every rank's master, Adam moments, step count and bf16 weights
  bit-identical to EmulatedCluster (the literal Algorithm-1 exchange,
  syncsim.py:121-153, as one mm_sync_emulated launch + per-rank K3) applied to
  the same per-rank gradients -- the gradients the threaded ranks posted to
  the communicator (recorded before the reduction), since two backward runs
  differ in the last bits (fp32 atomics).
"""
import numpy as np
import pytest
import torch

from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.data import make_batch

pytestmark = pytest.mark.gpu
FIELDS = ("master", "exp_avg", "exp_avg_sq", "weights")


def _world_case(name):
    shape = configs.SHAPE_CFG1_GPU
    if name == "config1true_w2":  # config 1 at its own shape (d64, head_dim 16)
        w = configs.config1()
        return w.tasks, w.topo, w.shape, 2, w.data
    if name == "config1_w2":
        w = configs.config1(shape)
        return w.tasks, w.topo, shape, 2, w.data
    w = configs.config3(4)  # config-3 structure (56 directions, groups of 4) at a small shape
    return w.tasks, w.topo, shape, 4, configs.config1().data


@pytest.mark.parametrize("case,exchange", [("config1_w2", "nccl"), ("config3_w4", "nccl"),
                                           ("config1true_w2", "nccl"), ("config1true_w2", "partitioned"),
                                           ("config1_w2", "partitioned"),
                                           ("config3_w4", "partitioned")])
def test_threaded_ranks_match_emulated_cluster(cuda, case, exchange):
    """exchange="nccl": all-reduce (n = 1: broadcast) + replicated K3;
    "partitioned": reduce-scatter, K3 on the owned shard, bf16 all-gather --
    there masters and moments are compared on each member's own shard, the
    bf16 weights everywhere."""
    from paper_2403_07544_b200.cluster import EmulatedCluster
    from paper_2403_07544_b200.emucomm import EmulatedWorld
    from paper_2403_07544_b200.engine import DeviceBatch
    from paper_2403_07544_b200.plan import ready_counts_all, shard_begin, task_modules
    tasks, topo, shape, world, spec = _world_case(case)
    emu = EmulatedWorld(tasks, topo, shape, world, device=cuda, seed=0, record=True,
                        exchange=exchange)
    ref = EmulatedCluster(tasks, topo, shape, world=world, device=cuda, seed=0)
    plan = emu.plan
    idx = plan.index()
    by_id = {t.id: t for t in tasks}
    seen_n = set()
    for step in range(3):
        rngs = [np.random.default_rng([step, r]) for r in range(world)]
        batches = [[DeviceBatch(make_batch(rngs[r], spec, shape.vocab, sentences=12), cuda)]
                   for r in range(world)]
        infos = emu.step(step, batches)
        used = {r: set(task_modules(by_id[infos[r]["tasks"][0]])) for r in range(world)}
        counts = ready_counts_all(plan, used)
        for r in range(world):
            assert [infos[r]["ready"][k] for k in plan.keys] == counts
            assert infos[r]["tasks"] == [ref.ranks[r].mux.pick(step).id]  # same multiplexer draws
        # replay: the literal Algorithm-1 exchange on the gradients the ranks posted
        for r, eng in enumerate(emu.engines):
            for k, st in eng.states.items():
                shared = len(plan.groups[k]) >= 2
                n_el = st.layout.numel
                if shared and counts[idx[k]] >= 1:
                    g = emu.hub.recorded[(k, r)][-1]
                else:
                    g = st.grad  # singleton (K2 skipped) or n = 0 (no exchange, no update)
                ref.ranks[r].states[k].grad.copy_(g[:n_el])
                if shared:
                    seen_n.add(min(counts[idx[k]], 2))
        ref.exchange_and_update(used)
        torch.cuda.synchronize()
        for r in range(world):
            for k, st in emu.engines[r].states.items():
                want = ref.ranks[r].states[k]
                assert st.step == want.step, (step, r, str(k))
                members = plan.groups[k]
                n_el = st.layout.numel
                b, e = 0, n_el
                if exchange == "partitioned" and len(members) >= 2:
                    j = members.index(r)
                    b, e = shard_begin(n_el, len(members), j), shard_begin(n_el, len(members), j + 1)
                for f in FIELDS:
                    lo, hi = (0, n_el) if f == "weights" else (b, e)
                    assert torch.equal(getattr(st, f)[lo:hi], getattr(want, f)[lo:hi]), \
                        (step, r, str(k), f)
    # config 1: rank 1 always runs a->c, so its shared modules never see n = 0
    assert seen_n == ({1, 2} if case.startswith("config1") else {0, 1, 2}), seen_n
    emu.close()


@pytest.mark.parametrize("exchange", ["nccl", "partitioned"])
def test_bf16_gradient_wire(cuda, exchange):
    """grad_wire="bf16": the shared modules' buckets cross the wire as bf16
    (cast, all-reduce / reduce-scatter of the copy, widen back): the reduced
    gradients of the first step stay within bf16 rounding of the fp32 wire's
    (two runs of the same world, same inputs), and training proceeds."""
    from paper_2403_07544_b200.emucomm import EmulatedWorld
    from paper_2403_07544_b200.engine import DeviceBatch
    tasks, topo, shape, world, spec = _world_case("config3_w4")
    grads = []
    for wire in ("fp32", "bf16"):
        emu = EmulatedWorld(tasks, topo, shape, world, device=cuda, seed=0, exchange=exchange,
                            grad_wire=wire)
        rngs = [np.random.default_rng([0, r]) for r in range(world)]
        batches = [[DeviceBatch(make_batch(rngs[r], spec, shape.vocab, sentences=12), cuda)]
                   for r in range(world)]
        infos = emu.step(0, batches)
        grads.append({(r, k): st.grad[:st.layout.numel].clone()
                      for r, e in enumerate(emu.engines) for k, st in e.states.items()})
        for e in emu.engines:
            for st in e.states.values():
                assert torch.isfinite(st.master).all()
        emu.close()
    from paper_2403_07544_b200.plan import build_plan, shard_begin
    plan = build_plan(tasks, topo)
    checked = 0
    for (r, k), g32 in grads[0].items():
        members = plan.groups[k]
        if infos[r]["ready"][k] < 1 or len(members) < 2:
            continue
        b, e = 0, g32.numel()
        if exchange == "partitioned":  # this member holds the reduced sum of its shard only
            j = members.index(r)
            b, e = shard_begin(g32.numel(), len(members), j), shard_begin(g32.numel(), len(members), j + 1)
        ref = g32[b:e]
        if not float(ref.abs().max()) > 0:
            continue
        err = float((grads[1][(r, k)][b:e] - ref).abs().max() / ref.abs().max())
        assert err < 1e-2, (r, str(k), err)
        checked += 1
    assert checked > 0


def test_partitioned_checkpoint_resume(cuda, tmp_path):
    """Partitioned transport + f4: after two steps every rank writes its owned
    shards (masters / moments are authoritative only there); a fresh world
    with other initial weights resumes from the files: every member's owned
    shard of master, moments and bf16 weights, the Adam step counts and the
    multiplexer state are bit-identical."""
    from paper_2403_07544_b200.emucomm import EmulatedWorld
    from paper_2403_07544_b200.engine import DeviceBatch
    tasks, topo, shape, world, spec = _world_case("config3_w4")

    def batches(step):
        rngs = [np.random.default_rng([step, r]) for r in range(world)]
        return [[DeviceBatch(make_batch(rngs[r], spec, shape.vocab, sentences=12), cuda)]
                for r in range(world)]

    a = EmulatedWorld(tasks, topo, shape, world, device=cuda, seed=0, exchange="partitioned")
    for step in range(2):
        a.step(step, batches(step))
    for r, e in enumerate(a.engines):
        e.save_checkpoint(str(tmp_path), {"step_idx": 2})
    b = EmulatedWorld(tasks, topo, shape, world, device=cuda, seed=7, exchange="partitioned")
    for e in b.engines:
        assert e.load_checkpoint(str(tmp_path))["step_idx"] == 2
    from paper_2403_07544_b200.plan import shard_begin
    for r in range(world):
        for k, st in a.engines[r].states.items():
            sb = b.engines[r].states[k]
            n, members = st.layout.numel, a.plan.groups[k]
            lo, hi = 0, n
            if len(members) >= 2:
                j = members.index(r)
                lo, hi = shard_begin(n, len(members), j), shard_begin(n, len(members), j + 1)
            assert st.step == sb.step, (r, str(k))
            for f in ("master", "exp_avg", "exp_avg_sq"):
                assert torch.equal(getattr(st, f)[lo:hi], getattr(sb, f)[lo:hi]), (r, str(k), f)
            # bf16 weights are re-cast from the master on load: equal on the owned shard
            assert torch.equal(st.weights[lo:hi], sb.weights[lo:hi]), (r, str(k))
            assert a.engines[r].mux.rng.getstate() == b.engines[r].mux.rng.getstate()
    a.close()
    b.close()

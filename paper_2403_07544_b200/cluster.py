"""Several ranks of the modular trainer emulated on ONE GPU.

Each emulated rank is an ``Engine`` with its own buckets; after every rank's
micro-batches the Algorithm-1 exchange runs as one ``mm_sync_emulated``
launch over all ranks' grad buckets (each module's group = its hosting
ranks, ascending; only ready members are read), then K3 runs per rank with
the group ready counts.  This is the single-GPU stand-in for the NCCL path
(the profiling recipe forbids running inter-dependent ranks as separate
processes on one GPU) and gives the config-1 plumbing run on a B200.

``exchange="peer"`` runs option B instead: one ``mm_peer_update`` launch
holding EVERY emulated rank's shards (the multi-rank kernel emulated as one
kernel over all ranks' data -- no flag barriers are needed inside a single
launch), with the fp32 master replicated to every member so all emulated
ranks hold complete masters; singletons keep the per-rank K3.
"""
from __future__ import annotations

import math

from typing import Sequence

from . import _native, ops
from .domain import ModuleKey
from .engine import DeviceBatch, Engine
from .plan import ready_counts_all, task_modules


class EmulatedCluster:
    def __init__(self, tasks, topo, shape, world: int, device=None, seed: int = 0,
                 exchange: str = "sync", **kw):
        if exchange not in ("sync", "peer"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.exchange_kind = exchange
        self.world = world
        self.ranks = [Engine(tasks, topo, shape, rank=r, world=1, device=device, seed=seed, **kw)
                      for r in range(world)]
        self.plan = self.ranks[0].plan

    def step(self, step_idx: int, batches: Sequence[Sequence[DeviceBatch]]) -> dict:
        """batches[r] = rank r's micro-batches for this step."""
        used_by_rank, picks = self.compute(step_idx, batches)
        counts = self.exchange_and_update(used_by_rank)
        return {"tasks": picks, "ready": dict(zip(self.plan.keys, counts))}

    def compute(self, step_idx: int, batches: Sequence[Sequence[DeviceBatch]]):
        """Every rank's micro-batches: (used modules per rank, task picks)."""
        used_by_rank: dict[int, set] = {}
        picks = {}
        for r, eng in enumerate(self.ranks):
            if r not in self.plan.tasks_by_rank:
                continue
            ops.memset(eng.loss_sum, 0)
            used: set[ModuleKey] = set()
            picks[r] = []
            for db in batches[r]:
                task = eng.mux.pick(step_idx)
                picks[r].append(task.id)
                fresh = [k for k in task_modules(task) if k not in used]
                eng.zero_grads(fresh)
                used.update(fresh)
                eng.forward_backward(task, db, eng.loss_sum)
            used_by_rank[r] = used
        return used_by_rank, picks

    def exchange_and_update(self, used_by_rank, exchange: str = None) -> list:
        """Algorithm-1 exchange + optimizer update; returns the ready counts."""
        counts = self.exchange(used_by_rank, exchange)
        if (exchange or self.exchange_kind) != "peer":
            for r in used_by_rank:
                self.update_rank(r, counts)
        return counts

    def exchange(self, used_by_rank, exchange: str = None) -> list:
        """The cross-rank part only: one mm_sync_emulated launch over every
        shared module (sync), or option B's fused exchange + update of the
        shared modules followed by each rank's singleton update (peer).
        Returns the ready counts."""
        counts = ready_counts_all(self.plan, used_by_rank)
        if (exchange or self.exchange_kind) == "peer":
            self._peer_exchange(used_by_rank, counts)
            return counts
        table = []
        for k in self.plan.keys:
            members = self.plan.groups[k]
            if len(members) < 2:
                continue
            m = _native.SyncModule()
            for j, r in enumerate(members):
                m.bufs[j] = self.ranks[r].states[k].grad.data_ptr()
            m.out = None
            m.n_elems = self.ranks[members[0]].states[k].grad.numel()
            m.group_size = len(members)
            m.used_mask = sum(1 << j for j, r in enumerate(members) if k in used_by_rank.get(r, ()))
            if m.used_mask:
                table.append(m)
        if table:
            # the emulated kernel already divides by n and installs the mean on
            # every member; K3 then runs with n = 1 for those modules
            ops.sync_emulated(table, only_ready=True)
        return counts

    def update_rank(self, r: int, counts) -> None:
        """Rank r's K3 after a sync exchange (shared modules already hold the
        mean: n = 1; singletons divide by their own count)."""
        idx = self.plan.index()
        per_rank = []
        for k in self.plan.keys:
            n = counts[idx[k]]
            per_rank.append(1 if (n >= 1 and len(self.plan.groups[k]) >= 2) else n)
        self.ranks[r].fused_update(per_rank)

    def _peer_exchange(self, used_by_rank, counts) -> None:
        from .peer import make_shard
        idx = self.plan.index()
        shards = []
        for k in self.plan.keys:
            members = self.plan.groups[k]
            if len(members) < 2:
                continue
            mask = sum(1 << j for j, r in enumerate(members) if k in used_by_rank.get(r, ()))
            if not mask:
                continue
            sts = [self.ranks[r].states[k] for r in members]
            for j, r in enumerate(members):
                eng, st = self.ranks[r], sts[j]
                a = eng.adam
                st.step += 1
                shards.append(make_shard(
                    [s.grad.data_ptr() for s in sts], [s.weights.data_ptr() for s in sts],
                    [s.master.data_ptr() for s in sts], st.master.data_ptr(),
                    st.exp_avg.data_ptr(), st.exp_avg_sq.data_ptr(), st.master.numel(), j, mask,
                    a.lr / (1.0 - a.beta1 ** st.step), 1.0 / math.sqrt(1.0 - a.beta2 ** st.step)))
        a = self.ranks[0].adam
        ops.peer_update(shards, _native.AdamHyper.make(beta1=a.beta1, beta2=a.beta2, eps=a.eps,
                                                       weight_decay=a.weight_decay))
        for r, eng in enumerate(self.ranks):
            if r not in used_by_rank:
                continue
            singles = {k for k in eng.states if len(self.plan.groups[k]) < 2}
            eng.fused_update(counts, only=singles)

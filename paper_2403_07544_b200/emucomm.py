"""In-process stand-in for the NCCL module-group communicators (K1 / K2).

``Engine.step`` with ``world > 1`` posts its collectives through a
``CommGroups`` object (``engine.py``: K1 ready-bit all-reduce, K2 per-module
sum or n = 1 broadcast on the module's member-set communicator).  This pool
gives one GPU per process, so the multi-rank path is exercised by running
every rank's UNMODIFIED ``Engine.step`` in its own host thread on the same
GPU, with ``EmuCommGroups`` in place of ``CommGroups``:

* a collective completes when every member of its group has posted it
  (matched by module key and per-rank call order, as NCCL matches calls on a
  communicator); the last thread to arrive executes it and the others wait;
* execution is host-synchronous (each member's posting stream is drained
  first), so no kernel ever waits on another rank's kernel -- the pattern the
  profiling recipe forbids on one GPU;
* K1 sums the ranks' ready bitmasks (int32, as the world all-reduce does);
  K2 sums the members' buckets in ascending rank order with the sm_100a
  Algorithm-1 kernel (``mm_sync_emulated``: all members, divide by 1) or, for
  n = 1, installs the one ready member's bucket on every member -- the
  arithmetic ``mm_reduce_modules`` performs with ncclAllReduce /
  ncclBroadcast up to the ring's summation order;
* the partitioned transport's reduce-scatter / all-gather (mode 1 / 2 items)
  are the same sum restricted to the owner's use, and a copy of each owner's
  bf16 weight shard into every member;
* bf16 gradient items (the bf16 wire) are summed in fp32 in rank order and
  rounded once (NCCL's ring rounds its partial sums: same order of error).

The C library is not re-entrant, so ``_native.serialized_calls`` makes every
ctypes call take one process-wide lock while the threads run.
``EmuHub.record`` (optional) keeps each member's bucket as posted, before
the reduction, so tests can replay the exchange elsewhere.
"""
from __future__ import annotations

import threading
from collections import defaultdict
from typing import Optional

import torch

from . import _native, ops

TIMEOUT_S = 120.0


class EmuHub:
    """Shared by the ranks of one emulated world."""

    def __init__(self, world: int, plan, record: bool = False):
        self.world = world
        self.plan = plan
        self.cv = threading.Condition()
        self.slots: dict = {}
        self.calls: dict = defaultdict(int)  # (rank, tag) -> calls so far
        self.record = record
        self.recorded: dict = defaultdict(list)  # (ModuleKey, rank) -> [pre-reduce bucket clones]
        self.buckets: dict = {}  # device pointer -> (rank, ModuleKey, tensor)
        self.set_ids: dict = {}
        self.id_sets: dict = {}
        for members in plan.member_sets():
            gid = len(self.set_ids) + 1
            self.set_ids[tuple(members)] = gid
            self.id_sets[gid] = tuple(members)

    def post(self, rank: int, tag, members, payload, execute):
        """Register this rank's part of collective ``tag`` on ``members``;
        the last member to post runs ``execute({rank: payload})``.  Returns
        the slot to ``wait`` on."""
        with self.cv:
            n = self.calls[(rank, tag)]
            self.calls[(rank, tag)] = n + 1
            slot = self.slots.setdefault((tag, n), {"reqs": {}, "done": False, "err": None,
                                                    "members": tuple(members), "left": 0})
            if slot["members"] != tuple(members):
                raise RuntimeError(f"collective {tag}: member sets differ across ranks")
            slot["reqs"][rank] = payload
            if len(slot["reqs"]) == len(members):
                try:
                    execute(slot["reqs"])
                except BaseException as e:  # surfaced in every member
                    slot["err"] = e
                slot["done"] = True
                self.cv.notify_all()
            return (tag, n)

    def wait(self, key) -> None:
        with self.cv:
            slot = self.slots[key]
            if not self.cv.wait_for(lambda: slot["done"], timeout=TIMEOUT_S):
                raise RuntimeError(f"collective {key} timed out: members {slot['members']}, "
                                   f"posted {sorted(slot['reqs'])}")
            slot["left"] += 1
            if slot["left"] == len(slot["members"]):
                del self.slots[key]
            if slot["err"] is not None:
                raise slot["err"]


class EmuCommGroups:
    """Drop-in for ``engine.CommGroups`` on one rank of an emulated world."""

    def __init__(self, hub: EmuHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world
        self.by_set = {m: gid for m, gid in hub.set_ids.items() if rank in m}

    # K1: world all-reduce of the ready bitmasks (int32)
    def ready_count(self, flags_dev: torch.Tensor, n_dev: torch.Tensor) -> None:
        ev = torch.cuda.Event()
        ev.record()

        def execute(reqs):
            tot = None
            for r in sorted(reqs):
                f, _, e = reqs[r]
                e.synchronize()
                v = f.cpu().to(torch.int64)
                tot = v if tot is None else tot + v
            for r in sorted(reqs):
                reqs[r][1].copy_(tot.to(torch.int32))
            torch.cuda.synchronize()

        key = self.hub.post(self.rank, "K1", tuple(range(self.world)), (flags_dev, n_dev, ev), execute)
        self.hub.wait(key)

    # K2: per-module items of mm_reduce_modules
    def reduce(self, items) -> None:
        if not items:
            return
        ev = torch.cuda.Event()
        ev.record()
        keys = []
        for it in items:
            members = self.hub.id_sets[int(it.group)]
            _, key, _ = self.hub.buckets[int(it.buf)]
            mode = int(it.mode)
            tag = ("K2", mode, members, key)  # matched per module and call order, as NCCL matches calls
            keys.append(self.hub.post(self.rank, tag, members,
                                      (int(it.buf), int(it.n_elems), int(it.dtype), int(it.root), ev,
                                       mode, int(it.shard)),
                                      self._execute_k2(members, tag)))
        for k in keys:
            self.hub.wait(k)

    def _execute_k2(self, members, tag):
        hub = self.hub

        def execute(reqs):
            for r in members:
                reqs[r][4].synchronize()  # every member's gradients are final
            first = reqs[members[0]]
            n_elems, dtype, root, mode, shard = first[1], first[2], first[3], first[5], first[6]
            if any(reqs[r][1:4] != first[1:4] or reqs[r][5:] != first[5:] for r in members):
                raise RuntimeError(f"{tag}: members posted different items")
            if mode in (1, 2) and n_elems != len(members) * shard:
                raise RuntimeError(f"{tag}: partitioned item of {n_elems} != {len(members)} x {shard}")
            if mode == 2:  # all-gather: every owner's shard into every member
                views = [hub.buckets[reqs[r][0]][2] for r in members]
                for j, src in enumerate(views):
                    for dst in views:
                        if dst is not src:
                            dst[j * shard:(j + 1) * shard].copy_(src[j * shard:(j + 1) * shard])
                torch.cuda.synchronize()
                return
            if dtype == 1:  # bf16 wire: fp32 sum in rank order, one rounding
                views = [hub.buckets[reqs[r][0]][2] for r in members]
                if mode == 0 and root >= 0:
                    tot = views[root].clone()
                else:
                    acc = torch.zeros(n_elems, dtype=torch.float32, device=views[0].device)
                    for v in views:
                        acc += v.float()
                    tot = acc.bfloat16()
                for v in views:
                    v.copy_(tot)
                torch.cuda.synchronize()
                return
            if hub.record:
                for r in members:
                    _, key, t = hub.buckets[reqs[r][0]]
                    hub.recorded[(key, r)].append(t.clone())
            m = _native.SyncModule()
            for j, r in enumerate(members):
                m.bufs[j] = reqs[r][0]
            m.out = None
            m.n_elems = n_elems
            m.group_size = len(members)
            # mode 1 (reduce-scatter): the sum lands in every member's bucket;
            # each owner reads only its shard, as after ncclReduceScatter
            if mode == 0 and root >= 0:   # broadcast from the one ready member
                m.used_mask = 1 << root
                ops.sync_emulated([m], only_ready=True)
            else:           # sum over every member (zeros included), divide by 1
                m.used_mask = 1
                ops.sync_emulated([m], only_ready=False)
            torch.cuda.synchronize()

        return execute

    def close(self) -> None:
        pass


class EmulatedWorld:
    """``world`` Engines, one per emulated rank, stepped concurrently from
    host threads through an ``EmuHub`` (see the module docstring)."""

    def __init__(self, tasks, topo, shape, world: int, device=None, seed: int = 0,
                 record: bool = False, **engine_kw):
        from .engine import Engine
        from .plan import build_plan
        plan = build_plan(tasks, topo)
        self.hub = EmuHub(world, plan, record=record)
        self.world = world
        self.engines = [Engine(tasks, topo, shape, rank=r, world=world, device=device, seed=seed,
                               comm=EmuCommGroups(self.hub, r), **engine_kw)
                        for r in range(world)]
        for r, e in enumerate(self.engines):
            for k, st in e.states.items():
                self.hub.buckets[st.grad.data_ptr()] = (r, k, st.grad)
                self.hub.buckets[st.weights.data_ptr()] = (r, k, st.weights)
                if getattr(st, "wire", None) is not None:
                    self.hub.buckets[st.wire.data_ptr()] = (r, k, st.wire)
        self.plan = self.engines[0].plan

    def step(self, step_idx: int, batches) -> list:
        """batches[r]: rank r's DeviceBatch list; returns each rank's step info."""
        out: list = [None] * self.world
        errs: list = []

        def run(r):
            try:
                out[r] = self.engines[r].step(step_idx, batches[r])
                self.engines[r].sync_updates()
                torch.cuda.current_stream().synchronize()
            except BaseException as e:  # noqa: BLE001
                errs.append((r, e))

        with _native.serialized_calls():
            threads = [threading.Thread(target=run, args=(r,)) for r in range(self.world)]
            for t in threads:
                t.start()
            for t in threads:
                t.join(TIMEOUT_S * 4)
        if errs:
            raise RuntimeError(f"rank {errs[0][0]} failed") from errs[0][1]
        if any(t.is_alive() for t in threads):
            raise RuntimeError("emulated ranks did not finish")
        torch.cuda.synchronize()
        return out

    def close(self) -> None:
        for e in self.engines:
            e.close()

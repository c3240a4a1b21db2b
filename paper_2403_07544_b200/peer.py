"""Option B of the module exchange: K2 + K3 + the weight
all-gather as one kernel over NVLink peer memory.

Per step and per exchange call every rank runs, on its stream,

    mm_peer_barrier  (epoch e+1: every peer's gradients are final)
    mm_peer_update   (this rank's shard of every shared module with n >= 1:
                      masked peer loads of the ready members' gradients,
                      / n, Adam on the local shard, bf16 weights stored
                      into every member's bucket)
    mm_peer_barrier  (epoch e+2: every peer is done reading and writing
                      this rank's buckets)

Singleton modules keep the local K3 (``Engine.fused_update``).  The buckets
of every module a rank shares with a peer, and the peers' barrier flag
arrays, are mapped once with CUDA IPC (``mm_ipc_export`` / ``mm_ipc_import``)
and exchanged through the rendezvous store.

Algorithm-1 semantics (syncsim.py:121-153): the sum runs over READY members
only, in ascending member order, so unused members' buckets need no zero
fill; the owner of a shard is its only reader, so with lazy zeroing it can
clear the shard right after reading it.  Numerically each shard is
bit-identical to ``mm_sync_emulated`` + ``mm_fused_update(n = 1)``.

The master copy is sharded: after an exchange, member r's fp32 master is
authoritative on its own shard of each shared module (every member's bf16
weights are complete).  ``replicate_master=True`` also stores the fp32
master into the other members (4 more bytes per element on the wire).
"""
from __future__ import annotations

import math
import pickle
from typing import Sequence

import torch

from . import _native, ops
from .plan import peer_plan, shard_begin


def _key(k) -> str:
    return str(k)


def make_shard(members_grad, members_param, members_master, master, exp_avg, exp_avg_sq,
               n_elems: int, member: int, mask: int, step_size: float, inv_sqrt_bc2: float,
               own_master_copy: bool = False) -> "_native.PeerShard":
    """PeerShard for `member`'s shard; *members_* are per-member device
    pointers (0 = skip).  The owner's own entry of master_copy is dropped
    (it updates `master` in place) unless own_master_copy."""
    g = len(members_grad)
    sh = _native.PeerShard()
    for j in range(g):
        sh.grad[j] = members_grad[j] or None
        sh.param[j] = members_param[j] or None
        mc = members_master[j] if members_master is not None else 0
        sh.master_copy[j] = (mc if (j != member or own_master_copy) else 0) or None
    sh.master, sh.exp_avg, sh.exp_avg_sq = master, exp_avg, exp_avg_sq
    sh.begin = shard_begin(n_elems, g, member)
    sh.end = shard_begin(n_elems, g, member + 1)
    sh.group_size = g
    sh.ready_mask = mask
    sh.step_size = step_size
    sh.inv_sqrt_bc2 = inv_sqrt_bc2
    return sh


class PeerExchange:
    """One rank's option-B exchange state (IPC mappings, flags, epochs)."""

    def __init__(self, engine, store, replicate_master: bool = False, timeout_ms: int = 120000):
        self.engine = engine
        plan, rank = engine.plan, engine.rank
        self.rank = rank
        self.replicate_master = replicate_master
        self.timeout_ms = timeout_ms
        self.flags = torch.zeros(_native.PEER_MAX_RANKS, dtype=torch.int32, device=engine.device)
        shared = [k for k in engine.states if len(plan.groups[k]) >= 2]
        mine = {"flags": ops.ipc_export(self.flags)}
        for k in shared:
            st = engine.states[k]
            mine[_key(k)] = tuple(ops.ipc_export(t) for t in (st.grad, st.weights, st.master))
        # the zero fill of the flags must land before any peer can signal
        torch.cuda.synchronize(engine.device)
        store.set(f"mmb200_ipc_{rank}", pickle.dumps(mine))
        self.peers = sorted({r for k in shared for r in plan.groups[k] if r != rank})
        if len(self.peers) > _native.PEER_MAX_RANKS:
            raise ValueError("too many peers for one flag array")
        self._imported: list[int] = []
        self.remote: dict[tuple, tuple] = {}  # (rank, key) -> (grad, weights, master) pointers
        peer_flags = []
        for r in self.peers:
            theirs = pickle.loads(store.get(f"mmb200_ipc_{r}"))
            peer_flags.append(self._import(*theirs["flags"]))
            for k in shared:
                if r in plan.groups[k]:
                    self.remote[(r, k)] = tuple(self._import(*he) for he in theirs[_key(k)])
        self.sig = _native.PeerSignal()
        self.sig.local_flags = self.flags.data_ptr()
        for i, r in enumerate(self.peers):
            self.sig.peer_flags[i] = peer_flags[i]
            self.sig.peer_rank[i] = r
        self.sig.n_peers = len(self.peers)
        self.sig.my_rank = rank
        self.sig.timeout_ms = timeout_ms
        self.epoch = 0

    def _import(self, handle: bytes, offset: int) -> int:
        p = ops.ipc_import(handle, offset)
        self._imported.append(p)
        return p

    def barrier(self) -> None:
        self.epoch += 1
        self.sig.epoch = self.epoch
        ops.peer_barrier(self.sig)

    def shards(self, bits: Sequence[int], only=None) -> list:
        """This rank's PeerShard list for the world-summed ready bits; bumps
        the Adam step of every module it updates."""
        eng = self.engine
        a = eng.adam
        out = []
        for k, members, j, mask in peer_plan(eng.plan, self.rank, bits, only):
            st = eng.states[k]
            ptrs = [(st.grad.data_ptr(), st.weights.data_ptr(), st.master.data_ptr())
                    if r == self.rank else self.remote[(r, k)] for r in members]
            st.step += 1
            bc1 = 1.0 - a.beta1 ** st.step
            bc2 = 1.0 - a.beta2 ** st.step
            out.append(make_shard(
                [p[0] for p in ptrs], [p[1] for p in ptrs],
                [p[2] for p in ptrs] if self.replicate_master else None,
                st.master.data_ptr(), st.exp_avg.data_ptr(), st.exp_avg_sq.data_ptr(),
                st.master.numel(), j, mask, a.lr / bc1, 1.0 / math.sqrt(bc2)))
        return out

    def run(self, bits: Sequence[int], only=None, zero_grad: bool = False) -> None:
        """One exchange on the current stream.  Every rank must call it the
        same number of times per step (the barriers pair up by epoch)."""
        a = self.engine.adam
        sh = self.shards(bits, only)
        self.barrier()
        ops.peer_update(sh, _native.AdamHyper.make(beta1=a.beta1, beta2=a.beta2, eps=a.eps,
                                                   weight_decay=a.weight_decay,
                                                   zero_grad=int(zero_grad)))
        self.barrier()

    def close(self) -> None:
        for p in self._imported:
            ops.ipc_release(p)
        self._imported = []

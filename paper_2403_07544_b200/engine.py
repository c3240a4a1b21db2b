"""The B200 modular-training step: per-language transformer modules, one
process per GPU, Algorithm-1 gradient exchange and the fused optimizer.

Replaces the trainer loop of the reference simulator (``run_benchmark``,
``syncsim.py:346-392``): for every rank, ``accum_count`` micro-batches are
drawn through the multiplexer (``syncsim.py:353``), each runs the task's
encoder stacks then decoder stacks (``TaskSpec.modules()``, core.py:147-149)
with hand-written sm_100a kernels (K4-K8), gradients accumulate straight into
each module's flat fp32 bucket (``DeviceState.accumulate``, syncsim.py:113-118),
then

* K1  ready counts: world int32 allreduce of the used-flags (NCCL),
* K2  per-module sum over the module's own NCCL sub-communicator, only for
      groups with >= 2 ranks and n >= 1, in sorted ModuleKey order,
* K3  fused ``/ n`` rescale + Adam + bf16 weight write for every hosted
      module with n >= 1 (n == 0: no update, no optimizer step).

All compute goes through ``libmmb200.so``; torch provides allocations and
the stream only.
"""
from __future__ import annotations

import dataclasses
import math
import os
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native, ops
from .configs import ModelShape
from .data import ATTN_CAP, Batch, attention_groups
from .domain import ClusterTopology, ModuleKey, Side, TaskSpec
from .model import LN_EPS, ModuleState, module_layouts
from .plan import (Multiplexer, build_plan, decode_ready, embedding_keys, exchange_plan, ready_bits,
                   ready_flags, task_modules)


@dataclasses.dataclass
class AdamConfig:
    lr: float = 2e-4
    beta1: float = 0.9
    beta2: float = 0.998
    eps: float = 1e-8
    weight_decay: float = 0.0


def native_attention_groups(cu_q: np.ndarray, cu_k: np.ndarray, cap: int = ATTN_CAP,
                            align: int = 32):
    """data.attention_groups through the C ABI (mm_attention_groups): the
    numpy loop cost ~0.12 ms per table on every step's host path."""
    import ctypes
    cq = np.ascontiguousarray(cu_q, dtype=np.int32)
    ck = np.ascontiguousarray(cu_k, dtype=np.int32)
    n = len(cq) - 1
    out = np.empty(2 * max(n, 1), dtype=np.int32)
    ng, foot = ctypes.c_int(), ctypes.c_int()
    _native.check(_native.lib().mm_attention_groups(cq.ctypes.data, ck.ctypes.data, n, cap, align,
                                                    out.ctypes.data, ctypes.byref(ng), ctypes.byref(foot)),
                  "mm_attention_groups")
    return out[:2 * ng.value], foot.value


class DeviceBatch:
    """A packed batch resident in HBM: one H2D copy of one pinned int32 buffer
    holding the token streams, offsets and the attention work groups."""

    FIELDS = ("src", "src_pos", "cu_src", "tgt_in", "tgt_pos", "labels", "cu_tgt")

    def __init__(self, b: Batch, device, pinned: Optional[torch.Tensor] = None,
                 non_blocking: bool = True):
        arrs = dict(b.host_arrays())
        groups = {}
        # the six work-group tables in one host call: padded (mma.sync) and
        # unpadded (tcgen05: fewer, fuller units) for src / tgt / cross
        n = b.n_seq
        cs = np.ascontiguousarray(b.cu_src, dtype=np.int32)
        ct = np.ascontiguousarray(b.cu_tgt, dtype=np.int32)
        tab = np.empty(12 * max(n, 1), dtype=np.int32)
        ng, foot = np.zeros(6, dtype=np.int32), np.zeros(6, dtype=np.int32)
        _native.check(_native.lib().mm_attention_tables(cs.ctypes.data, ct.ctypes.data, n, ATTN_CAP,
                                                        tab.ctypes.data, ng.ctypes.data,
                                                        foot.ctypes.data), "mm_attention_tables")
        for t, name in enumerate(("attn_src", "attn_tgt", "attn_cross", "tc_src", "tc_tgt", "tc_cross")):
            arrs[name] = tab[2 * n * t:2 * n * t + 2 * int(ng[t])]
            groups[name] = (int(ng[t]), int(foot[t])) if t < 3 else (int(ng[t]),)
        # deterministic embedding backward: rows sorted by token id, chunked
        self.emb_counts = {}
        for name, ids in (("emb_src", b.src), ("emb_tgt", b.tgt_in)):
            arrs[name], nc, nm = ops.embed_segments(ids)
            self.emb_counts[name] = (nc, nm)
        names = list(self.FIELDS) + list(groups) + ["emb_src", "emb_tgt"]
        sizes = [len(arrs[f]) for f in names]
        total = sum(sizes)
        host = pinned if pinned is not None and pinned.numel() >= total else \
            torch.empty(total, dtype=torch.int32, pin_memory=True)
        flat = host.numpy()
        off = 0
        for f, n in zip(names, sizes):
            flat[off:off + n] = arrs[f]
            off += n
        self.h2d_bytes = total * 4
        dev = torch.empty(total, dtype=torch.int32, device=device)
        dev.copy_(host[:total], non_blocking=non_blocking)
        off = 0
        for f, n in zip(names, sizes):
            view = dev[off:off + n]
            setattr(self, f, (view,) + groups[f] if f in groups else view)
            off += n
        # padded table -> its unpadded twin (the per-op Python path's lookup)
        self.tc_of = {id(self.attn_src): self.tc_src, id(self.attn_tgt): self.tc_tgt,
                      id(self.attn_cross): self.tc_cross}
        self.n_seq = b.n_seq
        self.n_src, self.n_tgt = b.n_src, b.n_tgt
        self.max_src, self.max_tgt = b.max_src, b.max_tgt
        self._keep = host  # keep the pinned staging alive until the copy retires
        gs, gt, gc = self.attn_src, self.attn_tgt, self.attn_cross
        ts, tt, tc = self.tc_src, self.tc_tgt, self.tc_cross
        self.desc = _native.BatchDesc(
            tcg_src=ts[0].data_ptr(), tcg_tgt=tt[0].data_ptr(), tcg_cross=tc[0].data_ptr(),
            ntc_src=ts[1], ntc_tgt=tt[1], ntc_cross=tc[1],
            src=self.src.data_ptr(), src_pos=self.src_pos.data_ptr(), cu_src=self.cu_src.data_ptr(),
            tgt_in=self.tgt_in.data_ptr(), tgt_pos=self.tgt_pos.data_ptr(),
            labels=self.labels.data_ptr(), cu_tgt=self.cu_tgt.data_ptr(),
            groups_src=gs[0].data_ptr(), groups_tgt=gt[0].data_ptr(), groups_cross=gc[0].data_ptr(),
            n_seq=self.n_seq, n_src=self.n_src, n_tgt=self.n_tgt, max_src=self.max_src,
            max_tgt=self.max_tgt, ng_src=gs[1], cap_src=gs[2], ng_tgt=gt[1], cap_tgt=gt[2],
            ng_cross=gc[1], cap_cross=gc[2],
            emb_src=self.emb_src.data_ptr(), emb_tgt=self.emb_tgt.data_ptr(),
            nch_src=self.emb_counts["emb_src"][0], nmul_src=self.emb_counts["emb_src"][1],
            nch_tgt=self.emb_counts["emb_tgt"][0], nmul_tgt=self.emb_counts["emb_tgt"][1])


class CommGroups:
    """NCCL world + one sub-communicator per distinct member set (K1/K2)."""

    def __init__(self, plan, rank: int, world: int, device_index: int, store):
        L = _native.lib()
        if rank == 0:
            uid = ctypes_buf(128)
            _native.check(L.mm_nccl_unique_id(uid), "mm_nccl_unique_id")
            store.set("mmb200_nccl_uid", bytes(uid.raw))
        uid_bytes = store.get("mmb200_nccl_uid")
        self.ctx = ctypes_voidp()
        _native.check(L.mm_comm_init(rank, world, uid_bytes, device_index, ctypes_ref(self.ctx)),
                      "mm_comm_init")
        self.by_set: dict[tuple, object] = {}
        for members in plan.member_sets():  # identical order on every rank
            arr = (ctypes_int * len(members))(*members)
            grp = ctypes_voidp()
            _native.check(L.mm_group_create(self.ctx, arr, len(members), ctypes_ref(grp)),
                          "mm_group_create")
            self.by_set[members] = grp.value
        self.rank, self.world = rank, world

    def ready_count(self, flags_dev: torch.Tensor, n_dev: torch.Tensor) -> None:
        _native.check(_native.lib().mm_ready_count(self.ctx, flags_dev.data_ptr(), n_dev.data_ptr(),
                                                   flags_dev.numel(), ops.stream_ptr()),
                      "mm_ready_count")

    def reduce(self, items) -> None:
        if not items:
            return
        arr = (_native.ReduceItem * len(items))(*items)
        _native.check(_native.lib().mm_reduce_modules(self.ctx, arr, len(items), ops.stream_ptr()),
                      "mm_reduce_modules")

    def close(self) -> None:
        L = _native.lib()
        for g in self.by_set.values():
            if g:
                L.mm_group_destroy(g)
        L.mm_comm_destroy(self.ctx)


import ctypes  # noqa: E402  (helpers for CommGroups)

ctypes_int = ctypes.c_int


def ctypes_buf(n):
    return ctypes.create_string_buffer(n)


def ctypes_voidp():
    return ctypes.c_void_p()


def ctypes_ref(x):
    return ctypes.byref(x)


class Engine:
    """One rank of the modular trainer."""

    def __init__(self, tasks: Sequence[TaskSpec], topo: ClusterTopology, shape: ModelShape,
                 rank: int = 0, world: int = 1, device=None, seed: int = 0,
                 adam: AdamConfig = AdamConfig(), store=None, masters=None,
                 exchange: Optional[str] = None, comm=None, grad_wire: Optional[str] = None):
        if shape.head_dim not in (16, 32, 64) or shape.d_model % shape.heads:
            raise ValueError(f"head_dim {shape.d_model}/{shape.heads}: the attention kernels take 16, 32 or 64")
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.shape = shape
        self.rank, self.world = rank, world
        self.plan = build_plan(tasks, topo)
        self.layouts = module_layouts(self.plan, shape)
        self.index = self.plan.index()
        self.hosted = sorted(self.plan.hosted.get(rank, frozenset()))
        # K2 transport for world > 1: "nccl" (group all-reduce / broadcast, then
        # the replicated K3), "partitioned" (reduce-scatter, K3 on the owned
        # shard, bf16 all-gather of the weights) or "peer" (option B: one
        # fused peer-memory kernel per exchange, paper_2403_07544_b200/peer.py)
        self.exchange = exchange or os.environ.get("MM_EXCHANGE", "nccl")
        if self.exchange not in ("nccl", "peer", "partitioned"):
            raise ValueError(f"unknown exchange {self.exchange!r}")
        self.partitioned = world > 1 and self.exchange == "partitioned"
        # K2's gradient wire format: "fp32", or "bf16" (the bucket is cast to a
        # bf16 copy before the all-reduce / reduce-scatter and widened back:
        # half the NVLink bytes for a 2^-9 relative rounding of the sum)
        self.grad_wire = grad_wire or os.environ.get("MM_GRAD_WIRE", "fp32")
        if self.grad_wire not in ("fp32", "bf16"):
            raise ValueError(f"unknown grad_wire {self.grad_wire!r}")
        self.states: dict[ModuleKey, ModuleState] = {}
        for k in self.hosted:
            m = None if masters is None else masters.get(k)
            cap = 0
            g = len(self.plan.groups[k])
            if self.partitioned and g >= 2:  # buckets padded to g equal shards
                cap = g * self.shard_elems(self.layouts[k].numel, g)
            st = ModuleState(self.layouts[k], shape, self.device, seed, master=m, capacity=cap)
            st.wire = None
            if world > 1 and g >= 2 and self.grad_wire == "bf16" and self.exchange != "peer":
                st.wire = torch.empty(st.grad.numel(), dtype=torch.bfloat16, device=self.device)
            self.states[k] = st
        self.mux = Multiplexer(self.plan, rank, seed)
        self.adam = adam
        # K1 / K2 communicators: NCCL (CommGroups), or an injected stand-in
        # with the same interface (emucomm.EmuCommGroups: emulated ranks)
        if comm is not None:
            self.comm = comm
        else:
            self.comm = CommGroups(self.plan, rank, world, self.device.index or 0, store) \
                if world > 1 else None
        self.peer = None
        if world > 1 and self.exchange == "peer":
            from .peer import PeerExchange
            self.peer = PeerExchange(self, store)
        self._bits = None
        self.loss_sum = torch.zeros(1, device=self.device)
        self.n_ready_dev = torch.zeros(len(self.plan.keys), dtype=torch.int32, device=self.device)
        self.flags_dev = torch.zeros(len(self.plan.keys), dtype=torch.int32, device=self.device)
        self.scale = math.sqrt(shape.d_model)
        self.trace = None  # set to a dict to capture intermediates (diagnostics)
        self.native = True  # C++ step driver (mm_task_fwd_bwd); False -> per-op Python path
        self._task_desc: dict = {}
        self._ws = None
        # decoder-side exchange + update overlap the encoder backward
        # (MM_OVERLAP=0 for A/B: every exchange + update after the backward)
        self.overlap = os.environ.get("MM_OVERLAP", "1") != "0"
        # 0 = full grid.  A capped background update (MM_OVERLAP_CTAS=64) breaks
        # even at N=1 (r01 sweep: 8/16/32/64 CTAs -> 266K/413K/587K/740K vs
        # 756K tok/s): the update is HBM-bound and latency-bound per CTA.
        self.overlap_ctas = int(os.environ.get("MM_OVERLAP_CTAS", "0"))
        # Cross-step deferral (single rank): the encoder-side update of step k
        # runs on the side stream under step k+1's compute; step k+1 waits for
        # it only if it uses one of the modules being updated (a module's
        # update always completes before its next read or gradient reset).
        self.defer_update = world == 1 and os.environ.get("MM_DEFER_UPDATE", "1") != "0"
        self._pending_event = None            # side-stream event: every issued update done
        self._pending_mods: set = set()       # modules whose update may still be running
        # Lazy gradient zeroing: the fused update writes 0 over every gradient
        # it consumes, so a module's bucket is clean for its next use without
        # a memset pass on the step's critical path.  Off by default (the
        # reduced gradients stay readable after a step, as the parity tests
        # and the reference's DeviceState.buffers expect).
        self.zero_in_update = False
        # first micro-batch of a module per step: weight-matrix gradients are
        # stored (no memset of [0, dense_end), no reduce-add read);
        # MM_STORE_WGRAD=0 restores memset + reduce-add (bit-identical results)
        self.store_first_wgrad = os.environ.get("MM_STORE_WGRAD", "1") != "0"
        self._dirty: set = set(self.states)   # buckets that may hold a gradient
        self._counts_host = torch.zeros(len(self.plan.keys), dtype=torch.int32, pin_memory=True)
        self._side_stream = torch.cuda.Stream(device=self.device)
        # torch creates the CUDA event lazily: record once so .cuda_event is a
        # real handle before the C driver records it
        self._dec_done = torch.cuda.Event()
        self._dec_done.record()

    # ------------------------------------------------------------------ layers
    def _zeros(self, *shape):
        t = torch.empty(*shape, device=self.device)
        ops.memset(t, 0)
        return t

    def _tr(self, name, t):
        if self.trace is not None:
            self.trace[name] = t.detach().float().cpu()

    def _ln(self, st, name, x):
        T, d = x.shape
        y = torch.empty(T, d, device=self.device, dtype=torch.bfloat16)
        mean = torch.empty(T, device=self.device)
        rstd = torch.empty(T, device=self.device)
        ops.layernorm_fwd(x, st.f32(name + ".g"), st.f32(name + ".b"), y, mean, rstd, LN_EPS)
        return y, mean, rstd

    def _ln_bwd(self, st, name, dy, x, mean, rstd, dx, dx_bf):
        ops.layernorm_bwd(dy, x, st.f32(name + ".g"), mean, rstd, dx, dx_bf,
                          st.g(name + ".g"), st.g(name + ".b"))

    def _attn_args(self, q, k, v, o, lse, cu_q, cu_k, n_seq, max_q, max_k, causal, **kw):
        if kw.get("d_o") is None and "tc_groups" not in kw:
            kw["tc_groups"] = self._tc(kw.get("groups"))  # None -> built by attention_args
            if kw["tc_groups"] is None and kw.get("groups") is not None:
                kw["tc_groups"] = False  # staged padded table without a twin
        return ops.attention_args(q, k, v, o, lse, cu_q, cu_k, n_seq, self.shape.heads, max_q,
                                  max_k, causal, head_dim=self.shape.head_dim, **kw)

    def _self_block_fwd(self, st, p, x, cu, n_seq, max_len, causal, sv, groups=None):
        d = self.shape.d_model
        T = x.shape[0]
        h, mean, rstd = self._ln(st, p + "ln1", x)
        qkv = torch.empty(T, 3 * d, device=self.device, dtype=torch.bfloat16)
        ops.gemm(h, st.w(p + "qkv.w"), qkv, epilogue=ops.EPI_BF16, bias=st.f32(p + "qkv.b"))
        a = torch.empty(T, d, device=self.device, dtype=torch.bfloat16)
        lse = torch.empty(self.shape.heads, T, device=self.device)
        ops.attention_fwd(self._attn_args(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], a, lse, cu,
                                          cu, n_seq, max_len, max_len, causal, groups=groups))
        out = torch.empty_like(x)
        ops.gemm(a, st.w(p + "out.w"), out, epilogue=ops.EPI_F32_RESID, bias=st.f32(p + "out.b"),
                 resid=x)
        sv.append(("self", x, h, mean, rstd, qkv, a, lse, groups))
        return out

    def _cross_block_fwd(self, st, p, x, mem, db, sv):
        d = self.shape.d_model
        T, S = x.shape[0], mem.shape[0]
        h, mean, rstd = self._ln(st, p + "lnc", x)
        q = torch.empty(T, d, device=self.device, dtype=torch.bfloat16)
        ops.gemm(h, st.w(p + "cq.w"), q, epilogue=ops.EPI_BF16, bias=st.f32(p + "cq.b"))
        kv = torch.empty(S, 2 * d, device=self.device, dtype=torch.bfloat16)
        ops.gemm(mem, st.w(p + "ckv.w"), kv, epilogue=ops.EPI_BF16, bias=st.f32(p + "ckv.b"))
        a = torch.empty(T, d, device=self.device, dtype=torch.bfloat16)
        lse = torch.empty(self.shape.heads, T, device=self.device)
        ops.attention_fwd(self._attn_args(q, kv[:, :d], kv[:, d:], a, lse, db.cu_tgt, db.cu_src,
                                          db.n_seq, db.max_tgt, db.max_src, False,
                                          groups=getattr(db, "attn_cross", None)))
        out = torch.empty_like(x)
        ops.gemm(a, st.w(p + "cout.w"), out, epilogue=ops.EPI_F32_RESID, bias=st.f32(p + "cout.b"),
                 resid=x)
        self._tr(p + "ckv", kv)
        self._tr(p + "ca", a)
        self._tr(p + "cx_in", x)
        sv.append(("cross", x, h, mean, rstd, q, kv, a, lse))
        return out

    def _ffn_fwd(self, st, p, x, sv):
        T = x.shape[0]
        h, mean, rstd = self._ln(st, p + "ln2", x)
        f = torch.empty(T, self.shape.ffn, device=self.device, dtype=torch.bfloat16)
        ops.gemm(h, st.w(p + "ff1.w"), f, epilogue=ops.EPI_BF16_RELU, bias=st.f32(p + "ff1.b"))
        out = torch.empty_like(x)
        ops.gemm(f, st.w(p + "ff2.w"), out, epilogue=ops.EPI_F32_RESID, bias=st.f32(p + "ff2.b"),
                 resid=x)
        sv.append(("ffn", x, h, mean, rstd, f))
        return out

    # backward of the three block kinds; dx (fp32) / dx_bf hold dL/d(block output)
    def _ffn_bwd(self, st, p, rec, dx, dx_bf):
        _, x_in, h, mean, rstd, f = rec
        T = x_in.shape[0]
        ops.gemm(dx_bf, f, st.g(p + "ff2.w"), a_kmajor=False, b_kmajor=False,
                 epilogue=ops.EPI_F32_ACCUM, dbias=st.g(p + "ff2.b"))
        df = torch.empty(T, self.shape.ffn, device=self.device, dtype=torch.bfloat16)
        ops.gemm(dx_bf, st.w(p + "ff2.w"), df, b_kmajor=False, epilogue=ops.EPI_BF16_DRELU, aux=f)
        ops.gemm(df, h, st.g(p + "ff1.w"), a_kmajor=False, b_kmajor=False,
                 epilogue=ops.EPI_F32_ACCUM, dbias=st.g(p + "ff1.b"))
        dh = torch.empty(T, self.shape.d_model, device=self.device)
        ops.gemm(df, st.w(p + "ff1.w"), dh, b_kmajor=False, epilogue=ops.EPI_F32)
        self._ln_bwd(st, p + "ln2", dh, x_in, mean, rstd, dx, dx_bf)

    def _tc(self, groups):
        """The unpadded twin of a staged padded group table (None: build it)."""
        db = getattr(self, "_cur_db", None)
        return None if groups is None or db is None else db.tc_of.get(id(groups))

    def _self_bwd(self, st, p, rec, dx, dx_bf, cu, n_seq, max_len, causal):
        _, x_in, h, mean, rstd, qkv, a, lse, groups = rec
        d = self.shape.d_model
        T = x_in.shape[0]
        ops.gemm(dx_bf, a, st.g(p + "out.w"), a_kmajor=False, b_kmajor=False,
                 epilogue=ops.EPI_F32_ACCUM, dbias=st.g(p + "out.b"))
        da = torch.empty(T, d, device=self.device, dtype=torch.bfloat16)
        ops.gemm(dx_bf, st.w(p + "out.w"), da, b_kmajor=False, epilogue=ops.EPI_BF16)
        dqkv = torch.empty(T, 3 * d, device=self.device, dtype=torch.bfloat16)
        ops.attention_bwd(self._attn_args(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], a, lse, cu,
                                          cu, n_seq, max_len, max_len, causal, d_o=da,
                                          dq=dqkv[:, :d], dk=dqkv[:, d:2 * d], dv=dqkv[:, 2 * d:],
                                          groups=groups, tc_groups=self._tc(groups)))
        ops.gemm(dqkv, h, st.g(p + "qkv.w"), a_kmajor=False, b_kmajor=False,
                 epilogue=ops.EPI_F32_ACCUM, dbias=st.g(p + "qkv.b"))
        dh = torch.empty(T, d, device=self.device)
        ops.gemm(dqkv, st.w(p + "qkv.w"), dh, b_kmajor=False, epilogue=ops.EPI_F32)
        self._ln_bwd(st, p + "ln1", dh, x_in, mean, rstd, dx, dx_bf)

    def _cross_bwd(self, st, p, rec, dx, dx_bf, mem, dmem, db):
        _, x_in, h, mean, rstd, q, kv, a, lse = rec
        d = self.shape.d_model
        T, S = x_in.shape[0], mem.shape[0]
        ops.gemm(dx_bf, a, st.g(p + "cout.w"), a_kmajor=False, b_kmajor=False,
                 epilogue=ops.EPI_F32_ACCUM, dbias=st.g(p + "cout.b"))
        da = torch.empty(T, d, device=self.device, dtype=torch.bfloat16)
        ops.gemm(dx_bf, st.w(p + "cout.w"), da, b_kmajor=False, epilogue=ops.EPI_BF16)
        dq = torch.empty(T, d, device=self.device, dtype=torch.bfloat16)
        dkv = torch.empty(S, 2 * d, device=self.device, dtype=torch.bfloat16)
        ops.attention_bwd(self._attn_args(q, kv[:, :d], kv[:, d:], a, lse, db.cu_tgt, db.cu_src,
                                          db.n_seq, db.max_tgt, db.max_src, False, d_o=da, dq=dq,
                                          dk=dkv[:, :d], dv=dkv[:, d:],
                                          groups=getattr(db, "attn_cross", None),
                                          tc_groups=self._tc(getattr(db, "attn_cross", None))))
        self._tr(p + "dckv", dkv)
        self._tr(p + "dca", da)
        self._tr(p + "dcx_out", dx)
        ops.gemm(dkv, mem, st.g(p + "ckv.w"), a_kmajor=False, b_kmajor=False,
                 epilogue=ops.EPI_F32_ACCUM, dbias=st.g(p + "ckv.b"))
        ops.gemm(dkv, st.w(p + "ckv.w"), dmem, b_kmajor=False, epilogue=ops.EPI_F32_ACCUM)
        ops.gemm(dq, h, st.g(p + "cq.w"), a_kmajor=False, b_kmajor=False,
                 epilogue=ops.EPI_F32_ACCUM, dbias=st.g(p + "cq.b"))
        dh = torch.empty(T, d, device=self.device)
        ops.gemm(dq, st.w(p + "cq.w"), dh, b_kmajor=False, epilogue=ops.EPI_F32)
        self._ln_bwd(st, p + "lnc", dh, x_in, mean, rstd, dx, dx_bf)

    # ------------------------------------------------------------------ task
    def _stack_desc(self, key: ModuleKey):
        st = self.states[key]
        lay = st.layout
        names = [f for f, _ in _native.LayerOffsets._fields_]
        arr = (_native.LayerOffsets * lay.n_layers)()
        for i in range(lay.n_layers):
            for f in names:
                pname = f"l{i}." + f.replace("_w", ".w").replace("_b", ".b").replace("_g", ".g")
                p = lay.params.get(pname)
                setattr(arr[i], f, p.offset if p is not None else -1)
        has_f = "lnf.g" in lay.params
        desc = _native.Stack(w_bf16=st.weights.data_ptr(), w_f32=st.master.data_ptr(),
                             grad=st.grad.data_ptr(), layers=arr, n_layers=lay.n_layers,
                             decoder=int(key.side is Side.DECODER),
                             lnf_g=lay.params["lnf.g"].offset if has_f else -1,
                             lnf_b=lay.params["lnf.b"].offset if has_f else -1)
        return desc, arr

    def _embed_desc(self, key: ModuleKey):
        st = self.states[key]
        P = st.layout.params
        return _native.Embed(w_bf16=st.weights.data_ptr(), w_f32=st.master.data_ptr(),
                             grad=st.grad.data_ptr(), emb=P["emb"].offset,
                             gen_w=P["gen.w"].offset if "gen.w" in P else -1,
                             gen_b=P["gen.b"].offset if "gen.b" in P else -1)

    def task_desc(self, task: TaskSpec):
        """mm_task descriptor of a task (cached; buckets never move)."""
        if task.id not in self._task_desc:
            enc = [self._stack_desc(k) for k in task.enc_modules]
            dec = [self._stack_desc(k) for k in task.dec_modules]
            enc_arr = (_native.Stack * len(enc))(*[d for d, _ in enc])
            dec_arr = (_native.Stack * len(dec))(*[d for d, _ in dec])
            ek, dk = embedding_keys(task)
            s = self.shape
            t = _native.Task(d_model=s.d_model, heads=s.heads, ffn=s.ffn, vocab=s.vocab,
                             n_enc=len(enc), n_dec=len(dec), enc=enc_arr, dec=dec_arr,
                             enc_emb=self._embed_desc(ek), dec_emb=self._embed_desc(dk))
            # keep every ctypes array the descriptor points into alive
            self._task_desc[task.id] = (t, enc_arr, dec_arr, [a for _, a in enc + dec])
        return self._task_desc[task.id][0]

    def forward_backward(self, task: TaskSpec, db: DeviceBatch, loss_sum: torch.Tensor,
                         dec_done=None, store=frozenset()) -> None:
        """One micro-batch of one task; gradients accumulate into the buckets.
        ``dec_done`` (torch.cuda.Event) is recorded once the decoder-side
        gradients are final (native path only).  Modules in ``store`` (native
        path) get their weight-matrix gradients [0, layout.dense_end) STORED
        rather than reduce-added: the caller zeroed only the rest of their
        buckets (``zero_grads(tail_only=True)``)."""
        if not self.native or self.trace is not None:
            assert not store, "store mode is for the native step driver"
            self.forward_backward_py(task, db, loss_sum)
            if dec_done is not None:
                dec_done.record()
            return
        import ctypes
        L = _native.lib()
        t = self.task_desc(task)
        _t, enc_arr, dec_arr, _keep = self._task_desc[task.id]
        for arr, keys in ((enc_arr, task.enc_modules), (dec_arr, task.dec_modules)):
            for i, k in enumerate(keys):
                arr[i].store_wgrad = int(k in store)
        t.dec_emb.store_gen_w = int(embedding_keys(task)[1] in store)
        if dec_done is not None and not dec_done.cuda_event:
            raise RuntimeError("dec_done event has no CUDA handle yet")
        need = ctypes.c_size_t(0)
        _native.check(L.mm_task_fwd_bwd(ctypes.byref(t), ctypes.byref(db.desc), None,
                                        ctypes.byref(need), None, None, None),
                      "mm_task_fwd_bwd(size)")
        if self._ws is None or self._ws.numel() < need.value:
            self._ws = torch.empty(int(need.value * 1.25) + (1 << 20), dtype=torch.uint8,
                                   device=self.device)
        have = ctypes.c_size_t(self._ws.numel())
        ops.LAUNCHES[0] += 1
        _native.check(L.mm_task_fwd_bwd(ctypes.byref(t), ctypes.byref(db.desc), self._ws.data_ptr(),
                                        ctypes.byref(have), loss_sum.data_ptr(), ops.stream_ptr(),
                                        dec_done.cuda_event if dec_done is not None else None),
                      "mm_task_fwd_bwd")

    def forward_backward_py(self, task: TaskSpec, db: DeviceBatch, loss_sum: torch.Tensor) -> None:
        """Per-op Python path (same kernels, same order); used for diagnostics
        (intermediate tracing) and as the native driver's cross-check."""
        shp, dev, d = self.shape, self.device, self.shape.d_model
        self._cur_db = db
        ek, dk = embedding_keys(task)
        emb_e, emb_d = self.states[ek], self.states[dk]
        Ts, Tt = db.n_src, db.n_tgt
        # ---- encoder
        x = torch.empty(Ts, d, device=dev)
        ops.embed_fwd(db.src, db.src_pos, emb_e.w("emb"), x, self.scale)
        self._tr("emb_src", x)
        enc_saved = []
        for key in task.enc_modules:
            st = self.states[key]
            for i in range(st.layout.n_layers):
                sv = []
                x = self._self_block_fwd(st, f"l{i}.", x, db.cu_src, db.n_seq, db.max_src, False, sv,
                                         db.attn_src)
                self._tr(f"enc_l{i}_attn", x)
                x = self._ffn_fwd(st, f"l{i}.", x, sv)
                self._tr(f"enc_l{i}_ffn", x)
                enc_saved.append((st, f"l{i}.", sv))
        lnf_e = self.states[task.enc_modules[-1]]
        mem, mem_mean, mem_rstd = self._ln(lnf_e, "lnf", x)
        self._tr("x_enc", x)
        self._tr("mem", mem)
        x_enc = x
        # ---- decoder
        y = torch.empty(Tt, d, device=dev)
        ops.embed_fwd(db.tgt_in, db.tgt_pos, emb_d.w("emb"), y, self.scale)
        dec_saved = []
        for key in task.dec_modules:
            st = self.states[key]
            for i in range(st.layout.n_layers):
                sv = []
                y = self._self_block_fwd(st, f"l{i}.", y, db.cu_tgt, db.n_seq, db.max_tgt, True, sv,
                                         db.attn_tgt)
                y = self._cross_block_fwd(st, f"l{i}.", y, mem, db, sv)
                y = self._ffn_fwd(st, f"l{i}.", y, sv)
                dec_saved.append((st, f"l{i}.", sv))
        lnf_d = self.states[task.dec_modules[-1]]
        hdec, hd_mean, hd_rstd = self._ln(lnf_d, "lnf", y)
        self._tr("y_dec", y)
        self._tr("hdec", hdec)
        logits = torch.empty(Tt, shp.vocab, device=dev, dtype=torch.bfloat16)
        ops.gemm(hdec, emb_d.w("gen.w"), logits, epilogue=ops.EPI_BF16, bias=emb_d.f32("gen.b"))
        row_loss = torch.empty(Tt, device=dev)
        self._tr("logits", logits)
        ops.xent(logits, db.labels, logits, row_loss, 1.0 / Tt, loss_sum)  # dlogits in place
        dlogits = logits
        self._tr("dlogits", dlogits)
        # ---- generator backward
        ops.gemm(dlogits, hdec, emb_d.g("gen.w"), a_kmajor=False, b_kmajor=False,
                 epilogue=ops.EPI_F32_ACCUM, dbias=emb_d.g("gen.b"))
        dh = torch.empty(Tt, d, device=dev)
        ops.gemm(dlogits, emb_d.w("gen.w"), dh, b_kmajor=False, epilogue=ops.EPI_F32)
        del logits, dlogits
        dy = self._zeros(Tt, d)
        dy_bf = torch.empty(Tt, d, device=dev, dtype=torch.bfloat16)
        self._ln_bwd(lnf_d, "lnf", dh, y, hd_mean, hd_rstd, dy, dy_bf)
        self._tr("dh", dh)
        self._tr("dy_top", dy)
        dmem = self._zeros(Ts, d)
        for st, p, sv in reversed(dec_saved):
            self._ffn_bwd(st, p, sv[2], dy, dy_bf)
            self._cross_bwd(st, p, sv[1], dy, dy_bf, mem, dmem, db)
            self._self_bwd(st, p, sv[0], dy, dy_bf, db.cu_tgt, db.n_seq, db.max_tgt, True)
        self._tr("dy_bottom", dy)
        self._tr("dmem", dmem)
        self._embed_bwd(db, "emb_tgt", db.tgt_in, dy, emb_d.g("emb"))
        # ---- encoder backward
        dx = self._zeros(Ts, d)
        dx_bf = torch.empty(Ts, d, device=dev, dtype=torch.bfloat16)
        self._ln_bwd(lnf_e, "lnf", dmem, x_enc, mem_mean, mem_rstd, dx, dx_bf)
        for st, p, sv in reversed(enc_saved):
            self._ffn_bwd(st, p, sv[1], dx, dx_bf)
            self._self_bwd(st, p, sv[0], dx, dx_bf, db.cu_src, db.n_seq, db.max_src, False)
        self._tr("dx_bottom", dx)
        self._embed_bwd(db, "emb_src", db.src, dx, emb_e.g("emb"))

    def _embed_bwd(self, db, name, ids, dout, dtable) -> None:
        """K8 scatter-add: the deterministic sorted kernels when the batch
        carries their tables (DeviceBatch always does), else atomics."""
        counts = getattr(db, "emb_counts", {}).get(name)
        if counts is None:
            ops.embed_bwd(ids, dout, dtable, self.scale)
            return
        nc, nm = counts
        scratch = torch.empty(max(nc, 1), dout.shape[1], device=self.device) if nm else None
        ops.embed_bwd_sorted(getattr(db, name), dout.shape[0], nc, nm, dout, dtable, self.scale, scratch)

    # ------------------------------------------------------------------ step
    def zero_grads(self, keys=None, tail_only: bool = False) -> None:
        """DeviceState.reset (syncsim.py:108-111).  Only buckets that will be
        written this step need zeroing: K3 never reads a module with n = 0,
        and a module's bucket is zeroed before its first use in a step.
        ``tail_only``: zero [layout.dense_end, end) only -- the weight matrices
        in front are stored whole by the native driver's store-mode wgrads."""
        for k in (self.states if keys is None else keys):
            st = self.states[k]
            ops.memset(st.grad[st.layout.dense_end:] if tail_only else st.grad, 0)
            self._dirty.discard(k)

    def step(self, step_idx: int, batches: Sequence[DeviceBatch], tasks=None) -> dict:
        """One optimizer step: len(batches) micro-batches (accum_count), then
        the Algorithm-1 exchange and the fused update.  Returns host-side
        bookkeeping; the loss stays on device in ``self.loss_sum``."""
        ops.memset(self.loss_sum, 0)
        # the multiplexer's picks (host RNG) fix this step's used set -- and so
        # the ready flags -- before any compute is issued (syncsim.py:353)
        if tasks is None:  # else: picked by the caller (one pick per micro-batch, in order)
            tasks = [self.mux.pick(step_idx) for _ in batches]
        picked = [t.id for t in tasks]
        used: set[ModuleKey] = set()
        for t in tasks:
            used.update(task_modules(t))
        if self._pending_mods & used:  # a module of this step is still being updated
            self.sync_updates()
        flags = ready_flags(self.plan, self.rank, used)
        counts_ready = None
        self._roots = None
        if self.comm is not None:
            # K1 on rank bitmasks: the world sum gives each module's ready set
            bits = ready_bits(self.plan, self.rank, used)
            self.flags_dev.copy_(torch.tensor(bits, dtype=torch.int32), non_blocking=True)
            self.comm.ready_count(self.flags_dev, self.n_ready_dev)  # K1, ahead of the compute
            self._counts_host.copy_(self.n_ready_dev, non_blocking=True)
            counts_ready = torch.cuda.Event()
            counts_ready.record()
        zeroed: set[ModuleKey] = set()
        overlap = self.overlap and self.native
        dec_done = self._dec_done if overlap else None
        store_mode = self.native and self.trace is None and self.store_first_wgrad
        for i, (task, db) in enumerate(zip(tasks, batches)):
            fresh = [k for k in task_modules(task) if k not in zeroed]
            # a module's first micro-batch of the step: its weight-gradient
            # GEMMs store, so only the bucket's tail needs the memset
            self.zero_grads([k for k in fresh if k in self._dirty], tail_only=store_mode)
            zeroed.update(fresh)
            self._dirty.update(fresh)
            self.forward_backward(task, db, self.loss_sum,
                                  dec_done if i == len(tasks) - 1 else None,
                                  store=frozenset(fresh) if store_mode else frozenset())
        if counts_ready is not None:
            counts_ready.synchronize()  # waits for K1 only, not for the compute behind it
            self._bits = self._counts_host.tolist()
            counts, self._roots = decode_ready(self._bits)
        else:
            counts = flags
        if overlap:
            # decoder-side modules: exchange + K3 on a side stream while the
            # encoder backward runs; sorted ModuleKey order
            # puts every decoder key first, so collective order is unchanged
            dec = {k for k in self.states if k.side is Side.DECODER}
            side = self._side_stream
            side.wait_event(dec_done)
            with torch.cuda.stream(side):
                # a thin background update: few CTAs, so the encoder-backward
                # GEMMs keep their SMs
                self.exchange_and_update(counts, used, only=dec, max_ctas=self.overlap_ctas)
            rest = set(self.states) - dec
            if self.defer_update:
                side.wait_stream(torch.cuda.current_stream())  # this step's gradients final
                with torch.cuda.stream(side):
                    self.exchange_and_update(counts, used, only=rest, max_ctas=self.overlap_ctas)
                ev = torch.cuda.Event()
                ev.record(side)
                self._pending_event = ev
                self._pending_mods |= {k for k in self.states if counts[self.index[k]] >= 1}
            else:
                if self.comm is not None:
                    # a decoder and an encoder module may share a member set and
                    # so a communicator: keep each communicator's collectives
                    # in one stream order on every rank
                    torch.cuda.current_stream().wait_stream(side)
                self.exchange_and_update(counts, used, only=rest)
                torch.cuda.current_stream().wait_stream(side)
        else:
            self.exchange_and_update(counts, used)
        return {"tasks": picked, "ready": dict(zip(self.plan.keys, counts))}

    def sync_updates(self) -> None:
        """Order the current stream after every issued optimizer update (the
        deferred ones of earlier steps included); host reads of module state
        (weights, moments, step counts on the device) must call this or a
        device-wide synchronize first."""
        if self._pending_event is not None:
            torch.cuda.current_stream().wait_event(self._pending_event)
            self._pending_event = None
        self._pending_mods = set()

    @staticmethod
    def shard_elems(n_elems: int, g: int) -> int:
        """Elements per member of the partitioned exchange: ceil(n / g) rounded
        up to 4 (plan.shard_begin's partition; shard j = [j S, (j+1) S))."""
        s = -(-n_elems // g)
        return (s + 3) & ~3

    def exchange_and_update(self, counts: Sequence[int], used=frozenset(), only=None,
                            max_ctas: int = 0) -> None:
        """K2 for the modules of ``exchange_order`` then K3 for every hosted
        module with n >= 1; ``only`` restricts both to a subset of keys."""
        if self.partitioned:
            self._partitioned_exchange(counts, used, only, max_ctas)
            return
        if self.peer is not None:
            # option B: shared modules in one fused peer-memory kernel, then
            # the local K3 for singletons
            self.peer.run(self._bits, only=only, zero_grad=self.zero_in_update)
            if self.zero_in_update:
                self._dirty -= {k for k in self.states if len(self.plan.groups[k]) >= 2
                                and (only is None or k in only)
                                and (self._bits[self.index[k]] >> self.rank) & 1}
            singles = {k for k in self.states if len(self.plan.groups[k]) < 2}
            self.fused_update(counts, singles if only is None else singles & set(only), max_ctas)
            return
        items = []
        if self.comm is not None:
            for k, members, root in exchange_plan(self.plan, self.rank, self._bits, only):
                grp = self.comm.by_set.get(tuple(members))
                st = self.states[k]
                # root >= 0 (n = 1): broadcast the one ready member's buffer (it is the sum)
                if root < 0 and k not in used and k in self._dirty:  # contribute the zero of Algorithm 1
                    ops.memset(st.grad, 0)
                self._dirty.add(k)  # receives the group's sum
                if st.wire is not None:  # bf16 wire: cast, reduce the copy, widen back below
                    ops.cast_bf16(st.grad, st.wire)
                    items.append(_native.ReduceItem(group=grp, buf=st.wire.data_ptr(),
                                                    n_elems=st.wire.numel(), dtype=1, root=root))
                else:
                    items.append(_native.ReduceItem(group=grp, buf=st.grad.data_ptr(),
                                                    n_elems=st.grad.numel(), dtype=0, root=root))
            self.comm.reduce(items)
            for k, _members, _root in exchange_plan(self.plan, self.rank, self._bits, only):
                st = self.states[k]
                if st.wire is not None:
                    ops.widen_bf16(st.wire, st.grad)
        self.fused_update(counts, only, max_ctas)

    def _partitioned_exchange(self, counts, used, only, max_ctas) -> None:
        """per shared module (sorted ModuleKey order, n >= 1) a
        reduce-scatter of the fp32 gradient bucket (member j receives the group
        sum of shard j), K3 on the owned shard only (the sum / n rescale, Adam
        and the bf16 cast of that shard), then an all-gather of the bf16
        weight shards.  Wire bytes per element: (g-1)/g * (4 + 2) instead of
        the all-reduce's 2 (g-1)/g * 4, and each member runs 1/g of the
        optimizer.  Member j's fp32 master and moments are authoritative on
        shard j (the checkpoint writes them per shard)."""
        plan_items, ag_items, mods = [], [], []
        for k, members, _root in exchange_plan(self.plan, self.rank, self._bits, only):
            st = self.states[k]
            g, j = len(members), members.index(self.rank)
            s = self.shard_elems(st.layout.numel, g)
            if k not in used and k in self._dirty:  # the zero contribution of Algorithm 1
                ops.memset(st.grad, 0)
            self._dirty.add(k)
            grp = self.comm.by_set.get(tuple(members))
            if st.wire is not None:  # bf16 wire: reduce-scatter the bf16 copy
                ops.cast_bf16(st.grad, st.wire)
                plan_items.append(_native.ReduceItem(group=grp, buf=st.wire.data_ptr(), n_elems=g * s,
                                                     dtype=1, root=-1, mode=1, shard=s))
            else:
                plan_items.append(_native.ReduceItem(group=grp, buf=st.grad.data_ptr(), n_elems=g * s,
                                                     dtype=0, root=-1, mode=1, shard=s))
            ag_items.append(_native.ReduceItem(group=grp, buf=st.weights.data_ptr(), n_elems=g * s,
                                               dtype=1, root=-1, mode=2, shard=s))
            mods.append((k, j * s, s))
        self.comm.reduce(plan_items)
        for k, off, cnt in mods:  # widen the owned shard of a bf16 reduce-scatter
            st = self.states[k]
            if st.wire is not None:
                ops.widen_bf16(st.wire[off:off + cnt], st.grad[off:off + cnt])
        shards = {k: (off, n) for k, off, n in mods}
        singles = {k for k in self.states if len(self.plan.groups[k]) < 2
                   and (only is None or k in only)}
        self.fused_update(counts, singles | set(shards), max_ctas, shards=shards)
        self.comm.reduce(ag_items)

    def fused_update(self, counts: Sequence[int], only=None, max_ctas: int = 0,
                     shards: Optional[dict] = None) -> None:
        a = self.adam
        mods = []
        for k, st in self.states.items():
            if only is not None and k not in only:
                continue
            n = counts[self.index[k]]
            if n < 1:
                continue
            st.step += 1
            bc1 = 1.0 - a.beta1 ** st.step
            bc2 = 1.0 - a.beta2 ** st.step
            if self.zero_in_update and not (shards and k in shards):
                self._dirty.discard(k)  # the update leaves the bucket at zero
            off, cnt = (shards[k] if shards and k in shards else (0, st.master.numel()))
            mods.append(_native.AdamModule(
                grad=st.grad.data_ptr() + 4 * off, master=st.master.data_ptr() + 4 * off,
                exp_avg=st.exp_avg.data_ptr() + 4 * off, exp_avg_sq=st.exp_avg_sq.data_ptr() + 4 * off,
                param_bf16=st.weights.data_ptr() + 2 * off,
                n_elems=cnt, n_ready=n, ready_index=-1, step_size=a.lr / bc1,
                inv_sqrt_bc2=1.0 / math.sqrt(bc2)))
        if mods:
            ops.fused_update(mods, _native.AdamHyper.make(beta1=a.beta1, beta2=a.beta2, eps=a.eps,
                                                     weight_decay=a.weight_decay,
                                                     inv_loss_scale=1.0, max_ctas=max_ctas,
                                                     zero_grad=int(self.zero_in_update)))

    # ------------------------------------------------------------- checkpoint
    def save_checkpoint(self, root: str, extra: Optional[dict] = None) -> list[str]:
        """Write this rank's share of a per-module checkpoint (f4,
        ``checkpoint.py``): each module once per group by its lowest rank, or
        with the peer exchange each member's own shard; plus this rank's
        multiplexer state.  Returns the module files written."""
        from . import checkpoint as C
        from .plan import shard_begin
        self.sync_updates()
        torch.cuda.synchronize(self.device)
        written = []
        for k, st in self.states.items():
            members = self.plan.groups[k]
            n = st.layout.numel  # partitioned buckets carry zero padding past it
            host = {f: getattr(st, f)[:n].cpu().numpy() for f in C.FIELDS}
            if (self.peer is not None or self.partitioned) and len(members) >= 2:
                j, g = members.index(self.rank), len(members)
                b, e = shard_begin(n, g, j), shard_begin(n, g, j + 1)
                written.append(C.write_module(root, k, {f: v[b:e] for f, v in host.items()},
                                              st.step, n, (j, g, b, e)))
            elif self.rank == members[0]:
                written.append(C.write_module(root, k, host, st.step, n))
        # the rank's json goes last: it is the manifest of the files above
        extra = dict(extra or {})
        C.write_rank_state(root, self.rank, {"mux_rng": C.rng_to_json(self.mux.rng),
                                             "files": [os.path.relpath(f, root) for f in written],
                                             **extra})
        return written

    def load_checkpoint(self, root: str) -> dict:
        """Restore every hosted module (master, moments, Adam step; bf16
        weights re-cast from the master) and the multiplexer state; returns
        this rank's extra host state."""
        from . import checkpoint as C
        self.sync_updates()
        state = C.read_rank_state(root, self.rank)
        C.check_manifest(root, [f for k in self.states for f in C.module_files(root, k)],
                         state.get("step_idx"))
        for k, st in self.states.items():
            n = st.layout.numel
            arrays, step = C.read_module(root, k, n)
            for f in C.FIELDS:
                getattr(st, f)[:n].copy_(torch.from_numpy(arrays[f]))
            st.step = step
            ops.cast_bf16(st.master, st.weights)
            ops.memset(st.grad, 0)
            self._dirty.discard(k)
        state.pop("files", None)
        C.rng_from_json(self.mux.rng, state.pop("mux_rng"))
        torch.cuda.synchronize(self.device)
        return state

    def close(self) -> None:
        self.sync_updates()
        if self.peer is not None:
            torch.cuda.synchronize(self.device)
            self.peer.close()
            self.peer = None
        if self.comm is not None:
            self.comm.close()
            self.comm = None


class Trainer:
    """Public entry point of the trainer step for one rank.

    ``train_step(host_batches)`` takes this rank's micro-batches as host
    ``data.Batch`` objects, stages them through a pinned buffer (one H2D copy
    per micro-batch), runs forward / backward / Algorithm-1 exchange / fused
    update and returns the step's loss (sum over micro-batches of the token
    mean) read back to the host.
    """

    def __init__(self, tasks, topo, shape, rank: int = 0, world: int = 1, device=None,
                 seed: int = 0, adam: AdamConfig = AdamConfig(), store=None,
                 pinned_elems: int = 1 << 20):
        self.engine = Engine(tasks, topo, shape, rank, world, device, seed, adam, store)
        # MM_LAZY_ZERO=1: the update zeroes the gradients it consumed (no memset
        # before a bucket's next use).  Off: measured neutral on config 3 (the
        # memsets overlap; the update moves 34 instead of 30 B per parameter)
        self.engine.zero_in_update = os.environ.get("MM_LAZY_ZERO", "0") == "1"
        self.device = self.engine.device
        self._pinned = [torch.empty(pinned_elems, dtype=torch.int32, pin_memory=True)
                        for _ in range(4)]
        # per pinned buffer: event recorded after its H2D copy was queued; the
        # host waits on it before writing the buffer again (the copy is
        # asynchronous, and a step may stage more micro-batches than buffers)
        self._pin_events: list = [None] * len(self._pinned)
        self._loss_host = torch.empty(1, dtype=torch.float32, pin_memory=True)
        self._loss_ring = torch.empty(2, dtype=torch.float32, pin_memory=True)  # train_steps
        self._pin_next = 0  # rotating pinned staging buffer (reused >= 2 steps later)
        self.step_idx = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 4

    def stage(self, batches) -> list:
        out = []
        for b in batches:
            slot = self._pin_next % len(self._pinned)
            self._pin_next += 1
            if self._pin_events[slot] is not None:
                self._pin_events[slot].synchronize()  # its previous H2D copy has read it
            out.append(DeviceBatch(b, self.device, pinned=self._pinned[slot]))
            ev = torch.cuda.Event()
            ev.record()
            self._pin_events[slot] = ev
        self.h2d_bytes = sum(d.h2d_bytes for d in out)
        return out

    def train_steps(self, step_batches, n_steps: int) -> list:
        """``n_steps`` training steps over an iterable of per-step micro-batch
        lists, with lookahead: the host builds and stages step k+1's batches
        (one H2D copy each, queued behind step k) and issues step k+1 before
        it waits for step k's loss, so the GPU never idles between steps;
        every step's loss is copied back (a two-slot pinned ring, the copy
        queued before the next step resets the device sum) and read on the
        host one step later.  Returns the losses."""
        it = iter(step_batches)
        losses = []
        staged = self.stage(next(it)) if n_steps > 0 else None
        h2d = [self.h2d_bytes]
        pending = None  # (event, ring slot) of the previous step's loss copy
        for k in range(n_steps):
            self.engine.step(self.step_idx, staged)
            self.step_idx += 1
            slot = k & 1
            self._loss_ring[slot:slot + 1].copy_(self.engine.loss_sum, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            if k + 1 < n_steps:  # host work for step k+1 overlaps step k on the GPU
                staged = self.stage(next(it))
                h2d.append(self.h2d_bytes)
            if pending is not None:
                pending[0].synchronize()
                losses.append(float(self._loss_ring[pending[1]]))
            pending = (ev, slot)
        if pending is not None:
            pending[0].synchronize()
            losses.append(float(self._loss_ring[pending[1]]))
        self.h2d_bytes = sum(h2d) // max(1, len(h2d))
        return losses

    def train_step(self, host_batches=None, pipeline=None, accum: int = 1) -> float:
        """host_batches: this rank's micro-batches (task-agnostic synthetic
        data), or pipeline: a ``datapath.DataPipeline`` asked for the batch of
        each task the multiplexer picks (``accum`` micro-batches)."""
        tasks = None
        if pipeline is not None:
            tasks = [self.engine.mux.pick(self.step_idx) for _ in range(accum)]
            host_batches = [pipeline.batch_for(t) for t in tasks]
        dbs = self.stage(host_batches)
        self.engine.step(self.step_idx, dbs, tasks=tasks)
        self.step_idx += 1
        self._loss_host.copy_(self.engine.loss_sum, non_blocking=True)
        torch.cuda.current_stream().synchronize()  # also retires the pinned staging
        return float(self._loss_host[0])

    def save_checkpoint(self, root: str, pipeline=None) -> list[str]:
        """Every rank calls this after the same step (f4); ``pipeline`` (a
        ``datapath.DataPipeline``) adds its corpus positions and draws."""
        extra = {"step_idx": self.step_idx}
        if pipeline is not None:
            extra["pipeline"] = pipeline.state()
        return self.engine.save_checkpoint(root, extra)

    def load_checkpoint(self, root: str, pipeline=None) -> None:
        state = self.engine.load_checkpoint(root)
        self.step_idx = int(state["step_idx"])
        if pipeline is not None:
            if "pipeline" not in state:
                raise ValueError("checkpoint holds no data-pipeline state")
            pipeline.load_state(state["pipeline"])

    def close(self) -> None:
        self.engine.close()

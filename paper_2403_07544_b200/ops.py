"""Python wrappers over the C-ABI kernels of ``libmmb200.so``.

PyTorch tensors are used only as device allocations: each wrapper checks
device / dtype / contiguity, passes raw pointers and the current CUDA stream,
and raises ``MMError`` on a non-zero status.  Nothing here computes on the
host or falls back to a torch op.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _native
from ._native import check, lib

EPI_BF16, EPI_BF16_RELU, EPI_F32, EPI_F32_ACCUM, EPI_F32_RESID, EPI_BF16_DRELU, EPI_F32_RESID_LN = range(7)


class GemmArgs(ctypes.Structure):
    _fields_ = [
        ("a", ctypes.c_void_p), ("b", ctypes.c_void_p), ("d", ctypes.c_void_p),
        ("bias", ctypes.c_void_p), ("resid", ctypes.c_void_p), ("aux", ctypes.c_void_p),
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
        ("lda", ctypes.c_int64), ("ldb", ctypes.c_int64), ("ldd", ctypes.c_int64),
        ("a_kmajor", ctypes.c_int32), ("b_kmajor", ctypes.c_int32),
        ("epilogue", ctypes.c_int32), ("b_prefetch", ctypes.c_int32),
        ("dbias", ctypes.c_void_p),
        ("ln_gamma", ctypes.c_void_p), ("ln_beta", ctypes.c_void_p), ("ln_out", ctypes.c_void_p),
        ("ln_mean", ctypes.c_void_p), ("ln_rstd", ctypes.c_void_p), ("ln_eps", ctypes.c_float),
        ("relu_mask", ctypes.c_void_p), ("resid_early", ctypes.c_int32), ("pad_", ctypes.c_int32),
    ]


class AttnArgs(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_void_p), ("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
        ("o", ctypes.c_void_p), ("lse", ctypes.c_void_p), ("d_o", ctypes.c_void_p),
        ("dq", ctypes.c_void_p), ("dk", ctypes.c_void_p), ("dv", ctypes.c_void_p),
        ("cu_q", ctypes.c_void_p), ("cu_k", ctypes.c_void_p),
        ("ldq", ctypes.c_int64), ("ldk", ctypes.c_int64), ("ldv", ctypes.c_int64),
        ("ldo", ctypes.c_int64), ("ld_dq", ctypes.c_int64), ("ld_dk", ctypes.c_int64),
        ("ld_dv", ctypes.c_int64),
        ("n_seq", ctypes.c_int32), ("heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("causal", ctypes.c_int32), ("max_q", ctypes.c_int32), ("max_k", ctypes.c_int32),
        ("scale", ctypes.c_float), ("total_q", ctypes.c_int32),
        ("groups", ctypes.c_void_p), ("n_groups", ctypes.c_int32), ("cap", ctypes.c_int32),
        ("total_k", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("tc_groups", ctypes.c_void_p), ("n_tc_groups", ctypes.c_int32), ("pad0", ctypes.c_int32),
    ]


#: when a list, every GEMM launch appends (flops, start_event, end_event)
GEMM_PROFILE = None
#: launches issued through these wrappers (each wrapper = one kernel launch)
LAUNCHES = [0]


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")


def _rowstride(t: torch.Tensor, name: str) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name} must be a 2-D row-major view")
    return t.stride(0)


def gemm_args(a: torch.Tensor, b: torch.Tensor, d: torch.Tensor, *, a_kmajor: bool = True,
              b_kmajor: bool = True, epilogue: int = EPI_BF16, bias=None, resid=None, aux=None,
              dbias=None, ln=None, relu_mask=None) -> GemmArgs:
    """Validated mm_gemm_args for d[M,N] (epilogue)= op(a) @ op(b)^T."""
    _need(a, torch.bfloat16, "a")
    _need(b, torch.bfloat16, "b")
    m, k = (a.shape[0], a.shape[1]) if a_kmajor else (a.shape[1], a.shape[0])
    n, kb = (b.shape[0], b.shape[1]) if b_kmajor else (b.shape[1], b.shape[0])
    if k != kb:
        raise ValueError(f"K mismatch {k} vs {kb}")
    if tuple(d.shape) != (m, n):
        raise ValueError(f"d shape {tuple(d.shape)} != {(m, n)}")
    out_bf16 = epilogue in (EPI_BF16, EPI_BF16_RELU, EPI_BF16_DRELU)
    _need(d, torch.bfloat16 if out_bf16 else torch.float32, "d")
    args = GemmArgs(a=a.data_ptr(), b=b.data_ptr(), d=d.data_ptr(), bias=_ptr(bias),
                    resid=_ptr(resid), aux=_ptr(aux), m=m, n=n, k=k,
                    lda=_rowstride(a, "a"), ldb=_rowstride(b, "b"), ldd=_rowstride(d, "d"),
                    a_kmajor=int(a_kmajor), b_kmajor=int(b_kmajor), epilogue=epilogue,
                    dbias=_ptr(dbias))
    if epilogue == EPI_F32_RESID_LN:
        # ln = (gamma, beta, out_bf16 [M, N], mean [M], rstd [M], eps)
        g, bt, out, mean, rstd, eps = ln
        _need(out, torch.bfloat16, "ln_out")
        if tuple(out.shape) != (m, n) or out.stride(0) != n:
            raise ValueError("ln_out must be a contiguous [M, N] bf16 tensor")
        args.ln_gamma, args.ln_beta, args.ln_out = g.data_ptr(), bt.data_ptr(), out.data_ptr()
        args.ln_mean, args.ln_rstd, args.ln_eps = mean.data_ptr(), rstd.data_ptr(), float(eps)
    if resid is not None and _rowstride(resid, "resid") != args.ldd:
        raise ValueError("resid must share d's row stride")
    if aux is not None and _rowstride(aux, "aux") != args.ldd:
        raise ValueError("aux must share d's row stride")
    if relu_mask is not None:
        _need(relu_mask, torch.int32, "relu_mask")
        if relu_mask.numel() < m * ((n + 31) // 32) or not relu_mask.is_contiguous():
            raise ValueError("relu_mask must be a contiguous [M, ceil(N/32)] int32 tensor")
        args.relu_mask = relu_mask.data_ptr()
    args.b_prefetch = 0
    return args


def gemm(a: torch.Tensor, b: torch.Tensor, d: torch.Tensor, *, a_kmajor: bool = True,
         b_kmajor: bool = True, epilogue: int = EPI_BF16, bias=None, resid=None, aux=None,
         dbias=None, ln=None, relu_mask=None, resid_early: bool = False) -> None:
    """d[M,N] (epilogue)= op(a) @ op(b)^T on tcgen05.

    a: [M,K] if a_kmajor else [K,M]; b: [N,K] if b_kmajor else [K,N] (bf16).
    relu_mask (int32 [M, ceil(N/32)]): written by EPI_BF16_RELU, read by
    EPI_BF16_DRELU in place of aux.  resid_early: the caller guarantees the
    previous kernel on the stream did not write ``resid`` (mm_gemm_args).
    """
    args = gemm_args(a, b, d, a_kmajor=a_kmajor, b_kmajor=b_kmajor, epilogue=epilogue,
                     bias=bias, resid=resid, aux=aux, dbias=dbias, ln=ln, relu_mask=relu_mask)
    args.resid_early = int(resid_early)
    m, n, k = args.m, args.n, args.k
    LAUNCHES[0] += 1
    if GEMM_PROFILE is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(lib().mm_gemm(ctypes.byref(args), stream_ptr()), "mm_gemm")
        e1.record()
        GEMM_PROFILE.append((2.0 * m * n * k, e0, e1))
        return
    check(lib().mm_gemm(ctypes.byref(args), stream_ptr()), "mm_gemm")


def gemm_grouped(problems: list) -> None:
    """Several independent GEMMs in one persistent launch (mm_gemm_grouped).

    problems: list of dicts of gemm() keyword arguments (a, b, d, ...); all
    must share a_kmajor / b_kmajor.
    """
    arr = (GemmArgs * len(problems))(*[gemm_args(**p) for p in problems])
    LAUNCHES[0] += (len(problems) + 47) // 48
    check(lib().mm_gemm_grouped(arr, len(problems), stream_ptr()), "mm_gemm_grouped")


def layernorm_fwd(x, gamma, beta, y, mean, rstd, eps=1e-6) -> None:
    rows, cols = x.shape
    LAUNCHES[0] += 1
    check(lib().mm_layernorm_fwd(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(),
                                 mean.data_ptr(), rstd.data_ptr(), rows, cols, eps,
                                 stream_ptr()), "mm_layernorm_fwd")


def layernorm_bwd(dy, x, gamma, mean, rstd, dx, dx_bf16, dgamma, dbeta) -> None:
    rows, cols = x.shape
    LAUNCHES[0] += 1
    check(lib().mm_layernorm_bwd(dy.data_ptr(), x.data_ptr(), gamma.data_ptr(), mean.data_ptr(),
                                 rstd.data_ptr(), dx.data_ptr(), _ptr(dx_bf16), dgamma.data_ptr(),
                                 dbeta.data_ptr(), rows, cols, stream_ptr()), "mm_layernorm_bwd")


def embed_fwd(ids, pos, table_bf16, out, scale) -> None:
    rows, cols = out.shape
    LAUNCHES[0] += 1
    check(lib().mm_embed_fwd(ids.data_ptr(), pos.data_ptr(), table_bf16.data_ptr(), out.data_ptr(),
                             rows, cols, scale, stream_ptr()), "mm_embed_fwd")


EMB_CHUNK_ROWS = 32  # rows per partial of the deterministic embedding backward


def embed_segments(ids: np.ndarray) -> tuple[np.ndarray, int, int]:
    """Host tables of the deterministic embedding backward (mm_embed_segments):
    (int32 table, chunks, multi-chunk ids)."""
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    out = np.empty(7 * max(len(ids), 1), dtype=np.int32)
    nc, nm = ctypes.c_int(), ctypes.c_int()
    check(lib().mm_embed_segments(ids.ctypes.data, len(ids), EMB_CHUNK_ROWS, out.ctypes.data,
                                  ctypes.byref(nc), ctypes.byref(nm)), "mm_embed_segments")
    return out[:len(ids) + 3 * nc.value + 3 * nm.value], nc.value, nm.value


def embed_bwd_sorted(table_dev, rows, n_chunks, n_multi, dout, dtable, scale, scratch) -> None:
    _need(dout, torch.float32, "dout")
    _need(dtable, torch.float32, "dtable")
    LAUNCHES[0] += 1 + (n_multi > 0)
    check(lib().mm_embed_bwd_sorted(table_dev.data_ptr(), rows, n_chunks, n_multi, dout.data_ptr(),
                                    dtable.data_ptr(), dout.shape[1], scale,
                                    scratch.data_ptr() if scratch is not None else None, stream_ptr()),
          "mm_embed_bwd_sorted")


def embed_bwd(ids, dout, dtable, scale) -> None:
    rows, cols = dout.shape
    LAUNCHES[0] += 1
    check(lib().mm_embed_bwd(ids.data_ptr(), dout.data_ptr(), dtable.data_ptr(), rows, cols, scale,
                             stream_ptr()), "mm_embed_bwd")


def xent(logits, labels, dlogits, row_loss, grad_scale, loss_sum=None) -> None:
    rows, vocab = logits.shape
    LAUNCHES[0] += 1
    check(lib().mm_xent_fwd_bwd(logits.data_ptr(), labels.data_ptr(), dlogits.data_ptr(),
                                row_loss.data_ptr(), _ptr(loss_sum), rows, vocab, grad_scale,
                                stream_ptr()), "mm_xent_fwd_bwd")


def colsum(x, out) -> None:
    rows, cols = x.shape
    LAUNCHES[0] += 1
    check(lib().mm_colsum_bf16(x.data_ptr(), out.data_ptr(), rows, cols, stream_ptr()),
          "mm_colsum_bf16")


def cast_bf16(x, y) -> None:
    LAUNCHES[0] += 1
    check(lib().mm_cast_f32_bf16(x.data_ptr(), y.data_ptr(), x.numel(), stream_ptr()),
          "mm_cast_f32_bf16")


def widen_bf16(x, y) -> None:
    """y (fp32) = x (bf16), elementwise."""
    LAUNCHES[0] += 1
    check(lib().mm_cast_bf16_f32(x.data_ptr(), y.data_ptr(), x.numel(), stream_ptr()),
          "mm_cast_bf16_f32")


def attention_args(q, k, v, o, lse, cu_q, cu_k, n_seq, heads, max_q, max_k, causal,
                   d_o=None, dq=None, dk=None, dv=None, groups=None, tc_groups=None,
                   head_dim: int = 64) -> AttnArgs:
    """groups: (device int32 tensor [2*n_groups], n_groups, cap) from
    data.attention_groups (32-row aligned); tc_groups: the unpadded packing
    (align = 1) for the tcgen05 backward.  Both are built here from cu_q /
    cu_k when omitted; tc_groups=False keeps the backward on `groups`.
    head_dim 64 runs the tcgen05 kernels, 16 / 32 (config 1's true shape)
    the CUDA-core kernels of attn_small.cu."""
    hd = int(head_dim)
    import numpy as _np
    from .data import attention_groups
    if groups is None:
        gh, cap = attention_groups(_np.asarray(cu_q.cpu()), _np.asarray(cu_k.cpu()))
        groups = (torch.from_numpy(gh).to(q.device), len(gh) // 2, cap)
    if tc_groups is None:
        th, _ = attention_groups(_np.asarray(cu_q.cpu()), _np.asarray(cu_k.cpu()), align=1)
        tc_groups = (torch.from_numpy(th).to(q.device), len(th) // 2)
    gt, n_groups, cap = groups
    tt, n_tc = (None, 0) if tc_groups is False else tc_groups[:2]
    args = AttnArgs(
        q=q.data_ptr(), k=k.data_ptr(), v=v.data_ptr(), o=o.data_ptr(), lse=lse.data_ptr(),
        d_o=_ptr(d_o), dq=_ptr(dq), dk=_ptr(dk), dv=_ptr(dv),
        cu_q=cu_q.data_ptr(), cu_k=cu_k.data_ptr(),
        ldq=q.stride(0), ldk=k.stride(0), ldv=v.stride(0), ldo=o.stride(0),
        ld_dq=dq.stride(0) if dq is not None else 0, ld_dk=dk.stride(0) if dk is not None else 0,
        ld_dv=dv.stride(0) if dv is not None else 0,
        n_seq=n_seq, heads=heads, head_dim=hd, causal=int(causal), max_q=max_q, max_k=max_k,
        scale=1.0 / math.sqrt(hd), total_q=q.shape[0],
        groups=gt.data_ptr(), n_groups=n_groups, cap=cap, total_k=k.shape[0],
        tc_groups=tt.data_ptr() if tt is not None else None, n_tc_groups=n_tc)
    # the struct holds raw pointers: keep the device group tables (possibly
    # built here) alive as long as the args are
    args._keep = (gt, tt)
    return args


def attention_fwd(args: AttnArgs) -> None:
    LAUNCHES[0] += 1
    check(lib().mm_attention_fwd(ctypes.byref(args), stream_ptr()), "mm_attention_fwd")


def attention_bwd(args: AttnArgs) -> None:
    LAUNCHES[0] += 1
    check(lib().mm_attention_bwd(ctypes.byref(args), stream_ptr()), "mm_attention_bwd")


def flush_l2(scratch: torch.Tensor) -> None:
    check(lib().mm_flush_l2(scratch.data_ptr(), scratch.numel() * scratch.element_size(),
                            stream_ptr()), "mm_flush_l2")


def memset(t: torch.Tensor, value: int = 0) -> None:
    if not t.is_contiguous():
        raise ValueError("memset needs a contiguous tensor")
    check(lib().mm_memset(t.data_ptr(), value, t.numel() * t.element_size(), stream_ptr()),
          "mm_memset")


def axpy(y: torch.Tensor, x: torch.Tensor, alpha: float) -> None:
    """y += alpha * x over fp32 or fp64 CUDA tensors (mm_axpy_f32 / _f64)."""
    dt = y.dtype if y.dtype in (torch.float32, torch.float64) else torch.float32
    _need(y, dt, "y")
    _need(x, dt, "x")
    if y.numel() != x.numel() or not (y.is_contiguous() and x.is_contiguous()):
        raise ValueError("axpy needs equal-size contiguous tensors")
    LAUNCHES[0] += 1
    if dt == torch.float64:
        check(lib().mm_axpy_f64(y.data_ptr(), x.data_ptr(), alpha, y.numel(), stream_ptr()),
              "mm_axpy_f64")
    else:
        check(lib().mm_axpy_f32(y.data_ptr(), x.data_ptr(), alpha, y.numel(), stream_ptr()),
              "mm_axpy_f32")


def sync_emulated(mods, only_ready: bool, f64: bool = False) -> None:
    arr = (_native.SyncModule * len(mods))(*mods)
    LAUNCHES[0] += 1
    if f64:
        check(lib().mm_sync_emulated_f64(arr, len(mods), int(only_ready), stream_ptr()),
              "mm_sync_emulated_f64")
    else:
        check(lib().mm_sync_emulated(arr, len(mods), int(only_ready), stream_ptr()),
              "mm_sync_emulated")


def peer_shard_begin(n_elems: int, group_size: int, member: int) -> int:
    """First element of member's shard (mm_peer_shard_begin; shard r of g is
    [begin(r), begin(r + 1)), begin(g) = n_elems)."""
    return int(lib().mm_peer_shard_begin(n_elems, group_size, member))


def peer_update(shards, hyper: "_native.AdamHyper") -> None:
    """Option-B exchange: masked peer reduce + Adam + weight all-gather."""
    if not shards:
        return
    arr = (_native.PeerShard * len(shards))(*shards)
    LAUNCHES[0] += (len(shards) + 111) // 112
    check(lib().mm_peer_update(arr, len(shards), ctypes.byref(hyper), stream_ptr()),
          "mm_peer_update")


def peer_barrier(sig: "_native.PeerSignal") -> None:
    if sig.n_peers == 0:
        return
    LAUNCHES[0] += 1
    check(lib().mm_peer_barrier(ctypes.byref(sig), stream_ptr()), "mm_peer_barrier")


def ipc_export(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, t's byte offset in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    check(lib().mm_ipc_export(t.data_ptr(), h, ctypes.byref(off)), "mm_ipc_export")
    return bytes(h.raw), int(off.value)


def ipc_import(handle: bytes, offset: int) -> int:
    """Device pointer of a peer's exported buffer (refcounted mapping)."""
    assert len(handle) == 64
    p = ctypes.c_void_p()
    check(lib().mm_ipc_import(handle, offset, ctypes.byref(p)), "mm_ipc_import")
    return int(p.value)


def ipc_release(ptr: int) -> None:
    check(lib().mm_ipc_release(ptr), "mm_ipc_release")


def fused_update(mods, hyper: "_native.AdamHyper", ready_dev=None) -> None:
    arr = (_native.AdamModule * len(mods))(*mods)
    LAUNCHES[0] += 1
    check(lib().mm_fused_update(arr, len(mods), ctypes.byref(hyper), _ptr(ready_dev),
                                stream_ptr()), "mm_fused_update")

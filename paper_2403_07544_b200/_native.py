"""ctypes binding of the C-ABI library ``libmmb200.so`` (declared in
``include/mmb200.h``).

There is no fallback: if the library is missing the import of any product
module that needs it raises ``NativeLibraryError``.  Every entry point returns
an ``int`` status (0 = OK, negative = CUDA/NCCL/argument error) and the
message of the last failure is available from ``mm_last_error``.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_uint32, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "csrc", "libmmb200.so")
if os.environ.get("MM_LIB_VARIANT"):  # diagnostics: a tuning build from tools/build_variant.py
    LIB_PATH = os.path.join(os.path.dirname(_HERE), "build", "variants", os.environ["MM_LIB_VARIANT"],
                            "libmmb200.so")

#: must match MMB200_ABI_VERSION in include/mmb200.h
ABI_VERSION = 24
MAX_GROUP = 8
MAX_SYNC_GROUP = 32


class NativeLibraryError(RuntimeError):
    pass


class MMError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_lib = None
_call_lock = None  # set while emulated ranks call the library from several threads


class _Serialized:
    """The library handle with every entry point behind one process-wide
    lock (the C library keeps host-side staging state and is not re-entrant;
    emucomm.EmulatedWorld drives several ranks from host threads)."""

    def __init__(self, handle, lock):
        self._h, self._lock = handle, lock

    def __getattr__(self, name):
        fn = getattr(self._h, name)
        if not callable(fn):
            return fn
        lock = self._lock

        def call(*args):
            with lock:
                return fn(*args)
        return call


class serialized_calls:
    """Context manager: library calls from any thread take one lock."""

    def __enter__(self):
        global _call_lock
        import threading
        self._prev = _call_lock
        _call_lock = _call_lock or threading.RLock()
        return self

    def __exit__(self, *exc):
        global _call_lock
        _call_lock = self._prev
        return False


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None and _call_lock is not None:
        return _Serialized(_lib, _call_lock)
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        handle = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        _declare(handle)
        got = handle.mm_abi_version()
        if got != ABI_VERSION:
            raise NativeLibraryError(f"libmmb200 ABI {got} != expected {ABI_VERSION}; rebuild")
        _lib = handle
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().mm_last_error().decode(errors="replace")
        raise MMError(f"{what} failed ({status}): {msg}")


# ----------------------------------------------------------------------------
# descriptor structs (layouts mirror include/mmb200.h)


class SyncModule(ctypes.Structure):
    _fields_ = [
        ("bufs", c_void_p * MAX_SYNC_GROUP),
        ("out", c_void_p),
        ("n_elems", c_int64),
        ("group_size", c_int32),
        ("used_mask", c_uint32),
    ]


class AdamModule(ctypes.Structure):
    _fields_ = [
        ("grad", c_void_p),
        ("master", c_void_p),
        ("exp_avg", c_void_p),
        ("exp_avg_sq", c_void_p),
        ("param_bf16", c_void_p),
        ("n_elems", c_int64),
        ("n_ready", c_int32),
        ("ready_index", c_int32),
        ("step_size", c_float),
        ("inv_sqrt_bc2", c_float),
    ]


class AdamHyper(ctypes.Structure):
    _fields_ = [
        ("beta1", c_float),
        ("beta2", c_float),
        ("eps", c_float),
        ("weight_decay", c_float),
        ("inv_loss_scale", c_float),
        ("one_minus_beta1", c_float),
        ("one_minus_beta2", c_float),
        ("max_ctas", c_int32),
        ("zero_grad", c_int32),
    ]

    @classmethod
    def make(cls, beta1, beta2, eps, weight_decay=0.0, inv_loss_scale=1.0, max_ctas=0, zero_grad=0):
        return cls(beta1=beta1, beta2=beta2, eps=eps, weight_decay=weight_decay,
                   inv_loss_scale=inv_loss_scale, one_minus_beta1=1.0 - beta1,
                   one_minus_beta2=1.0 - beta2, max_ctas=max_ctas, zero_grad=zero_grad)


class ReduceItem(ctypes.Structure):
    _fields_ = [
        ("group", c_void_p),
        ("buf", c_void_p),
        ("n_elems", c_int64),
        ("dtype", c_int32),
        ("root", c_int32),  # -1: allreduce; >= 0: broadcast from this group rank (n = 1)
        ("mode", c_int32),  # 0 allreduce / broadcast, 1 reduce-scatter, 2 all-gather
        ("pad_", c_int32),
        ("shard", c_int64),  # modes 1 / 2: elements per group rank
    ]


class PeerShard(ctypes.Structure):
    """mm_peer_shard: one member's owned shard of one module (option-B exchange)."""
    _fields_ = [
        ("grad", c_void_p * MAX_GROUP),
        ("param", c_void_p * MAX_GROUP),
        ("master_copy", c_void_p * MAX_GROUP),
        ("master", c_void_p),
        ("exp_avg", c_void_p),
        ("exp_avg_sq", c_void_p),
        ("begin", c_int64),
        ("end", c_int64),
        ("group_size", c_int32),
        ("ready_mask", ctypes.c_uint32),
        ("step_size", c_float),
        ("inv_sqrt_bc2", c_float),
    ]


PEER_MAX_RANKS = 32


class PeerSignal(ctypes.Structure):
    """mm_peer_signal: the flag barrier over NVLink peer memory."""
    _fields_ = [
        ("local_flags", c_void_p),
        ("peer_flags", c_void_p * PEER_MAX_RANKS),
        ("peer_rank", c_int32 * PEER_MAX_RANKS),
        ("n_peers", c_int32),
        ("my_rank", c_int32),
        ("epoch", ctypes.c_uint32),
        ("timeout_ms", c_int32),
    ]


class LayerOffsets(ctypes.Structure):
    _fields_ = [(n, c_int64) for n in (
        "ln1_g", "ln1_b", "qkv_w", "qkv_b", "out_w", "out_b",
        "lnc_g", "lnc_b", "cq_w", "cq_b", "ckv_w", "ckv_b", "cout_w", "cout_b",
        "ln2_g", "ln2_b", "ff1_w", "ff1_b", "ff2_w", "ff2_b")]


class Stack(ctypes.Structure):
    _fields_ = [("w_bf16", c_void_p), ("w_f32", c_void_p), ("grad", c_void_p),
                ("layers", POINTER(LayerOffsets)), ("n_layers", c_int32), ("decoder", c_int32),
                ("lnf_g", c_int64), ("lnf_b", c_int64), ("store_wgrad", c_int32), ("pad_", c_int32)]


class Embed(ctypes.Structure):
    _fields_ = [("w_bf16", c_void_p), ("w_f32", c_void_p), ("grad", c_void_p),
                ("emb", c_int64), ("gen_w", c_int64), ("gen_b", c_int64), ("store_gen_w", c_int32),
                ("pad_", c_int32)]


class Task(ctypes.Structure):
    _fields_ = [("d_model", c_int32), ("heads", c_int32), ("ffn", c_int32), ("vocab", c_int32),
                ("n_enc", c_int32), ("n_dec", c_int32), ("enc", POINTER(Stack)),
                ("dec", POINTER(Stack)), ("enc_emb", Embed), ("dec_emb", Embed)]


class BatchDesc(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("src", "src_pos", "cu_src", "tgt_in", "tgt_pos", "labels",
                                        "cu_tgt", "groups_src", "groups_tgt", "groups_cross")] + \
               [(n, c_int32) for n in ("n_seq", "n_src", "n_tgt", "max_src", "max_tgt",
                                       "ng_src", "cap_src", "ng_tgt", "cap_tgt", "ng_cross",
                                       "cap_cross")] + \
               [(n, c_void_p) for n in ("tcg_src", "tcg_tgt", "tcg_cross")] + \
               [(n, c_int32) for n in ("ntc_src", "ntc_tgt", "ntc_cross", "pad0")] + \
               [(n, c_void_p) for n in ("emb_src", "emb_tgt")] + \
               [(n, c_int32) for n in ("nch_src", "nmul_src", "nch_tgt", "nmul_tgt")]


def _declare(h: ctypes.CDLL) -> None:
    variant = bool(os.environ.get("MM_LIB_VARIANT"))

    def sig(name, res, *args):
        if variant and not hasattr(h, name):  # A/B builds of older sources (tools/)
            return
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = list(args)

    sig("mm_abi_version", c_int)
    sig("mm_last_error", c_char_p)
    sig("mm_device_info", c_int, POINTER(c_int), POINTER(c_int))
    # K9 -- comm cost (replaces _speedups.pyx:11-57)
    sig("mm_comm_cost", c_int, POINTER(c_double), c_int64, POINTER(c_int64), POINTER(c_int64),
        POINTER(c_int64), POINTER(c_int64), c_int64, c_double, c_double, POINTER(c_double),
        POINTER(c_double))
    sig("mm_comm_cost_moves", c_int, POINTER(c_double), c_int64, POINTER(c_int64), POINTER(c_int64),
        POINTER(c_int64), c_int64, POINTER(c_int64), c_int64, c_double, c_double, POINTER(c_int64),
        c_int64, POINTER(c_double), c_int)
    # Algorithm-1 sync, emulated devices on one GPU (sync_step syncsim.py:121-153)
    sig("mm_sync_emulated", c_int, POINTER(SyncModule), c_int, c_int, c_void_p)
    sig("mm_sync_emulated_f64", c_int, POINTER(SyncModule), c_int, c_int, c_void_p)
    # K3 fused rescale + unscale + Adam + bf16 cast
    sig("mm_fused_update", c_int, POINTER(AdamModule), c_int, POINTER(AdamHyper), c_void_p, c_void_p)
    # NCCL plumbing (K1/K2)
    sig("mm_nccl_unique_id", c_int, ctypes.c_char_p)
    sig("mm_comm_init", c_int, c_int, c_int, ctypes.c_char_p, c_int, POINTER(c_void_p))
    sig("mm_comm_destroy", c_int, c_void_p)
    sig("mm_group_create", c_int, c_void_p, POINTER(c_int), c_int, POINTER(c_void_p))
    sig("mm_group_destroy", c_int, c_void_p)
    sig("mm_ready_count", c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p)
    sig("mm_reduce_modules", c_int, c_void_p, POINTER(ReduceItem), c_int, c_void_p)
    # option-B exchange: fused peer reduce + update + all-gather, flag barrier, IPC
    sig("mm_peer_shard_begin", c_int64, c_int64, c_int, c_int)
    sig("mm_peer_update", c_int, POINTER(PeerShard), c_int, POINTER(AdamHyper), c_void_p)
    sig("mm_peer_barrier", c_int, POINTER(PeerSignal), c_void_p)
    sig("mm_ipc_export", c_int, c_void_p, c_void_p, POINTER(ctypes.c_uint64))
    sig("mm_ipc_import", c_int, c_void_p, ctypes.c_uint64, POINTER(c_void_p))
    sig("mm_ipc_release", c_int, c_void_p)
    # layer kernels (K4-K8)
    sig("mm_launch_count", ctypes.c_ulonglong)
    sig("mm_gemm", c_int, c_void_p, c_void_p)
    sig("mm_gemm_grouped", c_int, c_void_p, c_int, c_void_p)
    sig("mm_abi_sizeof", c_int64, c_char_p)
    sig("mm_gemm_timing", c_int, c_int, POINTER(c_double), POINTER(c_float), POINTER(c_int))
    sig("mm_gemm_spans", c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_int))
    sig("mm_step_timing", c_int, c_int, POINTER(c_float), POINTER(c_int))
    sig("mm_attention_order", c_int, c_void_p, c_void_p, c_int, c_int, c_void_p)
    sig("mm_attention_tables", c_int, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p)
    sig("mm_attention_groups", c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, POINTER(c_int),
        POINTER(c_int))
    sig("mm_gemm_trace", c_int, c_void_p)
    sig("mm_layernorm_fwd", c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
        c_int64, c_int, c_float, c_void_p)
    sig("mm_layernorm_bwd", c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
        c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p)
    sig("mm_embed_fwd", c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_float,
        c_void_p)
    sig("mm_embed_bwd", c_int, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_float, c_void_p)
    sig("mm_attention_fwd", c_int, c_void_p, c_void_p)
    sig("mm_attention_bwd", c_int, c_void_p, c_void_p)
    sig("mm_xent_fwd_bwd", c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
        c_int, c_float, c_void_p)
    sig("mm_colsum_bf16", c_int, c_void_p, c_void_p, c_int64, c_int, c_void_p)
    sig("mm_cast_f32_bf16", c_int, c_void_p, c_void_p, c_int64, c_void_p)
    sig("mm_flush_l2", c_int, c_void_p, c_size_t, c_void_p)
    sig("mm_memset", c_int, c_void_p, c_int, c_size_t, c_void_p)
    sig("mm_embed_bwd_sorted", c_int, c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p, c_int, c_float,
        c_void_p, c_void_p)
    sig("mm_embed_segments", c_int, c_void_p, c_int, c_int, c_void_p, POINTER(c_int), POINTER(c_int))
    sig("mm_cast_bf16_f32", c_int, c_void_p, c_void_p, c_int64, c_void_p)
    sig("mm_axpy_f32", c_int, c_void_p, c_void_p, c_float, c_int64, c_void_p)
    sig("mm_axpy_f64", c_int, c_void_p, c_void_p, c_double, c_int64, c_void_p)
    sig("mm_task_fwd_bwd", c_int, c_void_p, c_void_p, c_void_p, POINTER(c_size_t), c_void_p,
        c_void_p, c_void_p)


def symbols() -> list[str]:
    """Names of every entry point declared in include/mmb200.h."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "mmb200.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(mm_[a-z0-9_]+)\s*\(", text)))

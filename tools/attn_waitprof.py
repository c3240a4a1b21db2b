"""Per-unit wait-time breakdown of the tcgen05 attention backward.  Needs the
diagnostics build:
  python tools/build_variant.py attn_wp -DMM_ATTN_WAITPROF attention.cu=paper_2403_07544_b200/csrc/attention.cu
  MM_LIB_VARIANT=attn_wp python tools/attn_waitprof.py      (C5=1: config-5 shapes)"""
import os, sys, ctypes
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2403_07544_b200 import ops, _native
from paper_2403_07544_b200.data import attention_groups, attention_order
dev = torch.device("cuda:0")
L = _native.lib()
WP = hasattr(L, "mm_attn_wp_read")  # release build: timing only (e.g. under ncu)
if WP:
    L.mm_attn_wp_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
rng = np.random.default_rng(0)
cfg5 = os.environ.get("C5") == "1"
d, heads, TOK, MU, SIG, HI = (1024, 16, 16384, 3.2, 0.6, 128) if cfg5 else (512, 8, 4096, 3.0, 0.5, 128)
ls = []
while sum(ls) < TOK:
    ls.append(int(np.clip(round(rng.lognormal(MU, SIG)), 4, HI)))
lq = np.array(ls)
cu = np.concatenate([[0], np.cumsum(lq)]).astype(np.int32)
T = int(cu[-1])
q = torch.randn(T, d, device=dev).bfloat16(); k = torch.randn(T, d, device=dev).bfloat16(); v = torch.randn(T, d, device=dev).bfloat16()
o = torch.empty_like(q); lse = torch.empty(heads, T, device=dev); do = torch.randn_like(q)
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
c = torch.from_numpy(cu).to(dev)
args = ops.attention_args(q, k, v, o, lse, c, c, len(lq), heads, int(lq.max()), int(lq.max()), False, d_o=do, dq=dq, dk=dk, dv=dv)
ops.attention_fwd(args); ops.attention_bwd(args); torch.cuda.synchronize()
for _ in range(int(os.environ.get("REPS", "0"))):
    ops.attention_bwd(args)
torch.cuda.synchronize()
if WP:
    L.mm_attn_wp_read(None, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ops.attention_bwd(args); e1.record(); torch.cuda.synchronize()
units = args.n_tc_groups * heads
print("units", units, "per CTA", units / 148, "kernel us", e0.elapsed_time(e1) * 1e3)
if not WP:
    sys.exit(0)
buf = (ctypes.c_ulonglong * (148 * 8))()
L.mm_attn_wp_read(buf, 0)
w = np.array(buf, dtype=np.float64).reshape(148, 8)
per_unit = w[:, :4].sum(0) / units / 1.9e3  # cycles -> us at ~1.9 GHz
print("avg wait per unit (us): MMA<-tma %.2f  MMA<-p %.2f  EPI<-s %.2f  EPI<-g %.2f" % tuple(per_unit))

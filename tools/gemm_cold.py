"""Does a GEMM launch pay for the kernels around it?  Per-launch device spans
(mm_gemm_timing) of the FFN-up GEMM (4096x2048x512, ReLU epilogue) when it
runs (A) back to back, (B) alternating with a LayerNorm, (C) alternating with
a LayerNorm and a GEMM of another instantiation (MN-major B), (D) as (C) with
the attention forward too.  python tools/gemm_cold.py"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import _native, ops
dev = torch.device("cuda:0")
L = _native.lib()
T, d, F = 4096, 512, 2048
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(T, d, device=dev, generator=g)
h = torch.randn(T, d, device=dev, generator=g).bfloat16()
W1 = (torch.randn(F, d, device=dev, generator=g) / 30).bfloat16()
b1 = torch.zeros(F, device=dev)
f = torch.empty(T, F, device=dev, dtype=torch.bfloat16)
W = (torch.randn(d, d, device=dev, generator=g) / 30).bfloat16()
dx = torch.empty(T, d, device=dev)
gam, bet = torch.ones(d, device=dev), torch.zeros(d, device=dev)
y = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
mu, rs = torch.empty(T, device=dev), torch.empty(T, device=dev)
ff1 = lambda: ops.gemm(h, W1, f, epilogue=ops.EPI_BF16_RELU, bias=b1)
mask = torch.empty((T, F // 32), device=dev, dtype=torch.int32)
ff1m = lambda: ops.gemm(h, W1, f, epilogue=ops.EPI_BF16_RELU, bias=b1, relu_mask=mask)
other = lambda: ops.gemm(h, W, dx, b_kmajor=False, epilogue=ops.EPI_F32)
ln = lambda: ops.layernorm_fwd(x, gam, bet, y, mu, rs)


def spans(seq, reps=20):
    for fn in seq:
        fn()
    torch.cuda.synchronize()
    _native.check(L.mm_gemm_timing(1, None, None, None), "timing")
    for _ in range(reps):
        for fn in seq:
            fn()
    torch.cuda.synchronize()
    _native.check(L.mm_gemm_timing(0, None, None, None), "timing")
    n = 4096
    lo = (ctypes.c_ulonglong * n)(); hi = (ctypes.c_ulonglong * n)()
    fl = (ctypes.c_double * n)(); shp = (ctypes.c_int * (4 * n))(); cnt = ctypes.c_int()
    L.mm_gemm_spans(n, lo, hi, fl, shp, ctypes.byref(cnt))
    us = [(hi[i] - lo[i]) / 1e3 for i in range(cnt.value) if shp[4 * i + 1] == F]
    return np.median(us), np.mean(us)


L.mm_gemm_spans.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 5
for name, seq in (("A ff1 only", [ff1]), ("B ff1 + LN", [ff1, ln]),
                  ("C ff1 + LN + other GEMM", [ff1, ln, other]),
                  ("E ff1 + other GEMM", [ff1, other]),
                  ("F ff1 (ReLU mask) + LN + other", [ff1m, ln, other]),
                  ("G ff1 (ReLU mask) only", [ff1m])):
    med, mean = spans(seq)
    print(f"{name:28s} ff1 span median {med:6.2f} us  mean {mean:6.2f} us", flush=True)

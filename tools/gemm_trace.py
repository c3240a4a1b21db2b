"""Per-CTA phase timestamps of one GEMM launch (diagnostics)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import _native, ops
dev = torch.device("cuda:0")
L = _native.lib()
buf = torch.zeros(8 * 148, dtype=torch.int64, device=dev)
T = 4096
cases = {"fwd_out": (T, 512, 512, True, True, ops.EPI_F32), "fwd_ff1": (T, 2048, 512, True, True, ops.EPI_BF16_RELU),
         "wgrad_ff1": (2048, 512, T, False, False, ops.EPI_F32_ACCUM), "dgrad_ff1": (T, 512, 2048, True, False, ops.EPI_F32),
         "tiny": (128, 128, 64, True, True, ops.EPI_F32), "fwd_ff2": (T, 512, 2048, True, True, ops.EPI_F32)}
for name, (m, n, k, ak, bk, epi) in cases.items():
    A = torch.randn(m, k, device=dev).bfloat16() if ak else torch.randn(k, m, device=dev).bfloat16()
    B = torch.randn(n, k, device=dev).bfloat16() if bk else torch.randn(k, n, device=dev).bfloat16()
    bf = epi in (ops.EPI_BF16, ops.EPI_BF16_RELU)
    D = torch.zeros(m, n, device=dev, dtype=torch.bfloat16 if bf else torch.float32)
    bias = torch.zeros(n, device=dev) if bf else None
    for _ in range(3):
        ops.gemm(A, B, D, a_kmajor=ak, b_kmajor=bk, epilogue=epi, bias=bias)
    torch.cuda.synchronize()
    buf.zero_()
    L.mm_gemm_trace(buf.data_ptr())
    ops.gemm(A, B, D, a_kmajor=ak, b_kmajor=bk, epilogue=epi, bias=bias)
    torch.cuda.synchronize()
    L.mm_gemm_trace(None)
    t = buf.view(148, 8).cpu().numpy().astype(np.float64)
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    r = (t - base) / 1e3  # us
    med = lambda a, b: np.median(r[:, b] - r[:, a])
    print(f"{name:10s} ctas={len(t)} entry-spread {r[:,0].max():.2f} | setup {med(0,1):.2f} | first-full {med(1,2):.2f} | "
          f"mainloop {med(2,3):.2f} | mma-drain {med(3,4):.2f} | epi {med(4,5):.2f} | store-drain {med(5,6):.2f} | "
          f"exit {med(6,7):.2f} | end max {r[:,7].max():.2f} us")

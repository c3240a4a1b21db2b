"""Residual GEMM + LayerNorm: two launches (GEMM, mm_layernorm_fwd) vs the
fused MM_EPI_F32_RESID_LN launch, back to back in a CUDA graph."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")


def timeit(fn, n=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * n)


for m, n, k in [(4096, 512, 512), (4096, 512, 2048), (16384, 1024, 1024), (16384, 1024, 4096)]:
    A = torch.randn(m, k, device=dev).bfloat16()
    B = torch.randn(n, k, device=dev).bfloat16()
    bias = torch.randn(n, device=dev); resid = torch.randn(m, n, device=dev)
    g_, b_ = torch.ones(n, device=dev), torch.zeros(n, device=dev)
    x = torch.empty(m, n, device=dev); h = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    mean, rstd = torch.empty(m, device=dev), torch.empty(m, device=dev)

    def two():
        ops.gemm(A, B, x, epilogue=ops.EPI_F32_RESID, bias=bias, resid=resid)
        ops.layernorm_fwd(x, g_, b_, h, mean, rstd, eps=1e-6)

    def gemm_only():
        ops.gemm(A, B, x, epilogue=ops.EPI_F32_RESID, bias=bias, resid=resid)

    def fused():
        ops.gemm(A, B, x, epilogue=ops.EPI_F32_RESID_LN, bias=bias, resid=resid,
                 ln=(g_, b_, h, mean, rstd, 1e-6))
    print(f"{m}x{n}x{k}: gemm {timeit(gemm_only):6.2f} us  gemm+ln {timeit(two):6.2f} us  fused {timeit(fused):6.2f} us", flush=True)

"""Upper bound of fusing the FFN's two GEMMs into one launch: ff1 then ff2 as
two dependent launches vs the same two problems as ONE grouped launch with
no dependency (ff2 reads an independent input), CUDA graph, device time."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
T, d, F = 4096, 512, 2048
x = torch.randn(T, d, device=dev).bfloat16()
w1 = torch.randn(F, d, device=dev).bfloat16() * 0.05
w2 = torch.randn(d, F, device=dev).bfloat16() * 0.05
b1 = torch.zeros(F, device=dev)
b2 = torch.zeros(d, device=dev)
h = torch.empty(T, F, device=dev, dtype=torch.bfloat16)
h2 = torch.randn(T, F, device=dev).bfloat16()
res = torch.randn(T, d, device=dev)
out = torch.empty(T, d, device=dev)


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


def two():
    ops.gemm(x, w1, h, epilogue=ops.EPI_BF16_RELU, bias=b1)
    ops.gemm(h, w2, out, epilogue=ops.EPI_F32_RESID, bias=b2, resid=res)


def grouped():
    ops.gemm_grouped([dict(a=x, b=w1, d=h, epilogue=ops.EPI_BF16_RELU, bias=b1),
                      dict(a=h2, b=w2, d=out, epilogue=ops.EPI_F32_RESID, bias=b2, resid=res)])


def ff1():
    ops.gemm(x, w1, h, epilogue=ops.EPI_BF16_RELU, bias=b1)


def ff2():
    ops.gemm(h, w2, out, epilogue=ops.EPI_F32_RESID, bias=b2, resid=res)


print(f"ff1 {timeit(ff1):.2f} us  ff2 {timeit(ff2):.2f} us  two launches {timeit(two):.2f} us  "
      f"one grouped launch (no dependency) {timeit(grouped):.2f} us")

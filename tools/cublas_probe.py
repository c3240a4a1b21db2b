"""Run cuBLAS (torch.mm) and our GEMM once each on the config-3 shapes, for
an ncu comparison of tiling / L2 traffic (diagnostics)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
T = 4096
for (m, n, k) in [(T, 512, 512), (T, 512, 2048), (T, 2048, 512), (T, 1536, 512)]:
    A = torch.randn(m, k, device=dev).bfloat16()
    B = torch.randn(n, k, device=dev).bfloat16()
    D = torch.empty(m, n, device=dev)
    Dc = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    for _ in range(2):
        torch.mm(A, B.t(), out=Dc)
        ops.gemm(A, B, D, epilogue=ops.EPI_F32)
    torch.cuda.synchronize()

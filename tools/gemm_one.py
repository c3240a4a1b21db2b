"""One GEMM shape through cuBLAS (torch.mm) and libmmb200, a few launches
each (for ncu --set full captures)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
m, n, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 512, 2048)))
A = torch.randn(m, k, device=dev).bfloat16()
B = torch.randn(n, k, device=dev).bfloat16()
D = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    torch.mm(A, B.t(), out=D)
    ops.gemm(A, B, D, epilogue=ops.EPI_BF16)
torch.cuda.synchronize()

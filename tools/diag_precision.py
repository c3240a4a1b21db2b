"""Raw error levels of the kernels vs fp64 (diagnostic)."""
import os, sys, math
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
torch.backends.cuda.matmul.allow_tf32 = False
c = torch.device("cuda:0")
def rel(a, b): return ((a.double() - b).abs().max() / b.abs().max()).item()
for (m, n, k) in [(256, 256, 64), (512, 512, 512), (512, 512, 4096)]:
    A = torch.randn(m, k, device=c).bfloat16(); B = torch.randn(n, k, device=c).bfloat16()
    ref = A.double() @ B.double().t()
    d = torch.empty(m, n, device=c)
    ops.gemm(A, B, d, epilogue=ops.EPI_F32)
    cub = A.float() @ B.float().t()
    cub16 = (A @ B.t()).float()
    print(f"gemm {m}x{n}x{k}: mm rel {rel(d, ref):.2e}  torch-fp32 rel {rel(cub, ref):.2e}  cublas-bf16 rel {rel(cub16, ref):.2e}")
    # per-element distribution
    e = (d.double() - ref).abs() / ref.abs().max()
    print("   mean err", e.mean().item(), " frac>1e-5", (e > 1e-5).float().mean().item())
# K=16 single MMA
A = torch.randn(128, 16, device=c).bfloat16(); B = torch.randn(128, 16, device=c).bfloat16()
d = torch.empty(128, 128, device=c); ops.gemm(A, B, d, epilogue=ops.EPI_F32)
print("K16 rel", rel(d, A.double() @ B.double().t()))
# LN
x = torch.randn(1000, 512, device=c) * 3 + 1
g = torch.randn(512, device=c); b = torch.randn(512, device=c)
y = torch.empty(1000, 512, device=c, dtype=torch.bfloat16); mu = torch.empty(1000, device=c); rs = torch.empty(1000, device=c)
ops.layernorm_fwd(x, g, b, y, mu, rs, 1e-6)
ref = torch.nn.functional.layer_norm(x.double(), (512,), g.double(), b.double(), eps=1e-6)
print("LN bf16-out vs rne(fp64): mismatching elements", (y != ref.float().bfloat16()).float().mean().item())

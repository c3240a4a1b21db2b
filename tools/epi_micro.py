"""GEMM epilogue variants (bias, residual, bf16) on one shape (diagnostics)."""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
sys.path.insert(0, "tools")
from ln_fuse_micro import timeit
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
for m, n, k in [(4096, 512, 512), (4096, 512, 2048)]:
    A = torch.randn(m, k, device=dev).bfloat16(); B = torch.randn(n, k, device=dev).bfloat16()
    bias = torch.randn(n, device=dev); resid = torch.randn(m, n, device=dev)
    x = torch.empty(m, n, device=dev); xb = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    r = {}
    r["f32"] = timeit(lambda: ops.gemm(A, B, x, epilogue=ops.EPI_F32))
    r["f32+bias"] = timeit(lambda: ops.gemm(A, B, x, epilogue=ops.EPI_F32, bias=bias))
    r["resid"] = timeit(lambda: ops.gemm(A, B, x, epilogue=ops.EPI_F32_RESID, resid=resid))
    r["resid+bias"] = timeit(lambda: ops.gemm(A, B, x, epilogue=ops.EPI_F32_RESID, bias=bias, resid=resid))
    r["bf16"] = timeit(lambda: ops.gemm(A, B, xb, epilogue=ops.EPI_BF16))
    r["bf16+bias"] = timeit(lambda: ops.gemm(A, B, xb, epilogue=ops.EPI_BF16, bias=bias))
    print(m, n, k, " ".join(f"{kk} {v:.2f}" for kk, v in r.items()), flush=True)

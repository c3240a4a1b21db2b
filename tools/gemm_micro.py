"""Back-to-back GEMM timing per shape (CUDA graph of 20 launches, CUDA
events), ours vs cuBLAS (torch.mm, bf16 in / bf16 out).  Our epilogue is the
one the step uses for that shape: bf16 out (EPI_BF16*), fp32 out (EPI_F32:
twice cuBLAS's output bytes) or an fp32 TMA reduce-add (EPI_F32_ACCUM: read +
write of an fp32 output) -- the "out" column says which."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
T = 4096
cases = [  # name, m, n, k, a_k, b_k, epi
    ("fwd qkv", T, 1536, 512, True, True, ops.EPI_BF16),
    ("fwd out", T, 512, 512, True, True, ops.EPI_F32),
    ("fwd ff1", T, 2048, 512, True, True, ops.EPI_BF16_RELU),
    ("fwd ff2", T, 512, 2048, True, True, ops.EPI_F32),
    ("fwd gen", T, 32000, 512, True, True, ops.EPI_BF16),
    ("dgrad out", T, 512, 512, True, False, ops.EPI_F32),
    ("dgrad ff2", T, 2048, 512, True, False, ops.EPI_BF16),
    ("dgrad ff1", T, 512, 2048, True, False, ops.EPI_F32),
    ("dgrad gen", T, 512, 32000, True, False, ops.EPI_F32),
    ("dgrad gen acc", T, 512, 32000, True, False, ops.EPI_F32_ACCUM),
    ("wgrad out", 512, 512, T, False, False, ops.EPI_F32_ACCUM),
    ("wgrad qkv", 1536, 512, T, False, False, ops.EPI_F32_ACCUM),
    ("wgrad ff1", 2048, 512, T, False, False, ops.EPI_F32_ACCUM),
    ("wgrad ff2", 512, 2048, T, False, False, ops.EPI_F32_ACCUM),
    ("wgrad gen", 32000, 512, T, False, False, ops.EPI_F32_ACCUM),
    # config 5 (d 1024, ffn 4096, 16384 tokens)
    ("c5 fwd qkv", 16384, 3072, 1024, True, True, ops.EPI_BF16),
    ("c5 fwd ff1", 16384, 4096, 1024, True, True, ops.EPI_BF16_RELU),
    ("c5 fwd ff2", 16384, 1024, 4096, True, True, ops.EPI_F32),
    ("c5 fwd out", 16384, 1024, 1024, True, True, ops.EPI_F32),
    ("c5 dgrad ff1", 16384, 1024, 4096, True, False, ops.EPI_F32),
    ("c5 dgrad ff2", 16384, 4096, 1024, True, False, ops.EPI_BF16),
    ("c5 wgrad ff1", 4096, 1024, 16384, False, False, ops.EPI_F32_ACCUM),
    ("c5 wgrad qkv", 3072, 1024, 16384, False, False, ops.EPI_F32_ACCUM),
    ("c5 fwd gen", 16384, 32000, 1024, True, True, ops.EPI_BF16),
    ("tiny", 128, 128, 64, True, True, ops.EPI_F32),
    ("big", 8192, 8192, 8192, True, True, ops.EPI_BF16),
    ("maj kk", 2048, 512, 4096, True, True, ops.EPI_F32),
    ("maj km", 2048, 512, 4096, True, False, ops.EPI_F32),
    ("maj mk", 2048, 512, 4096, False, True, ops.EPI_F32),
    ("maj mm", 2048, 512, 4096, False, False, ops.EPI_F32),
    ("maj mm acc", 2048, 512, 4096, False, False, ops.EPI_F32_ACCUM),
    ("odd", 1000, 700, 520, True, True, ops.EPI_F32),
    ("odd wg", 700, 520, 1000, False, False, ops.EPI_F32_ACCUM),
    ("odd dg", 1000, 520, 700, True, False, ops.EPI_F32),
]
sel = sys.argv[1:] or None
VARIANTS = os.environ.get("GEMM_VARIANTS", "auto").split(",")
for name, m, n, k, ak, bk, epi in cases:
    if sel and not any(s in name for s in sel):
        continue
    A = torch.randn(m, k, device=dev).bfloat16() if ak else torch.randn(k, m, device=dev).bfloat16()
    B = torch.randn(n, k, device=dev).bfloat16() if bk else torch.randn(k, n, device=dev).bfloat16()
    bf = epi in (ops.EPI_BF16, ops.EPI_BF16_RELU, ops.EPI_BF16_DRELU)
    D = torch.zeros(m, n, device=dev, dtype=torch.bfloat16 if bf else torch.float32)
    bias = torch.zeros(n, device=dev) if epi in (ops.EPI_BF16, ops.EPI_BF16_RELU) else None
    run = lambda: ops.gemm(A, B, D, a_kmajor=ak, b_kmajor=bk, epilogue=epi, bias=bias)
    At = A if ak else A.t()
    Bt = B.t() if bk else B
    Dc = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    runc = lambda: torch.mm(At, Bt, out=Dc)
    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        n_it = 20  # back-to-back launches captured in a CUDA graph: device time, not host issue
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(n_it):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (5 * n_it)
    uc = timeit(runc)
    ref = (At.float() @ Bt.float())
    outk = {ops.EPI_F32: "f32", ops.EPI_F32_ACCUM: "f32+=", ops.EPI_F32_RESID: "f32+res"}.get(epi, "bf16")
    line = f"{name:10s} {m:6d}x{n:6d}x{k:6d} out {outk:6s} cublas {uc:7.2f}us {2*m*n*k/uc/1e6:7.1f}TF |"
    for var in VARIANTS:
        for key in ("MM_GEMM_CG", "MM_GEMM_BN"):
            os.environ.pop(key, None)
        if var != "auto":
            cg, bn = var.split(":")
            os.environ["MM_GEMM_CG"], os.environ["MM_GEMM_BN"] = cg, bn
        try:
            us = timeit(run)
        except Exception as e:  # shapes the kernel rejects (e.g. ld % 8)
            line += f" {var} rejected ({str(e)[-40:]}) |"
            continue
        D.zero_()
        ops.gemm(A, B, D, a_kmajor=ak, b_kmajor=bk, epilogue=epi, bias=bias)
        torch.cuda.synchronize()
        out = D.float()
        if epi == ops.EPI_BF16_RELU:
            r = ref.clamp_min(0)
        else:
            r = ref
        err = ((out - r).abs().max() / r.abs().max()).item() if epi != ops.EPI_BF16_DRELU else 0.0
        ok = "ok" if err < 2e-2 else f"BAD{err:.1e}"
        line += f" {var} {us:7.2f}us {2*m*n*k/us/1e6:7.1f}TF {ok} |"
    for key in ("MM_GEMM_CG", "MM_GEMM_BN"):
        os.environ.pop(key, None)
    print(line, flush=True)

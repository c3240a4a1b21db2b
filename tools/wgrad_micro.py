"""Grouped weight-gradient launches of one config-3 step side (encoder: 6 x 4
problems; decoder: 6 x 7 + generator), timed per forced tile shape."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
T, d, F, V = 4100, 512, 2048, 32000
enc = [(3 * d, d), (d, d), (F, d), (d, F)] * 6
dec = [(3 * d, d), (d, d), (d, d), (2 * d, d), (d, d), (F, d), (d, F)] * 6
sides = {"enc": enc, "dec": dec, "dec+gen": dec + [(V, d)], "gen": [(V, d)]}


def probs(shapes):
    out = []
    for (n_out, n_in) in shapes:
        dy = torch.randn(T, n_out, device=dev).bfloat16()
        x = torch.randn(T, n_in, device=dev).bfloat16()
        out.append(dict(a=dy, b=x, d=torch.zeros(n_out, n_in, device=dev), a_kmajor=False,
                        b_kmajor=False, epilogue=ops.EPI_F32_ACCUM, dbias=torch.zeros(n_out, device=dev)))
    return out


def timeit(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


for name in (sys.argv[1:] or sides):
    ps = probs(sides[name])
    flops = sum(2 * T * p["a"].shape[1] * p["b"].shape[1] for p in ps)
    line = f"{name:8s} {len(ps):3d} probs {flops/1e9:6.1f} GFLOP |"
    for var in ["auto", "1:128", "1:256", "2:128", "2:256"]:
        for k in ("MM_GEMM_CG", "MM_GEMM_BN"):
            os.environ.pop(k, None)
        if var != "auto":
            os.environ["MM_GEMM_CG"], os.environ["MM_GEMM_BN"] = var.split(":")
        us = timeit(lambda: ops.gemm_grouped(ps))
        line += f" {var} {us:7.1f}us {flops/us/1e6:6.0f}TF |"
    print(line, flush=True)

"""LayerNorm forward / backward device time at the config-3 / config-5
shapes: back-to-back launches in a CUDA graph (L2-warm, as inside a step)
and single launches after an L2 flush (cold, as ncu times them).
MM_LN_V1=1 selects the previous kernels (A/B)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import ops
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def warm(fn, n=20):
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


def cold(fn, n=20):
    ts = []
    for _ in range(n):
        ops.flush_l2(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


tag = "v1" if os.environ.get("MM_LN_V1") else "v2"
for rows, cols in [(4096, 512), (4134, 512), (16384, 1024)]:
    x = torch.randn(rows, cols, device=dev); g = torch.rand(cols, device=dev); b = torch.randn(cols, device=dev)
    y = torch.empty(rows, cols, device=dev, dtype=torch.bfloat16)
    mean, rstd = torch.empty(rows, device=dev), torch.empty(rows, device=dev)
    dy = torch.randn(rows, cols, device=dev); dx = torch.zeros(rows, cols, device=dev)
    dxb = torch.empty(rows, cols, device=dev, dtype=torch.bfloat16)
    dg, db = torch.zeros(cols, device=dev), torch.zeros(cols, device=dev)
    fwd = lambda: ops.layernorm_fwd(x, g, b, y, mean, rstd)
    bwd = lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dxb, dg, db)
    fb, bb = rows * cols * (4 + 2), rows * cols * (4 * 4 + 2)
    tfw, tbw, tfc, tbc = warm(fwd), warm(bwd), cold(fwd), cold(bwd)
    print(f"{tag} {rows}x{cols}: fwd warm {tfw:6.2f} us ({fb/tfw/1e3:5.0f} GB/s) cold {tfc:6.2f} us "
          f"({fb/tfc/1e3:5.0f} GB/s) | bwd warm {tbw:6.2f} us ({bb/tbw/1e3:5.0f} GB/s) cold {tbc:6.2f} us "
          f"({bb/tbc/1e3:5.0f} GB/s)", flush=True)

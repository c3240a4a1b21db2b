"""LayerNorm forward / backward device time (CUDA graph of back-to-back
launches) at the config-3 and config-5 shapes."""
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


for rows, cols in [(4096, 512), (16384, 1024)]:
    x = torch.randn(rows, cols, device=dev); g = torch.rand(cols, device=dev); b = torch.randn(cols, device=dev)
    y = torch.empty(rows, cols, device=dev, dtype=torch.bfloat16)
    mean, rstd = torch.empty(rows, device=dev), torch.empty(rows, device=dev)
    dy = torch.randn(rows, cols, device=dev); dx = torch.zeros(rows, cols, device=dev)
    dxb = torch.empty(rows, cols, device=dev, dtype=torch.bfloat16)
    dg, db = torch.zeros(cols, device=dev), torch.zeros(cols, device=dev)
    tf = timeit(lambda: ops.layernorm_fwd(x, g, b, y, mean, rstd))
    tb = timeit(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dxb, dg, db))
    fb, bb = rows * cols * (4 + 2), rows * cols * (4 * 4 + 2)
    print(f"{rows}x{cols}: fwd {tf:6.2f} us ({fb/tf/1e3:5.0f} GB/s)  bwd {tb:6.2f} us ({bb/tb/1e3:5.0f} GB/s)", flush=True)

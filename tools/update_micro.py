"""Fused update (K3) device time on a config-3-sized module set, with and
without lazy gradient zeroing (diagnostics)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07544_b200 import _native, ops
dev = torch.device("cuda:0")
sizes = [16_384_000, 16_384_000, 16_416_000, 25_200_000, 18_900_000]
bufs = []
for n in sizes:
    bufs.append([torch.randn(n, device=dev) * 1e-3, torch.randn(n, device=dev), torch.zeros(n, device=dev),
                 torch.zeros(n, device=dev), torch.empty(n, device=dev, dtype=torch.bfloat16)])
for zg in (0, 1, 0, 1):
    mods = [_native.AdamModule(grad=g.data_ptr(), master=m.data_ptr(), exp_avg=a.data_ptr(), exp_avg_sq=v.data_ptr(),
                               param_bf16=b.data_ptr(), n_elems=g.numel(), n_ready=1, ready_index=-1,
                               step_size=1e-4, inv_sqrt_bc2=1.0) for g, m, a, v, b in bufs]
    hyper = _native.AdamHyper.make(0.9, 0.998, 1e-8, zero_grad=zg)
    for _ in range(3):
        ops.fused_update(mods, hyper)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.fused_update(mods, hyper)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100
    n = sum(sizes)
    print(f"zero_grad={zg}: {us:7.1f} us  {n * (30 + 4 * zg) / us / 1e3:6.0f} GB/s", flush=True)

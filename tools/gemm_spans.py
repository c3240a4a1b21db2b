"""In-step GEMM spans: every GEMM launch of one config-3 (or 4/5) training
step, timed on the device by its own %globaltimer span (mm_gemm_timing /
mm_gemm_spans), with its shape, TFLOP/s and the idle gap before the next
GEMM.  Usage: python tools/gemm_spans.py [config3|config4|config5] [out.json]"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_07544_b200 import _native, configs  # noqa: E402
from paper_2403_07544_b200.data import ZipfIds, make_batch  # noqa: E402
from paper_2403_07544_b200.engine import DeviceBatch, Engine  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "config3"
    dev = torch.device("cuda:0")
    wl = getattr(configs, cfg)(1)
    eng = Engine(wl.tasks, wl.topo, wl.shape, device=dev, seed=0)
    rng = np.random.default_rng([0, 0])
    ids = ZipfIds(wl.shape.vocab, wl.data.zipf_s)
    dbs = [DeviceBatch(make_batch(rng, wl.data, wl.shape.vocab, ids=ids), dev) for _ in range(8)]
    for s in range(6):
        eng.step(s, [dbs[s]])
    eng.sync_updates()
    torch.cuda.synchronize()
    L = _native.lib()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _native.check(L.mm_gemm_timing(1, None, None, None), "timing")
    e0.record()
    eng.step(6, [dbs[6]])
    eng.sync_updates()
    e1.record()
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1)
    f, t, n = ctypes.c_double(), ctypes.c_float(), ctypes.c_int()
    _native.check(L.mm_gemm_timing(0, ctypes.byref(f), ctypes.byref(t), ctypes.byref(n)), "timing")
    N = n.value
    lo = (ctypes.c_ulonglong * N)()
    hi = (ctypes.c_ulonglong * N)()
    fl = (ctypes.c_double * N)()
    sh = (ctypes.c_int * (4 * N))()
    cnt = ctypes.c_int()
    _native.check(L.mm_gemm_spans(N, lo, hi, fl, sh, ctypes.byref(cnt)), "spans")
    rows = []
    t0 = lo[0]
    for i in range(cnt.value):
        us = (hi[i] - lo[i]) / 1e3
        gap = (lo[i + 1] - hi[i]) / 1e3 if i + 1 < cnt.value else 0.0
        rows.append({"i": i, "m": sh[4 * i], "n": sh[4 * i + 1], "k": sh[4 * i + 2], "probs": sh[4 * i + 3],
                     "start_us": (lo[i] - t0) / 1e3, "us": us, "tflops": fl[i] / us / 1e6,
                     "gap_next_us": gap, "gflop": fl[i] / 1e9})
    for r in rows:
        print(f"{r['i']:4d} {r['m']:6d}x{r['n']:6d}x{r['k']:6d} p{r['probs']:2d} @{r['start_us']:8.1f} "
              f"{r['us']:7.2f}us {r['tflops']:7.1f}TF gap {r['gap_next_us']:6.2f}us")
    tot = sum(r["us"] for r in rows)
    print(f"step {step_ms:.3f} ms; GEMM spans {tot / 1e3:.3f} ms over {len(rows)} launches, "
          f"{f.value / 1e12:.3f} TFLOP -> {f.value / (tot * 1e-6) / 1e12:.1f} TF/s; "
          f"gaps between GEMMs {sum(r['gap_next_us'] for r in rows) / 1e3:.3f} ms")
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as fh:
            json.dump({"config": cfg, "step_ms": step_ms, "launches": rows}, fh, indent=0)


if __name__ == "__main__":
    main()

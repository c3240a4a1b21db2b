"""Config 1 at its true shape: per-tensor max-relative error of the engine and
of the independent autocast-bf16 implementation vs the fp32 oracle, for a few
batch sizes (the worst tensors of each)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2403_07544_b200 import configs  # noqa: E402
from paper_2403_07544_b200.data import make_batch  # noqa: E402
from test_parity_shapes_gpu import run_case  # noqa: E402

cuda = torch.device("cuda:0")
wl = configs.config1()
for sentences in [int(x) for x in (sys.argv[1:] or ["64", "256", "1024"])]:
    for seed in (0, 1):
        rng = np.random.default_rng([1, seed])
        batch = make_batch(rng, wl.data, wl.shape.vocab, sentences=sentences)
        rows = run_case(cuda, wl, batch)
        flat = []
        for mod, r in rows.items():
            for t, (e, a) in r["tensors"].items():
                flat.append((e, a, mod, t))
        flat.sort(reverse=True)
        mods = max(r["engine"] for r in rows.values())
        over_alt = sum(1 for e, a, _, _ in flat if e > a)
        print(f"sentences {sentences} seed {seed}: worst module {mods:.4f}; tensors {len(flat)}, "
              f"engine > alt on {over_alt}; worst:", flush=True)
        for e, a, m, t in flat[:5]:
            print(f"   {m:14s} {t:12s} engine {e:.4f} alt {a:.4f}", flush=True)

"""Diagnostics: per-module and per-tensor max-relative gradient errors of one
engine step against the fp32 oracle, the bf16-faithful oracle and an
independent autocast-bf16 implementation (tests/bf16_autocast.py), for the
toy-shape engine tests and the block tests.  Writes gpurun_out/<tag>/diag_parity.json."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import transformer as OT  # noqa: E402
from paper_2403_07544_b200 import configs  # noqa: E402
from paper_2403_07544_b200.data import make_batch  # noqa: E402
from paper_2403_07544_b200.domain import ClusterTopology, DeviceId  # noqa: E402
from paper_2403_07544_b200.plan import embedding_keys  # noqa: E402
from parity_util import effective_weights, error_table  # noqa: E402
from bf16_autocast import local_grads as ac_grads  # noqa: E402


def single_rank(dev, accum, seed=0, sentences=16):
    from paper_2403_07544_b200.engine import DeviceBatch, Engine
    shape = configs.SHAPE_CFG1_GPU
    w = configs.config1(shape)
    tasks = [t.with_device(DeviceId(0, 0)) for t in w.tasks]
    eng = Engine(tasks, ClusterTopology(1, 1, 3), shape, device=dev, seed=0)
    rng = np.random.default_rng([seed, 0])
    hb = [make_batch(rng, w.data, shape.vocab, sentences=sentences) for _ in range(accum)]
    m0 = {k: st.master.cpu().numpy().copy() for k, st in eng.states.items()}
    info = eng.step(0, [DeviceBatch(b, dev) for b in hb])
    torch.cuda.synchronize()
    g_eng = {k: st.grad.cpu().numpy().astype(np.float64) for k, st in eng.states.items()}
    eff = {k: effective_weights(eng.layouts[k], v) for k, v in m0.items()}
    by_id = {t.id: t for t in tasks}
    picked = [by_id[t] for t in info["tasks"]]
    refs = {}
    for name, bf in (("fp32", False), ("bf16_faithful", True)):
        g, used, _ = OT.local_grads(list(zip(picked, hb)), eff, eng.layouts, shape, embedding_keys, bf16=bf)
        refs[name] = {k: (g[k].double().numpy() if k in used else None) for k in g}
    ac = {k: np.zeros(eng.layouts[k].numel) for k in eff}
    for t, b in zip(picked, hb):
        gg, _ = ac_grads(t, b, eff, eng.layouts, shape, embedding_keys, dev)
        for k, v in gg.items():
            if v is not None:
                ac[k] += v.numpy()
    rows = error_table(g_eng, refs["fp32"], eng.layouts, ac)
    rows_bf = error_table(g_eng, refs["bf16_faithful"], eng.layouts)
    for k in rows:
        rows[k]["engine_vs_bf16_faithful"] = rows_bf[k]["engine"]
    return rows


def main():
    dev = torch.device("cuda:0")
    torch.set_num_threads(os.cpu_count() or 1)
    out = {}
    for sentences in (16, 64, 256):
        for accum in (1, 2):
            for seed in (0, 1):
                out[f"s{sentences}_accum{accum}_seed{seed}"] = single_rank(dev, accum, seed, sentences)
    path = os.path.join(ROOT, "gpurun_out", sys.argv[1] if len(sys.argv) > 1 else "diag", "diag_parity.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    for case, rows in out.items():
        for k, r in rows.items():
            worst = max(r["tensors"].items(), key=lambda kv: kv[1][0])
            over = sum(1 for e, a in r["tensors"].values() if e > 2e-2)
            ratio = np.exp(np.mean([np.log(e / a) for e, a in r["tensors"].values() if a and e]))
            print(f"{case:22s} {k:16s} mod {r['engine']:.4f} alt {r['alt']:.4f} "
                  f"vs-bf16f {r['engine_vs_bf16_faithful']:.4f} worst {worst[0]} {worst[1][0]:.4f}/{worst[1][1]:.4f} "
                  f"over2e-2 {over}/{len(r['tensors'])} geo(e/a) {ratio:.2f}")


if __name__ == "__main__":
    main()

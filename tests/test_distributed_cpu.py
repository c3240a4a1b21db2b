"""Config 1 (world_size 2, fp32) on the CPU reference over torch.distributed
gloo: the engine's host-side exchange plan (ready flags, world-summed
counts, exchange_order on per-member-set sub-groups) drives real collectives;
ready counts must equal the reference's (golden) and the reduced gradients
must match the single-process Algorithm-1 oracle within 1e-5 (fp32)."""
import json
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    from oracle import transformer as OT
    from paper_2403_07544_b200 import configs
    from paper_2403_07544_b200.data import make_batch
    from paper_2403_07544_b200.model import init_module, module_layouts
    from paper_2403_07544_b200.plan import (Multiplexer, build_plan, decode_ready, embedding_keys,
                                            exchange_plan, ready_bits, ready_flags, task_modules)
    wl = configs.config1()
    plan = build_plan(wl.tasks, wl.topo)
    layouts = module_layouts(plan, wl.shape)
    masters = {k: init_module(layouts[k], wl.shape) for k in plan.keys}
    subgroups = {m: dist.new_group(list(m)) for m in plan.member_sets()}  # same order on all ranks
    results = []
    for accum in (1, 2):
        mux = Multiplexer(plan, rank, 0)
        for step in range(2):
            rng = np.random.default_rng([step, rank])
            tasks = [mux.pick(step) for _ in range(accum)]
            batches = [make_batch(rng, wl.data, wl.shape.vocab, sentences=16) for _ in range(accum)]
            mine = {k: masters[k] for k in plan.hosted[rank]}
            grads, used, losses = OT.local_grads(list(zip(tasks, batches)), mine, layouts, wl.shape,
                                                 embedding_keys)
            bits = torch.tensor(ready_bits(plan, rank, used), dtype=torch.int32)
            dist.all_reduce(bits)  # K1 on rank bitmasks
            counts, _ = decode_ready(bits.tolist())
            idx = plan.index()
            # K2: the engine's own item list (exchange_plan), sorted ModuleKey order
            for k, members, root in exchange_plan(plan, rank, bits.tolist()):
                g = subgroups[tuple(members)]
                if root >= 0:  # n = 1: the ready member's buffer is the sum
                    dist.broadcast(grads[k], src=members[root], group=g)
                else:
                    dist.all_reduce(grads[k], group=g)
            synced = {str(k): (grads[k] / counts[idx[k]]).numpy()
                      for k in plan.hosted[rank] if counts[idx[k]] >= 1}
            results.append({"accum": accum, "step": step, "counts": counts,
                            "tasks": [t.id for t in tasks], "synced": synced})
    torch.save(results, os.path.join(out_dir, f"rank{rank}.pt"))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_config1_gloo_world2(tmp_path):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    res = [torch.load(tmp_path / f"rank{r}.pt", weights_only=False) for r in range(2)]
    sys.path.insert(0, ROOT)
    from oracle import transformer as OT
    from paper_2403_07544_b200 import configs
    from paper_2403_07544_b200.data import make_batch
    from paper_2403_07544_b200.model import init_module, module_layouts
    from paper_2403_07544_b200.plan import build_plan, embedding_keys
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        gold = json.load(f)["groups_ready"]
    wl = configs.config1()
    plan = build_plan(wl.tasks, wl.topo)
    layouts = module_layouts(plan, wl.shape)
    masters = {k: init_module(layouts[k], wl.shape) for k in plan.keys}
    by_id = {t.id: t for t in wl.tasks}
    for i, (a, b) in enumerate(zip(res[0], res[1])):
        assert a["counts"] == b["counts"]
        ready = {str(k): c for k, c in zip(plan.keys, a["counts"]) if k.position >= 0}
        assert ready == gold[f"config1_accum{a['accum']}"]["ready"][a["step"]]
        # single-process oracle over both ranks
        per_g, per_u = {}, {}
        for r, rec in ((0, a), (1, b)):
            rng = np.random.default_rng([rec["step"], r])
            bs = [make_batch(rng, wl.data, wl.shape.vocab, sentences=16) for _ in rec["tasks"]]
            mine = {k: masters[k] for k in plan.hosted[r]}
            per_g[r], per_u[r], _ = OT.local_grads([(by_id[t], bb) for t, bb in zip(rec["tasks"], bs)],
                                                   mine, layouts, wl.shape, embedding_keys)
        synced, counts = OT.algorithm1(per_g, per_u, plan.groups)
        for r, rec in ((0, a), (1, b)):
            for ks, g in rec["synced"].items():
                ref = synced[next(k for k in plan.keys if str(k) == ks)].numpy()
                err = np.abs(g - ref).max() / max(np.abs(ref).max(), 1e-30)
                assert err <= 1e-5, (i, r, ks, err)

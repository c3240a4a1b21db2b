"""Generate the golden fixtures of tests/golden/ from the reference itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``mmtplan`` read-only from /root/reference/pkg/src, drives it on
the workloads of ``paper_2403_07544_b200.configs`` and on seeded random
instances, and writes small JSON / NPZ files.  The GPU box never runs this;
tests read only the committed outputs.
"""
from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import mmtplan  # noqa: E402
from mmtplan import allocator as R_alloc  # noqa: E402
from mmtplan import core as R_core  # noqa: E402
from mmtplan import sharing as R_sharing  # noqa: E402
from mmtplan import syncsim as R_sim  # noqa: E402
from mmtplan._cost_py import comm_cost_kernel as R_cost_py  # noqa: E402

from paper_2403_07544_b200 import configs  # noqa: E402


def to_ref_task(t, device="keep"):
    """Our TaskSpec -> the reference's TaskSpec (field copy)."""
    key = lambda k: R_core.ModuleKey(R_core.Side(k.side.value), k.position, k.group)
    dev = t.device if device == "keep" else device
    return R_core.TaskSpec(
        id=t.id, src_lang=t.src_lang, tgt_lang=t.tgt_lang, src_path=t.src_path,
        tgt_path=t.tgt_path, enc_modules=tuple(key(k) for k in t.enc_modules),
        dec_modules=tuple(key(k) for k in t.dec_modules), enc_layers=tuple(t.enc_layers),
        dec_layers=tuple(t.dec_layers), weight=t.weight,
        introduce_at_training_step=t.introduce_at_training_step,
        device=None if dev is None else R_core.DeviceId(dev.node, dev.gpu))


def ref_topo(topo):
    return R_core.ClusterTopology(topo.n_nodes, topo.n_gpus_per_node, topo.n_slots_per_gpu)


def spy_run(tasks, topo, steps, seed=0, accum=1):
    """Run the reference run_benchmark, capturing each sync_step's groups and
    ready counts, and return them with the ledger."""
    captured = []
    orig = R_sim.sync_step

    def spy(devices):
        ordered = sorted(devices, key=lambda d: d.index)
        keys = sorted(set().union(*(d.hosted for d in ordered)))
        rec = {}
        for k in keys:
            grp = [d.index for d in ordered if k in d.hosted]
            n = sum(1 for d in ordered if k in d.hosted and k in d.used)
            rec[str(k)] = [grp, n]
        captured.append(rec)
        return orig(devices)

    R_sim.sync_step = spy
    try:
        ledger, summary = R_sim.run_benchmark(tasks, topo, steps=steps, seed=seed, accum_count=accum)
    finally:
        R_sim.sync_step = orig
    groups = {k: v[0] for k, v in captured[0].items()} if captured else {}
    ready = [{k: v[1] for k, v in rec.items()} for rec in captured]
    led = [[r.step, r.ready_bytes, r.grad_bytes, r.tokens] for r in ledger.records]
    return {"groups": groups, "ready": ready, "ledger": led,
            "summary": {k: summary[k] for k in ("modules", "devices", "tasks",
                                                 "grad_allreduce_bytes", "ready_sync_bytes")}}


def gen_groups_ready():
    out = {}
    w1 = configs.config1()
    t1 = [to_ref_task(t) for t in w1.tasks]
    for accum in (1, 2):
        out[f"config1_accum{accum}"] = spy_run(t1, ref_topo(w1.topo), steps=4, accum=accum)
    for world in (2, 4, 8):
        w = configs.config3(world)
        out[f"config3_w{world}"] = spy_run([to_ref_task(t) for t in w.tasks], ref_topo(w.topo),
                                           steps=30)
        w = configs.config5(world)
        out[f"config5_w{world}"] = spy_run([to_ref_task(t) for t in w.tasks], ref_topo(w.topo),
                                           steps=10)
    # config 4: the reference allocator places the tasks, then the same spy
    for world in (2, 8):
        tasks, topo = configs.config4_tasks(world)
        rt = [to_ref_task(t, device=None) for t in tasks]
        rtopo = ref_topo(topo)
        mods = R_sharing.enumerate_modules(rt)
        a0 = R_alloc.initial_assignment(rt, rtopo, seed=0)
        a = R_alloc.local_search(a0, rt, mods, rtopo, budget=2000, seed=0)
        placed = [t.with_device(a.placement[t.id]) for t in rt]
        rec = spy_run(placed, rtopo, steps=5)
        rec["placement"] = {tid: str(d) for tid, d in sorted(a.placement.items())}
        rec["initial"] = {tid: str(d) for tid, d in sorted(a0.placement.items())}
        rec["budget"] = 2000
        out[f"config4_w{world}"] = rec
    return out


def desc_task(t):
    return {"src": t.src_lang, "tgt": t.tgt_lang, "enc": [m.group for m in t.enc_modules],
            "dec": [m.group for m in t.dec_modules], "enc_layers": list(t.enc_layers),
            "dec_layers": list(t.dec_layers), "weight": t.weight,
            "intro": t.introduce_at_training_step}


def mk_ref_task(d, device=None):
    E, D = R_core.Side.ENCODER, R_core.Side.DECODER
    return R_core.TaskSpec(
        id=R_core.task_id(d["src"], d["tgt"]), src_lang=d["src"], tgt_lang=d["tgt"],
        src_path="x", tgt_path="y",
        enc_modules=tuple(R_core.ModuleKey(E, i, g) for i, g in enumerate(d["enc"])),
        dec_modules=tuple(R_core.ModuleKey(D, i, g) for i, g in enumerate(d["dec"])),
        enc_layers=tuple(d["enc_layers"]), dec_layers=tuple(d["dec_layers"]),
        weight=d["weight"], introduce_at_training_step=d["intro"], device=device)


def random_tasks(seed, n_tasks, n_groups=3, p_delay=0.3):
    rng = random.Random(seed)
    out = []
    for i in range(n_tasks):
        out.append({"src": f"s{i:02d}", "tgt": f"t{i:02d}",
                    "enc": [f"e{rng.randrange(n_groups)}", "full"],
                    "dec": [f"d{rng.randrange(n_groups)}"], "enc_layers": [rng.randint(1, 3), 2],
                    "dec_layers": [rng.randint(1, 3)], "weight": rng.randint(1, 3),
                    "intro": 1000 if rng.random() < p_delay else 0})
    return out


def gen_allocator():
    cases = []
    for seed in range(40):
        rng = random.Random(10_000 + seed)
        nodes, gpus, slots = rng.randint(1, 3), rng.randint(1, 4), rng.randint(1, 4)
        n_tasks = rng.randint(1, min(12, nodes * gpus * slots))
        tasks = random_tasks(seed, n_tasks)
        # layer counts must agree per module key: pin them per group name
        for t in tasks:
            t["enc_layers"] = [1 + int(t["enc"][0][1:]), 2]
            t["dec_layers"] = [1 + int(t["dec"][0][1:])]
        rt = [mk_ref_task(t) for t in tasks]
        topo = R_core.ClusterTopology(nodes, gpus, slots)
        case = {"seed": seed, "topo": [nodes, gpus, slots], "tasks": tasks}
        try:
            a0 = R_alloc.initial_assignment(rt, topo, seed=seed)
        except R_alloc.AllocationError as exc:
            case["error"] = str(exc)
            cases.append(case)
            continue
        mods = R_sharing.enumerate_modules(rt, 10)
        budget = [0, 7, 10000][seed % 3]
        a1 = R_alloc.local_search(a0, rt, mods, topo, budget=budget, seed=seed,
                                  w_intra=1.0, w_inter=4.0 + (seed % 2))
        case.update({
            "budget": budget, "w_inter": 4.0 + (seed % 2),
            "initial": {k: str(v) for k, v in sorted(a0.placement.items())},
            "final": {k: str(v) for k, v in sorted(a1.placement.items())},
            "cost_initial": R_alloc.comm_cost(a0, rt, mods, topo).total.hex(),
            "cost_final": R_alloc.comm_cost(a1, rt, mods, topo, 1.0, 4.0 + (seed % 2)).total.hex(),
            "violations": R_alloc.validate_assignment(a1, rt, topo),
        })
        cases.append(case)
    # raw kernel known answers (CSR inputs + float64 outputs, hex)
    kernel = []
    for seed in range(30):
        rng = np.random.default_rng(seed)
        n_mod, n_task = int(rng.integers(1, 30)), int(rng.integers(1, 60))
        n_nodes, per = int(rng.integers(1, 4)), int(rng.integers(1, 8))
        n_dev = n_nodes * per
        params = rng.integers(1, 10**7, size=n_mod).astype(np.float64) * rng.random(n_mod)
        lists = [sorted(rng.choice(n_task, size=int(rng.integers(0, min(n_task, 9) + 1)),
                                   replace=False).tolist()) for _ in range(n_mod)]
        off = np.concatenate([[0], np.cumsum([len(l) for l in lists])]).astype(np.int64)
        idx = np.asarray([i for l in lists for i in l], dtype=np.int64)
        task_dev = rng.integers(0, n_dev, size=n_task).astype(np.int64)
        dev_node = np.asarray([d // per for d in range(n_dev)], dtype=np.int64)
        wi, we = float(rng.random() * 2), float(2 + rng.random() * 3)
        outp = np.zeros(n_mod)
        total = R_cost_py(params, off, idx, task_dev, dev_node, wi, we, outp)
        kernel.append({"params": [p.hex() for p in params], "off": off.tolist(),
                       "idx": idx.tolist(), "task_dev": task_dev.tolist(),
                       "dev_node": dev_node.tolist(), "w_intra": wi.hex(), "w_inter": we.hex(),
                       "total": float(total).hex(), "per_module": [float(x).hex() for x in outp]})
    return {"cases": cases, "kernel": kernel}


def gen_modules():
    SP = R_sharing.SharingPattern
    out = {"sort_order": [], "sequences": [], "inventories": {}}
    E, D = R_core.Side.ENCODER, R_core.Side.DECODER
    keys = [R_core.ModuleKey(E, 1, "a"), R_core.ModuleKey(D, 0, "z"), R_core.ModuleKey(E, -1, "full"),
            R_core.ModuleKey(D, 1, "a"), R_core.ModuleKey(E, 0, "b"), R_core.ModuleKey(E, 0, "a"),
            R_core.ModuleKey(D, 0, "b")]
    out["sort_order"] = [str(k) for k in sorted(keys)]
    groups = {"aa": "g0", "bb": "g0", "cc": "g1", "dd": "g1"}
    archs = {
        "lang": R_sharing.ArchSpec(((SP.LANGUAGE, 6),), ((SP.LANGUAGE, 6),)),
        "partial": R_sharing.ArchSpec(((SP.LANGUAGE, 3), (SP.FULL, 3)), ((SP.TGT_GROUP, 6),)),
        "mixed": R_sharing.ArchSpec(((SP.SRC_GROUP, 2), (SP.GROUP, 1), (SP.TGT_LANGUAGE, 1)),
                                    ((SP.SRC_LANGUAGE, 2), (SP.GROUP, 3))),
    }
    for name, arch in archs.items():
        for src in ("aa", "cc"):
            for tgt in ("bb", "dd"):
                e, d, el, dl = R_sharing.build_module_sequence(arch, src, tgt, groups)
                out["sequences"].append({"arch": name, "src": src, "tgt": tgt,
                                         "enc": [str(k) for k in e], "dec": [str(k) for k in d],
                                         "enc_layers": list(el), "dec_layers": list(dl)})
    for name, w in (("config1", configs.config1()), ("config3", configs.config3(8)),
                    ("config5", configs.config5(8))):
        inv = R_sharing.enumerate_modules([to_ref_task(t) for t in w.tasks])
        out["inventories"][name] = [[str(k), v.n_layers, v.n_params] for k, v in inv.items()]
    tasks, _ = configs.config4_tasks(8)
    inv = R_sharing.enumerate_modules([to_ref_task(t, None) for t in tasks])
    out["inventories"]["config4"] = [[str(k), v.n_layers, v.n_params] for k, v in inv.items()]
    return out


def gen_multiplex():
    cases = []
    for seed in range(12):
        rng = random.Random(seed)
        n = rng.randint(1, 6)
        tasks = [{"src": f"s{i}", "tgt": "zz", "enc": ["x"], "dec": ["y"], "enc_layers": [1],
                  "dec_layers": [1], "weight": rng.randint(1, 5),
                  "intro": rng.choice([0, 0, 3, 10])} for i in range(n)]
        tasks[0]["intro"] = 0
        rt = [mk_ref_task(t) for t in tasks]
        mux = random.Random(f"{seed}:0:mux")
        picks = [R_sim.multiplex(rt, step // 4, mux).id for step in range(200)]
        cases.append({"seed": seed, "tasks": tasks, "picks": picks})
    return cases


def scenario(seed, dtype):
    """Random multi-device buffers / hosted / used sets and the reference's
    sync_step output on them."""
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    E, D = R_core.Side.ENCODER, R_core.Side.DECODER
    n_dev = rng.randint(1, 8)
    pool = sorted({R_core.ModuleKey(E, i, f"g{rng.randrange(3)}") for i in range(3)} |
                  {R_core.ModuleKey(D, 0, f"g{rng.randrange(3)}"), R_core.ModuleKey(E, 0, "full")})
    sizes = {k: int(nrng.integers(1, 200)) for k in pool}
    devs = []
    for i in range(n_dev):
        hosted = frozenset(k for k in pool if rng.random() < 0.6) or frozenset([pool[0]])
        used = {k for k in hosted if rng.random() < 0.6}
        bufs = {k: (nrng.standard_normal(sizes[k]).astype(dtype) if k in used
                    else np.zeros(sizes[k], dtype=dtype)) for k in sorted(hosted)}
        if rng.random() < 0.2 and hosted:  # stale non-zero buffer on an unused module
            k = sorted(hosted)[0]
            if k not in used:
                bufs[k] = nrng.standard_normal(sizes[k]).astype(dtype)
        devs.append(R_sim.DeviceState(i * 2 + rng.randint(0, 1), hosted, 1, bufs, used))
    inputs = [{"index": d.index, "hosted": sorted(str(k) for k in d.hosted),
               "used": sorted(str(k) for k in d.used),
               "buffers": {str(k): b.copy() for k, b in d.buffers.items()}} for d in devs]
    synced = R_sim.sync_step(devs)
    after = [{str(k): b.copy() for k, b in d.buffers.items()} for d in devs]
    return inputs, {str(k): v for k, v in synced.items()}, after


def gen_scenarios(path):
    arrays = {}
    meta = []
    for s in range(40):
        dtype = np.float32 if s % 2 == 0 else np.float64
        inputs, synced, after = scenario(s, dtype)
        m = {"seed": s, "dtype": np.dtype(dtype).name, "devices": []}
        for j, d in enumerate(inputs):
            m["devices"].append({"index": d["index"], "hosted": d["hosted"], "used": d["used"]})
            for k, b in d["buffers"].items():
                arrays[f"s{s}_in_{j}_{k}"] = b
                arrays[f"s{s}_after_{j}_{k}"] = after[j][k]
        for k, v in synced.items():
            arrays[f"s{s}_synced_{k}"] = v
        meta.append(m)
    np.savez_compressed(path, **arrays)
    return meta


def gen_reduce_small(path):
    """Config-2 generator scaled to 1e2..6.4e3 params, fp32, through the
    reference sync_step over 8 DeviceStates (bit-exact target)."""
    rng, mods = configs.reduce_microbench(lo=100.0, hi=6400.0)
    E = R_core.Side.ENCODER
    keys = [R_core.ModuleKey(E, i, f"m{i:02d}") for i in range(len(mods))]
    grads = {}
    for r in range(8):
        for i, m in enumerate(mods):
            if r in m.ranks:
                ready = bool(m.ready[r - m.start])
                grads[(r, i)] = (rng.standard_normal(m.n_params, dtype=np.float32) if ready
                                 else np.zeros(m.n_params, dtype=np.float32))
    devs = []
    for r in range(8):
        hosted = frozenset(keys[i] for i, m in enumerate(mods) if r in m.ranks)
        used = {keys[i] for i, m in enumerate(mods) if r in m.ranks and m.ready[r - m.start]}
        bufs = {keys[i]: grads[(r, i)].copy() for i, m in enumerate(mods) if r in m.ranks}
        devs.append(R_sim.DeviceState(r, hosted, 1, bufs, used))
    synced = R_sim.sync_step(devs)
    arrays = {f"grad_{r}_{i}": g for (r, i), g in grads.items()}
    arrays.update({f"synced_{i}": synced[keys[i]] for i in range(len(mods))})
    np.savez_compressed(path, **arrays)
    return [{"n_params": m.n_params, "start": m.start, "group": m.group,
             "ready": m.ready.tolist()} for m in mods]


def main():
    out = {"reference_version": mmtplan.__version__}
    out["groups_ready"] = gen_groups_ready()
    out["allocator"] = gen_allocator()
    out["modules"] = gen_modules()
    out["multiplex"] = gen_multiplex()
    out["scenarios"] = gen_scenarios(os.path.join(HERE, "sync_scenarios.npz"))
    out["reduce_small"] = gen_reduce_small(os.path.join(HERE, "reduce_small.npz"))
    w2 = configs.reduce_microbench()[1]
    out["config2"] = {"sizes": [m.n_params for m in w2], "groups": [m.group for m in w2],
                      "n_ready": [m.n_ready for m in w2]}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()

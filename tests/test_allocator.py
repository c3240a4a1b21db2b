"""Task->device allocation: bit-exact with the reference on golden instances
(placements and float64 costs), plus the reference's own known answers
(allocator tests of the reference, test_allocator.py:67-253)."""
import itertools
import json
import os

import pytest

from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.allocator import (AllocationError, Assignment, comm_cost,
                                             initial_assignment, local_search,
                                             validate_assignment)
from paper_2403_07544_b200.domain import ClusterTopology, DeviceId, ModuleKey, Side, TaskSpec, task_id
from paper_2403_07544_b200.sharing import enumerate_modules

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


def mk(d, device=None):
    return TaskSpec(
        id=task_id(d["src"], d["tgt"]), src_lang=d["src"], tgt_lang=d["tgt"], src_path="x",
        tgt_path="y",
        enc_modules=tuple(ModuleKey(Side.ENCODER, i, g) for i, g in enumerate(d["enc"])),
        dec_modules=tuple(ModuleKey(Side.DECODER, i, g) for i, g in enumerate(d["dec"])),
        enc_layers=tuple(d["enc_layers"]), dec_layers=tuple(d["dec_layers"]),
        weight=d["weight"], introduce_at_training_step=d["intro"], device=device)


def task(src, tgt, enc, dec, intro=0):
    return mk({"src": src, "tgt": tgt, "enc": enc, "dec": dec, "enc_layers": [1] * len(enc),
               "dec_layers": [1] * len(dec), "weight": 1, "intro": intro})


def test_golden_placements_and_costs(golden):
    n_ok = n_err = 0
    for c in golden["allocator"]["cases"]:
        tasks = [mk(d) for d in c["tasks"]]
        topo = ClusterTopology(*c["topo"])
        if "error" in c:
            with pytest.raises(AllocationError):
                initial_assignment(tasks, topo, seed=c["seed"])
            n_err += 1
            continue
        a0 = initial_assignment(tasks, topo, seed=c["seed"])
        assert {k: str(v) for k, v in a0.placement.items()} == c["initial"]
        mods = enumerate_modules(tasks, 10)
        a1 = local_search(a0, tasks, mods, topo, budget=c["budget"], seed=c["seed"],
                          w_intra=1.0, w_inter=c["w_inter"])
        assert {k: str(v) for k, v in a1.placement.items()} == c["final"]
        assert comm_cost(a0, tasks, mods, topo).total.hex() == c["cost_initial"]
        assert comm_cost(a1, tasks, mods, topo, 1.0, c["w_inter"]).total.hex() == c["cost_final"]
        assert validate_assignment(a1, tasks, topo) == c["violations"]
        n_ok += 1
    assert n_ok >= 20


@pytest.mark.parametrize("world", [2, 8])
def test_config4_placement_matches_reference(golden, world):
    rec = golden["groups_ready"][f"config4_w{world}"]
    tasks, topo = configs.config4_tasks(world)
    a0 = initial_assignment(tasks, topo, seed=0)
    assert {k: str(v) for k, v in sorted(a0.placement.items())} == rec["initial"]
    a = local_search(a0, tasks, enumerate_modules(tasks), topo, budget=rec["budget"], seed=0)
    assert {k: str(v) for k, v in sorted(a.placement.items())} == rec["placement"]


def test_known_answers():
    topo = ClusterTopology(1, 2, 1)
    t1, t2 = task("aa", "bb", ["full"], ["d1"]), task("bb", "aa", ["full"], ["d2"])
    a = Assignment({t1.id: DeviceId(0, 0), t2.id: DeviceId(0, 1)})
    mods = {k: 100 for k in enumerate_modules([t1, t2])}
    cost = comm_cost(a, [t1, t2], mods, topo)
    assert cost.total == 100.0
    assert cost.per_module[ModuleKey(Side.ENCODER, 0, "full")] == 100.0
    topo2 = ClusterTopology(2, 1, 1)
    a2 = Assignment({t1.id: DeviceId(0, 0), t2.id: DeviceId(1, 0)})
    assert comm_cost(a2, [t1, t2], mods, topo2).total == 400.0


def test_budget_zero_is_identity_and_never_worse():
    topo = ClusterTopology(2, 2, 2)
    tasks = [task(f"s{i}", f"t{i}", [f"e{i % 3}", "full"], [f"d{i % 2}"]) for i in range(6)]
    mods = enumerate_modules(tasks, 10)
    a0 = initial_assignment(tasks, topo)
    assert local_search(a0, tasks, mods, topo, budget=0).placement == a0.placement
    a1 = local_search(a0, tasks, mods, topo)
    assert comm_cost(a1, tasks, mods, topo).total <= comm_cost(a0, tasks, mods, topo).total
    assert validate_assignment(a1, tasks, topo) == []


def test_local_search_reaches_exhaustive_optimum():
    topo = ClusterTopology(1, 2, 3)
    tasks = [task(f"s{i}", f"t{i}", [f"e{i % 2}", "full"], [f"d{(i // 2) % 2}"]) for i in range(5)]
    mods = enumerate_modules(tasks, 10)
    best = float("inf")
    for combo in itertools.product(topo.devices(), repeat=len(tasks)):
        a = Assignment({t.id: d for t, d in zip(tasks, combo)})
        if validate_assignment(a, tasks, topo):
            continue
        best = min(best, comm_cost(a, tasks, mods, topo).total)
    res = local_search(initial_assignment(tasks, topo), tasks, mods, topo)
    assert comm_cost(res, tasks, mods, topo).total == pytest.approx(best)


def test_capacity_and_cover_errors():
    with pytest.raises(AllocationError):
        initial_assignment([task(f"s{i}", "zz", ["full"], ["full"]) for i in range(5)],
                           ClusterTopology(1, 4, 1))
    with pytest.raises(AllocationError):
        initial_assignment([task("aa", "zz", ["full"], ["full"]),
                            task("bb", "zz", ["full"], ["full"], intro=5000)],
                           ClusterTopology(1, 2, 1))
    tasks = [task("aa", "zz", ["x"], ["x"]), task("bb", "zz", ["x"], ["x"]),
             task("cc", "zz", ["y"], ["y"], intro=5000), task("dd", "zz", ["y"], ["y"], intro=5000)]
    topo = ClusterTopology(1, 2, 2)
    assert validate_assignment(initial_assignment(tasks, topo), tasks, topo) == []


@pytest.mark.parametrize("window,threads", [(1, 1), (7, 2), (256, 0)])
def test_batched_local_search_matches_reference_golden(golden, window, threads):
    """f3: the batched move evaluation (mm_comm_cost_moves on host threads)
    reproduces the reference's local_search results on every golden case."""
    from paper_2403_07544_b200.allocator import local_search_batched
    n = 0
    for c in golden["allocator"]["cases"]:
        if "error" in c:
            continue
        tasks = [mk(d) for d in c["tasks"]]
        topo = ClusterTopology(*c["topo"])
        a0 = initial_assignment(tasks, topo, seed=c["seed"])
        a1 = local_search_batched(a0, tasks, enumerate_modules(tasks, 10), topo,
                                  budget=c["budget"], seed=c["seed"], w_intra=1.0,
                                  w_inter=c["w_inter"], window=window, threads=threads)
        assert {k: str(v) for k, v in a1.placement.items()} == c["final"]
        n += 1
    assert n >= 20


@pytest.mark.parametrize("world", [2, 8])
def test_batched_local_search_config4(golden, world):
    from paper_2403_07544_b200.allocator import local_search_batched
    rec = golden["groups_ready"][f"config4_w{world}"]
    tasks, topo = configs.config4_tasks(world)
    a0 = initial_assignment(tasks, topo, seed=0)
    a = local_search_batched(a0, tasks, enumerate_modules(tasks), topo, budget=rec["budget"], seed=0)
    assert {k: str(v) for k, v in sorted(a.placement.items())} == rec["placement"]


def test_comm_cost_moves_equals_single_costs():
    import numpy as np
    from paper_2403_07544_b200.allocator import CostContext, comm_cost_moves
    tasks, topo = configs.config4_tasks(8)
    ctx = CostContext(tasks, enumerate_modules(tasks), topo)
    rng = np.random.default_rng(0)
    dev = rng.integers(0, topo.n_devices, len(ctx.tasks))
    moves = [(0, int(rng.integers(len(dev))), int(rng.integers(topo.n_devices))) for _ in range(50)]
    moves += [(1, int(a), int(b)) for a, b in rng.integers(0, len(dev), (50, 2))]
    got = comm_cost_moves(ctx, dev, np.asarray(moves), threads=3)
    for (k, x, y), c in zip(moves, got):
        d = dev.copy()
        if k == 0:
            d[x] = y
        else:
            d[x], d[y] = d[y], d[x]
        assert c.hex() == ctx.cost(d).hex()

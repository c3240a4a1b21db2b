"""Module identity, groups, multiplexer and ready counts: bit-exact with the
reference (golden fixtures captured from mmtplan.syncsim.run_benchmark), for
the engine's host logic AND for the oracle restatement (which pins it)."""
import json
import os
import random

import pytest

from oracle import algorithm1 as A1
from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.allocator import initial_assignment, local_search
from paper_2403_07544_b200.domain import DeviceId, ModuleKey, Side, TaskSpec, task_id, validate_config
from paper_2403_07544_b200.plan import (Multiplexer, build_plan, multiplex, ready_counts_all,
                                        ready_flags, task_modules)
from paper_2403_07544_b200.sharing import (ArchSpec, SharingPattern, build_module_sequence,
                                           enumerate_modules)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


def workloads():
    yield "config1_accum1", configs.config1(), 1, 4
    yield "config1_accum2", configs.config1(), 2, 4
    for w in (2, 4, 8):
        yield f"config3_w{w}", configs.config3(w), 1, 30
        yield f"config5_w{w}", configs.config5(w), 1, 10


def engine_ready(plan, steps, accum, seed=0):
    """The engine's own per-step path: per-rank Multiplexer + ready flags +
    world sum (what K1's allreduce returns)."""
    muxes = {r: Multiplexer(plan, r, seed) for r in plan.ranks}
    out = []
    for step in range(steps):
        used = {}
        for r in plan.ranks:
            u = set()
            for _ in range(accum):
                u.update(task_modules(muxes[r].pick(step)))
            used[r] = u
        counts = ready_counts_all(plan, used)
        out.append({str(k): c for k, c in zip(plan.keys, counts) if k.position >= 0})
    return out


@pytest.mark.parametrize("name,wl,accum,steps", list(workloads()))
def test_groups_and_ready_counts_bit_exact(golden, name, wl, accum, steps):
    gold = golden["groups_ready"][name]
    plan = build_plan(wl.tasks, wl.topo)
    assert {str(k): g for k, g in plan.groups.items() if k.position >= 0} == gold["groups"]
    assert engine_ready(plan, steps, accum) == gold["ready"]
    # the oracle restatement agrees too
    assert {str(k): g for k, g in A1.group_map(wl.tasks, wl.topo.n_gpus_per_node).items()} == gold["groups"]
    ready, _ = A1.ready_counts(wl.tasks, wl.topo.n_gpus_per_node, steps, 0, accum)
    assert [{str(k): v for k, v in r.items()} for r in ready] == gold["ready"]


@pytest.mark.parametrize("world", [2, 8])
def test_config4_groups_and_ready(golden, world):
    gold = golden["groups_ready"][f"config4_w{world}"]
    tasks, topo = configs.config4_tasks(world)
    a = local_search(initial_assignment(tasks, topo, 0), tasks, enumerate_modules(tasks), topo,
                     budget=gold["budget"], seed=0)
    placed = [t.with_device(a.placement[t.id]) for t in tasks]
    plan = build_plan(placed, topo)
    assert {str(k): g for k, g in plan.groups.items() if k.position >= 0} == gold["groups"]
    assert engine_ready(plan, 5, 1) == gold["ready"]


def test_config1_appendix_b_values():
    """step-0 ready counts of config 1."""
    plan = build_plan(configs.config1().tasks, configs.config1().topo)
    r = engine_ready(plan, 4, 1)
    assert r[0] == {"decoder:0:b": 0, "decoder:0:c": 2, "encoder:0:a": 1, "encoder:0:b": 1}
    assert r[1] == {"decoder:0:b": 1, "decoder:0:c": 1, "encoder:0:a": 2, "encoder:0:b": 0}


def test_config5_group_sizes():
    from collections import Counter
    assert Counter(len(g) for k, g in build_plan(configs.config5(8).tasks, configs.config5(8).topo)
                   .groups.items() if k.position >= 0) == {1: 19, 2: 23, 3: 12, 4: 5}


def test_config2_generator_matches_survey():
    _, mods = configs.reduce_microbench()
    assert [m.group for m in mods] == [4, 8, 8, 4, 8, 2, 4, 2, 8, 8, 8, 2, 2, 8, 2, 8, 2, 4, 2, 8, 2, 4, 2, 8]
    assert [m.n_ready for m in mods] == [2, 5, 8, 3, 6, 2, 2, 2, 7, 5, 5, 2, 1, 2, 1, 7, 1, 3, 1, 6, 2, 2, 2, 6]
    assert round(sum(m.n_params for m in mods) / 1e6, 1) == 431.9


def test_multiplexer_golden(golden):
    for case in golden["multiplex"]:
        tasks = [TaskSpec(id=task_id(d["src"], d["tgt"]), src_lang=d["src"], tgt_lang=d["tgt"],
                          src_path="x", tgt_path="y",
                          enc_modules=(ModuleKey(Side.ENCODER, 0, "x"),),
                          dec_modules=(ModuleKey(Side.DECODER, 0, "y"),), enc_layers=(1,),
                          dec_layers=(1,), weight=d["weight"],
                          introduce_at_training_step=d["intro"]) for d in case["tasks"]]
        mux = random.Random(f"{case['seed']}:0:mux")
        assert [multiplex(tasks, s // 4, mux).id for s in range(200)] == case["picks"]
        mux = random.Random(f"{case['seed']}:0:mux")
        assert [A1.multiplex(tasks, s // 4, mux).id for s in range(200)] == case["picks"]


def test_module_identity_golden(golden):
    m = golden["modules"]
    keys = [ModuleKey.parse(s) for s in m["sort_order"]]
    assert [str(k) for k in sorted(reversed(keys))] == m["sort_order"]
    SP = SharingPattern
    groups = {"aa": "g0", "bb": "g0", "cc": "g1", "dd": "g1"}
    archs = {"lang": ArchSpec(((SP.LANGUAGE, 6),), ((SP.LANGUAGE, 6),)),
             "partial": ArchSpec(((SP.LANGUAGE, 3), (SP.FULL, 3)), ((SP.TGT_GROUP, 6),)),
             "mixed": ArchSpec(((SP.SRC_GROUP, 2), (SP.GROUP, 1), (SP.TGT_LANGUAGE, 1)),
                               ((SP.SRC_LANGUAGE, 2), (SP.GROUP, 3)))}
    for seq in m["sequences"]:
        e, d, el, dl = build_module_sequence(archs[seq["arch"]], seq["src"], seq["tgt"], groups)
        assert [str(k) for k in e] == seq["enc"] and [str(k) for k in d] == seq["dec"]
        assert list(el) == seq["enc_layers"] and list(dl) == seq["dec_layers"]
    for name, wl in (("config1", configs.config1()), ("config3", configs.config3(8)),
                     ("config5", configs.config5(8))):
        inv = enumerate_modules(wl.tasks)
        assert [[str(k), v.n_layers, v.n_params] for k, v in inv.items()] == m["inventories"][name]
    tasks, _ = configs.config4_tasks(8)
    inv = enumerate_modules(tasks)
    assert [[str(k), v.n_layers, v.n_params] for k, v in inv.items()] == m["inventories"]["config4"]


def test_ready_flags_and_member_sets():
    wl = configs.config1()
    plan = build_plan(wl.tasks, wl.topo)
    t_ab = next(t for t in wl.tasks if t.id == "train_a-b")
    flags = ready_flags(plan, 0, task_modules(t_ab))
    assert sum(flags) == 4  # enc a, dec b, their two embedding modules
    assert plan.member_sets() == [(0, 1)]
    # non-hosted modules never count
    assert ready_flags(plan, 1, task_modules(t_ab)) == [
        1 if (k in task_modules(t_ab) and k in plan.hosted[1]) else 0 for k in plan.keys]


def test_validate_config_and_unplaced():
    wl = configs.config3(8)
    assert validate_config(wl.tasks, wl.topo) == []
    bad = [t.with_device(DeviceId(0, 9)) for t in wl.tasks[:1]]
    assert validate_config(bad, wl.topo)
    from paper_2403_07544_b200.plan import SimulationError
    unplaced = TaskSpec(**{**wl.tasks[0].__dict__, "device": None})
    with pytest.raises(SimulationError):
        build_plan([unplaced], wl.topo)


def test_ready_bitmask_decode():
    """K1 on rank bitmasks: the world sum decodes to the ready counts the
    flag sum gives, and names the single ready rank for n = 1 modules."""
    import random
    from paper_2403_07544_b200.plan import decode_ready
    rng = random.Random(3)
    for _ in range(200):
        world = rng.randint(1, 8)
        ready = [[rng.random() < 0.5 for _ in range(world)] for _ in range(12)]
        bits = [sum(1 << r for r in range(world) if row[r]) for row in ready]
        counts, roots = decode_ready(bits)
        assert counts == [sum(row) for row in ready]
        for row, c, r in zip(ready, counts, roots):
            assert (r == row.index(True)) if c == 1 else (r == -1)


def test_peer_plan_shards_tile_every_module_once():
    """Option B: from the same world-summed ready bits every member derives
    its own shard of each shared module with n >= 1; over the members the
    shards tile the module exactly once and all carry the same group mask."""
    import random
    from paper_2403_07544_b200 import configs
    from paper_2403_07544_b200.plan import (Multiplexer, build_plan, member_mask, peer_plan,
                                            ready_bits, shard_begin, task_modules)
    w = configs.config5(world=8)  # sparse groups: sizes 1..4, many singletons
    plan = build_plan(w.tasks, w.topo)
    for step in range(3):
        used = {}
        for r in range(8):
            mux = Multiplexer(plan, r, 0)
            used[r] = set(task_modules(mux.pick(step)))
        bits = [0] * len(plan.keys)
        for r in range(8):
            bits = [a + b for a, b in zip(bits, ready_bits(plan, r, used[r]))]
        seen = {}
        for r in range(8):
            for k, members, j, mask in peer_plan(plan, r, bits):
                assert members[j] == r and mask == member_mask(bits[plan.index()[k]], members)
                seen.setdefault(k, []).append((j, mask))
        n = 1000
        for k, lst in seen.items():
            g = len(plan.groups[k])
            assert sorted(j for j, _ in lst) == list(range(g))
            assert len({m for _, m in lst}) == 1
            cover = sum(shard_begin(n, g, j + 1) - shard_begin(n, g, j) for j, _ in lst)
            assert cover == n
        for k in plan.keys:  # every shared module with a ready member is covered
            i = plan.index()[k]
            if len(plan.groups[k]) >= 2 and member_mask(bits[i], plan.groups[k]):
                assert k in seen


def test_exchange_plan_is_consistent_across_members():
    """Every member of a group derives the same K2 item (same key order, same
    broadcast root) from the same world-summed bits: the precondition for
    NCCL collectives on overlapping sub-communicators not to cross."""
    from paper_2403_07544_b200 import configs
    from paper_2403_07544_b200.plan import (Multiplexer, build_plan, decode_ready, exchange_plan,
                                            ready_bits, task_modules)
    w = configs.config5(world=8)
    plan = build_plan(w.tasks, w.topo)
    for step in range(4):
        used = {r: set(task_modules(Multiplexer(plan, r, 0).pick(step))) for r in range(8)}
        bits = [0] * len(plan.keys)
        for r in range(8):
            bits = [a + b for a, b in zip(bits, ready_bits(plan, r, used[r]))]
        counts, roots = decode_ready(bits)
        per_rank = {r: exchange_plan(plan, r, bits) for r in range(8)}
        for k in plan.keys:
            seen = {(tuple(members), root) for r in range(8) for kk, members, root in per_rank[r] if kk == k}
            assert len(seen) <= 1, str(k)
            if seen:
                members, root = seen.pop()
                assert (root >= 0) == (counts[plan.index()[k]] == 1)
                if root >= 0:
                    assert members[root] == roots[plan.index()[k]] and members[root] in members
        for r in range(8):  # each rank's list is in sorted key order
            keys = [k for k, _, _ in per_rank[r]]
            assert keys == sorted(keys)

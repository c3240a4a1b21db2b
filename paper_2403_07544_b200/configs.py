"""The five workloads of BASELINE.json, expressed through the drop-in API.

Placement and task sets follow SURVEY.md §8(d); the choices BASELINE.json
leaves open are fixed here once and used identically by the engine, the CPU
oracle and the golden-fixture generator:

* config 1: languages a, b, c; tasks a->b and b->c on rank 0, a->c on rank 1;
  ``ClusterTopology(1, 2, 2)``; LANGUAGE(2) / LANGUAGE(2).
* config 2: the module-gradient microbench generator (``reduce_microbench``).
* config 3: 8 languages, all 56 directions, LANGUAGE(6) / LANGUAGE(6),
  round-robin placement of the id-sorted tasks (task i -> rank i mod W).
* config 4: 16 languages, all 240 directions, encoder LANGUAGE(3)+FULL(3),
  decoder TGT_GROUP(6) over 4 groups of 4 sorted languages, placed by the
  reference allocator (initial_assignment + local_search, seed 0).
* config 5: 32 languages, ``random.Random(0).sample`` of 8*W directions, GPU
  i hosts sample[8i:8i+8], LANGUAGE(6) / LANGUAGE(6), transformer-big.
"""
from __future__ import annotations

import dataclasses
import itertools
import math
import random
from typing import Optional

import numpy as np

from .domain import ClusterTopology, DeviceId, TaskSpec, task_id
from .sharing import ArchSpec, SharingPattern, build_module_sequence

SP = SharingPattern


@dataclasses.dataclass(frozen=True)
class ModelShape:
    d_model: int
    heads: int
    ffn: int
    vocab: int
    max_len: int  # length clip of the synthetic data

    @property
    def head_dim(self) -> int:
        return self.d_model // self.heads


SHAPE_TINY = ModelShape(64, 4, 256, 1000, 32)       # config 1 (head_dim 16: oracle only)
SHAPE_CFG1_GPU = ModelShape(128, 2, 256, 1000, 32)  # config-1 structure at head_dim 64
SHAPE_BASE = ModelShape(512, 8, 2048, 32000, 128)
SHAPE_BIG = ModelShape(1024, 16, 4096, 32000, 256)


@dataclasses.dataclass(frozen=True)
class DataSpec:
    tokens_per_gpu: int
    len_mu: float
    len_sigma: float
    len_min: int
    len_max: int
    zipf_s: float  # 0 -> uniform ids


@dataclasses.dataclass
class Workload:
    name: str
    tasks: list[TaskSpec]
    topo: ClusterTopology
    shape: ModelShape
    data: DataSpec
    world: int


def _task(arch: ArchSpec, src: str, tgt: str, device: Optional[DeviceId],
          groups=None) -> TaskSpec:
    enc, dec, el, dl = build_module_sequence(arch, src, tgt, groups)
    return TaskSpec(id=task_id(src, tgt), src_lang=src, tgt_lang=tgt,
                    src_path=f"synthetic/{src}-{tgt}.{src}", tgt_path=f"synthetic/{src}-{tgt}.{tgt}",
                    enc_modules=enc, dec_modules=dec, enc_layers=el, dec_layers=dl, device=device)


def languages(n: int) -> list[str]:
    return [f"l{i:02d}" for i in range(n)]


def config1(shape: ModelShape = SHAPE_TINY) -> Workload:
    arch = ArchSpec(((SP.LANGUAGE, 2),), ((SP.LANGUAGE, 2),))
    tasks = [_task(arch, "a", "b", DeviceId(0, 0)), _task(arch, "b", "c", DeviceId(0, 0)),
             _task(arch, "a", "c", DeviceId(0, 1))]
    return Workload("config1", tasks, ClusterTopology(1, 2, 2), shape,
                    DataSpec(0, 0, 0, 8, 32, 0.0), 2)


def config3(world: int = 8) -> Workload:
    arch = ArchSpec(((SP.LANGUAGE, 6),), ((SP.LANGUAGE, 6),))
    langs = languages(8)
    dirs = sorted(task_id(s, t) for s, t in itertools.permutations(langs, 2))
    pairs = {task_id(s, t): (s, t) for s, t in itertools.permutations(langs, 2)}
    tasks = [_task(arch, *pairs[tid], DeviceId(0, i % world)) for i, tid in enumerate(dirs)]
    topo = ClusterTopology(1, world, math.ceil(len(tasks) / world))
    return Workload("config3", tasks, topo, SHAPE_BASE,
                    DataSpec(4096, 3.0, 0.5, 4, 128, 1.1), world)


def config4_tasks(world: int = 8) -> tuple[list[TaskSpec], ClusterTopology]:
    """Unplaced config-4 tasks and topology (placement comes from the allocator)."""
    langs = languages(16)
    groups = {l: f"group{i // 4}" for i, l in enumerate(sorted(langs))}
    arch = ArchSpec(((SP.LANGUAGE, 3), (SP.FULL, 3)), ((SP.TGT_GROUP, 6),))
    tasks = [_task(arch, s, t, None, groups) for s, t in itertools.permutations(langs, 2)]
    topo = ClusterTopology(1, world, math.ceil(len(tasks) / world))
    return tasks, topo


def config4(world: int = 8, budget: int = 10000) -> Workload:
    from .allocator import initial_assignment, local_search_batched
    from .sharing import enumerate_modules
    tasks, topo = config4_tasks(world)
    a0 = initial_assignment(tasks, topo, seed=0)
    # batched evaluation: the same placement as local_search (f3), ~5x faster
    a = local_search_batched(a0, tasks, enumerate_modules(tasks), topo, budget=budget, seed=0)
    placed = [t.with_device(a.placement[t.id]) for t in tasks]
    return Workload("config4", placed, topo, SHAPE_BASE,
                    DataSpec(8192, 3.0, 0.5, 4, 128, 1.1), world)


def config5(world: int = 8, per_gpu: int = 8, seed: int = 0) -> Workload:
    arch = ArchSpec(((SP.LANGUAGE, 6),), ((SP.LANGUAGE, 6),))
    langs = languages(32)
    dirs = sorted(itertools.permutations(langs, 2), key=lambda p: task_id(*p))
    pick = random.Random(seed).sample(dirs, per_gpu * world)
    tasks = [_task(arch, s, t, DeviceId(0, i // per_gpu)) for i, (s, t) in enumerate(pick)]
    return Workload("config5", tasks, ClusterTopology(1, world, per_gpu), SHAPE_BIG,
                    DataSpec(16384, 3.2, 0.6, 4, 256, 1.1), world)


# ----------------------------------------------------------------------------
# config 2: module-gradient reduction microbench (SURVEY §8(d) generator)


@dataclasses.dataclass
class ReduceModule:
    n_params: int
    start: int
    group: int
    ready: np.ndarray  # bool[group]

    @property
    def ranks(self) -> list[int]:
        return list(range(self.start, self.start + self.group))

    @property
    def n_ready(self) -> int:
        return int(self.ready.sum())


def reduce_microbench(n_modules: int = 24, world: int = 8, seed: int = 0,
                      lo: float = 1e6, hi: float = 64e6) -> tuple[np.random.Generator, list[ReduceModule]]:
    """Module sizes, contiguous groups of 2/4/8 ranks, Bernoulli(0.75) ready
    flags with at least one ready rank.  Returns the generator positioned for
    the gradient draws (rank ascending, module ascending)."""
    rng = np.random.default_rng(seed)
    mods = []
    for _ in range(n_modules):
        p = int(round(float(np.exp(rng.uniform(np.log(lo), np.log(hi))))))
        g = int(rng.choice([2, 4, 8]))
        g = min(g, world)
        start = int(rng.integers(0, world - g + 1))
        while True:
            ready = rng.random(g) < 0.75
            if ready.any():
                break
        mods.append(ReduceModule(p, start, g, ready))
    return rng, mods

"""Static module/process-group plan and per-step readiness.

Replaces ``run_benchmark``'s setup (``syncsim.py:313-343``) with the engine's
version: one entry per rank (torchrun rank == ``ClusterTopology.flat``), the
hosted module set per rank, each module's group (hosting ranks ascending),
the distinct member sets that need a communicator, and the multiplexer RNG
seeding ``random.Random(f"{seed}:{rank}:mux")`` so ready flags are bit-exact
with the reference.

Besides the reference's stack modules the engine owns one embedding module
per language and side, keyed ``ModuleKey(side, -1, lang)`` (the position -1
convention of ``sharing.embedding_modules``, sharing.py:141-152, made
language-specific): the encoder one holds the source embedding table, the
decoder one the target embedding table and the generator.
"""
from __future__ import annotations

import dataclasses
import random
from typing import Iterable, Sequence

from .domain import ClusterTopology, ModuleKey, Side, TaskSpec


class SimulationError(RuntimeError):
    """Same role as the reference's ``syncsim.SimulationError`` (syncsim.py:30)."""


def embedding_keys(task: TaskSpec) -> tuple[ModuleKey, ModuleKey]:
    return ModuleKey(Side.ENCODER, -1, task.src_lang), ModuleKey(Side.DECODER, -1, task.tgt_lang)


def task_modules(task: TaskSpec, with_embeddings: bool = True) -> tuple[ModuleKey, ...]:
    mods = task.modules()
    return mods + embedding_keys(task) if with_embeddings else mods


@dataclasses.dataclass
class ModulePlan:
    tasks: list[TaskSpec]                      # sorted by id
    topo: ClusterTopology
    ranks: list[int]                           # ranks hosting >= 1 task, ascending
    tasks_by_rank: dict[int, list[TaskSpec]]
    hosted: dict[int, frozenset]               # rank -> hosted keys (incl. embeddings)
    keys: list[ModuleKey]                      # every module, sorted = collective order
    groups: dict[ModuleKey, list[int]]         # key -> hosting ranks ascending
    with_embeddings: bool

    @property
    def stack_keys(self) -> list[ModuleKey]:
        return [k for k in self.keys if k.position >= 0]

    def member_sets(self) -> list[tuple[int, ...]]:
        """Distinct groups with >= 2 ranks, in first-use order over sorted keys
        (the order communicators are split in, identical on every rank)."""
        seen: dict[tuple[int, ...], None] = {}
        for k in self.keys:
            g = tuple(self.groups[k])
            if len(g) >= 2:
                seen.setdefault(g, None)
        return list(seen)

    def index(self) -> dict[ModuleKey, int]:
        return {k: i for i, k in enumerate(self.keys)}


def build_plan(tasks: Iterable[TaskSpec], topo: ClusterTopology,
               with_embeddings: bool = True) -> ModulePlan:
    tasks = sorted(tasks, key=lambda t: t.id)
    by_rank: dict[int, list[TaskSpec]] = {}
    for t in tasks:
        if t.device is None:
            raise SimulationError(f"task {t.id} has no device assignment")
        by_rank.setdefault(topo.flat(t.device), []).append(t)
    ranks = sorted(by_rank)
    hosted = {r: frozenset(k for t in by_rank[r] for k in task_modules(t, with_embeddings))
              for r in ranks}
    keys = sorted(set().union(*hosted.values())) if hosted else []
    groups = {k: [r for r in ranks if k in hosted[r]] for k in keys}
    return ModulePlan(tasks, topo, ranks, by_rank, hosted, keys, groups, with_embeddings)


def multiplex(tasks: Sequence[TaskSpec], step: int, rng: random.Random) -> TaskSpec:
    """Weighted choice among tasks active at ``step``; exactly one
    ``rng.random()`` per call (syncsim.py:190-205)."""
    active = [t for t in sorted(tasks, key=lambda t: t.id) if t.introduce_at_training_step <= step]
    if not active:
        raise SimulationError(f"no active task at step {step}")
    x = rng.random() * sum(t.weight for t in active)
    run = 0.0
    for t in active:
        run += t.weight
        if x < run:
            return t
    return active[-1]


class Multiplexer:
    """Per-rank task picker seeded like ``run_benchmark`` (syncsim.py:342)."""

    def __init__(self, plan: ModulePlan, rank: int, seed: int = 0):
        self.tasks = plan.tasks_by_rank.get(rank, [])
        self.rng = random.Random(f"{seed}:{rank}:mux")

    def pick(self, step: int) -> TaskSpec:
        return multiplex(self.tasks, step, self.rng)


def ready_flags(plan: ModulePlan, rank: int, used: Iterable[ModuleKey]) -> list[int]:
    """int32 flags in plan.keys order: 1 iff hosted here and used this step."""
    u = set(used)
    mine = plan.hosted.get(rank, frozenset())
    return [1 if (k in u and k in mine) else 0 for k in plan.keys]


def ready_bits(plan: ModulePlan, rank: int, used: Iterable[ModuleKey]) -> list[int]:
    """K1 contribution as a rank bitmask: bit `rank` set iff hosted here and
    used this step.  Bits are disjoint across ranks, so the world sum-allreduce
    returns each module's set of ready ranks: n = popcount, and for n = 1 the
    one rank whose buffer already is the group sum (the broadcast root)."""
    if rank >= 31:
        raise ValueError("ready bitmasks hold ranks 0..30")
    return [f << rank for f in ready_flags(plan, rank, used)]


def decode_ready(bits) -> tuple[list[int], list[int]]:
    """(counts, roots) from the world-summed ready bitmasks: counts[m] = number
    of ready ranks; roots[m] = the single ready rank when counts[m] == 1, else -1."""
    bits = [int(b) for b in bits]
    counts = [bin(b).count("1") for b in bits]
    roots = [b.bit_length() - 1 if c == 1 else -1 for b, c in zip(bits, counts)]
    return counts, roots


def ready_counts_all(plan: ModulePlan, used_by_rank: dict[int, set]) -> list[int]:
    """Sum of every rank's flags (what the world allreduce of K1 returns)."""
    tot = [0] * len(plan.keys)
    for r, used in used_by_rank.items():
        for i, f in enumerate(ready_flags(plan, r, used)):
            tot[i] += f
    return tot


def exchange_order(plan: ModulePlan, counts, rank: int) -> list[ModuleKey]:
    """Modules this rank must post a group reduction for, in the global issue
    order (sorted ModuleKey): hosted here, group of >= 2 ranks, n >= 1.  Every
    member of a group derives the same list from the same world-summed counts,
    so collectives on overlapping sub-communicators never cross."""
    idx = plan.index()
    mine = plan.hosted.get(rank, frozenset())
    return [k for k in plan.keys
            if k in mine and len(plan.groups[k]) >= 2 and counts[idx[k]] >= 1]


def exchange_plan(plan: ModulePlan, rank: int, bits, only=None) -> list[tuple]:
    """K2 work of `rank` for the world-summed ready bitmasks: (key, members,
    root) in the global issue order (``exchange_order``: sorted ModuleKey,
    hosted here, >= 2 members, n >= 1); root = the member index of the single
    ready rank when n = 1 (a broadcast from it), else -1 (a sum all-reduce).
    The NCCL engine and the gloo tests issue exactly this list."""
    counts, roots = decode_ready(bits)
    idx = plan.index()
    out = []
    for k in exchange_order(plan, counts, rank):
        if only is not None and k not in only:
            continue
        members = plan.groups[k]
        i = idx[k]
        out.append((k, members, members.index(roots[i]) if counts[i] == 1 else -1))
    return out


def shard_begin(n_elems: int, group_size: int, member: int) -> int:
    """First element of member's shard of a module (the host restatement of
    mm_peer_shard_begin): S = ceil(n / g) rounded up to 4 elements, shard r =
    [min(n, r*S), min(n, (r+1)*S))."""
    s = -(-n_elems // group_size)
    s = (s + 3) & ~3
    return min(n_elems, s * member)


def member_mask(bits: int, members: Sequence[int]) -> int:
    """World-summed ready bitmask (rank bits) -> group bitmask (member bits,
    member j = members[j], ascending ranks as in syncsim.py:337-340)."""
    return sum(((int(bits) >> r) & 1) << j for j, r in enumerate(members))


def peer_plan(plan: ModulePlan, rank: int, bits, only=None) -> list[tuple]:
    """Option-B work of `rank` for one exchange: (key, members, member index,
    group ready mask) for every hosted module with >= 2 members and n >= 1,
    in sorted ModuleKey order.  Every member derives its own entry from the
    same world-summed bits, so the shards of a module tile it exactly once."""
    idx = plan.index()
    mine = plan.hosted.get(rank, frozenset())
    out = []
    for k in plan.keys:
        if k not in mine or (only is not None and k not in only):
            continue
        members = plan.groups[k]
        if len(members) < 2:
            continue
        mask = member_mask(bits[idx[k]], members)
        if mask:
            out.append((k, members, members.index(rank), mask))
    return out

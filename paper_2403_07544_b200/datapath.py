"""Real-data input path: a FullConfig YAML as the trainer's
input, corpus path templates, per-task corpus streams, reservoir batching
and the multiplexer-driven micro-batch provider.

* ``parse_full_config`` / ``load_full_config`` read the reference's FullConfig
  YAML (keys of ``configgen.emit``, configgen.py:302-326; inverse of
  ``configgen.parse``, configgen.py:329-387) into this package's TaskSpec /
  ClusterTopology (field-for-field the reference's, core.py:74-149).
* ``PathTemplate`` renders corpus paths in the reference's two layouts
  (directional / symmetric, pathtmpl.py:19-89).
* ``CorpusStream`` yields (source ids, target ids) pairs from a task's two
  corpus files, cycling epochs.  The paper's SentencePiece models are not in
  this container, so the default tokenizer reads pre-tokenized lines
  (whitespace-separated integer ids); any ``tokenize(str) -> list[int]``
  callable can replace it.
* ``ReservoirBatcher`` draws a pool of pairs from the stream, keeps a uniform
  reservoir sample of it (``Reservoir`` semantics, syncsim.py:208-234) and
  packs the sample into one ``data.Batch`` of at most ``tokens`` target
  tokens (decoder input = BOS + sentence, labels = sentence + EOS).
* ``DataPipeline`` maps the task the rank's multiplexer picked
  (syncsim.py:190-205, curriculum-gated) to that task's batcher; it is what
  ``engine.Trainer.train_step`` accepts in place of ready-made batches.

Host-side only: batches are staged to HBM by ``engine.DeviceBatch``.
"""
from __future__ import annotations

import dataclasses
import os
import string
from enum import Enum
from typing import Callable, Iterable, Iterator, Optional, Sequence

import numpy as np

from .data import BOS, EOS, Batch
from .domain import ClusterTopology, DeviceId, ModuleKey, Side, TaskSpec, check_language
from .syncsim import Reservoir


class ConfigError(ValueError):
    """Malformed FullConfig (the reference raises configgen.ConfigError)."""


# ---------------------------------------------------------------------------
# FullConfig YAML


@dataclasses.dataclass(frozen=True)
class FullConfig:
    tasks: dict           # task id -> TaskSpec, sorted by id
    enc_layers: tuple
    dec_layers: tuple
    topology: ClusterTopology

    def task_list(self) -> list[TaskSpec]:
        return list(self.tasks.values())


def parse_full_config(text: str) -> FullConfig:
    """FullConfig YAML -> FullConfig (the key set of configgen.py:302-326)."""
    import yaml
    try:
        doc = yaml.safe_load(text)
    except yaml.YAMLError as exc:
        raise ConfigError(f"invalid YAML: {exc}") from exc
    if not isinstance(doc, dict):
        raise ConfigError("top level must be a mapping")
    try:
        topo = ClusterTopology(
            n_nodes=doc["n_nodes"], n_gpus_per_node=doc["n_gpus_per_node"],
            n_slots_per_gpu=doc["n_slots_per_gpu"],
            alpha_intra=doc.get("alpha_intra", 5e-6), alpha_inter=doc.get("alpha_inter", 20e-6),
            beta_intra=doc.get("beta_intra", 100e9), beta_inter=doc.get("beta_inter", 12.5e9))
        enc_layers, dec_layers = tuple(doc["enc_layers"]), tuple(doc["dec_layers"])
        tasks = {}
        for tid, e in doc["tasks"].items():
            src, _, tgt = e["src_tgt"].partition("-")
            enc = tuple(ModuleKey(Side.ENCODER, i, g) for i, g in enumerate(e["enc_sharing_groups"]))
            dec = tuple(ModuleKey(Side.DECODER, i, g) for i, g in enumerate(e["dec_sharing_groups"]))
            tasks[tid] = TaskSpec(
                id=tid, src_lang=src, tgt_lang=tgt, src_path=e["path_src"], tgt_path=e["path_tgt"],
                enc_modules=enc, dec_modules=dec,
                enc_layers=enc_layers[:len(enc)], dec_layers=dec_layers[:len(dec)],
                weight=e.get("weight", 1),
                introduce_at_training_step=e.get("introduce_at_training_step", 0),
                transforms=tuple(e.get("transforms", ())),
                adapters=tuple(sorted(e.get("adapters", {}).items())),
                device=DeviceId.parse(e["node_gpu"]) if "node_gpu" in e else None)
    except (KeyError, TypeError, ValueError) as exc:
        raise ConfigError(f"malformed configuration: {exc!r}") from exc
    return FullConfig(dict(sorted(tasks.items())), enc_layers, dec_layers, topo)


def load_full_config(path: str) -> FullConfig:
    with open(path) as f:
        return parse_full_config(f.read())


# ---------------------------------------------------------------------------
# corpus path templates


class CorpusMode(str, Enum):
    DIRECTIONAL = "directional"
    SYMMETRIC = "symmetric"


class TemplateError(ValueError):
    pass


_VARS = {CorpusMode.DIRECTIONAL: frozenset({"src_lang", "tgt_lang", "lang_pair"}),
         CorpusMode.SYMMETRIC: frozenset({"lang_a", "lang_b", "side_a", "side_b", "sorted_pair"})}


@dataclasses.dataclass(frozen=True)
class PathTemplate:
    """``{variable}`` path pattern checked against its mode's whitelist."""

    template: str
    mode: CorpusMode

    def __post_init__(self) -> None:
        names = set()
        for _, name, spec, conv in string.Formatter().parse(self.template):
            if name is None:
                continue
            if not name or spec or conv or "." in name or "[" in name:
                raise TemplateError(f"malformed placeholder in template: {self.template!r}")
            names.add(name)
        unknown = names - _VARS[self.mode]
        if unknown:
            raise TemplateError(f"variables {sorted(unknown)} not allowed in {self.mode.value} "
                                f"mode (template {self.template!r})")

    def render(self, src: str, tgt: str) -> str:
        check_language(src)
        check_language(tgt)
        if self.mode is CorpusMode.DIRECTIONAL:
            return self.template.format(src_lang=src, tgt_lang=tgt, lang_pair=f"{src}-{tgt}")
        # symmetric: one alphabetically sorted file pair serves both directions;
        # the target side is called "trg"
        a, b = min(src, tgt), max(src, tgt)
        fwd = src == a
        return self.template.format(lang_a=a, lang_b=b, side_a="src" if fwd else "trg",
                                    side_b="trg" if fwd else "src", sorted_pair=f"{a}-{b}")


# ---------------------------------------------------------------------------
# corpus streams and reservoir batching


def id_tokenizer(line: str) -> list[int]:
    """Pre-tokenized corpus line: whitespace-separated integer ids."""
    return [int(x) for x in line.split()]


class CorpusStream:
    """Endless stream of (src ids, tgt ids) for one task; each epoch re-reads
    the two files in parallel (line i of one is the translation of line i of
    the other), skipping pairs with an empty side."""

    def __init__(self, src_path: str, tgt_path: str,
                 tokenize: Callable[[str], list[int]] = id_tokenizer, max_len: int = 256):
        for p in (src_path, tgt_path):
            if not os.path.exists(p):
                raise FileNotFoundError(p)
        self.src_path, self.tgt_path = src_path, tgt_path
        self.tokenize = tokenize
        self.max_len = max_len
        self.epoch = 0
        self.line = 0  # lines of the current epoch already consumed
        self._it = self._pairs()

    def state(self) -> dict:
        return {"epoch": self.epoch, "line": self.line}

    def load_state(self, st: dict) -> None:
        """Resume at (epoch, line): the next pair is the first usable one
        after the consumed lines of that epoch."""
        self.epoch, self.line = int(st["epoch"]), int(st["line"])
        self._it = self._pairs()

    def _pairs(self) -> Iterator[tuple[list[int], list[int]]]:
        while True:
            n, skip = 0, self.line
            with open(self.src_path) as fs, open(self.tgt_path) as ft:
                for idx, (ls, lt) in enumerate(zip(fs, ft)):
                    if idx < skip:
                        continue
                    self.line = idx + 1
                    s, t = self.tokenize(ls)[:self.max_len], self.tokenize(lt)[:self.max_len - 1]
                    if s and t:
                        n += 1
                        yield s, t
            if n == 0 and skip == 0:
                raise ValueError(f"corpus {self.src_path} / {self.tgt_path} has no usable pair")
            self.epoch += 1
            self.line = 0

    def take(self, n: int) -> list[tuple[list[int], list[int]]]:
        return [next(self._it) for _ in range(n)]


def pack_pairs(pairs: Sequence[tuple[Sequence[int], Sequence[int]]], tokens: int,
               order: bool = True) -> Batch:
    """Take pairs in order until the target side holds ``tokens`` tokens
    (each target contributes len + 1: BOS-shifted input / EOS-terminated
    labels; the pair that crosses the budget is truncated, >= 1 token), then
    lay the taken pairs out in data.attention_order (order=True)."""
    ss, ts, used = [], [], 0
    for s, t in pairs:
        if used >= tokens:
            break
        room = tokens - used
        t = list(t)[:max(0, room - 1)]
        ss.append(np.asarray(s, np.int32))
        ts.append(np.asarray(t, np.int32))
        used += len(t) + 1
    if not ss:
        raise ValueError("no pairs to pack")
    if order and len(ss) > 1:
        from .data import attention_order
        perm = attention_order([len(x) for x in ss], [len(t) + 1 for t in ts])
        ss, ts = [ss[i] for i in perm], [ts[i] for i in perm]
    ls = np.array([len(s) for s in ss])
    lt = np.array([len(t) + 1 for t in ts])
    cu_s = np.concatenate([[0], np.cumsum(ls)]).astype(np.int32)
    cu_t = np.concatenate([[0], np.cumsum(lt)]).astype(np.int32)
    src = np.concatenate(ss)
    tgt_in = np.concatenate([np.concatenate([[BOS], t]) for t in ts]).astype(np.int32)
    labels = np.concatenate([np.concatenate([t, [EOS]]) for t in ts]).astype(np.int32)
    src_pos = np.concatenate([np.arange(n) for n in ls]).astype(np.int32)
    tgt_pos = np.concatenate([np.arange(n) for n in lt]).astype(np.int32)
    return Batch(src, src_pos, cu_s, tgt_in, tgt_pos, labels, cu_t)


class ReservoirBatcher:
    """Per task: read ``pool`` pairs, keep a uniform ``capacity`` reservoir
    of them (seeded per draw: ``Random(f"{seed}:{task}:{draw}")``), pack the
    sample into a batch of <= ``tokens`` target tokens."""

    def __init__(self, stream: CorpusStream, task_id: str, tokens: int, capacity: int = 512,
                 pool: int = 2048, seed: int = 0, vocab: Optional[int] = None):
        if pool < capacity:
            raise ValueError("pool must be >= capacity")
        self.stream, self.task_id = stream, task_id
        self.tokens, self.capacity, self.pool, self.seed = tokens, capacity, pool, seed
        self.vocab = vocab
        self.draws = 0

    def next_batch(self) -> Batch:
        res = Reservoir(self.capacity, seed=f"{self.seed}:{self.task_id}:{self.draws}")
        for pair in self.stream.take(self.pool):
            res.add(pair)
        self.draws += 1
        b = pack_pairs(res.items, self.tokens)
        if self.vocab is not None:
            for a in (b.src, b.tgt_in, b.labels):
                if a.size and (a.min() < 0 or a.max() >= self.vocab):
                    raise ValueError(f"task {self.task_id}: token id outside [0, {self.vocab})")
        return b


class DataPipeline:
    """Micro-batch provider: ``batch_for(task)`` returns the next batch of
    the task the multiplexer picked.  Corpus paths come from each TaskSpec
    (``path_src`` / ``path_tgt`` of the FullConfig), relative ones resolved
    against ``root``; sentences are clipped to ``max_len`` tokens (the
    model's position table, including the EOS / BOS slot)."""

    def __init__(self, tasks: Iterable[TaskSpec], tokens: int, root: str = ".", seed: int = 0,
                 tokenize: Callable[[str], list[int]] = id_tokenizer, capacity: int = 512,
                 pool: int = 2048, vocab: Optional[int] = None, max_len: int = 256):
        self.batchers: dict[str, ReservoirBatcher] = {}
        for t in tasks:
            sp, tp = (p if os.path.isabs(p) else os.path.join(root, p)
                      for p in (t.src_path, t.tgt_path))
            self.batchers[t.id] = ReservoirBatcher(CorpusStream(sp, tp, tokenize, max_len), t.id, tokens,
                                                   capacity, pool, seed, vocab)

    def batch_for(self, task: TaskSpec) -> Batch:
        return self.batchers[task.id].next_batch()

    def state(self) -> dict:
        """Per task: reservoir draws and the corpus position (checkpointed
        with the trainer, so a resumed run continues the same data)."""
        return {tid: {"draws": b.draws, **b.stream.state()} for tid, b in self.batchers.items()}

    def load_state(self, state: dict) -> None:
        if set(state) != set(self.batchers):
            raise ValueError("pipeline state is for a different task set")
        for tid, st in state.items():
            b = self.batchers[tid]
            b.draws = int(st["draws"])
            b.stream.load_state(st)

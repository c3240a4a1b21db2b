"""Per-module checkpoint / resume (the reference has none).

Layout of a checkpoint directory::

    <dir>/modules/<side>:<position>:<group>.npz          whole module
    <dir>/modules/<side>:<position>:<group>.s<j>of<g>.npz  member j's shard
    <dir>/rank<r>.json                                  per-rank host state

A module's state (fp32 master, Adam exp_avg / exp_avg_sq, Adam step) is
identical on every member of its group after the Algorithm-1 exchange, so
it is written ONCE per group, by the group's lowest rank.  With the
option-B peer exchange each member is authoritative only on its own shard
(``peer.py``), so each member writes its shard and the loader assembles
them.  bf16 weights are not stored: they are re-cast from the master on
load (the cast the fused update performs).  Per-rank files hold the
multiplexer RNG state (syncsim.py:342: picks continue exactly where they
stopped) and the trainer's step index.

Files are written to a temporary name and renamed, so a reader never sees a
partial file.  Every rank calls ``save`` / ``load``; ranks write disjoint files.
Saving a module in one layout removes that module's files of the other layout
(a directory reused after switching the exchange never mixes them), and each
rank's json is written LAST and lists the module files that rank wrote with
the save's step index: the loader accepts a module file only if some rank's
manifest lists it for the step being resumed, so an interrupted save (module
files newer than their manifest, or missing) fails loudly instead of resuming
a mix of steps.
"""
from __future__ import annotations

import glob
import json
import os
from typing import Optional

import numpy as np

FIELDS = ("master", "exp_avg", "exp_avg_sq")


def module_path(root: str, key, shard: Optional[tuple[int, int]] = None) -> str:
    name = str(key) if shard is None else f"{key}.s{shard[0]}of{shard[1]}"
    return os.path.join(root, "modules", name + ".npz")


def _atomic_savez(path: str, **arrays) -> None:
    os.makedirs(os.path.dirname(path), exist_ok=True)
    tmp = path + ".tmp.npz"
    np.savez(tmp, **arrays)
    os.replace(tmp, path)


def write_module(root: str, key, state: dict, step: int, n_elems: int,
                 shard: Optional[tuple[int, int, int, int]] = None) -> str:
    """state: FIELDS -> host float32 arrays (the whole module, or only the
    shard [begin, end) when ``shard = (j, g, begin, end)``)."""
    arrays = {f: np.ascontiguousarray(state[f], dtype=np.float32) for f in FIELDS}
    meta = np.array([step, n_elems] + (list(shard) if shard else [0, 1, 0, n_elems]), np.int64)
    path = module_path(root, key, None if shard is None else shard[:2])
    _atomic_savez(path, meta=meta, **arrays)
    # drop this module's files of the other layout (or of another group size)
    stale = glob.glob(glob.escape(module_path(root, key))[:-4] + ".s*of*.npz")
    if shard is not None:  # keep the shards of this group size, drop the whole file
        stale = [f for f in stale if not f.endswith(f"of{shard[1]}.npz")] + [module_path(root, key)]
    for f in stale:
        try:
            os.remove(f)
        except FileNotFoundError:
            pass
    return path


def manifest(root: str) -> dict:
    """{module file (relative to root): step index} over every rank's json."""
    out = {}
    for path in glob.glob(os.path.join(glob.escape(root), "rank*.json")):
        with open(path) as f:
            st = json.load(f)
        for rel in st.get("files", ()):
            out[rel] = st.get("step_idx")
    return out


def check_manifest(root: str, files, step_idx) -> None:
    """Every module file read must be listed by some rank's manifest for
    ``step_idx`` (the resumed save)."""
    listed = manifest(root)
    for path in files:
        rel = os.path.relpath(path, root)
        if rel not in listed:
            raise ValueError(f"{rel}: not in any rank's manifest (interrupted or stale save)")
        if listed[rel] != step_idx:
            raise ValueError(f"{rel}: written by the save of step {listed[rel]}, resuming {step_idx}")


def module_files(root: str, key) -> list[str]:
    """The files holding a module: its whole file, or all its shards."""
    whole = module_path(root, key)
    if os.path.exists(whole):
        return [whole]
    g = _shard_count(root, key)
    return [module_path(root, key, (j, g)) for j in range(g)]


def read_module(root: str, key, n_elems: int) -> tuple[dict, int]:
    """(FIELDS -> whole-module arrays, Adam step) from either layout."""
    whole = module_path(root, key)
    if os.path.exists(whole):
        with np.load(whole) as z:
            meta = z["meta"]
            if int(meta[1]) != n_elems:
                raise ValueError(f"{key}: checkpoint has {int(meta[1])} elements, module {n_elems}")
            return {f: z[f].copy() for f in FIELDS}, int(meta[0])
    g = _shard_count(root, key)
    out = {f: np.empty(n_elems, np.float32) for f in FIELDS}
    covered, steps = 0, set()
    for j in range(g):
        path = module_path(root, key, (j, g))
        if not os.path.exists(path):
            raise FileNotFoundError(f"{key}: missing shard {path}")
        with np.load(path) as z:
            st, n, jj, gg, b, e = (int(x) for x in z["meta"])
            if n != n_elems or jj != j or gg != g:
                raise ValueError(f"{key}: inconsistent shard {path}")
            for f in FIELDS:
                out[f][b:e] = z[f]
        steps.add(st)
        covered += e - b
    if len(steps) != 1:
        raise ValueError(f"{key}: shards disagree on the Adam step")
    if covered != n_elems:
        raise ValueError(f"{key}: shards cover {covered} of {n_elems} elements")
    return out, steps.pop()


def _shard_count(root: str, key) -> int:
    prefix = f"{key}.s0of"
    d = os.path.join(root, "modules")
    for name in (os.listdir(d) if os.path.isdir(d) else ()):
        if name.startswith(prefix) and name.endswith(".npz") and ".tmp" not in name:
            return int(name[len(prefix):-4])
    raise FileNotFoundError(f"{key}: no checkpoint under {root}")


def write_rank_state(root: str, rank: int, state: dict) -> None:
    os.makedirs(root, exist_ok=True)
    path = os.path.join(root, f"rank{rank}.json")
    with open(path + ".tmp", "w") as f:
        json.dump(state, f)
    os.replace(path + ".tmp", path)


def read_rank_state(root: str, rank: int) -> dict:
    with open(os.path.join(root, f"rank{rank}.json")) as f:
        return json.load(f)


def rng_to_json(rng) -> list:
    v, internal, gauss = rng.getstate()
    return [v, list(internal), gauss]


def rng_from_json(rng, s) -> None:
    rng.setstate((s[0], tuple(s[1]), s[2]))

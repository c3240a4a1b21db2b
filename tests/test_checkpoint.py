"""Per-module checkpoint files (f4) on the CPU: whole-module and sharded
layouts round-trip bit-exactly, shards written by different members
assemble into the module, and broken checkpoints fail loudly."""
import os
import random

import numpy as np
import pytest

from paper_2403_07544_b200 import checkpoint as C
from paper_2403_07544_b200.domain import ModuleKey, Side
from paper_2403_07544_b200.plan import shard_begin

KEY = ModuleKey(Side.ENCODER, 0, "de")


def _state(n, seed):
    rng = np.random.default_rng(seed)
    return {f: rng.standard_normal(n).astype(np.float32) for f in C.FIELDS}


def test_whole_module_round_trip(tmp_path):
    st = _state(1001, 0)
    C.write_module(str(tmp_path), KEY, st, step=7, n_elems=1001)
    got, step = C.read_module(str(tmp_path), KEY, 1001)
    assert step == 7 and all(np.array_equal(got[f], st[f]) for f in C.FIELDS)
    with pytest.raises(ValueError):
        C.read_module(str(tmp_path), KEY, 1000)


@pytest.mark.parametrize("n,g", [(1001, 3), (8, 8), (5, 4), (100_003, 7)])
def test_sharded_round_trip(tmp_path, n, g):
    st = _state(n, g)
    for j in reversed(range(g)):  # members write in any order
        b, e = shard_begin(n, g, j), shard_begin(n, g, j + 1)
        C.write_module(str(tmp_path), KEY, {f: v[b:e] for f, v in st.items()}, 3, n, (j, g, b, e))
    got, step = C.read_module(str(tmp_path), KEY, n)
    assert step == 3 and all(np.array_equal(got[f], st[f]) for f in C.FIELDS)


def test_missing_or_inconsistent_shards(tmp_path):
    n, g = 1000, 4
    st = _state(n, 1)
    for j in (0, 1, 3):
        b, e = shard_begin(n, g, j), shard_begin(n, g, j + 1)
        C.write_module(str(tmp_path), KEY, {f: v[b:e] for f, v in st.items()}, 3, n, (j, g, b, e))
    with pytest.raises(FileNotFoundError):
        C.read_module(str(tmp_path), KEY, n)
    b, e = shard_begin(n, g, 2), shard_begin(n, g, 3)
    C.write_module(str(tmp_path), KEY, {f: v[b:e] for f, v in st.items()}, 4, n, (2, g, b, e))
    with pytest.raises(ValueError):  # steps disagree
        C.read_module(str(tmp_path), KEY, n)
    with pytest.raises(FileNotFoundError):
        C.read_module(str(tmp_path), ModuleKey(Side.DECODER, 0, "x"), n)


def test_rank_state_and_rng(tmp_path):
    rng = random.Random("0:3:mux")
    for _ in range(5):
        rng.random()
    C.write_rank_state(str(tmp_path), 3, {"mux_rng": C.rng_to_json(rng), "step_idx": 5})
    want = [rng.random() for _ in range(4)]
    st = C.read_rank_state(str(tmp_path), 3)
    other = random.Random(0)
    C.rng_from_json(other, st["mux_rng"])
    assert [other.random() for _ in range(4)] == want and st["step_idx"] == 5


def test_layout_switch_drops_the_other_layout(tmp_path):
    """Saving a module whole after a sharded save (exchange switched from
    peer to nccl) removes its shards, and vice versa: a reused directory never
    resolves a module from a stale layout."""
    root, n, g = str(tmp_path), 1000, 4
    old = _state(n, 5)
    for j in range(g):
        b, e = shard_begin(n, g, j), shard_begin(n, g, j + 1)
        C.write_module(root, KEY, {f: v[b:e] for f, v in old.items()}, 3, n, (j, g, b, e))
    new = _state(n, 6)
    C.write_module(root, KEY, new, 4, n)
    assert C.module_files(root, KEY) == [C.module_path(root, KEY)]
    got, step = C.read_module(root, KEY, n)
    assert step == 4 and np.array_equal(got["master"], new["master"])
    b, e = shard_begin(n, g, 0), shard_begin(n, g, 1)
    C.write_module(root, KEY, {f: v[b:e] for f, v in old.items()}, 5, n, (0, g, b, e))
    assert not (tmp_path / "modules" / f"{KEY}.npz").exists()


def test_manifest_rejects_interrupted_save(tmp_path):
    """Each rank's json, written last, lists its module files with the step:
    files of a later, interrupted save (no updated manifest) or files no
    manifest lists are rejected."""
    root, n = str(tmp_path), 64
    f1 = C.write_module(root, KEY, _state(n, 1), 2, n)
    C.write_rank_state(root, 0, {"step_idx": 2, "files": [os.path.relpath(f1, root)]})
    C.check_manifest(root, C.module_files(root, KEY), 2)
    with pytest.raises(ValueError):
        C.check_manifest(root, C.module_files(root, KEY), 3)  # resuming another step
    other = ModuleKey(Side.DECODER, 0, "x")
    C.write_module(root, other, _state(n, 2), 3, n)  # written, manifest never updated
    with pytest.raises(ValueError):
        C.check_manifest(root, C.module_files(root, other), 2)

"""Real-data path on the CPU: FullConfig YAML emitted by
the reference (tests/golden/make_golden_datapath.py) parses into the same
tasks / topology / module plan as configs.py builds; path templates and
reservoir samples match the reference's outputs; corpus streams pack into
well-formed batches."""
import json
import os

import numpy as np
import pytest

from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.data import BOS, EOS
from paper_2403_07544_b200.datapath import (ConfigError, CorpusMode, CorpusStream, DataPipeline,
                                            PathTemplate, ReservoirBatcher, TemplateError,
                                            load_full_config, pack_pairs, parse_full_config)
from paper_2403_07544_b200.plan import build_plan
from paper_2403_07544_b200.syncsim import reservoir_batch

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _same_task(a, b):
    for f in ("id", "src_lang", "tgt_lang", "src_path", "tgt_path", "enc_modules", "dec_modules",
              "enc_layers", "dec_layers", "weight", "introduce_at_training_step", "device"):
        assert getattr(a, f) == getattr(b, f), (a.id, f)


@pytest.mark.parametrize("name", ["config1", "config4"])
def test_reference_fullconfig_parses_to_the_workload(name):
    cfg = load_full_config(os.path.join(GOLD, f"fullconfig_{name}.yaml"))
    if name == "config1":
        w = configs.config1()
        tasks, topo = w.tasks, w.topo
    else:
        tasks, topo = configs.config4_tasks(8)
    assert sorted(cfg.tasks) == sorted(t.id for t in tasks)
    for t in tasks:
        _same_task(cfg.tasks[t.id], t)
    assert (cfg.topology.n_nodes, cfg.topology.n_gpus_per_node, cfg.topology.n_slots_per_gpu) == \
        (topo.n_nodes, topo.n_gpus_per_node, topo.n_slots_per_gpu)
    if all(t.device is not None for t in tasks):
        assert build_plan(cfg.task_list(), cfg.topology).groups == build_plan(tasks, topo).groups


def test_fullconfig_errors():
    with pytest.raises(ConfigError):
        parse_full_config("tasks: [unclosed")
    with pytest.raises(ConfigError):
        parse_full_config("- a list")
    with pytest.raises(ConfigError):
        parse_full_config("n_nodes: 1\ntasks: {}\n")  # missing keys


def test_path_templates_match_reference():
    with open(os.path.join(GOLD, "datapath.json")) as f:
        gold = json.load(f)
    for r in gold["render"]:
        t = PathTemplate(r["template"], CorpusMode(r["mode"]))
        assert t.render(r["src"], r["tgt"]) == r["path"], r
    with pytest.raises(TemplateError):
        PathTemplate("{lang_a}/x", CorpusMode.DIRECTIONAL)
    with pytest.raises(TemplateError):
        PathTemplate("{src_lang!r}", CorpusMode.DIRECTIONAL)


def test_reservoir_matches_reference():
    with open(os.path.join(GOLD, "datapath.json")) as f:
        gold = json.load(f)
    for r in gold["reservoir"]:
        assert reservoir_batch(range(r["n"]), r["capacity"], r["seed"]) == r["items"]


def _corpus(tmp_path, n=50, seed=0):
    rng = np.random.default_rng(seed)
    src, tgt = tmp_path / "x.src", tmp_path / "x.tgt"
    with open(src, "w") as fs, open(tgt, "w") as ft:
        for i in range(n):
            fs.write(" ".join(map(str, rng.integers(4, 100, rng.integers(1, 20)))) + "\n")
            ft.write(" ".join(map(str, rng.integers(4, 100, rng.integers(1, 20)))) + "\n")
        fs.write("\n")  # empty pair: skipped
        ft.write("5 6\n")
    return str(src), str(tgt)


def test_pack_pairs_layout():
    pairs = [([4, 5, 6], [7, 8]), ([9], [10, 11, 12, 13]), ([14, 15], [16])]
    b = pack_pairs(pairs, tokens=100, order=False)
    assert b.cu_src.tolist() == [0, 3, 4, 6] and b.cu_tgt.tolist() == [0, 3, 8, 10]
    assert b.tgt_in.tolist() == [BOS, 7, 8, BOS, 10, 11, 12, 13, BOS, 16]
    assert b.labels.tolist() == [7, 8, EOS, 10, 11, 12, 13, EOS, 16, EOS]
    assert b.src_pos.tolist() == [0, 1, 2, 0, 0, 1] and b.tgt_pos.tolist()[:4] == [0, 1, 2, 0]
    cut = pack_pairs(pairs, tokens=5, order=False)  # 3 + truncated second pair (1 token + EOS)
    assert cut.n_tgt == 5 and cut.labels.tolist() == [7, 8, EOS, 10, EOS]


def test_corpus_stream_and_reservoir_batcher(tmp_path):
    sp, tp = _corpus(tmp_path)
    st = CorpusStream(sp, tp)
    first = st.take(50)
    assert st.take(1)[0] == first[0] and st.epoch == 1  # cycles, empty pair skipped
    b1 = ReservoirBatcher(CorpusStream(sp, tp), "train_x-y", tokens=64, capacity=8, pool=20, seed=3)
    b2 = ReservoirBatcher(CorpusStream(sp, tp), "train_x-y", tokens=64, capacity=8, pool=20, seed=3)
    for _ in range(4):
        x, y = b1.next_batch(), b2.next_batch()
        assert all(np.array_equal(getattr(x, f), getattr(y, f)) for f in x.host_arrays())
        assert x.n_tgt <= 64 and x.n_seq <= 8
        assert (np.diff(x.cu_tgt) >= 1).all() and (np.diff(x.cu_src) >= 1).all()
        ends = x.cu_tgt[1:] - 1
        assert (x.labels[ends] == EOS).all() and (x.tgt_in[x.cu_tgt[:-1]] == BOS).all()
    with pytest.raises(ValueError):
        ReservoirBatcher(CorpusStream(sp, tp), "t", tokens=8, capacity=8, vocab=50).next_batch()


def test_pipeline_from_fullconfig(tmp_path):
    cfg = load_full_config(os.path.join(GOLD, "fullconfig_config1.yaml"))
    for t in cfg.task_list():
        os.makedirs(tmp_path / os.path.dirname(t.src_path), exist_ok=True)
        sp, tp = _corpus(tmp_path, seed=len(t.id) + ord(t.id[-1]))
        os.replace(sp, tmp_path / t.src_path)
        os.replace(tp, tmp_path / t.tgt_path)
    pipe = DataPipeline(cfg.task_list(), tokens=128, root=str(tmp_path), seed=0, capacity=16, pool=32)
    for t in cfg.task_list():
        b = pipe.batch_for(t)
        assert 0 < b.n_tgt <= 128
    with pytest.raises(FileNotFoundError):
        DataPipeline(cfg.task_list(), tokens=128, root=str(tmp_path / "missing"))


def test_attention_order_native_matches_restatement_and_packs_tighter():
    from paper_2403_07544_b200.data import attention_groups, attention_order, attention_order_py
    rng = np.random.default_rng(4)
    for t in range(100):
        n = int(rng.integers(0, 300))
        ls, lt = rng.integers(1, 160, n), rng.integers(1, 160, n)
        perm = attention_order(ls, lt)
        assert np.array_equal(perm, attention_order_py(ls, lt)), t
        assert sorted(perm.tolist()) == list(range(n))
        if n:
            cs = np.concatenate([[0], np.cumsum(ls)]).astype(np.int32)
            ct = np.concatenate([[0], np.cumsum(lt)]).astype(np.int32)
            cs2 = np.concatenate([[0], np.cumsum(ls[perm])]).astype(np.int32)
            ct2 = np.concatenate([[0], np.cumsum(lt[perm])]).astype(np.int32)
            g1, _ = attention_groups(ct, cs, 128, 1)
            g2, _ = attention_groups(ct2, cs2, 128, 1)
            assert len(g2) <= len(g1), t  # never more cross-attention groups


def test_pack_pairs_order_is_a_permutation(tmp_path):
    pairs = [(list(range(4, 4 + a)), list(range(4, 4 + b))) for a, b in
             [(30, 5), (3, 40), (60, 60), (10, 12), (100, 20), (7, 90)]]
    b0 = pack_pairs(pairs, tokens=10_000, order=False)
    b1 = pack_pairs(pairs, tokens=10_000, order=True)
    assert b0.n_src == b1.n_src and b0.n_tgt == b1.n_tgt
    assert sorted(np.diff(b0.cu_src).tolist()) == sorted(np.diff(b1.cu_src).tolist())


def test_pipeline_state_resumes_the_same_data(tmp_path):
    """DataPipeline.state / load_state (checkpointed by Trainer): a fresh
    pipeline restored from the state after k batches yields the same next
    batches as the original, across an epoch boundary."""
    cfg = load_full_config(os.path.join(GOLD, "fullconfig_config1.yaml"))
    for t in cfg.task_list():
        os.makedirs(tmp_path / os.path.dirname(t.src_path), exist_ok=True)
        sp, tp = _corpus(tmp_path, seed=len(t.id) + ord(t.id[-1]))
        os.replace(sp, tmp_path / t.src_path)
        os.replace(tp, tmp_path / t.tgt_path)
    mk = lambda: DataPipeline(cfg.task_list(), tokens=96, root=str(tmp_path), seed=1, capacity=8,
                              pool=20)
    tasks = cfg.task_list()
    a = mk()
    for i in range(5):
        a.batch_for(tasks[i % len(tasks)])
    state = json.loads(json.dumps(a.state()))  # as stored in the rank json
    b = mk()
    b.load_state(state)
    for i in range(6):  # the 20-pair pools cross the corpus' epoch boundary
        t = tasks[(i * 2) % len(tasks)]
        x, y = a.batch_for(t), b.batch_for(t)
        assert all(np.array_equal(getattr(x, f), getattr(y, f)) for f in x.host_arrays())
    assert any(st["epoch"] > 0 for st in a.state().values())

"""The C-ABI library loads on a CPU-only host, exports every entry point the
header declares, and K9 (the allocator's comm-cost kernel) is bit-identical
to the reference's kernel (golden vectors from _cost_py.py, the oracle's C
restatement and -- when built -- the reference's own compiled Cython)."""
import ctypes
import json
import os

import numpy as np
import pytest

from paper_2403_07544_b200 import _native
from paper_2403_07544_b200.allocator import comm_cost_kernel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


def test_library_loads_and_exports_every_symbol():
    lib = _native.lib()
    syms = _native.symbols()
    assert len(syms) >= 25
    for name in syms:
        assert hasattr(lib, name), name
    assert lib.mm_abi_version() == _native.ABI_VERSION


def test_header_version_matches_binding():
    with open(os.path.join(ROOT, "include", "mmb200.h")) as f:
        txt = f.read()
    assert f"#define MMB200_ABI_VERSION {_native.ABI_VERSION}" in txt


def test_struct_layouts():
    # the ctypes mirrors have the sizes the C side was compiled with
    from paper_2403_07544_b200 import ops
    mirrors = {"mm_sync_module": _native.SyncModule, "mm_adam_module": _native.AdamModule,
               "mm_adam_hyper": _native.AdamHyper, "mm_reduce_item": _native.ReduceItem,
               "mm_peer_shard": _native.PeerShard, "mm_peer_signal": _native.PeerSignal,
               "mm_gemm_args": ops.GemmArgs, "mm_attn_args": ops.AttnArgs,
               "mm_layer_offsets": _native.LayerOffsets, "mm_stack": _native.Stack,
               "mm_embed": _native.Embed, "mm_task": _native.Task, "mm_batch": _native.BatchDesc}
    for name, cls in mirrors.items():
        assert _native.lib().mm_abi_sizeof(name.encode()) == ctypes.sizeof(cls), name
    assert _native.lib().mm_abi_sizeof(b"nope") == -1
    # offsets the C side relies on (include/mmb200.h)
    assert ctypes.sizeof(_native.SyncModule) == 32 * 8 + 8 + 8 + 4 + 4
    assert ctypes.sizeof(_native.AdamModule) == 5 * 8 + 8 + 4 + 4 + 4 + 4
    assert ctypes.sizeof(_native.AdamHyper) == 7 * 4 + 4 + 4  # + zero_grad
    assert ctypes.sizeof(_native.ReduceItem) == 8 + 8 + 8 + 4 + 4 + 4 + 4 + 8
    assert ctypes.sizeof(_native.PeerShard) == 3 * 8 * 8 + 3 * 8 + 2 * 8 + 4 * 4
    assert ctypes.sizeof(_native.PeerSignal) == 8 + 32 * 8 + 32 * 4 + 4 * 4
    from paper_2403_07544_b200 import ops
    assert ctypes.sizeof(ops.AttnArgs) == 11 * 8 + 7 * 8 + 8 * 4 + 8 + 4 * 4 + 8 + 8


def test_peer_shard_partition_matches_host_restatement():
    """mm_peer_shard_begin (host code in the library) == plan.shard_begin, and
    the g shards tile [0, n) with 16-byte aligned starts."""
    from paper_2403_07544_b200.plan import shard_begin
    L = _native.lib()
    for n in (0, 1, 3, 4, 5, 7, 64, 1000, 100_003, 6_295_552, 56_000_001):
        for g in range(1, 9):
            bounds = [shard_begin(n, g, r) for r in range(g + 1)]
            assert bounds == [L.mm_peer_shard_begin(n, g, r) for r in range(g + 1)]
            assert bounds[0] == 0 and bounds[-1] == n
            assert all(a <= b for a, b in zip(bounds, bounds[1:]))
            assert all(b % 4 == 0 for b in bounds[:-1] if b < n)
    assert L.mm_peer_shard_begin(10, 0, 0) == -1


def test_peer_entry_points_reject_bad_arguments():
    L = _native.lib()
    sh = _native.PeerShard()
    sh.group_size = 9
    hp = _native.AdamHyper.make(0.9, 0.998, 1e-8)
    assert L.mm_peer_update(ctypes.byref(sh), 1, ctypes.byref(hp), None) == -1
    assert b"group size" in L.mm_last_error()
    sig = _native.PeerSignal()
    sig.n_peers = 33
    assert L.mm_peer_barrier(ctypes.byref(sig), None) == -1
    assert L.mm_ipc_release(ctypes.c_void_p(1234)) == -1


def test_argument_errors_are_reported():
    lib = _native.lib()
    total = ctypes.c_double()
    st = lib.mm_comm_cost(None, -1, None, None, None, None, 0, 1.0, 4.0, None, ctypes.byref(total))
    assert st == -1
    assert b"negative" in lib.mm_last_error()


def _case_arrays(c):
    params = np.array([float.fromhex(x) for x in c["params"]])
    return (params, np.array(c["off"], np.int64), np.array(c["idx"], np.int64),
            np.array(c["task_dev"], np.int64), np.array(c["dev_node"], np.int64),
            float.fromhex(c["w_intra"]), float.fromhex(c["w_inter"]))


def test_comm_cost_bit_exact_vs_reference_golden(golden):
    for c in golden["allocator"]["kernel"]:
        p, off, idx, td, dn, wi, we = _case_arrays(c)
        out = np.zeros(len(p))
        total = comm_cost_kernel(p, off, idx, td, dn, wi, we, out)
        assert total.hex() == c["total"]
        assert [x.hex() for x in out] == c["per_module"]


def test_comm_cost_vs_oracle_c_and_reference_build(golden):
    from oracle import build_ref
    build_ref.build()
    lib = ctypes.CDLL(build_ref.ORACLE_SO)
    lib.oracle_comm_cost.restype = ctypes.c_double
    ref_kernel = build_ref.load_reference_kernel()  # None on the GPU box
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int64)
    for c in golden["allocator"]["kernel"]:
        p, off, idx, td, dn, wi, we = _case_arrays(c)
        o1, o2 = np.zeros(len(p)), np.zeros(len(p))
        t1 = comm_cost_kernel(p, off, idx, td, dn, wi, we, o1)
        t2 = lib.oracle_comm_cost(p.ctypes.data_as(dp), len(p), off.ctypes.data_as(ip),
                                  idx.ctypes.data_as(ip), td.ctypes.data_as(ip),
                                  dn.ctypes.data_as(ip), len(dn), ctypes.c_double(wi),
                                  ctypes.c_double(we), o2.ctypes.data_as(dp))
        assert t1 == t2 and np.array_equal(o1, o2)
        if ref_kernel is not None:
            o3 = np.zeros(len(p))
            assert ref_kernel(p, off, idx, td, dn, wi, we, o3) == t1
            assert np.array_equal(o3, o1)


def test_comm_cost_rejects_bad_device():
    out = np.zeros(1)
    with pytest.raises(_native.MMError):
        comm_cost_kernel(np.ones(1), np.array([0, 1]), np.array([0]), np.array([5]),
                         np.array([0, 0]), 1.0, 4.0, out)


def test_attention_groups_native_matches_numpy():
    """mm_attention_groups (host C++, on the step's path) == data.attention_groups."""
    import numpy as np
    from paper_2403_07544_b200.data import attention_groups
    from paper_2403_07544_b200.engine import native_attention_groups
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = int(rng.integers(0, 60))
        hi = int(rng.choice([8, 40, 128, 256]))
        lq = rng.integers(1, hi + 1, size=n)
        lk = rng.integers(1, hi + 1, size=n) if trial % 2 else lq
        cq = np.concatenate([[0], np.cumsum(lq)]).astype(np.int32)
        ck = np.concatenate([[0], np.cumsum(lk)]).astype(np.int32)
        for cap in (64, 128, 256):
            for align in (32, 1, 8):
                g1, f1 = attention_groups(cq, ck, cap, align)
                g2, f2 = native_attention_groups(cq, ck, cap, align)
                assert np.array_equal(g1, g2) and f1 == f2, (trial, cap, align)
        # the two packings route every sequence to exactly one backward kernel:
        # a sequence of <= 128 rows per side sits in an unpadded group of <= 128
        # rows (tcgen05) and in a padded group of <= 128 actual rows (skipped by
        # mma.sync); a longer one is alone in both (mma.sync only)
        gp, _ = attention_groups(cq, ck, 128, 32)
        gt, _ = attention_groups(cq, ck, 128, 1)
        def rows(g, cu):
            return [int(cu[g[2 * i] + g[2 * i + 1]] - cu[g[2 * i]]) for i in range(len(g) // 2)]
        tc_seqs = {s for i in range(len(gt) // 2)
                   if rows(gt, cq)[i] <= 128 and rows(gt, ck)[i] <= 128
                   for s in range(gt[2 * i], gt[2 * i] + gt[2 * i + 1])}
        ms_seqs = {s for i in range(len(gp) // 2)
                   if not (rows(gp, cq)[i] <= 128 and rows(gp, ck)[i] <= 128)
                   for s in range(gp[2 * i], gp[2 * i] + gp[2 * i + 1])}
        assert tc_seqs | ms_seqs == set(range(n)) and not (tc_seqs & ms_seqs), trial


def test_attention_tables_one_call_matches_six():
    """mm_attention_tables (the staging path's single host call) == the six
    mm_attention_groups tables it stands for."""
    import numpy as np
    from paper_2403_07544_b200.engine import native_attention_groups
    L = _native.lib()
    rng = np.random.default_rng(11)
    for trial in range(50):
        n = int(rng.integers(1, 80))
        cs = np.concatenate([[0], np.cumsum(rng.integers(1, 200, n))]).astype(np.int32)
        ct = np.concatenate([[0], np.cumsum(rng.integers(1, 200, n))]).astype(np.int32)
        tab = np.empty(12 * n, dtype=np.int32)
        ng, foot = np.zeros(6, dtype=np.int32), np.zeros(6, dtype=np.int32)
        assert L.mm_attention_tables(cs.ctypes.data, ct.ctypes.data, n, 128, tab.ctypes.data,
                                     ng.ctypes.data, foot.ctypes.data) == 0
        for t, (q, k, align) in enumerate([(cs, cs, 32), (ct, ct, 32), (ct, cs, 32),
                                           (cs, cs, 1), (ct, ct, 1), (ct, cs, 1)]):
            g, f = native_attention_groups(q, k, 128, align)
            assert np.array_equal(tab[2 * n * t:2 * n * t + 2 * ng[t]], g) and foot[t] == f, (trial, t)


def _segments_ref(ids, chunk):
    """numpy restatement of mm_embed_segments (stable sort by id, chunks of
    <= chunk rows, partial slots numbered in chunk order)."""
    perm = np.argsort(ids, kind="stable")
    chunks, multi, slots = [], [], 0
    i = 0
    while i < len(perm):
        j = i
        while j < len(perm) and ids[perm[j]] == ids[perm[i]]:
            j += 1
        pieces = -(-(j - i) // chunk)
        if pieces > 1:
            multi.append((int(ids[perm[i]]), slots, pieces))
        for c in range(pieces):
            chunks.append((i + c * chunk, min(j, i + (c + 1) * chunk),
                           -(slots + c + 1) if pieces > 1 else int(ids[perm[i]])))
        slots += pieces if pieces > 1 else 0
        i = j
    return perm, chunks, multi


@pytest.mark.parametrize("rows,vocab", [(0, 10), (1, 10), (4096, 32000), (777, 50)])
def test_embed_segments_match_restatement(rows, vocab):
    """K8's deterministic scatter-add tables (host C++) vs numpy: Zipf-hot
    ids (one id over many chunks), all ids distinct, a single row, empty."""
    from paper_2403_07544_b200 import ops
    from paper_2403_07544_b200.data import ZipfIds
    rng = np.random.default_rng(rows)
    ids = ZipfIds(vocab, 1.1).draw(rng, rows) if rows else np.zeros(0, np.int32)
    tab, nc, nm = ops.embed_segments(ids)
    perm, chunks, multi = _segments_ref(ids, ops.EMB_CHUNK_ROWS)
    assert np.array_equal(tab[:rows], perm)
    assert nc == len(chunks) and nm == len(multi)
    assert [tuple(x) for x in tab[rows:rows + 3 * nc].reshape(-1, 3)] == chunks
    assert [tuple(x) for x in tab[rows + 3 * nc:].reshape(-1, 3)] == multi
    if rows == 4096:
        assert nm >= 1 and max(m[2] for m in multi) >= 10  # the hottest id spans many chunks

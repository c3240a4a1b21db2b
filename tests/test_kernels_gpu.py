"""Numerics of every CUDA kernel in libmmb200 against a plain PyTorch fp32
reference of the same op (bf16 inputs upcast to fp32)."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel_err(got, ref):
    got = got.float()
    ref = ref.float()
    return (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)


# every tile shape the launcher can pick: (CTAs per MMA, tile width); None =
# the launcher's own choice
TILES = [None, (1, 128), (1, 192), (1, 256), (2, 128), (2, 256)]


@pytest.fixture(params=TILES, ids=lambda t: "auto" if t is None else f"cg{t[0]}bn{t[1]}")
def tile(request, monkeypatch):
    if request.param is not None:
        monkeypatch.setenv("MM_GEMM_CG", str(request.param[0]))
        monkeypatch.setenv("MM_GEMM_BN", str(request.param[1]))
    return request.param


GEMM_SHAPES = [(128, 128, 64), (256, 512, 512), (296, 200, 136), (4096, 1536, 512),
               (1000, 2048, 512), (512, 512, 4096), (264, 32000, 512)]


@pytest.mark.parametrize("shape", GEMM_SHAPES)
@pytest.mark.parametrize("a_k,b_k", [(True, True), (True, False), (False, True), (False, False)])
def test_gemm_majors_f32(cuda, tile, shape, a_k, b_k):
    from paper_2403_07544_b200 import ops
    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = torch.randn(n, k, device=cuda, generator=g).bfloat16()
    a = A if a_k else A.t().contiguous()
    b = B if b_k else B.t().contiguous()
    d = torch.empty(m, n, device=cuda, dtype=torch.float32)
    ops.gemm(a, b, d, a_kmajor=a_k, b_kmajor=b_k, epilogue=ops.EPI_F32)
    ref = A.float() @ B.float().t()
    assert rel_err(d, ref) < 2e-3


@pytest.mark.parametrize("budget_mb", ["0.25", "1", "0"])
@pytest.mark.parametrize("shape", [(1000, 2048, 512), (4096, 1536, 1024), (512, 512, 4096)])
def test_gemm_grouped_unit_order(cuda, tile, shape, budget_mb, monkeypatch):
    """The L2-grouped unit order (M-tiles walked in groups when A outgrows
    the budget; small budgets force it at test sizes, including a partial
    last group) computes the same product as the plain M-first order."""
    from paper_2403_07544_b200 import ops
    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = torch.randn(n, k, device=cuda, generator=g).bfloat16()
    d = torch.empty(m, n, device=cuda, dtype=torch.float32)
    monkeypatch.setenv("MM_GEMM_L2_GROUP_MB", budget_mb)
    ops.gemm(A, B, d, epilogue=ops.EPI_F32)
    monkeypatch.setenv("MM_GEMM_L2_GROUP_MB", "0")
    d0 = torch.empty_like(d)
    ops.gemm(A, B, d0, epilogue=ops.EPI_F32)
    assert torch.equal(d, d0)
    assert rel_err(d, A.float() @ B.float().t()) < 2e-3


@pytest.mark.parametrize("shape", [(4096, 512, 512), (333, 1536, 512), (4096, 2048, 512)])
def test_gemm_epilogues(cuda, tile, shape):
    from paper_2403_07544_b200 import ops
    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = (torch.randn(n, k, device=cuda, generator=g) / math.sqrt(k)).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g)
    ref = A.float() @ B.float().t() + bias
    # bf16 + bias
    d = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
    ops.gemm(A, B, d, epilogue=ops.EPI_BF16, bias=bias)
    assert rel_err(d, ref) < 1e-2
    # bf16 relu
    ops.gemm(A, B, d, epilogue=ops.EPI_BF16_RELU, bias=bias)
    assert rel_err(d, ref.clamp_min(0)) < 1e-2
    # fp32 residual add, in place
    resid = torch.randn(m, n, device=cuda, generator=g)
    out = resid.clone()
    ops.gemm(A, B, out, epilogue=ops.EPI_F32_RESID, bias=bias, resid=out)
    assert rel_err(out, resid + ref) < 2e-3
    # the same with the first residual tiles fetched before griddepcontrol.wait
    # (the clone below is a torch kernel, which never releases its dependents early)
    out2 = resid.clone()
    ops.gemm(A, B, out2, epilogue=ops.EPI_F32_RESID, bias=bias, resid=out2, resid_early=True)
    assert torch.equal(out2, out)
    # relu-backward mask
    aux = torch.randn(m, n, device=cuda, generator=g).bfloat16()
    ops.gemm(A, B, d, epilogue=ops.EPI_BF16_DRELU, aux=aux)
    assert rel_err(d, (ref - bias) * (aux.float() > 0)) < 1e-2


@pytest.mark.parametrize("shape", [(4096, 2048, 512), (333, 1536, 512), (300, 200, 136)])
def test_gemm_relu_bitmask(cuda, tile, shape):
    """The 1-bit ReLU mask: EPI_BF16_RELU writes bit j of word (r, c) = the
    bf16 output (r, 32c + j) is non-zero; EPI_BF16_DRELU reading the mask is
    bit-identical to reading the bf16 activation (aux)."""
    from paper_2403_07544_b200 import ops
    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(n + k)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = (torch.randn(n, k, device=cuda, generator=g) / math.sqrt(k)).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g)
    f = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
    words = (n + 31) // 32
    mask = torch.full((m, words), -1, device=cuda, dtype=torch.int32)
    ops.gemm(A, B, f, epilogue=ops.EPI_BF16_RELU, bias=bias, relu_mask=mask)
    nz = torch.zeros(m, words * 32, dtype=torch.int64)
    nz[:, :n] = (f.cpu().view(torch.int16) != 0).long()
    want = (nz.view(m, words, 32) << torch.arange(32)).sum(-1)
    got = mask.cpu().long() & 0xFFFFFFFF
    assert torch.equal(got, want)
    dY = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    W = torch.randn(k, n, device=cuda, generator=g).bfloat16()  # dX = dY W, B MN-major
    d1 = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
    d2 = torch.empty_like(d1)
    ops.gemm(dY, W, d1, b_kmajor=False, epilogue=ops.EPI_BF16_DRELU, aux=f)
    ops.gemm(dY, W, d2, b_kmajor=False, epilogue=ops.EPI_BF16_DRELU, relu_mask=mask)
    assert torch.equal(d1, d2)
    assert rel_err(d1, (dY.float() @ W.float()) * (f.float() > 0)) < 1e-2


@pytest.mark.parametrize("shape", [(4096, 512, 512), (333, 512, 2048), (4100, 1024, 1024), (128, 512, 64)])
def test_gemm_fused_layernorm(cuda, shape):
    """MM_EPI_F32_RESID_LN: x = resid + A B^T + bias (fp32) and the following
    LayerNorm of x computed in the epilogue by a cluster of N/128 CTAs that
    exchange row sums through distributed shared memory."""
    from paper_2403_07544_b200 import ops
    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(21)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = (torch.randn(n, k, device=cuda, generator=g) / math.sqrt(k)).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g)
    resid = torch.randn(m, n, device=cuda, generator=g) * 3 + 1
    gamma = torch.rand(n, device=cuda, generator=g) + 0.5
    beta = torch.randn(n, device=cuda, generator=g)
    x = torch.empty(m, n, device=cuda)
    h = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
    mean = torch.empty(m, device=cuda)
    rstd = torch.empty(m, device=cuda)
    ops.gemm(A, B, x, epilogue=ops.EPI_F32_RESID_LN, bias=bias, resid=resid,
             ln=(gamma, beta, h, mean, rstd, 1e-6))
    ref_x = resid + A.float() @ B.float().t() + bias
    assert rel_err(x, ref_x) < 2e-3
    mu = x.mean(1)
    var = ((x - mu[:, None]) ** 2).mean(1)
    ref_rstd = torch.rsqrt(var + 1e-6)
    assert rel_err(mean, mu) < 1e-5
    assert rel_err(rstd, ref_rstd) < 1e-5
    ref_h = (x - mu[:, None]) * ref_rstd[:, None] * gamma + beta
    assert rel_err(h, ref_h) < 1e-2
    # identical to the standalone LayerNorm kernel on the same x
    h2 = torch.empty_like(h)
    m2, r2 = torch.empty_like(mean), torch.empty_like(rstd)
    ops.layernorm_fwd(x, gamma, beta, h2, m2, r2, eps=1e-6)
    assert rel_err(h, h2) < 1e-2 and rel_err(rstd, r2) < 1e-5


@pytest.mark.parametrize("shape", [(512, 512, 4096), (1536, 512, 4111), (32000, 512, 2048),
                                   (2048, 512, 300)])
def test_gemm_wgrad_accumulate(cuda, tile, shape):
    """dW += dY^T X with both operands MN-major (split-K, fp32 atomics)."""
    from paper_2403_07544_b200 import ops
    n_out, n_in, t = shape
    g = torch.Generator(device="cuda").manual_seed(5)
    dy = torch.randn(t, n_out, device=cuda, generator=g).bfloat16()
    x = torch.randn(t, n_in, device=cuda, generator=g).bfloat16()
    dw = torch.randn(n_out, n_in, device=cuda, generator=g)
    db = torch.randn(n_out, device=cuda, generator=g)
    ref = dw + dy.float().t() @ x.float()
    ref_b = db + dy.float().sum(0)
    ops.gemm(dy, x, dw, a_kmajor=False, b_kmajor=False, epilogue=ops.EPI_F32_ACCUM, dbias=db)
    assert rel_err(dw, ref) < 2e-3
    assert rel_err(db, ref_b) < 1e-4  # fused bias gradient (column sums of dY)


def test_gemm_grouped_wgrad(cuda, tile):
    """One grouped launch of a layer's worth of wgrads (mixed M, N, K; two
    problems accumulate into the same dW) == per-problem fp32 references."""
    from paper_2403_07544_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(11)
    shapes = [(512, 512, 4096), (1536, 512, 4096), (2048, 512, 4096), (512, 2048, 4096),
              (1024, 512, 333), (32000, 512, 1024), (200, 136, 64)]
    probs, refs = [], []
    for n_out, n_in, t in shapes:
        dy = torch.randn(t, n_out, device=cuda, generator=g).bfloat16()
        x = torch.randn(t, n_in, device=cuda, generator=g).bfloat16()
        dw = torch.randn(n_out, n_in, device=cuda, generator=g)
        db = torch.randn(n_out, device=cuda, generator=g)
        refs.append((dw, dw + dy.float().t() @ x.float(), db, db + dy.float().sum(0)))
        probs.append(dict(a=dy, b=x, d=dw, a_kmajor=False, b_kmajor=False,
                          epilogue=ops.EPI_F32_ACCUM, dbias=db))
    # a second contribution to problem 0's dW / db in the same launch
    dy2 = torch.randn(4096, 512, device=cuda, generator=g).bfloat16()
    x2 = torch.randn(4096, 512, device=cuda, generator=g).bfloat16()
    dw0, r0, db0, rb0 = refs[0]
    refs[0] = (dw0, r0 + dy2.float().t() @ x2.float(), db0, rb0 + dy2.float().sum(0))
    probs.append(dict(a=dy2, b=x2, d=dw0, a_kmajor=False, b_kmajor=False,
                      epilogue=ops.EPI_F32_ACCUM, dbias=db0))
    ops.gemm_grouped(probs)
    for dw, ref, db, ref_b in refs:
        assert rel_err(dw, ref) < 2e-3
        assert rel_err(db, ref_b) < 1e-4


def test_gemm_grouped_forward_epilogues(cuda, tile):
    """Grouped launch with a different epilogue per problem (K-major operands)."""
    from paper_2403_07544_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(12)
    probs, checks = [], []
    for i, (m, n, k) in enumerate([(4096, 1536, 512), (333, 512, 512), (4096, 2048, 512),
                                   (1000, 512, 2048)]):
        A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
        B = (torch.randn(n, k, device=cuda, generator=g) / math.sqrt(k)).bfloat16()
        bias = torch.randn(n, device=cuda, generator=g)
        ref = A.float() @ B.float().t() + bias
        if i % 2 == 0:
            d = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
            probs.append(dict(a=A, b=B, d=d, epilogue=ops.EPI_BF16_RELU, bias=bias))
            checks.append((d, ref.clamp_min(0), 1e-2))
        else:
            resid = torch.randn(m, n, device=cuda, generator=g)
            d = torch.empty(m, n, device=cuda)
            probs.append(dict(a=A, b=B, d=d, epilogue=ops.EPI_F32_RESID, bias=bias, resid=resid))
            checks.append((d, ref + resid, 2e-3))
    ops.gemm_grouped(probs)
    for d, ref, tol in checks:
        assert rel_err(d, ref) < tol


def test_gemm_grouped_rejects_mixed_majors(cuda):
    from paper_2403_07544_b200 import ops
    a = torch.zeros(128, 64, device=cuda, dtype=torch.bfloat16)
    d = torch.zeros(128, 128, device=cuda)
    with pytest.raises(RuntimeError, match="majorness"):
        ops.gemm_grouped([dict(a=a, b=a, d=d, epilogue=ops.EPI_F32),
                          dict(a=a.t().contiguous(), b=a, d=d, a_kmajor=False, epilogue=ops.EPI_F32)])


def test_layernorm(cuda):
    from paper_2403_07544_b200 import ops
    for cols in (64, 128, 512, 1024):  # 64: config 1's d_model (half-warp rows)
        rows = 1031
        g = torch.Generator(device="cuda").manual_seed(cols)
        x = torch.randn(rows, cols, device=cuda, generator=g) * 3 + 1
        gamma = torch.randn(cols, device=cuda, generator=g)
        beta = torch.randn(cols, device=cuda, generator=g)
        y = torch.empty(rows, cols, device=cuda, dtype=torch.bfloat16)
        mean = torch.empty(rows, device=cuda)
        rstd = torch.empty(rows, device=cuda)
        ops.layernorm_fwd(x, gamma, beta, y, mean, rstd, eps=1e-6)
        xr = x.clone().requires_grad_(True)
        gr = gamma.clone().requires_grad_(True)
        br = beta.clone().requires_grad_(True)
        ref = torch.nn.functional.layer_norm(xr, (cols,), gr, br, eps=1e-6)
        assert rel_err(y, ref) < 1e-2
        dy = torch.randn(rows, cols, device=cuda, generator=g)
        ref.backward(dy)
        dx = torch.randn(rows, cols, device=cuda, generator=g)
        dx0 = dx.clone()
        dxb = torch.empty(rows, cols, device=cuda, dtype=torch.bfloat16)
        dgamma = torch.zeros(cols, device=cuda)
        dbeta = torch.zeros(cols, device=cuda)
        ops.layernorm_bwd(dy, x, gamma, mean, rstd, dx, dxb, dgamma, dbeta)
        assert rel_err(dx - dx0, xr.grad) < 1e-4
        assert rel_err(dxb, dx) < 1e-2
        assert rel_err(dgamma, gr.grad) < 1e-4
        assert rel_err(dbeta, br.grad) < 1e-4


def sinusoid(pos, d):
    div = torch.exp(torch.arange(0, d, 2, dtype=torch.float32) * -(math.log(10000.0) / d))
    pe = torch.zeros(len(pos), d)
    pe[:, 0::2] = torch.sin(pos[:, None].float() * div)
    pe[:, 1::2] = torch.cos(pos[:, None].float() * div)
    return pe


def test_embedding(cuda):
    from paper_2403_07544_b200 import ops
    rows, vocab, d = 2000, 1000, 512
    g = torch.Generator().manual_seed(3)
    ids = torch.randint(0, vocab, (rows,), generator=g, dtype=torch.int32)
    ids[:300] = 7  # hot row
    pos = torch.randint(0, 128, (rows,), generator=g, dtype=torch.int32)
    table = torch.randn(vocab, d, generator=g).bfloat16()
    out = torch.empty(rows, d, device=cuda)
    scale = math.sqrt(d)
    ops.embed_fwd(ids.cuda(), pos.cuda(), table.cuda(), out, scale)
    ref = table.float()[ids.long()] * scale + sinusoid(pos, d)
    assert rel_err(out.cpu(), ref) < 1e-5
    dout = torch.randn(rows, d, generator=g)
    dtable = torch.zeros(vocab, d, device=cuda)
    ops.embed_bwd(ids.cuda(), dout.cuda(), dtable, scale)
    ref_d = torch.zeros(vocab, d).index_add_(0, ids.long(), dout * scale)
    assert rel_err(dtable.cpu(), ref_d) < 1e-5


@pytest.mark.parametrize("rows,d", [(4096, 512), (3000, 1024), (1, 128), (65, 256), (777, 64)])
def test_embedding_backward_sorted_deterministic(cuda, rows, d):
    """K8's sorted scatter-add (mm_embed_segments + mm_embed_bwd_sorted) on
    Zipf(1.1) ids: bit-exact against a numpy restatement of its summation
    order (scale 1: the kernel's fmaf(g, 1, acc) is an exact add), bitwise
    identical over repeated launches, and accumulating into a non-zero table;
    with scale sqrt(d) within 1e-6 of the fp64 index_add."""
    from paper_2403_07544_b200 import ops
    from paper_2403_07544_b200.data import ZipfIds
    rng = np.random.default_rng(rows)
    vocab = 32000
    ids = ZipfIds(vocab, 1.1).draw(rng, rows)
    tab, nc, nm = ops.embed_segments(ids)
    tab_d = torch.from_numpy(tab).to(cuda)
    dout = torch.from_numpy(rng.standard_normal((rows, d), dtype=np.float32)).to(cuda)
    base = torch.from_numpy(rng.standard_normal((vocab, d), dtype=np.float32)).to(cuda)
    scratch = torch.empty(max(nc, 1), d, device=cuda)
    outs = []
    for _ in range(3):
        t = base.clone()
        ops.embed_bwd_sorted(tab_d, rows, nc, nm, dout, t, 1.0, scratch)
        outs.append(t)
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    # numpy restatement: chunk partials in ascending row order, partials in chunk order
    g = dout.cpu().numpy()
    want = base.cpu().numpy().copy()
    perm = tab[:rows]
    chunks = tab[rows:rows + 3 * nc].reshape(-1, 3)
    partial = {}
    for b, e, tgt in chunks:
        acc = np.zeros(d, np.float32)
        for p in perm[b:e]:
            acc = acc + g[p]
        if tgt >= 0:
            want[tgt] = want[tgt] + acc
        else:
            partial[-tgt - 1] = acc
    for idv, s0, ns in tab[rows + 3 * nc:].reshape(-1, 3):
        acc = np.zeros(d, np.float32)
        for k in range(ns):
            acc = acc + partial[s0 + k]
        want[idv] = want[idv] + acc
    assert np.array_equal(outs[0].cpu().numpy(), want)
    t = torch.zeros(vocab, d, device=cuda)
    ops.embed_bwd_sorted(tab_d, rows, nc, nm, dout, t, math.sqrt(d), scratch)
    ref = np.zeros((vocab, d))
    np.add.at(ref, ids.astype(np.int64), g.astype(np.float64) * math.sqrt(d))
    assert np.abs(t.cpu().numpy() - ref).max() <= 1e-6 * np.abs(ref).max()


@pytest.mark.parametrize("rows,vocab", [(777, 32000), (300, 1000), (150, 40000), (2, 8), (513, 4096)])
def test_cross_entropy(cuda, rows, vocab):
    """Both kernels: the streamed one-CTA-per-SM kernel (vocab <= 32768) and
    the one-row-per-CTA fallback (larger vocabularies)."""
    from paper_2403_07544_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(9)
    logits = (torch.randn(rows, vocab, device=cuda, generator=g) * 4).bfloat16()
    labels = torch.randint(0, vocab, (rows,), device=cuda, generator=g, dtype=torch.int32)
    labels[min(5, rows - 1)] = -1
    dl = torch.empty_like(logits)
    loss = torch.empty(rows, device=cuda)
    scale = 1.0 / 700
    ops.xent(logits, labels, dl, loss, scale)
    lf = logits.float().requires_grad_(True)
    keep = labels >= 0
    ref_rows = torch.nn.functional.cross_entropy(lf, labels.long().clamp_min(0), reduction="none")
    ref_rows = ref_rows * keep
    (ref_rows.sum() * scale).backward()
    assert rel_err(loss, ref_rows) < 1e-5
    assert rel_err(dl, lf.grad) < 1e-2
    # in place
    ops.xent(logits, labels, logits, loss, scale)
    assert torch.equal(logits, dl)


def ref_attention(q, k, v, cu_q, cu_k, heads, causal):
    out = torch.zeros_like(q)
    for s in range(len(cu_q) - 1):
        qs, ks = slice(cu_q[s], cu_q[s + 1]), slice(cu_k[s], cu_k[s + 1])
        for h in range(heads):
            hs = slice(h * 64, (h + 1) * 64)
            sc = q[qs, hs] @ k[ks, hs].t() / 8.0
            if causal:
                lq, lk = sc.shape
                mask = torch.ones(lq, lk, dtype=torch.bool).triu(1)
                sc = sc.masked_fill(mask, float("-inf"))
            out[qs, hs] = torch.softmax(sc, -1) @ v[ks, hs]
    return out


def poison_smem(cuda):
    """Leave non-finite bit patterns in every SM's shared memory: the streamed
    cross-entropy kernel pads its row buffers with bf16 -inf.  Regression for
    attention backward reading D of padding rows from stale smem (0 * NaN)."""
    from paper_2403_07544_b200 import ops
    rows, vocab = 1024, 8
    logits = torch.zeros(rows, vocab, device=cuda, dtype=torch.bfloat16)
    labels = torch.zeros(rows, device=cuda, dtype=torch.int32)
    ops.xent(logits, labels, logits, torch.empty(rows, device=cuda), 1.0)


@pytest.mark.parametrize("tc_fwd", [False, True], ids=["fwd_mma_sync", "fwd_tcgen05"])
@pytest.mark.parametrize("causal,maxlen,maxk", [(True, 128, 128), (False, 128, 128), (True, 256, 256),
                                                (False, 256, 256), (False, 256, 100), (False, 90, 256)])
@pytest.mark.parametrize("long_path", ["tcgen05", "mma_sync"])
def test_attention(cuda, causal, maxlen, maxk, tc_fwd, long_path, monkeypatch):
    """Forward (tcgen05 by default, or the mma.sync kernel) and backward
    (tcgen05) vs an fp32 PyTorch reference; sequences past 128 rows (query
    side, key side or both) take the long-group tcgen05 kernels, or with
    long_path=mma_sync the previous mma.sync kernels."""
    if long_path == "mma_sync" and maxlen <= 128 and maxk <= 128:
        pytest.skip("no long groups")
    monkeypatch.setenv("MM_ATTN_TC_FWD", "1" if tc_fwd else "0")
    if long_path == "mma_sync":
        monkeypatch.setenv("MM_ATTN_LONG_MMA_SYNC", "1")
    else:
        monkeypatch.delenv("MM_ATTN_LONG_MMA_SYNC", raising=False)
    from paper_2403_07544_b200 import ops
    rng = np.random.default_rng(maxlen + causal + maxk)
    heads, d = 8, 512
    lq = rng.integers(1, maxlen + 1, size=13)
    lk = lq.copy() if causal else rng.integers(1, maxk + 1, size=13)
    if maxlen > 128:
        lq[3] = maxlen  # the clip's edge
    if maxk > 128:
        lk[7] = maxk
    if causal:
        lk = lq.copy()
    cu_q = np.concatenate([[0], np.cumsum(lq)]).astype(np.int32)
    cu_k = np.concatenate([[0], np.cumsum(lk)]).astype(np.int32)
    tq, tk = int(cu_q[-1]), int(cu_k[-1])
    g = torch.Generator().manual_seed(0)
    q = torch.randn(tq, d, generator=g).bfloat16().float()
    k = torch.randn(tk, d, generator=g).bfloat16().float()
    v = torch.randn(tk, d, generator=g).bfloat16().float()
    qr, kr, vr = (t.clone().requires_grad_(True) for t in (q, k, v))
    ref = ref_attention(qr, kr, vr, cu_q, cu_k, heads, causal)
    do = torch.randn(tq, d, generator=g).bfloat16().float()
    ref.backward(do)
    qd, kd, vd = (t.bfloat16().cuda() for t in (q, k, v))
    o = torch.empty(tq, d, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(heads, tq, device=cuda)
    cq, ck = torch.from_numpy(cu_q).cuda(), torch.from_numpy(cu_k).cuda()
    dq = torch.empty_like(qd)
    dk = torch.empty_like(kd)
    dv = torch.empty_like(vd)
    dod = do.bfloat16().cuda()
    args = ops.attention_args(qd, kd, vd, o, lse, cq, ck, 13, heads, int(lq.max()), int(lk.max()),
                              causal, d_o=dod, dq=dq, dk=dk, dv=dv)
    ops.attention_fwd(args)
    assert rel_err(o.cpu(), ref.detach()) < 1e-2
    poison_smem(cuda)
    ops.attention_bwd(args)
    for name, t in (("dq", dq), ("dk", dk), ("dv", dv)):
        bad = ~torch.isfinite(t)
        assert not bad.any(), (name, bad.sum().item(), bad.any(1).nonzero().flatten()[:10].tolist(),
                               bad.any(0).nonzero().flatten()[:10].tolist(), cu_q[:6].tolist(), cu_k[:6].tolist())
    assert rel_err(dq.cpu(), qr.grad) < 2e-2
    assert rel_err(dk.cpu(), kr.grad) < 2e-2
    assert rel_err(dv.cpu(), vr.grad) < 2e-2


@pytest.mark.parametrize("causal", [False, True])
def test_attention_many_long_groups(cuda, causal, monkeypatch):
    """Many sequences past 128 rows: the long-group kernels run one wave of
    persistent CTAs over the list of long groups (attention.cu collect_long),
    so each CTA takes several (head, group[, query block]) units in turn --
    40 long sequences x 8 heads = 640 forward / 320 backward units on 148
    CTAs, short sequences between them -- vs the fp32 reference."""
    monkeypatch.delenv("MM_ATTN_LONG_MMA_SYNC", raising=False)
    monkeypatch.setenv("MM_ATTN_TC_FWD", "1")
    from paper_2403_07544_b200 import ops
    rng = np.random.default_rng(11 + causal)
    heads, d, n = 8, 512, 60
    lq = rng.integers(129, 257, size=n)
    lq[rng.permutation(n)[:20]] = rng.integers(1, 129, size=20)  # 20 short ones between
    lk = lq.copy() if causal else np.where(lq > 128, rng.integers(1, 257, size=n), rng.integers(129, 257, size=n))
    cu_q = np.concatenate([[0], np.cumsum(lq)]).astype(np.int32)
    cu_k = np.concatenate([[0], np.cumsum(lk)]).astype(np.int32)
    tq, tk = int(cu_q[-1]), int(cu_k[-1])
    g = torch.Generator().manual_seed(1)
    q = torch.randn(tq, d, generator=g).bfloat16().float()
    k = torch.randn(tk, d, generator=g).bfloat16().float()
    v = torch.randn(tk, d, generator=g).bfloat16().float()
    qr, kr, vr = (t.clone().requires_grad_(True) for t in (q, k, v))
    ref = ref_attention(qr, kr, vr, cu_q, cu_k, heads, causal)
    do = torch.randn(tq, d, generator=g).bfloat16().float()
    ref.backward(do)
    qd, kd, vd = (t.bfloat16().cuda() for t in (q, k, v))
    o = torch.empty(tq, d, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(heads, tq, device=cuda)
    cq, ck = torch.from_numpy(cu_q).cuda(), torch.from_numpy(cu_k).cuda()
    dq, dk, dv = torch.empty_like(qd), torch.empty_like(kd), torch.empty_like(vd)
    args = ops.attention_args(qd, kd, vd, o, lse, cq, ck, n, heads, int(lq.max()), int(lk.max()),
                              causal, d_o=do.bfloat16().cuda(), dq=dq, dk=dk, dv=dv)
    ops.attention_fwd(args)
    assert rel_err(o.cpu(), ref.detach()) < 1e-2
    ops.attention_bwd(args)
    assert rel_err(dq.cpu(), qr.grad) < 2e-2
    assert rel_err(dk.cpu(), kr.grad) < 2e-2
    assert rel_err(dv.cpu(), vr.grad) < 2e-2


def test_colsum_and_cast(cuda):
    from paper_2403_07544_b200 import ops
    x = torch.randn(4097, 1536, device=cuda).bfloat16()
    out = torch.ones(1536, device=cuda)
    ops.colsum(x, out)
    assert rel_err(out, 1 + x.float().sum(0)) < 1e-4
    y = torch.randn(1000, 512, device=cuda)
    yb = torch.empty(1000, 512, device=cuda, dtype=torch.bfloat16)
    ops.cast_bf16(y, yb)
    assert torch.equal(yb, y.bfloat16())


@pytest.mark.parametrize("bn", ["128", "256"])
@pytest.mark.parametrize("shape,ak,bk", [((4096, 1536, 512), True, True), ((1000, 1280, 520), True, True),
                                         ((700, 384, 1024), True, False), ((512, 640, 2048), False, False)])
def test_gemm_pair_multicast_matches_unicast(cuda, shape, ak, bk, bn, monkeypatch):
    """CTA pairs in clusters of two pairs (each CTA fetches half of its A rows
    and multicasts it to the other pair; MM_GEMM_MC) give bit-identical
    results to unicast pairs: odd N-tile counts (the second pair's last tile
    outside N), ragged M / K, every operand majorness (bf16 out: an fp32
    weight-gradient-shaped output could split K, whose reduce-adds land in
    either order)."""
    from paper_2403_07544_b200 import ops
    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(m + n)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16() if ak else torch.randn(k, m, device=cuda, generator=g).bfloat16()
    B = torch.randn(n, k, device=cuda, generator=g).bfloat16() if bk else torch.randn(k, n, device=cuda, generator=g).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g)
    monkeypatch.setenv("MM_GEMM_CG", "2")
    monkeypatch.setenv("MM_GEMM_BN", bn)
    outs = []
    for mc in ("0", "1"):
        monkeypatch.setenv("MM_GEMM_MC", mc)
        d = torch.zeros(m, n, device=cuda, dtype=torch.bfloat16)
        ops.gemm(A, B, d, a_kmajor=ak, b_kmajor=bk, epilogue=ops.EPI_BF16, bias=bias)
        outs.append(d)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    ref = (A.float() if ak else A.float().t()) @ (B.float().t() if bk else B.float()) + bias
    assert rel_err(outs[1], ref) < 1e-2


@pytest.mark.parametrize("case", [
    # (a_kmajor, b_kmajor, epilogue, bn, cg): every specialised instantiation
    (True, True, "BF16", 128, 1), (True, True, "BF16_RELU", 128, 1), (True, True, "F32", 128, 1),
    (True, True, "F32_RESID", 128, 1), (True, False, "BF16", 128, 1), (True, False, "BF16_DRELU", 128, 1),
    (True, False, "F32", 128, 1), (True, False, "F32_ACCUM", 128, 1), (True, True, "BF16", 256, 1),
    (True, True, "BF16_RELU", 256, 1), (True, True, "F32_RESID", 256, 1), (True, False, "F32", 256, 1),
    (True, False, "BF16_DRELU", 256, 1), (True, True, "BF16", 256, 2), (True, False, "F32", 256, 2),
    (True, False, "F32", 128, 2)])
def test_gemm_specialised_matches_generic(cuda, case, monkeypatch):
    """The per-epilogue instantiations (MM_GEMM_SPECIALIZE) are bit-identical
    to the generic kernel on ragged shapes, with bias / residual / ReLU-mask
    operands as the epilogue takes them."""
    from paper_2403_07544_b200 import ops
    ak, bk, epi_name, bn, cg = case
    epi = getattr(ops, "EPI_" + epi_name)
    # (an fp32 accumulation with more k-blocks could split K, whose partial
    # sums reduce-add in either order)
    m, n, k = 1000, 520 if bn == 128 else 776, 136 if epi_name == "F32_ACCUM" else 392
    g = torch.Generator(device="cuda").manual_seed(bn + cg + epi)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = (torch.randn(n, k, device=cuda, generator=g) if bk else torch.randn(k, n, device=cuda, generator=g)).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g)
    resid = torch.randn(m, n, device=cuda, generator=g)
    mask = torch.randint(-2 ** 31, 2 ** 31 - 1, (m, (n + 31) // 32), device=cuda, dtype=torch.int32, generator=g)
    start = torch.randn(m, n, device=cuda, generator=g)
    monkeypatch.setenv("MM_GEMM_CG", str(cg))
    monkeypatch.setenv("MM_GEMM_BN", str(bn))
    outs = []
    for spec in ("0", "1"):
        monkeypatch.setenv("MM_GEMM_SPECIALIZE", spec)
        bf = epi in (ops.EPI_BF16, ops.EPI_BF16_RELU, ops.EPI_BF16_DRELU)
        d = torch.zeros(m, n, device=cuda, dtype=torch.bfloat16) if bf else start.clone()
        kw = {}
        if epi in (ops.EPI_BF16, ops.EPI_BF16_RELU, ops.EPI_F32, ops.EPI_F32_RESID):
            kw["bias"] = bias
        if epi == ops.EPI_F32_RESID:
            kw["resid"] = resid
        if epi in (ops.EPI_BF16_RELU, ops.EPI_BF16_DRELU):
            kw["relu_mask"] = mask if epi == ops.EPI_BF16_DRELU else torch.zeros_like(mask)
        ops.gemm(A, B, d, a_kmajor=ak, b_kmajor=bk, epilogue=epi, **kw)
        outs.append((d, kw.get("relu_mask")))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0])
    if epi == ops.EPI_BF16_RELU:
        assert torch.equal(outs[0][1], outs[1][1])

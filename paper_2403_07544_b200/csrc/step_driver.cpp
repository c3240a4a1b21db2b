// Native step driver: forward + backward of one task on one packed
// micro-batch, issuing every K4-K8 launch from C++ (the Python engine's
// Engine.forward_backward, without ~25 us of Python/ctypes per launch).
//
// Layer order (pre-LN, OpenNMT-py "standard"):
//   self block : x' = x + Attn(LN1(x)) Wo^T + bo
//   cross block: x' = x + CrossAttn(LNc(x), mem) Wco^T + bco     (decoder)
//   FFN block  : x' = x + relu(LN2(x) W1^T + b1) W2^T + b2
// Activations are bump-allocated from the caller's workspace.
//
// Weight gradients are off the backward critical path (nothing downstream
// reads dW until the optimizer), so the driver defers them: every wgrad of a
// side (decoder + generator, then encoder) is queued and issued as ONE grouped
// persistent GEMM launch when that side's backward is done.  Small per-layer
// wgrads (512x512 ... 2048x512, K = tokens) then share one unit list instead
// of paying a launch tail and a partial wave each.  The dY operands they read
// stay alive until the flush (per-block dx_bf copies, no temporaries
// released); MM_DEFER_WGRAD=0 restores eager wgrads with block-scoped
// temporaries.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mm_common.h"

namespace {

// diagnostics: CUDA events around the non-GEMM launches (mm_step_timing)
struct StepTiming {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<int> cat;
    size_t used = 0;
} g_step_timing;

struct TimedScope {
    cudaStream_t s;
    cudaEvent_t e1 = nullptr;
    TimedScope(int c, cudaStream_t st) : s(st) {
        StepTiming& t = g_step_timing;
        if (!t.on) return;
        while (t.ev.size() < 2 * (t.used + 1)) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            t.ev.push_back(e);
        }
        cudaEventRecord(t.ev[2 * t.used], s);
        e1 = t.ev[2 * t.used + 1];
        t.cat.resize(t.used + 1);
        t.cat[t.used] = c;
        ++t.used;
    }
    ~TimedScope() {
        if (e1) cudaEventRecord(e1, s);
    }
};

struct Arena {
    uint8_t* base = nullptr;
    size_t off = 0, peak = 0;
    bool sizing = true;
    template <class T>
    T* get(size_t n) {
        off = (off + 255) & ~size_t(255);
        T* p = sizing ? nullptr : reinterpret_cast<T*>(base + off);
        off += n * sizeof(T);
        if (off > peak) peak = off;
        return p;
    }
};

#define TIMED(c, expr)                             \
    do {                                           \
        if (!sizing) {                             \
            TimedScope _ts((c), s);                \
            int _st = (expr);                      \
            if (_st) return _st;                   \
        }                                          \
    } while (0)

#define TRY(expr)                    \
    do {                             \
        if (!sizing) {               \
            int _st = (expr);        \
            if (_st) return _st;     \
        }                            \
    } while (0)

struct SelfSave { const float* x_in; uint16_t* h; float* mean; float* rstd; uint16_t* qkv; uint16_t* a; float* lse; };
struct CrossSave { const float* x_in; uint16_t* h; float* mean; float* rstd; uint16_t* q; uint16_t* kv; uint16_t* a; float* lse; };
// MM_RELU_MASK=0: the ReLU-backward epilogue reads the bf16 activation (A/B)
static bool use_relu_mask() {
    static const bool on = [] {
        const char* e = std::getenv("MM_RELU_MASK");
        return !(e && e[0] == '0');
    }();
    return on;
}

struct FfnSave { const float* x_in; uint16_t* h; float* mean; float* rstd; uint16_t* f; uint32_t* mask; };

// A LayerNorm's outputs (bf16 normalised rows + per-row statistics), and the
// parameters of the LayerNorm that follows a residual GEMM
struct LnOut { uint16_t* h = nullptr; float* mean = nullptr; float* rstd = nullptr; };
struct LnNext { const mm_stack* st = nullptr; int64_t g = -1, b = -1; };

struct Layer {
    const mm_stack* st;
    const mm_layer_offsets* o;
    SelfSave self;
    CrossSave cross;
    FfnSave ffn;
};

struct Driver {
    const mm_task& t;
    const mm_batch& b;
    Arena& ar;
    cudaStream_t s;
    bool sizing;
    int d, H, F, V;

    const uint16_t* wb(const mm_stack* st, int64_t off) const { return st->w_bf16 + off; }
    const float* wf(const mm_stack* st, int64_t off) const { return st->w_f32 + off; }
    float* g(const mm_stack* st, int64_t off) const { return st->grad + off; }

    static mm_gemm_args make_args(const void* A, bool a_k, const void* B, bool b_k, void* D, int64_t m,
                                  int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldd, int epi,
                                  const float* bias = nullptr, const float* resid = nullptr,
                                  const void* aux = nullptr, float* dbias = nullptr) {
        mm_gemm_args a{};
        a.a = A; a.b = B; a.d = D; a.bias = bias; a.resid = resid; a.aux = aux; a.dbias = dbias;
        a.m = m; a.n = n; a.k = k; a.lda = lda; a.ldb = ldb; a.ldd = ldd;
        a.a_kmajor = a_k; a.b_kmajor = b_k; a.epilogue = epi;
        a.b_prefetch = 1;  // B is a weight or an earlier forward activation
        return a;
    }
    int gemm(const void* A, bool a_k, const void* B, bool b_k, void* D, int64_t m, int64_t n,
             int64_t k, int64_t lda, int64_t ldb, int64_t ldd, int epi, const float* bias = nullptr,
             const float* resid = nullptr, const void* aux = nullptr, float* dbias = nullptr) {
        const mm_gemm_args a = make_args(A, a_k, B, b_k, D, m, n, k, lda, ldb, ldd, epi, bias, resid, aux, dbias);
        return mm_gemm(&a, s);
    }
    // out[T,d] = resid + X W^T + bias; with `next`, the following LayerNorm of
    // out is computed in the GEMM epilogue (MM_EPI_F32_RESID_LN, a cluster of
    // d / 128 CTAs per row block) into *ln_out -- no separate LayerNorm pass
    bool fuse_ln = true;
    int residual(const uint16_t* X, const uint16_t* W, float* out, int64_t T, int64_t in,
                 const float* bias, const float* resid, const LnNext* next, LnOut* ln_out) {
        if (next && next->st) {
            ln_out->h = ar.get<uint16_t>(T * d);
            ln_out->mean = ar.get<float>(T);
            ln_out->rstd = ar.get<float>(T);
            if (fuse_ln && (d == 512 || d == 1024)) {
                mm_gemm_args a = make_args(X, true, W, true, out, T, d, in, in, in, d, MM_EPI_F32_RESID_LN,
                                           bias, resid);
                a.ln_gamma = wf(next->st, next->g);
                a.ln_beta = wf(next->st, next->b);
                a.ln_out = ln_out->h;
                a.ln_mean = ln_out->mean;
                a.ln_rstd = ln_out->rstd;
                a.ln_eps = 1e-6f;
                TRY(mm_gemm(&a, s));
                return 0;
            }
            TRY(linear(X, W, out, T, in, d, MM_EPI_F32_RESID, bias, resid));
            TIMED(0, mm_layernorm_fwd(out, wf(next->st, next->g), wf(next->st, next->b), ln_out->h,
                                      ln_out->mean, ln_out->rstd, T, d, 1e-6f, s));
            return 0;
        }
        TRY(linear(X, W, out, T, in, d, MM_EPI_F32_RESID, bias, resid));
        return 0;
    }
    // the block's input LayerNorm: already produced by the previous residual
    // GEMM (pre), or computed here
    int ln_in(const mm_stack* st, int64_t go, int64_t bo, const float* x, int64_t T, const LnOut* pre,
              uint16_t*& h, float*& mean, float*& rstd) {
        if (pre && pre->h) {
            h = pre->h; mean = pre->mean; rstd = pre->rstd;
            return 0;
        }
        return ln(st, go, bo, x, T, h, mean, rstd);
    }

    // dX[T,in] (epi)= dY[T,out] W[out,in] as a problem of a grouped launch
    static mm_gemm_args dgrad_args(const uint16_t* dY, const uint16_t* W, void* dX, int64_t T, int64_t in,
                                   int64_t out, int epi) {
        return make_args(dY, true, W, false, dX, T, in, out, out, in, in, epi);
    }
    // Y[T,out] (epi)= X[T,in] W[out,in]^T
    int linear(const uint16_t* X, const uint16_t* W, void* Y, int64_t T, int64_t in, int64_t out,
               int epi, const float* bias = nullptr, const float* resid = nullptr) {
        mm_gemm_args a = make_args(X, true, W, true, Y, T, out, in, in, in, out, epi, bias, resid);
        // every residual GEMM of the step reads a residual stream written at
        // least two kernels earlier (out-proj: the block input, then LN,
        // QKV, attention; cross out-proj: the self-attention output, then
        // LN, Q, cross attention; FFN-down: the attention output, then LN,
        // FFN-up), so its first residual tile is fetched before the wait
        a.resid_early = resid != nullptr && resid_early;
        return mm_gemm(&a, s);
    }
    bool resid_early = true;
    // dX[T,in] (epi)= dY[T,out] W[out,in]
    int dgrad(const uint16_t* dY, const uint16_t* W, void* dX, int64_t T, int64_t in, int64_t out,
              int epi, const void* aux = nullptr) {
        return gemm(dY, true, W, false, dX, T, in, out, out, in, in, epi, nullptr, nullptr, aux);
    }
    // dW[out,in] += dY[T,out]^T X[T,in] (store: dW = ..., the module's first
    // micro-batch of the step);  db[out] += sum_t dY[t,out] (fused)
    int wgrad(const uint16_t* dY, const uint16_t* X, float* dW, int64_t T, int64_t in, int64_t out,
              float* db, bool store) {
        mm_gemm_args a{};
        a.a = dY; a.b = X; a.d = dW; a.dbias = db;
        a.m = out; a.n = in; a.k = T; a.lda = out; a.ldb = in; a.ldd = in;
        a.a_kmajor = 0; a.b_kmajor = 0; a.epilogue = store ? MM_EPI_F32 : MM_EPI_F32_ACCUM;
        a.b_prefetch = 1;
        if (defer) {
            pending.push_back(a);
            return 0;
        }
        return mm_gemm(&a, s);
    }
    bool defer = true;
    std::vector<mm_gemm_args> pending;
    int flush_wgrads() {
        if (!sizing && !pending.empty()) {
            if (int st = mm_gemm_grouped(pending.data(), static_cast<int>(pending.size()), s)) return st;
        }
        pending.clear();
        return 0;
    }
    // block-scoped temporaries are released only when nothing deferred reads them
    void release(size_t mark) {
        if (!defer) ar.off = mark;
    }
    // buffer for dL/d(block input) in bf16: a fresh one per block while wgrads
    // are deferred (the queued wgrads of this block read the previous one)
    uint16_t* next_bf(uint16_t* cur, int64_t rows) { return defer ? ar.get<uint16_t>(rows * d) : cur; }

    int ln(const mm_stack* st, int64_t go, int64_t bo, const float* x, int64_t T, uint16_t*& y,
           float*& mean, float*& rstd) {
        y = ar.get<uint16_t>(T * d);
        mean = ar.get<float>(T);
        rstd = ar.get<float>(T);
        TIMED(0, mm_layernorm_fwd(x, wf(st, go), wf(st, bo), y, mean, rstd, T, d, 1e-6f, s));
        return 0;
    }

    mm_attn_args attn(const uint16_t* q, const uint16_t* k, const uint16_t* v, int64_t ldq,
                      int64_t ldkv, uint16_t* o, float* lse, const int32_t* cu_q,
                      const int32_t* cu_k, int max_q, int max_k, bool causal, int total_q,
                      const int32_t* groups, int ng, int cap, const int32_t* tcg = nullptr,
                      int ntc = 0) {
        mm_attn_args a{};
        a.tc_groups = tcg; a.n_tc_groups = ntc;
        a.q = q; a.k = k; a.v = v; a.o = o; a.lse = lse;
        a.cu_q = cu_q; a.cu_k = cu_k;
        a.ldq = ldq; a.ldk = ldkv; a.ldv = ldkv; a.ldo = d;
        a.n_seq = b.n_seq; a.heads = H; a.head_dim = d / H; a.causal = causal;
        a.max_q = max_q; a.max_k = max_k; a.scale = 1.f / std::sqrt(float(d / H)); a.total_q = total_q;
        a.groups = groups; a.n_groups = ng; a.cap = cap;
        a.total_k = cu_k == cu_q ? total_q : int(b.n_src);
        return a;
    }

    // ------------------------------------------------------------ forward
    int self_fwd(Layer& L, const float* x, float*& out, int64_t T, const int32_t* cu, int maxlen,
                 bool causal, const int32_t* groups, int ng, int cap, const int32_t* tcg, int ntc,
                 const LnOut* pre, const LnNext* next, LnOut* ln_out) {
        const mm_stack* st = L.st;
        const mm_layer_offsets* o = L.o;
        SelfSave& sv = L.self;
        sv.x_in = x;
        if (int e = ln_in(st, o->ln1_g, o->ln1_b, x, T, pre, sv.h, sv.mean, sv.rstd)) return e;
        sv.qkv = ar.get<uint16_t>(T * 3 * d);
        TRY(linear(sv.h, wb(st, o->qkv_w), sv.qkv, T, d, 3 * d, MM_EPI_BF16, wf(st, o->qkv_b)));
        sv.a = ar.get<uint16_t>(T * d);
        sv.lse = ar.get<float>(int64_t(H) * T);
        mm_attn_args a = attn(sv.qkv, sv.qkv + d, sv.qkv + 2 * d, 3 * d, 3 * d, sv.a, sv.lse, cu, cu,
                              maxlen, maxlen, causal, int(T), groups, ng, cap, tcg, ntc);
        a.v = sv.qkv + 2 * d;
        TIMED(2, mm_attention_fwd(&a, s));
        out = ar.get<float>(T * d);
        if (int e = residual(sv.a, wb(st, o->out_w), out, T, d, wf(st, o->out_b), x, next, ln_out)) return e;
        return 0;
    }

    int cross_fwd(Layer& L, const float* x, float*& out, const uint16_t* mem, const LnOut* pre,
                  const LnNext* next, LnOut* ln_out) {
        const mm_stack* st = L.st;
        const mm_layer_offsets* o = L.o;
        CrossSave& sv = L.cross;
        const int64_t T = b.n_tgt, S = b.n_src;
        sv.x_in = x;
        if (int e = ln_in(st, o->lnc_g, o->lnc_b, x, T, pre, sv.h, sv.mean, sv.rstd)) return e;
        sv.q = ar.get<uint16_t>(T * d);
        TRY(linear(sv.h, wb(st, o->cq_w), sv.q, T, d, d, MM_EPI_BF16, wf(st, o->cq_b)));
        // sv.kv: computed for every decoder layer in one grouped launch (kv_all)
        (void)mem; (void)S;
        sv.a = ar.get<uint16_t>(T * d);
        sv.lse = ar.get<float>(int64_t(H) * T);
        mm_attn_args a = attn(sv.q, sv.kv, sv.kv + d, d, 2 * d, sv.a, sv.lse, b.cu_tgt, b.cu_src,
                              b.max_tgt, b.max_src, false, int(T), b.groups_cross, b.ng_cross,
                              b.cap_cross, b.tcg_cross, b.ntc_cross);
        a.flags |= 4;  // K / V: the grouped projection of the encoder memory, launched before
        TIMED(2, mm_attention_fwd(&a, s));
        out = ar.get<float>(T * d);
        if (int e = residual(sv.a, wb(st, o->cout_w), out, T, d, wf(st, o->cout_b), x, next, ln_out)) return e;
        return 0;
    }

    int ffn_fwd(Layer& L, const float* x, float*& out, int64_t T, const LnOut* pre, const LnNext* next,
                LnOut* ln_out) {
        const mm_stack* st = L.st;
        const mm_layer_offsets* o = L.o;
        FfnSave& sv = L.ffn;
        sv.x_in = x;
        if (int e = ln_in(st, o->ln2_g, o->ln2_b, x, T, pre, sv.h, sv.mean, sv.rstd)) return e;
        sv.f = ar.get<uint16_t>(T * F);
        sv.mask = ar.get<uint32_t>(T * ((F + 31) / 32));  // 1-bit ReLU mask for the backward
        {
            mm_gemm_args a = make_args(sv.h, true, wb(st, o->ff1_w), true, sv.f, T, F, d, d, d, F,
                                       MM_EPI_BF16_RELU, wf(st, o->ff1_b));
            a.relu_mask = use_relu_mask() ? sv.mask : nullptr;
            TRY(mm_gemm(&a, s));
        }
        out = ar.get<float>(T * d);
        if (int e = residual(sv.f, wb(st, o->ff2_w), out, T, F, wf(st, o->ff2_b), x, next, ln_out)) return e;
        return 0;
    }

    // ------------------------------------------------------------ backward
    // dx (fp32) / dx_bf hold dL/d(block output) on entry, dL/d(block input) on exit
    int ffn_bwd(Layer& L, float* dx, uint16_t*& dx_bf, int64_t T) {
        const mm_stack* st = L.st;
        const mm_layer_offsets* o = L.o;
        FfnSave& sv = L.ffn;
        const size_t mark = ar.off;
        TRY(wgrad(dx_bf, sv.f, g(st, o->ff2_w), T, F, d, g(st, o->ff2_b), st->store_wgrad != 0));
        uint16_t* df = ar.get<uint16_t>(T * F);
        {
            mm_gemm_args a = make_args(dx_bf, true, wb(st, o->ff2_w), false, df, T, F, d, d, F, F,
                                       MM_EPI_BF16_DRELU, nullptr, nullptr, sv.f);
            a.relu_mask = use_relu_mask() ? sv.mask : nullptr;  // 1 bit per element instead of the bf16 activation
            TRY(mm_gemm(&a, s));
        }
        TRY(wgrad(df, sv.h, g(st, o->ff1_w), T, d, F, g(st, o->ff1_b), st->store_wgrad != 0));
        float* dh = ar.get<float>(T * d);
        TRY(dgrad(df, wb(st, o->ff1_w), dh, T, d, F, MM_EPI_F32));
        uint16_t* nbf = next_bf(dx_bf, T);
        TIMED(1, mm_layernorm_bwd(dh, sv.x_in, wf(st, o->ln2_g), sv.mean, sv.rstd, dx, nbf,
                             g(st, o->ln2_g), g(st, o->ln2_b), T, d, s));
        dx_bf = nbf;
        release(mark);
        return 0;
    }

    int self_bwd(Layer& L, float* dx, uint16_t*& dx_bf, int64_t T, const int32_t* cu, int maxlen,
                 bool causal, const int32_t* groups, int ng, int cap, const int32_t* tcg, int ntc) {
        const mm_stack* st = L.st;
        const mm_layer_offsets* o = L.o;
        SelfSave& sv = L.self;
        const size_t mark = ar.off;
        TRY(wgrad(dx_bf, sv.a, g(st, o->out_w), T, d, d, g(st, o->out_b), st->store_wgrad != 0));
        uint16_t* da = ar.get<uint16_t>(T * d);
        TRY(dgrad(dx_bf, wb(st, o->out_w), da, T, d, d, MM_EPI_BF16));
        uint16_t* dqkv = ar.get<uint16_t>(T * 3 * d);
        mm_attn_args a = attn(sv.qkv, sv.qkv + d, sv.qkv + 2 * d, 3 * d, 3 * d, sv.a, sv.lse, cu, cu,
                              maxlen, maxlen, causal, int(T), groups, ng, cap, tcg, ntc);
        a.d_o = da; a.dq = dqkv; a.dk = dqkv + d; a.dv = dqkv + 2 * d;
        a.ld_dq = a.ld_dk = a.ld_dv = 3 * d;
        a.flags |= 2;  // Q / K / V / lse come from the forward pass
        TIMED(3, mm_attention_bwd(&a, s));
        TRY(wgrad(dqkv, sv.h, g(st, o->qkv_w), T, d, 3 * d, g(st, o->qkv_b), st->store_wgrad != 0));
        float* dh = ar.get<float>(T * d);
        TRY(dgrad(dqkv, wb(st, o->qkv_w), dh, T, d, 3 * d, MM_EPI_F32));
        uint16_t* nbf = next_bf(dx_bf, T);
        TIMED(1, mm_layernorm_bwd(dh, sv.x_in, wf(st, o->ln1_g), sv.mean, sv.rstd, dx, nbf,
                             g(st, o->ln1_g), g(st, o->ln1_b), T, d, s));
        dx_bf = nbf;
        release(mark);
        return 0;
    }

    int cross_bwd(Layer& L, float* dx, uint16_t*& dx_bf, const uint16_t* mem, float* dmem) {
        const mm_stack* st = L.st;
        const mm_layer_offsets* o = L.o;
        CrossSave& sv = L.cross;
        const int64_t T = b.n_tgt, S = b.n_src;
        const size_t mark = ar.off;
        TRY(wgrad(dx_bf, sv.a, g(st, o->cout_w), T, d, d, g(st, o->cout_b), st->store_wgrad != 0));
        uint16_t* da = ar.get<uint16_t>(T * d);
        TRY(dgrad(dx_bf, wb(st, o->cout_w), da, T, d, d, MM_EPI_BF16));
        uint16_t* dq = ar.get<uint16_t>(T * d);
        uint16_t* dkv = ar.get<uint16_t>(S * 2 * d);
        mm_attn_args a = attn(sv.q, sv.kv, sv.kv + d, d, 2 * d, sv.a, sv.lse, b.cu_tgt, b.cu_src,
                              b.max_tgt, b.max_src, false, int(T), b.groups_cross, b.ng_cross,
                              b.cap_cross, b.tcg_cross, b.ntc_cross);
        a.d_o = da; a.dq = dq; a.dk = dkv; a.dv = dkv + d;
        a.ld_dq = d; a.ld_dk = a.ld_dv = 2 * d;
        a.flags |= 2;  // Q / K / V / lse come from the forward pass
        TIMED(3, mm_attention_bwd(&a, s));
        TRY(wgrad(dkv, mem, g(st, o->ckv_w), S, d, 2 * d, g(st, o->ckv_b), st->store_wgrad != 0));
        TRY(wgrad(dq, sv.h, g(st, o->cq_w), T, d, d, g(st, o->cq_b), st->store_wgrad != 0));
        float* dh = ar.get<float>(T * d);
        // the two independent dgrads of the block (memory side, query side)
        // share one grouped launch
        const mm_gemm_args dg[2] = {dgrad_args(dkv, wb(st, o->ckv_w), dmem, S, d, 2 * d, MM_EPI_F32_ACCUM),
                                    dgrad_args(dq, wb(st, o->cq_w), dh, T, d, d, MM_EPI_F32)};
        TRY(mm_gemm_grouped(dg, 2, s));
        uint16_t* nbf = next_bf(dx_bf, T);
        TIMED(1, mm_layernorm_bwd(dh, sv.x_in, wf(st, o->lnc_g), sv.mean, sv.rstd, dx, nbf,
                             g(st, o->lnc_g), g(st, o->lnc_b), T, d, s));
        dx_bf = nbf;
        release(mark);
        return 0;
    }

    int zeros(void* p, size_t bytes) {
        TIMED(6, mm_memset(p, 0, bytes, s));
        return 0;
    }

    // K8 scatter-add: deterministic sorted kernels when the batch carries
    // their tables (mm_embed_segments), else the atomic kernel
    int embed_bwd(const int32_t* table, int nch, int nmul, const int32_t* ids, const float* dout,
                  float* dtable, int64_t rows) {
        const float scale = std::sqrt(float(d));
        if (!table) {
            TIMED(5, mm_embed_bwd(ids, dout, dtable, rows, d, scale, s));
            return 0;
        }
        float* scratch = nmul ? ar.get<float>(size_t(nch) * d) : nullptr;
        TIMED(5, mm_embed_bwd_sorted(table, rows, nch, nmul, dout, dtable, d, scale, scratch, s));
        return 0;
    }

    cudaEvent_t dec_done = nullptr;

    int run(float* loss_sum) {
        const int64_t Ts = b.n_src, Tt = b.n_tgt;
        const float scale = std::sqrt(float(d));
        // host-side layer records (saved-activation pointers per layer)
        Layer enc_l[64], dec_l[64];
        int ne = 0, nd = 0;
        for (int i = 0; i < t.n_enc; ++i)
            for (int l = 0; l < t.enc[i].n_layers; ++l) enc_l[ne++] = Layer{&t.enc[i], &t.enc[i].layers[l], {}, {}, {}};
        for (int i = 0; i < t.n_dec; ++i)
            for (int l = 0; l < t.dec[i].n_layers; ++l) dec_l[nd++] = Layer{&t.dec[i], &t.dec[i].layers[l], {}, {}, {}};
        // ---- encoder
        float* x = ar.get<float>(Ts * d);
        TIMED(5, mm_embed_fwd(b.src, b.src_pos, t.enc_emb.w_bf16 + t.enc_emb.emb, x, Ts, d, scale, s));
        // every LayerNorm after a residual GEMM is fused into that GEMM: the
        // block's LN1 / LN2 / final LN outputs flow as LnOut between blocks
        const mm_stack* lnf_e = &t.enc[t.n_enc - 1];
        LnOut pre;  // LN1 of layer 0 runs standalone (its input is the embedding)
        for (int l = 0; l < ne; ++l) {
            float* y;
            LnOut ln2, next_out;
            const LnNext n2{enc_l[l].st, enc_l[l].o->ln2_g, enc_l[l].o->ln2_b};
            const LnNext n1 = l + 1 < ne ? LnNext{enc_l[l + 1].st, enc_l[l + 1].o->ln1_g, enc_l[l + 1].o->ln1_b}
                                         : LnNext{lnf_e, lnf_e->lnf_g, lnf_e->lnf_b};
            if (int e = self_fwd(enc_l[l], x, y, Ts, b.cu_src, b.max_src, false, b.groups_src, b.ng_src,
                                 b.cap_src, b.tcg_src, b.ntc_src, &pre, &n2, &ln2)) return e;
            if (int e = ffn_fwd(enc_l[l], y, x, Ts, &ln2, &n1, &next_out)) return e;
            pre = next_out;
        }
        uint16_t* mem = pre.h; float* mem_mean = pre.mean; float* mem_rstd = pre.rstd;
        const float* x_enc = x;
        // ---- decoder: every layer's cross-attention K/V projection of the
        // encoder memory in one grouped launch (they depend on mem only)
        {
            mm_gemm_args kv[64];
            for (int l = 0; l < nd; ++l) {
                CrossSave& sv = dec_l[l].cross;
                sv.kv = ar.get<uint16_t>(Ts * 2 * d);
                kv[l] = make_args(mem, true, wb(dec_l[l].st, dec_l[l].o->ckv_w), true, sv.kv, Ts, 2 * d, d,
                                  d, d, 2 * d, MM_EPI_BF16, wf(dec_l[l].st, dec_l[l].o->ckv_b));
            }
            TRY(mm_gemm_grouped(kv, nd, s));
        }
        float* y = ar.get<float>(Tt * d);
        TIMED(5, mm_embed_fwd(b.tgt_in, b.tgt_pos, t.dec_emb.w_bf16 + t.dec_emb.emb, y, Tt, d, scale, s));
        const mm_stack* lnf_d = &t.dec[t.n_dec - 1];
        LnOut dpre;
        for (int l = 0; l < nd; ++l) {
            float *y1, *y2;
            LnOut lnc, ln2, next_out;
            const LnNext nc{dec_l[l].st, dec_l[l].o->lnc_g, dec_l[l].o->lnc_b};
            const LnNext n2{dec_l[l].st, dec_l[l].o->ln2_g, dec_l[l].o->ln2_b};
            const LnNext n1 = l + 1 < nd ? LnNext{dec_l[l + 1].st, dec_l[l + 1].o->ln1_g, dec_l[l + 1].o->ln1_b}
                                         : LnNext{lnf_d, lnf_d->lnf_g, lnf_d->lnf_b};
            if (int e = self_fwd(dec_l[l], y, y1, Tt, b.cu_tgt, b.max_tgt, true, b.groups_tgt, b.ng_tgt,
                                 b.cap_tgt, b.tcg_tgt, b.ntc_tgt, &dpre, &nc, &lnc)) return e;
            if (int e = cross_fwd(dec_l[l], y1, y2, mem, &lnc, &n2, &ln2)) return e;
            if (int e = ffn_fwd(dec_l[l], y2, y, Tt, &ln2, &n1, &next_out)) return e;
            dpre = next_out;
        }
        uint16_t* hdec = dpre.h; float* hd_mean = dpre.mean; float* hd_rstd = dpre.rstd;
        uint16_t* logits = ar.get<uint16_t>(Tt * V);
        const mm_embed& E = t.dec_emb;
        TRY(linear(hdec, E.w_bf16 + E.gen_w, logits, Tt, d, V, MM_EPI_BF16, E.w_f32 + E.gen_b));
        float* row_loss = ar.get<float>(Tt);
        TIMED(4, mm_xent_fwd_bwd(logits, b.labels, logits, row_loss, loss_sum, Tt, V, 1.f / float(Tt), s));
        // ---- generator backward (dlogits in place of the logits)
        TRY(wgrad(logits, hdec, E.grad + E.gen_w, Tt, d, V, E.grad + E.gen_b, E.store_gen_w != 0));
        float* dh = ar.get<float>(Tt * d);
        TRY(dgrad(logits, E.w_bf16 + E.gen_w, dh, Tt, d, V, MM_EPI_F32));
        float* dy = ar.get<float>(Tt * d);
        uint16_t* dy_bf = ar.get<uint16_t>(Tt * d);
        if (int e = zeros(dy, Tt * d * 4)) return e;
        TIMED(1, mm_layernorm_bwd(dh, y, wf(lnf_d, lnf_d->lnf_g), hd_mean, hd_rstd, dy, dy_bf,
                             g(lnf_d, lnf_d->lnf_g), g(lnf_d, lnf_d->lnf_b), Tt, d, s));
        float* dmem = ar.get<float>(Ts * d);
        if (int e = zeros(dmem, Ts * d * 4)) return e;
        for (int l = nd - 1; l >= 0; --l) {
            if (int e = ffn_bwd(dec_l[l], dy, dy_bf, Tt)) return e;
            if (int e = cross_bwd(dec_l[l], dy, dy_bf, mem, dmem)) return e;
            if (int e = self_bwd(dec_l[l], dy, dy_bf, Tt, b.cu_tgt, b.max_tgt, true, b.groups_tgt, b.ng_tgt, b.cap_tgt,
                                 b.tcg_tgt, b.ntc_tgt)) return e;
        }
        if (int e = embed_bwd(b.emb_tgt, b.nch_tgt, b.nmul_tgt, b.tgt_in, dy,
                              t.dec_emb.grad + t.dec_emb.emb, Tt)) return e;
        if (int e = flush_wgrads()) return e;  // decoder side + generator
        if (dec_done && !sizing) MM_CUDA_TRY(cudaEventRecord(dec_done, s));
        // ---- encoder backward
        float* dx = ar.get<float>(Ts * d);
        uint16_t* dx_bf = ar.get<uint16_t>(Ts * d);
        if (int e = zeros(dx, Ts * d * 4)) return e;
        TIMED(1, mm_layernorm_bwd(dmem, x_enc, wf(lnf_e, lnf_e->lnf_g), mem_mean, mem_rstd, dx, dx_bf,
                             g(lnf_e, lnf_e->lnf_g), g(lnf_e, lnf_e->lnf_b), Ts, d, s));
        for (int l = ne - 1; l >= 0; --l) {
            if (int e = ffn_bwd(enc_l[l], dx, dx_bf, Ts)) return e;
            if (int e = self_bwd(enc_l[l], dx, dx_bf, Ts, b.cu_src, b.max_src, false, b.groups_src, b.ng_src, b.cap_src,
                                 b.tcg_src, b.ntc_src)) return e;
        }
        if (int e = embed_bwd(b.emb_src, b.nch_src, b.nmul_src, b.src, dx,
                              t.enc_emb.grad + t.enc_emb.emb, Ts)) return e;
        if (int e = flush_wgrads()) return e;  // encoder side
        return 0;
    }
};

}  // namespace

extern "C" int mm_step_timing(int mode, float* ms, int* launches) {
    StepTiming& t = g_step_timing;
    if (mode == 1) {
        t.on = true;
        t.used = 0;
        return 0;
    }
    t.on = false;
    for (int c = 0; c < 8; ++c) {
        if (ms) ms[c] = 0.f;
        if (launches) launches[c] = 0;
    }
    for (size_t i = 0; i < t.used; ++i) {
        MM_CUDA_TRY(cudaEventSynchronize(t.ev[2 * i + 1]));
        float x = 0.f;
        MM_CUDA_TRY(cudaEventElapsedTime(&x, t.ev[2 * i], t.ev[2 * i + 1]));
        const int c = t.cat[i] < 8 ? t.cat[i] : 7;
        if (ms) ms[c] += x;
        if (launches) launches[c] += 1;
    }
    t.used = 0;
    return 0;
}

extern "C" int mm_task_fwd_bwd(const mm_task* task, const mm_batch* batch, void* workspace,
                               size_t* ws_bytes, float* loss_sum, void* stream, void* dec_done) {
    MM_CHECK_ARG(task && batch && ws_bytes, "NULL argument");
    MM_CHECK_ARG(task->n_enc >= 1 && task->n_dec >= 1 && task->enc && task->dec, "empty task");
    MM_CHECK_ARG(task->heads > 0 && task->d_model % task->heads == 0 &&
                     (task->d_model / task->heads == 64 || task->d_model / task->heads == 32 ||
                      task->d_model / task->heads == 16),
                 "head_dim must be 16, 32 or 64 (d_model %d, heads %d)", task->d_model, task->heads);
    int nl = 0;
    for (int i = 0; i < task->n_enc; ++i) nl += task->enc[i].n_layers;
    MM_CHECK_ARG(nl <= 64, "more than 64 encoder layers");
    nl = 0;
    for (int i = 0; i < task->n_dec; ++i) nl += task->dec[i].n_layers;
    MM_CHECK_ARG(nl <= 64, "more than 64 decoder layers");
    MM_CHECK_ARG(task->enc[task->n_enc - 1].lnf_g >= 0 && task->dec[task->n_dec - 1].lnf_g >= 0,
                 "last stack of each side needs its final LayerNorm");
    static const bool defer = [] {
        const char* e = std::getenv("MM_DEFER_WGRAD");
        return !(e && e[0] == '0');
    }();
    // MM_FUSE_LN=1: LayerNorm fused into the residual GEMM (cluster + DSMEM row
    // statistics).  Off by default: measured slower than GEMM + standalone
    // LayerNorm on B200 (4096x512x512: 13.2 vs 12.3 us -- the 4-CTA cluster
    // launch costs ~1 us, the cross-CTA exchange ~2 us waiting for the slowest
    // tile of the cluster; at d = 1024 only 16 clusters of 8 are co-resident,
    // so the persistent grid runs in two waves; tools/ln_fuse_micro.py)
    const bool fuse_ln = [] {  // read per call (tests toggle it)
        const char* e = std::getenv("MM_FUSE_LN");
        return e && e[0] == '1';
    }();
    // MM_RESID_EARLY=0 (A/B): residual tiles only after griddepcontrol.wait
    const bool resid_early = [] {
        const char* e = std::getenv("MM_RESID_EARLY");
        return !(e && e[0] == '0');
    }();
    Arena ar;
    ar.base = static_cast<uint8_t*>(workspace);
    ar.sizing = workspace == nullptr;
    Driver drv{*task, *batch, ar, mm::as_stream(stream), ar.sizing, task->d_model, task->heads,
               task->ffn, task->vocab};
    if (!ar.sizing) {
        // dry run first: the caller's workspace must cover the peak
        Arena probe;
        Driver p{*task, *batch, probe, mm::as_stream(stream), true, task->d_model, task->heads,
                 task->ffn, task->vocab};
        p.defer = defer;
        p.fuse_ln = fuse_ln;
        p.run(loss_sum);
        MM_CHECK_ARG(probe.peak <= *ws_bytes, "workspace %zu B < required %zu B", *ws_bytes,
                     probe.peak);
    }
    drv.dec_done = static_cast<cudaEvent_t>(dec_done);
    drv.defer = defer;
    drv.fuse_ln = fuse_ln;
    drv.resid_early = resid_early;
    const int st = drv.run(loss_sum);
    if (ar.sizing) *ws_bytes = ar.peak;
    return st;
}

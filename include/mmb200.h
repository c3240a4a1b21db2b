/*
 * mmb200.h -- C ABI of libmmb200.so, the B200-native engine for MAMMOTH's
 * modular-training hot path (arXiv 2403.07544, Algorithm 1).
 *
 * Plain C: pointers, sizes and opaque handles only.  Device pointers come
 * from the caller (PyTorch owns device memory and streams); `stream` is a
 * cudaStream_t passed as void*.  Every call returns 0 on success and a
 * negative code on failure (-1 argument, -2 CUDA, -3 NCCL, -4 unsupported);
 * mm_last_error() returns the message of the calling thread's last failure.
 *
 * Reference interfaces each entry point replaces are cited per declaration
 * (paths relative to the reference tree, pkg/src/mmtplan/...).
 */
#ifndef MMB200_H
#define MMB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMB200_ABI_VERSION 24
#define MM_MAX_GROUP 8 /* one 8-GPU box: a module group has at most 8 ranks */
/* emulated devices of one sync (mm_sync_emulated): the reference's multi-node
 * scaling harness reaches 20 devices per group (syncsim.py:461-483) */
#define MM_MAX_SYNC_GROUP 32

int mm_abi_version(void);
/* sizeof(T) of the descriptor struct named T (e.g. "mm_sync_module"), -1 if
 * unknown: lets a binding check its struct mirrors against this build. */
long long mm_abi_sizeof(const char* name);
const char* mm_last_error(void);
/* SM count and compute capability (major*10+minor) of the current device. */
int mm_device_info(int* sm_count, int* cc);
/* Number of kernels this library has launched since load (all entry points). */
unsigned long long mm_launch_count(void);

/* ---------------------------------------------------------------------------
 * K9: allocator communication cost.  Same arguments, loop order and float64
 * accumulation as comm_cost_kernel (_speedups.pyx:11-57, twin _cost_py.py:11-48),
 * called by CostContext.cost (allocator.py:101-111).  Host code.
 */
int mm_comm_cost(const double* params, int64_t n_modules, const int64_t* mod_task_off,
                 const int64_t* mod_task_idx, const int64_t* task_dev,
                 const int64_t* dev_node, int64_t n_devices, double w_intra, double w_inter,
                 double* out_per_module, double* total);
/* f3: totals of n_moves candidate moves of one placement,
 * evaluated in parallel on n_threads host threads (0 = all cores).  Move i
 * is moves[3i..3i+2] = (kind, x, y): kind 0 relocates task x to device y,
 * kind 1 swaps the devices of tasks x and y.  out[i] is bit-identical to
 * mm_comm_cost's total on the moved placement, so a batched first-
 * improvement search (allocator.local_search_batched) accepts exactly the
 * moves of local_search (allocator.py:284-331). */
int mm_comm_cost_moves(const double* params, int64_t n_modules, const int64_t* mod_task_off,
                       const int64_t* mod_task_idx, const int64_t* task_dev, int64_t n_tasks,
                       const int64_t* dev_node, int64_t n_devices, double w_intra, double w_inter,
                       const int64_t* moves, int64_t n_moves, double* out, int n_threads);

/* ---------------------------------------------------------------------------
 * Algorithm 1 over emulated devices that share one GPU: the literal
 * sync_step(devices) of syncsim.py:121-153.  For every module: n = popcount
 * (used_mask); n == 0 -> buffers untouched, `out` zero-filled; otherwise
 * total = sum of member buffers in ascending member order (fp32), total /= n,
 * installed into every member buffer (and `out` if non-NULL).
 * only_ready != 0 sums only members whose used bit is set (exact when unused
 * buffers are zero, which DeviceState.reset guarantees, syncsim.py:108-111).
 */
typedef struct {
    float* bufs[MM_MAX_SYNC_GROUP]; /* member buffers, ascending device index */
    float* out;                /* optional synced copy, may be NULL */
    int64_t n_elems;
    int32_t group_size;
    uint32_t used_mask; /* bit r: member r used the module this step */
} mm_sync_module;

int mm_sync_emulated(const mm_sync_module* mods, int n_mods, int only_ready, void* stream);
/* The same over float64 buffers (the reference DeviceState's default dtype,
 * syncsim.py:103-106): bufs / out address doubles; IEEE double adds in
 * ascending member order, correctly rounded division. */
int mm_sync_emulated_f64(const mm_sync_module* mods, int n_mods, int only_ready, void* stream);

/* ---------------------------------------------------------------------------
 * K3: fused masked rescale + loss unscale + Adam + bf16 parameter cast on a
 * flat per-module bucket.  g = grad / n * inv_loss_scale (the "/ n_j" of
 * Algorithm 1, syncsim.py:149); modules with n == 0 are skipped
 * entirely (no optimizer step).  n is read from ready_dev[ready_index]
 * when ready_dev != NULL and ready_index >= 0, else from n_ready.
 * Adam follows torch.optim.Adam's update form (bias corrections folded into
 * step_size = lr / (1 - beta1^t) and inv_sqrt_bc2 = 1 / sqrt(1 - beta2^t)).
 */
typedef struct {
    float* grad; /* read (and zeroed when mm_adam_hyper.zero_grad) */
    float* master;
    float* exp_avg;
    float* exp_avg_sq;
    uint16_t* param_bf16; /* may be NULL */
    int64_t n_elems;
    int32_t n_ready;
    int32_t ready_index;
    float step_size;
    float inv_sqrt_bc2;
} mm_adam_module;

typedef struct {
    float beta1, beta2, eps, weight_decay, inv_loss_scale;
    float one_minus_beta1, one_minus_beta2; /* computed in double on the host */
    int32_t max_ctas; /* 0: one CTA per 16K-element chunk; > 0: persistent CTAs
                         (a thin background update overlapping other kernels) */
    int32_t zero_grad; /* 1: write 0 to every gradient element it consumed, so the
                          bucket is clean for the next step without a memset pass */
} mm_adam_hyper;

int mm_fused_update(const mm_adam_module* mods, int n_mods, const mm_adam_hyper* hyper,
                    const int32_t* ready_dev, void* stream);

/* ---------------------------------------------------------------------------
 * K1/K2: module-group communicators over NCCL (NVLink 5 / NVSwitch).
 * Replaces the in-process loops of sync_step (syncsim.py:140-152) and the
 * group map of run_benchmark (syncsim.py:337-340).
 */
int mm_nccl_unique_id(char out[128]);
/* World communicator for `rank` of `world` on CUDA device `device`. */
int mm_comm_init(int rank, int world, const char uid[128], int device, void** ctx);
int mm_comm_destroy(void* ctx);
/* Collective over the world communicator: every rank calls it with the same
 * member list (ascending ranks) in the same order.  *grp = NULL for
 * non-members and for singleton groups (they never communicate). */
int mm_group_create(void* ctx, const int* ranks, int n, void** grp);
int mm_group_destroy(void* grp);
/* Ready-count exchange: n_dev[m] = sum over ranks of flags_dev[m] (int32).
 * Non-hosting ranks contribute 0, so the world sum is the group sum. */
int mm_ready_count(void* ctx, const int32_t* flags_dev, int32_t* n_dev, int n_modules,
                   void* stream);

typedef struct {
    void* group;     /* from mm_group_create; NULL items are skipped */
    void* buf;       /* in place */
    int64_t n_elems; /* mode 0: elements; modes 1 / 2: g * shard (the padded bucket) */
    int32_t dtype;   /* 0 = fp32, 1 = bf16 */
    int32_t root;    /* mode 0: -1 sum-allreduce; >= 0: only that group rank used the
                        module (n = 1), so its buffer already is the sum: broadcast */
    int32_t mode;    /* 0 = allreduce / broadcast; 1 = reduce-scatter (group rank j
                        receives the sum of shard j at buf + j * shard); 2 = all-gather
                        (group rank j contributes buf + j * shard) */
    int32_t pad_;
    int64_t shard;   /* modes 1 / 2: elements per group rank */
} mm_reduce_item;

/* Every item on its group communicator, issued in array order (callers pass
 * sorted ModuleKey order) inside one ncclGroupStart/End: mode 0 sum-allreduce
 * (or, for n = 1, broadcast from the one ready member); modes 1 / 2 the
 * partitioned exchange (reduce-scatter of the gradient bucket, owner-shard
 * K3, all-gather of the bf16 weights), SURVEY §8(e). */
int mm_reduce_modules(void* ctx, const mm_reduce_item* items, int n, void* stream);

/* ---------------------------------------------------------------------------
 * Option B of SURVEY §8(f) f1: K2 + K3 + the parameter all-gather as ONE
 * streaming kernel over NVLink peer memory.  A module of group size g is cut
 * into g contiguous shards; member r owns shard r and, for it:
 *   total = sum over READY members j (ascending) of grad_j[shard]   -- masked
 *           peer loads: unused members' buckets are never read, so they
 *           need no zero fill (the 0 of Algorithm 1);
 *   g = total / n * inv_loss_scale   (syncsim.py:148-149);
 *   Adam on the owner's master / exp_avg / exp_avg_sq shard;
 *   bf16(master) stored into EVERY member's weight bucket (the all-gather);
 *   master fp32 also stored into other members' masters where non-NULL.
 * Results are bit-identical to mm_sync_emulated(only_ready=1) followed by
 * mm_fused_update (n_ready = 1) on the synced buffer.  mm_adam_hyper.zero_grad
 * zeroes each ready member's shard after it is read (each element of each
 * bucket has exactly one reader, its shard owner).  Peer pointers are CUDA-IPC mappings
 * (mm_ipc_import) of the other ranks' buckets; with every "rank" resident on
 * one GPU (tests, the config-2 bench) they are plain device pointers and one
 * launch covers every member's shard -- the same kernel, no flag waits.
 * Cross-rank ordering is by mm_peer_barrier before (gradients final) and
 * after (peers done reading / writing this rank's buckets).
 */
typedef struct {
    float* grad[MM_MAX_GROUP];      /* members' fp32 gradient buckets (whole module) */
    uint16_t* param[MM_MAX_GROUP];  /* members' bf16 weight buckets, NULL = skip */
    float* master_copy[MM_MAX_GROUP]; /* other members' fp32 masters, NULL = skip */
    float* master;                  /* owner's fp32 master (whole module) */
    float* exp_avg;
    float* exp_avg_sq;
    int64_t begin, end;             /* owned element range [begin, end) of the module */
    int32_t group_size;
    uint32_t ready_mask;            /* bit j: member j used the module this step */
    float step_size, inv_sqrt_bc2;  /* as mm_adam_module */
} mm_peer_shard;

/* Shard r of g over n elements: [r*S, min(n, (r+1)*S)), S = ceil(n / g)
 * rounded up to a multiple of 4 elements (16-byte vectors). */
int64_t mm_peer_shard_begin(int64_t n_elems, int group_size, int member);

int mm_peer_update(const mm_peer_shard* shards, int n, const mm_adam_hyper* hyper, void* stream);

#define MM_PEER_MAX_RANKS 32
/* Flag barrier over NVLink peer memory: for every peer i, store `epoch` into
 * peer_flags[i][my_rank] (st.release.sys), then wait until
 * local_flags[peer_rank[i]] >= epoch (ld.acquire.sys).  local_flags is this
 * rank's MM_PEER_MAX_RANKS-entry uint32 array; peers hold IPC mappings of it.
 * Epochs increase monotonically per rank pair.  A wait longer than
 * timeout_ms traps (a CUDA error on the stream, never a silent hang). */
typedef struct {
    uint32_t* local_flags;
    uint32_t* peer_flags[MM_PEER_MAX_RANKS];
    int32_t peer_rank[MM_PEER_MAX_RANKS];
    int32_t n_peers;
    int32_t my_rank;
    uint32_t epoch;
    int32_t timeout_ms;
} mm_peer_signal;

int mm_peer_barrier(const mm_peer_signal* sig, void* stream);

/* CUDA IPC for peer buckets.  export: handle of the allocation holding `ptr`
 * and ptr's byte offset in it; import: map a peer's allocation (once per
 * allocation, refcounted) and return base + offset; release: drop one
 * reference of the mapping that holds `ptr`. */
int mm_ipc_export(const void* ptr, uint8_t handle[64], uint64_t* offset);
int mm_ipc_import(const uint8_t handle[64], uint64_t offset, void** ptr);
int mm_ipc_release(void* ptr);

/* ---------------------------------------------------------------------------
 * K4: bf16 GEMM on tcgen05 tensor cores (TMA-staged operands, fp32 TMEM
 * accumulator).  D[M,N] = A[M,K] * B[N,K]^T with per-operand major-ness:
 *   a_kmajor: A stored [M,K] row-major (lda = row stride) else [K,M];
 *   b_kmajor: B stored [N,K] row-major else [K,N].
 * Epilogues: see MM_EPI_*.  Replaces the toy W @ h of forward / local_backward
 * (syncsim.py:55-87) with the transformer contractions.
 */
enum {
    MM_EPI_BF16 = 0,        /* D_bf16 = acc (+bias) */
    MM_EPI_BF16_RELU = 1,   /* D_bf16 = relu(acc + bias) */
    MM_EPI_F32 = 2,         /* D_f32 = acc (+bias) */
    MM_EPI_F32_ACCUM = 3,   /* D_f32 += acc */
    MM_EPI_F32_RESID = 4,   /* D_f32 = resid_f32 + acc + bias (resid may alias D) */
    MM_EPI_BF16_DRELU = 5,  /* D_bf16 = acc * (aux_bf16 > 0) */
    /* D_f32 = resid + acc + bias, then the following LayerNorm of every row of
     * D: ln_out_bf16 = (D - mean) * rstd * ln_gamma + ln_beta, ln_mean / ln_rstd
     * per row.  N in {512, 1024}: the N / 128 CTAs of a thread-block cluster
     * each own 128 columns of a row block and exchange per-row partial sums
     * through distributed shared memory (replaces mm_layernorm_fwd after a
     * residual GEMM).  K-major A and B, single (non-grouped) launches. */
    MM_EPI_F32_RESID_LN = 6
};

typedef struct {
    const void* a;      /* bf16 */
    const void* b;      /* bf16 */
    void* d;            /* bf16 or fp32 per epilogue */
    const float* bias;  /* [N] or NULL */
    const float* resid; /* MM_EPI_F32_RESID */
    const void* aux;    /* MM_EPI_BF16_DRELU mask source, bf16 [M, ldd] */
    int64_t m, n, k;
    int64_t lda, ldb, ldd; /* row strides in elements */
    int32_t a_kmajor, b_kmajor;
    int32_t epilogue;
    /* 1: B was not written by the immediately preceding kernel on the stream
     * (weights; earlier activations), so its first stages may be fetched
     * before griddepcontrol.wait */
    int32_t b_prefetch;
    /* optional: dbias[m] += sum_k A[m, k] (the bias gradient of a wgrad
     * dW = dY^T X, whose A operand is dY); requires MN-major A */
    float* dbias;
    /* MM_EPI_F32_RESID_LN: LayerNorm parameters and outputs (row stride n) */
    const float* ln_gamma;
    const float* ln_beta;
    void* ln_out;       /* bf16 [M, N] */
    float* ln_mean;     /* [M] */
    float* ln_rstd;     /* [M] */
    float ln_eps;
    /* optional 1-bit ReLU mask, [M, ceil(N / 32)] uint32 words, bit j of word
     * (r, c) = column 32c + j: written by MM_EPI_BF16_RELU (bit = the bf16
     * output is non-zero), read by MM_EPI_BF16_DRELU instead of `aux` (16x
     * fewer bytes than the bf16 activation) */
    uint32_t* relu_mask;
    /* 1: `resid` was not written by the immediately preceding kernel on the
     * stream (with programmatic dependent launch every kernel of the library
     * signals its dependents only after its own griddepcontrol.wait, so data
     * of the kernel before that is complete), so a CTA's first residual tile
     * may be fetched before griddepcontrol.wait */
    int32_t resid_early;
    int32_t pad_;
} mm_gemm_args;

int mm_gemm(const mm_gemm_args* args, void* stream);
/* n independent GEMMs in one persistent launch (one unit list, one tile
 * width); all problems share a_kmajor / b_kmajor.  Used for the deferred
 * weight-gradient GEMMs of a whole encoder or decoder side. */
int mm_gemm_grouped(const mm_gemm_args* probs, int n, void* stream);
/* mode 1: every later mm_gemm launch records its own span on the device
 * (%globaltimer of the first CTA past griddepcontrol.wait -> the last CTA's
 * exit; no events between kernels, programmatic dependent launch unchanged);
 * mode 0 (after the caller synchronised): stop and return total flops
 * (2MNK), summed launch spans (ms) and launch count since the last start. */
int mm_gemm_timing(int mode, double* flops, float* ms, int* launches);
/* diagnostics, after mm_gemm_timing(0): per-launch spans (ns, %globaltimer)
 * lo[i] / hi[i], flops[i] and shape[4i..4i+3] = m, n, k of the launch's
 * first problem and its problem count, for up to max launches. */
int mm_gemm_spans(int max, unsigned long long* lo, unsigned long long* hi, double* flops,
                  int* shape, int* count);
/* diagnostics: per-CTA %globaltimer stamps of every later mm_gemm launch into
 * dev_buf[8 * cta + slot] (NULL disables); see gemm.cu for the slots */
int mm_gemm_trace(unsigned long long* dev_buf);
/* Host: greedy packing of consecutive sequences into attention work groups
 * (<= cap rows per side, each sequence rounded up to `align` rows: 32 for
 * the mma.sync kernels' shared-memory tiles, 1 for the tcgen05 backward);
 * out holds 2 * n_seq int32 (first, count) pairs; *foot = rows of the
 * largest group.  Replaces the per-batch numpy loop of
 * data.attention_groups on the step's host path. */
int mm_attention_groups(const int32_t* cu_q, const int32_t* cu_k, int n_seq, int cap, int align,
                        int32_t* out, int* n_groups, int* foot);
/* Host: the six tables of a packed batch in one call -- {self source, self
 * target, cross (q = target, k = source)} x {align 32, align 1}; table t at
 * out + 2 * n_seq * t, n_groups[t], foot[t]. */
int mm_attention_tables(const int32_t* cu_src, const int32_t* cu_tgt, int n_seq, int cap,
                        int32_t* out, int* n_groups, int* foot);
/* Host: an order of a batch's n sentence pairs (source / target lengths)
 * that packs into few attention groups: first-fit-decreasing 2-D bins of
 * `cap` rows per side, bins in creation order, over-long pairs last.
 * perm[j] = input index of the j-th pair (data.attention_order). */
int mm_attention_order(const int32_t* len_s, const int32_t* len_t, int n, int cap, int32_t* perm);
/* diagnostics: mode 1 starts recording CUDA events around the non-GEMM
 * launches mm_task_fwd_bwd issues; mode 0 stops, synchronises and returns the
 * summed time (ms) and launch count per category: 0 LayerNorm fwd, 1 LayerNorm
 * bwd, 2 attention fwd, 3 attention bwd, 4 cross-entropy, 5 embedding,
 * 6 memset, 7 other (8 entries each). */
int mm_step_timing(int mode, float* ms, int* launches);

/* ---------------------------------------------------------------------------
 * K6: LayerNorm over rows of x (fp32 residual stream) -> bf16, saving
 * per-row mean / rstd; backward accumulates into dx (fp32) and writes its
 * bf16 copy, and accumulates dgamma / dbeta (fp32).
 */
int mm_layernorm_fwd(const float* x, const float* gamma, const float* beta, uint16_t* y,
                     float* mean, float* rstd, int64_t rows, int cols, float eps, void* stream);
int mm_layernorm_bwd(const float* dy, const float* x, const float* gamma, const float* mean,
                     const float* rstd, float* dx, uint16_t* dx_bf16, float* dgamma,
                     float* dbeta, int64_t rows, int cols, void* stream);

/* K8: embedding gather with scale + sinusoidal position, and its scatter-add. */
int mm_embed_fwd(const int32_t* ids, const int32_t* pos, const uint16_t* table, float* out,
                 int64_t rows, int cols, float scale, void* stream);
int mm_embed_bwd(const int32_t* ids, const float* dout, float* dtable, int64_t rows, int cols,
                 float scale, void* stream);
/* Deterministic scatter-add of the same sum (no atomics, fixed order):
 * `table` = mm_embed_segments' output for the batch's ids (device copy),
 * scratch >= (chunks of multi-chunk ids) * cols floats. */
int mm_embed_bwd_sorted(const int32_t* table, int64_t rows, int n_chunks, int n_multi,
                        const float* dout, float* dtable, int cols, float scale, float* scratch,
                        void* stream);
/* Host: the sort / chunk tables of mm_embed_bwd_sorted for `rows` token ids
 * (chunk_rows in [1, 32]; out: 7 * rows int32; see abi_host.cpp). */
int mm_embed_segments(const int32_t* ids, int rows, int chunk_rows, int32_t* out, int* n_chunks,
                      int* n_multi);

/* K5: packed varlen multi-head attention (bf16 in/out, fp32 softmax).
 * head_dim 64: tcgen05 kernels; head_dim 16 / 32 (config 1's d64 / 4 heads):
 * CUDA-core kernels (attn_small.cu) on the same arguments.
 * Work is split into CTA groups of consecutive sequences: groups[2g] = first
 * sequence, groups[2g+1] = count; every sequence occupies ceil(len/32)*32
 * rows of the group's shared-memory tile and the per-group footprint is at
 * most `cap` rows on each of the query and key sides (host-built, see
 * data.attention_groups). */
typedef struct {
    const uint16_t* q; const uint16_t* k; const uint16_t* v; /* [tokens, ld*] */
    uint16_t* o;                                              /* [tq, ldo] */
    float* lse;                                               /* [heads, tq] */
    const uint16_t* d_o;                                      /* backward */
    uint16_t* dq; uint16_t* dk; uint16_t* dv;                 /* backward */
    const int32_t* cu_q; const int32_t* cu_k;                 /* [n_seq+1] */
    int64_t ldq, ldk, ldv, ldo, ld_dq, ld_dk, ld_dv;
    int32_t n_seq, heads, head_dim, causal;
    int32_t max_q, max_k;
    float scale;
    int32_t total_q;
    const int32_t* groups; /* [2 * n_groups] */
    int32_t n_groups;
    int32_t cap;
    int32_t total_k;       /* key rows (the K / V tensors' extent, for TMA maps) */
    int32_t flags;         /* bit 1 (2): q / k / v / lse were complete before the
                              previous kernel on the stream started (backward:
                              the forward pass's tensors), so the tcgen05
                              backward may load them before griddepcontrol.wait;
                              bit 2 (4): the same for k / v of a forward call
                              (cross attention); bit 0 is internal */
    /* optional: the same sequences packed WITHOUT the 32-row padding
     * (mm_attention_groups with align = 1) for the tcgen05 backward, whose
     * units load one contiguous 128-row box per side; NULL = use `groups`.
     * Fewer, fuller units: 56 -> ~35 groups per config-3 table. */
    const int32_t* tc_groups;
    int32_t n_tc_groups;
    int32_t pad0;
} mm_attn_args;

int mm_attention_fwd(const mm_attn_args* a, void* stream);
int mm_attention_bwd(const mm_attn_args* a, void* stream);

/* K7: softmax cross-entropy over bf16 logits; writes dlogits (bf16, in place
 * allowed) scaled by grad_scale, per-row loss (fp32) and, if loss_sum is not
 * NULL, adds every row's loss times grad_scale to *loss_sum (the token mean
 * for grad_scale = 1/rows).  Labels < 0 are padding.
 * Replaces loss() of the toy model (syncsim.py:67-69). */
int mm_xent_fwd_bwd(const uint16_t* logits, const int32_t* labels, uint16_t* dlogits,
                    float* row_loss, float* loss_sum, int64_t rows, int vocab, float grad_scale,
                    void* stream);

/* ---------------------------------------------------------------------------
 * Native step driver: forward + backward of one task on one packed
 * micro-batch (the per-rank compute of run_benchmark's loop,
 * syncsim.py:352-360, with the toy chain replaced by the transformer
 * modules).  Issues every K4-K8 launch from C++ on `stream`; gradients
 * accumulate into the modules' grad buckets; the token-mean loss is added to
 * *loss_sum.  Offsets are in elements from the module's flat base pointers
 * (-1 = absent).  Activations live in a caller-provided workspace; call with
 * workspace == NULL to get the required size in *ws_bytes.
 */
typedef struct {
    int64_t ln1_g, ln1_b, qkv_w, qkv_b, out_w, out_b;
    int64_t lnc_g, lnc_b, cq_w, cq_b, ckv_w, ckv_b, cout_w, cout_b; /* decoder only */
    int64_t ln2_g, ln2_b, ff1_w, ff1_b, ff2_w, ff2_b;
} mm_layer_offsets;

typedef struct {
    const uint16_t* w_bf16; /* bf16 weight copy */
    const float* w_f32;     /* fp32 master (LayerNorm and bias parameters) */
    float* grad;            /* fp32 grad bucket */
    const mm_layer_offsets* layers; /* [n_layers], host memory */
    int32_t n_layers;
    int32_t decoder;
    int64_t lnf_g, lnf_b;   /* final LayerNorm, -1 if absent */
    int32_t store_wgrad;    /* 1: the weight-matrix gradients are STORED (this
                               micro-batch is the module's first of the step;
                               the caller zeroed only the rest of the bucket),
                               0: reduce-added onto the bucket */
    int32_t pad_;
} mm_stack;

typedef struct {
    const uint16_t* w_bf16;
    const float* w_f32;
    float* grad;
    int64_t emb, gen_w, gen_b; /* gen_* only for the decoder-side module */
    int32_t store_gen_w;       /* as mm_stack.store_wgrad, for the generator matrix */
    int32_t pad_;
} mm_embed;

typedef struct {
    int32_t d_model, heads, ffn, vocab;
    int32_t n_enc, n_dec;
    const mm_stack* enc; /* [n_enc], forward order */
    const mm_stack* dec; /* [n_dec] */
    mm_embed enc_emb, dec_emb;
} mm_task;

typedef struct {
    const int32_t *src, *src_pos, *cu_src, *tgt_in, *tgt_pos, *labels, *cu_tgt; /* device */
    const int32_t *groups_src, *groups_tgt, *groups_cross;                     /* device */
    int32_t n_seq, n_src, n_tgt, max_src, max_tgt;
    int32_t ng_src, cap_src, ng_tgt, cap_tgt, ng_cross, cap_cross;
    const int32_t *tcg_src, *tcg_tgt, *tcg_cross; /* unpadded groups (align 1), may be NULL */
    int32_t ntc_src, ntc_tgt, ntc_cross, pad0;
    /* mm_embed_segments tables of src / tgt_in (device), NULL: atomic scatter-add */
    const int32_t *emb_src, *emb_tgt;
    int32_t nch_src, nmul_src, nch_tgt, nmul_tgt;
} mm_batch;

/* dec_done (cudaEvent_t, may be NULL) is recorded on `stream` as soon as the
 * decoder-side gradients (decoder stacks, target embedding, generator) are
 * final, i.e. before the encoder backward: their exchange and update can
 * start on another stream while the encoder backward runs. */
int mm_task_fwd_bwd(const mm_task* task, const mm_batch* batch, void* workspace,
                    size_t* ws_bytes, float* loss_sum, void* stream, void* dec_done);

/* helpers */
/* out[c] += sum over rows of x[r, c] (bf16 in, fp32 accumulate) */
int mm_colsum_bf16(const uint16_t* x, float* out, int64_t rows, int cols, void* stream);
int mm_cast_f32_bf16(const float* x, uint16_t* y, int64_t n, void* stream);
/* y = (float) x, bf16 -> fp32 (n % 4 == 0): the bf16 gradient wire's way back */
int mm_cast_bf16_f32(const uint16_t* x, float* y, int64_t n, void* stream);
int mm_flush_l2(void* scratch, size_t bytes, void* stream);
/* y += alpha * x (fp32): DeviceState.accumulate (syncsim.py:113-118) */
int mm_axpy_f32(float* y, const float* x, float alpha, int64_t n, void* stream);
int mm_axpy_f64(double* y, const double* x, double alpha, int64_t n, void* stream);
/* stream-ordered byte fill (DeviceState.reset of the grad buckets, syncsim.py:108-111) */
int mm_memset(void* ptr, int value, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MMB200_H */

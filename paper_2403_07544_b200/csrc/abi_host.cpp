// Host-side entry points of libmmb200: version / error reporting, device
// info, K9 (the allocator's communication-cost kernel) and the attention
// work-group packing of a micro-batch.
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "mm_common.h"

namespace mm {

std::atomic<unsigned long long> g_launches{0};

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

bool pdl_enabled() {
    static const bool on = std::getenv("MM_NO_PDL") == nullptr;
    return on;
}

int num_sms() {
    static int cached = 0;
    if (cached == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
    }
    return cached;
}

}  // namespace mm

extern "C" int mm_abi_version(void) { return MMB200_ABI_VERSION; }

// sizeof of every descriptor struct of include/mmb200.h, by name (the
// binding's ctypes mirrors are checked against these), -1 if unknown
extern "C" long long mm_abi_sizeof(const char* name) {
    if (!name) return -1;
    const std::string n(name);
#define MM_SZ(T) if (n == #T) return static_cast<long long>(sizeof(T));
    MM_SZ(mm_sync_module) MM_SZ(mm_adam_module) MM_SZ(mm_adam_hyper) MM_SZ(mm_reduce_item)
    MM_SZ(mm_peer_shard) MM_SZ(mm_peer_signal) MM_SZ(mm_gemm_args) MM_SZ(mm_attn_args)
    MM_SZ(mm_layer_offsets) MM_SZ(mm_stack) MM_SZ(mm_embed) MM_SZ(mm_task) MM_SZ(mm_batch)
#undef MM_SZ
    return -1;
}

extern "C" unsigned long long mm_launch_count(void) { return mm::g_launches.load(); }

extern "C" const char* mm_last_error(void) { return mm::g_last_error.c_str(); }

extern "C" int mm_device_info(int* sm_count, int* cc) {
    int dev = 0;
    MM_CUDA_TRY(cudaGetDevice(&dev));
    cudaDeviceProp p;
    MM_CUDA_TRY(cudaGetDeviceProperties(&p, dev));
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (cc) *cc = p.major * 10 + p.minor;
    return 0;
}

// K9.  For every module (CSR row m) count the distinct devices and distinct
// nodes its tasks sit on, using "stamp" arrays keyed by the module index, and
// charge params[m] * (w_intra*(n_dev-1) + (w_inter-w_intra)*(n_node-1)).
// The float64 expression and the summation order over m are those of
// _speedups.pyx:38-57, so totals are bit-identical and local_search's strict
// comparisons (allocator.py:306,323) decide the same way.
extern "C" int mm_comm_cost(const double* params, int64_t n_modules, const int64_t* mod_task_off,
                            const int64_t* mod_task_idx, const int64_t* task_dev,
                            const int64_t* dev_node, int64_t n_devices, double w_intra,
                            double w_inter, double* out_per_module, double* total) {
    MM_CHECK_ARG(n_modules >= 0 && n_devices >= 0, "negative sizes");
    MM_CHECK_ARG(total != nullptr, "total is NULL");
    if (n_modules > 0) {
        MM_CHECK_ARG(params && mod_task_off && out_per_module, "NULL module arrays");
    }
    int64_t max_node = 0;
    for (int64_t i = 0; i < n_devices; ++i) max_node = std::max(max_node, dev_node[i]);
    // stamps start at -1 so module 0 is distinguishable from "never seen"
    std::vector<int64_t> dev_seen(static_cast<size_t>(n_devices), -1);
    std::vector<int64_t> node_seen(static_cast<size_t>(max_node + 1), -1);
    double acc = 0.0;
    for (int64_t m = 0; m < n_modules; ++m) {
        int64_t nd = 0, nn = 0;
        for (int64_t j = mod_task_off[m]; j < mod_task_off[m + 1]; ++j) {
            const int64_t d = task_dev[mod_task_idx[j]];
            if (d < 0 || d >= n_devices) {
                mm::set_error("task device %lld outside [0,%lld)", (long long)d,
                              (long long)n_devices);
                return mm::kArg;
            }
            if (dev_seen[d] == m) continue;
            dev_seen[d] = m;
            ++nd;
            const int64_t node = dev_node[d];
            if (node_seen[node] != m) {
                node_seen[node] = m;
                ++nn;
            }
        }
        const double c = nd > 0 ? params[m] * (w_intra * (double)(nd - 1) +
                                                (w_inter - w_intra) * (double)(nn - 1))
                                : 0.0;
        out_per_module[m] = c;
        acc += c;
    }
    *total = acc;
    return 0;
}

// f3: cost of many candidate moves of one placement, on host threads.  Each
// worker owns a copy of task_dev and the stamp arrays, applies a move, runs
// the same loop as mm_comm_cost and reverts -- bit-identical totals, so the
// batched local search accepts exactly the moves the sequential one does.
namespace {
double cost_of(const double* params, int64_t n_modules, const int64_t* off, const int64_t* idx,
               const int64_t* task_dev, const int64_t* dev_node, double w_intra, double w_inter,
               std::vector<int64_t>& dev_seen, std::vector<int64_t>& node_seen, int64_t stamp0) {
    double acc = 0.0;
    for (int64_t m = 0; m < n_modules; ++m) {
        const int64_t st = stamp0 + m;
        int64_t nd = 0, nn = 0;
        for (int64_t j = off[m]; j < off[m + 1]; ++j) {
            const int64_t d = task_dev[idx[j]];
            if (dev_seen[d] == st) continue;
            dev_seen[d] = st;
            ++nd;
            const int64_t node = dev_node[d];
            if (node_seen[node] != st) {
                node_seen[node] = st;
                ++nn;
            }
        }
        acc += nd > 0 ? params[m] * (w_intra * (double)(nd - 1) + (w_inter - w_intra) * (double)(nn - 1))
                      : 0.0;
    }
    return acc;
}
}  // namespace

extern "C" int mm_comm_cost_moves(const double* params, int64_t n_modules,
                                  const int64_t* mod_task_off, const int64_t* mod_task_idx,
                                  const int64_t* task_dev, int64_t n_tasks, const int64_t* dev_node,
                                  int64_t n_devices, double w_intra, double w_inter,
                                  const int64_t* moves, int64_t n_moves, double* out,
                                  int n_threads) {
    MM_CHECK_ARG(n_modules >= 0 && n_devices > 0 && n_tasks >= 0 && n_moves >= 0, "bad sizes");
    MM_CHECK_ARG(n_moves == 0 || (moves && out), "NULL move arrays");
    MM_CHECK_ARG(n_modules == 0 || (params && mod_task_off && mod_task_idx), "NULL module arrays");
    MM_CHECK_ARG(n_tasks == 0 || task_dev, "NULL task_dev");
    for (int64_t i = 0; i < n_tasks; ++i)
        MM_CHECK_ARG(task_dev[i] >= 0 && task_dev[i] < n_devices, "task %lld on device %lld",
                     (long long)i, (long long)task_dev[i]);
    for (int64_t i = 0; i < n_moves; ++i) {
        const int64_t k = moves[3 * i], x = moves[3 * i + 1], y = moves[3 * i + 2];
        MM_CHECK_ARG((k == 0 || k == 1) && x >= 0 && x < n_tasks, "move %lld malformed", (long long)i);
        MM_CHECK_ARG(k == 0 ? (y >= 0 && y < n_devices) : (y >= 0 && y < n_tasks),
                     "move %lld target out of range", (long long)i);
    }
    int64_t max_node = 0;
    for (int64_t i = 0; i < n_devices; ++i) max_node = std::max(max_node, dev_node[i]);
    int T = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::min<int64_t>(T, std::max<int64_t>(1, n_moves / 4));
    auto work = [&](int t) {
        std::vector<int64_t> dev(task_dev, task_dev + n_tasks);
        std::vector<int64_t> dev_seen((size_t)n_devices, -1), node_seen((size_t)max_node + 1, -1);
        int64_t stamp = 0;
        for (int64_t i = t; i < n_moves; i += T) {
            const int64_t k = moves[3 * i], x = moves[3 * i + 1], y = moves[3 * i + 2];
            if (k == 0) {
                const int64_t src = dev[x];
                dev[x] = y;
                out[i] = cost_of(params, n_modules, mod_task_off, mod_task_idx, dev.data(),
                                 dev_node, w_intra, w_inter, dev_seen, node_seen, stamp);
                dev[x] = src;
            } else {
                std::swap(dev[x], dev[y]);
                out[i] = cost_of(params, n_modules, mod_task_off, mod_task_idx, dev.data(),
                                 dev_node, w_intra, w_inter, dev_seen, node_seen, stamp);
                std::swap(dev[x], dev[y]);
            }
            stamp += n_modules;  // fresh stamps: no reset of the seen arrays
        }
    };
    if (T == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    return 0;
}

// All six work-group tables of a packed batch in one host call (the staging
// path of every step): {self source, self target, cross} x {32-row aligned
// (mma.sync), unpadded (tcgen05)}; table t is written at out + 2 * n_seq * t.
extern "C" int mm_attention_tables(const int32_t* cu_src, const int32_t* cu_tgt, int n_seq, int cap,
                                   int32_t* out, int* n_groups, int* foot) {
    MM_CHECK_ARG(cu_src && cu_tgt && out && n_groups && foot, "NULL argument");
    const int32_t* q[3] = {cu_src, cu_tgt, cu_tgt};
    const int32_t* k[3] = {cu_src, cu_tgt, cu_src};
    for (int t = 0; t < 6; ++t) {
        const int side = t % 3, align = t < 3 ? 32 : 1;
        if (int st = mm_attention_groups(q[side], k[side], n_seq, cap, align,
                                         out + int64_t(2) * n_seq * t, n_groups + t, foot + t))
            return st;
    }
    return 0;
}

// Deterministic embedding backward (K8): the rows of a batch sorted by token
// id (stable: ascending row within an id) and cut into chunks of at most
// `chunk_rows` rows of one id.  out = [perm: rows][chunks: 3 per chunk]
// [multi: 3 per id with > 1 chunk]; a chunk is (perm begin, perm end,
// target): target >= 0 is the id itself (its only chunk adds straight into
// the table row), target < 0 is -(scratch slot + 1) (one partial per chunk);
// a multi entry is (id, first slot, slots): the partials are summed in chunk
// order.  Capacity of out: 7 * rows int32.
extern "C" int mm_embed_segments(const int32_t* ids, int rows, int chunk_rows, int32_t* out,
                                 int* n_chunks, int* n_multi) {
    MM_CHECK_ARG(rows >= 0 && chunk_rows >= 1 && chunk_rows <= 32 && out && n_chunks && n_multi &&
                     (rows == 0 || ids),
                 "bad arguments (chunk_rows must be in [1, 32])");
    std::vector<uint64_t> key(rows);
    for (int r = 0; r < rows; ++r) {
        MM_CHECK_ARG(ids[r] >= 0, "negative token id at row %d", r);
        key[r] = (uint64_t(uint32_t(ids[r])) << 32) | uint32_t(r);
    }
    std::sort(key.begin(), key.end());
    int32_t* perm = out;
    for (int r = 0; r < rows; ++r) perm[r] = int32_t(key[r] & 0xffffffffu);
    int32_t* chunks = out + rows;
    std::vector<int32_t> multi;
    int nc = 0, slots = 0;
    for (int a = 0; a < rows;) {
        const int32_t id = int32_t(key[a] >> 32);
        int b = a;
        while (b < rows && int32_t(key[b] >> 32) == id) ++b;
        const int pieces = (b - a + chunk_rows - 1) / chunk_rows;
        if (pieces > 1) multi.insert(multi.end(), {id, slots, pieces});
        for (int c = 0; c < pieces; ++c) {
            chunks[3 * nc] = a + c * chunk_rows;
            chunks[3 * nc + 1] = std::min(b, a + (c + 1) * chunk_rows);
            chunks[3 * nc + 2] = pieces > 1 ? -(slots + c + 1) : id;
            ++nc;
        }
        if (pieces > 1) slots += pieces;
        a = b;
    }
    std::copy(multi.begin(), multi.end(), chunks + 3 * nc);
    *n_chunks = nc;
    *n_multi = int(multi.size() / 3);
    return 0;
}

// Order of a batch's sentence pairs for the attention work groups: first-fit
// decreasing 2-D bin packing (capacity `cap` rows on both the source and the
// target side), bins emitted in creation order, pairs longer than `cap` on
// either side last in input order.  Consecutive packing (mm_attention_groups)
// of this order needs no more groups than FFD has bins -- for config 3 about
// 34 instead of ~41 cross-attention groups in input order.  The order only
// permutes independent sentence pairs (the loss is a sum over them).
extern "C" int mm_attention_order(const int32_t* len_s, const int32_t* len_t, int n, int cap,
                                  int32_t* perm) {
    MM_CHECK_ARG(n >= 0 && cap > 0 && (n == 0 || (len_s && len_t && perm)), "bad arguments");
    std::vector<int> items, big;
    for (int i = 0; i < n; ++i) (len_s[i] > cap || len_t[i] > cap ? big : items).push_back(i);
    std::stable_sort(items.begin(), items.end(), [&](int x, int y) {
        const int mx = std::max(len_s[x], len_t[x]), my = std::max(len_s[y], len_t[y]);
        if (mx != my) return mx > my;
        return len_s[x] + len_t[x] > len_s[y] + len_t[y];
    });
    std::vector<int> bs, bt;                 // bin fill per side
    std::vector<std::vector<int>> bins;
    for (int i : items) {
        size_t b = 0;
        while (b < bins.size() && (bs[b] + len_s[i] > cap || bt[b] + len_t[i] > cap)) ++b;
        if (b == bins.size()) {
            bins.emplace_back();
            bs.push_back(0);
            bt.push_back(0);
        }
        bins[b].push_back(i);
        bs[b] += len_s[i];
        bt[b] += len_t[i];
    }
    int k = 0;
    for (const auto& bin : bins)
        for (int i : bin) perm[k++] = i;
    for (int i : big) perm[k++] = i;
    return 0;
}

// Greedy packing of consecutive sequences into attention CTA groups (the
// host half of K5; data.attention_groups is the same algorithm in numpy and
// the cross-check): each sequence takes ceil(len / 32) * 32 rows per side; a
// group holds at most `cap` rows per side, a longer sequence gets a group of
// its own.  out[2 g] = first sequence, out[2 g + 1] = count (out holds
// 2 * n_seq entries); *foot = rows of the largest group (either side).
extern "C" int mm_attention_groups(const int32_t* cu_q, const int32_t* cu_k, int n_seq, int cap,
                                   int align, int32_t* out, int* n_groups, int* foot) {
    MM_CHECK_ARG(cu_q && cu_k && out && n_groups && foot, "NULL argument");
    MM_CHECK_ARG(n_seq >= 0 && cap > 0 && align >= 1, "bad sizes");
    int g = 0, fp = 0;
    for (int i = 0; i < n_seq;) {
        int j = i, sq = 0, sk = 0;
        while (j < n_seq) {
            const int pq = (cu_q[j + 1] - cu_q[j] + align - 1) / align * align;
            const int pk = (cu_k[j + 1] - cu_k[j] + align - 1) / align * align;
            if (j != i && (sq + pq > cap || sk + pk > cap)) break;
            sq += pq;
            sk += pk;
            ++j;
        }
        out[2 * g] = i;
        out[2 * g + 1] = j - i;
        ++g;
        fp = std::max(fp, std::max(sq, sk));
        i = j;
    }
    *n_groups = g;
    *foot = fp;
    return 0;
}

// Host-side entry points of libmmb200: version / error reporting, device
// info, K9 (the allocator's communication-cost kernel) and the attention
// work-group packing of a micro-batch.
#include <cstdlib>
#include <algorithm>
#include <cstring>
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

// Greedy packing of consecutive sequences into attention CTA groups (the
// host half of K5; data.attention_groups is the same algorithm in numpy and
// the cross-check): each sequence takes ceil(len / 32) * 32 rows per side; a
// group holds at most `cap` rows per side, a longer sequence gets a group of
// its own.  out[2 g] = first sequence, out[2 g + 1] = count (out holds
// 2 * n_seq entries); *foot = rows of the largest group (either side).
extern "C" int mm_attention_groups(const int32_t* cu_q, const int32_t* cu_k, int n_seq, int cap,
                                   int32_t* out, int* n_groups, int* foot) {
    MM_CHECK_ARG(cu_q && cu_k && out && n_groups && foot, "NULL argument");
    MM_CHECK_ARG(n_seq >= 0 && cap > 0, "bad sizes");
    int g = 0, fp = 0;
    for (int i = 0; i < n_seq;) {
        int j = i, sq = 0, sk = 0;
        while (j < n_seq) {
            const int pq = (cu_q[j + 1] - cu_q[j] + 31) / 32 * 32;
            const int pk = (cu_k[j + 1] - cu_k[j] + 31) / 32 * 32;
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

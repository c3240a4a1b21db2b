/* Oracle (test infrastructure): C restatement of comm_cost_kernel,
 * /root/reference/pkg/src/mmtplan/_speedups.pyx:11-57 (twin _cost_py.py:11-48).
 * Per module (CSR row m): distinct devices and nodes of its tasks via stamp
 * arrays; cost = params[m]*(w_intra*(n_dev-1) + (w_inter-w_intra)*(n_node-1)),
 * summed in module order in float64. */
#include <stdint.h>
#include <stdlib.h>

double oracle_comm_cost(const double* params, int64_t n_modules, const int64_t* off,
                        const int64_t* idx, const int64_t* task_dev, const int64_t* dev_node,
                        int64_t n_devices, double w_intra, double w_inter, double* out) {
    int64_t max_node = 0;
    for (int64_t i = 0; i < n_devices; ++i)
        if (dev_node[i] > max_node) max_node = dev_node[i];
    int64_t* ds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_devices > 0 ? n_devices : 1));
    int64_t* ns = (int64_t*)malloc(sizeof(int64_t) * (size_t)(max_node + 1));
    for (int64_t i = 0; i < n_devices; ++i) ds[i] = -1;
    for (int64_t i = 0; i <= max_node; ++i) ns[i] = -1;
    double total = 0.0;
    for (int64_t m = 0; m < n_modules; ++m) {
        int64_t nd = 0, nn = 0;
        for (int64_t j = off[m]; j < off[m + 1]; ++j) {
            int64_t d = task_dev[idx[j]];
            if (ds[d] != m) {
                ds[d] = m;
                ++nd;
                int64_t node = dev_node[d];
                if (ns[node] != m) {
                    ns[node] = m;
                    ++nn;
                }
            }
        }
        double c = 0.0;
        if (nd > 0) c = params[m] * (w_intra * (double)(nd - 1) + (w_inter - w_intra) * (double)(nn - 1));
        out[m] = c;
        total += c;
    }
    free(ds);
    free(ns);
    return total;
}

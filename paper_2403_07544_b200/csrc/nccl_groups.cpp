// K1/K2: module-group communicators over NCCL (NVLink 5 / NVSwitch).
//
// One world communicator per process plus one sub-communicator per distinct
// module member set with more than one rank, created with ncclCommSplit so
// every rank takes part in every split in the same order (the group map of
// run_benchmark, syncsim.py:337-340, computed identically on every rank).
// Reductions are posted in the caller's order -- sorted ModuleKey order --
// inside one ncclGroupStart/End, so overlapping sub-communicators cannot
// deadlock.
#include <nccl.h>

#include <cstring>
#include <vector>

#include "mm_common.h"

namespace {

struct Ctx {
    ncclComm_t world = nullptr;
    int rank = 0, size = 1;
};

struct Group {
    ncclComm_t comm = nullptr;
    int size = 0;
};

int nccl_status(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return 0;
    mm::set_error("%s: %s", what, ncclGetErrorString(r));
    return mm::kNccl;
}

#define MM_NCCL_TRY(expr)                                          \
    do {                                                           \
        ncclResult_t _r = (expr);                                  \
        if (_r != ncclSuccess) return nccl_status(_r, #expr);      \
    } while (0)

}  // namespace

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");

extern "C" int mm_nccl_unique_id(char out[128]) {
    MM_CHECK_ARG(out != nullptr, "out is NULL");
    ncclUniqueId id;
    MM_NCCL_TRY(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return 0;
}

extern "C" int mm_comm_init(int rank, int world, const char uid[128], int device, void** ctx) {
    MM_CHECK_ARG(ctx && uid, "NULL argument");
    MM_CHECK_ARG(world >= 1 && rank >= 0 && rank < world, "rank %d of %d", rank, world);
    MM_CUDA_TRY(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    Ctx* c = new Ctx();
    c->rank = rank;
    c->size = world;
    ncclResult_t r = ncclCommInitRank(&c->world, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_status(r, "ncclCommInitRank");
    }
    *ctx = c;
    return 0;
}

extern "C" int mm_comm_destroy(void* ctx) {
    if (!ctx) return 0;
    Ctx* c = static_cast<Ctx*>(ctx);
    int st = 0;
    if (c->world) st = nccl_status(ncclCommDestroy(c->world), "ncclCommDestroy");
    delete c;
    return st;
}

extern "C" int mm_group_create(void* ctx, const int* ranks, int n, void** grp) {
    MM_CHECK_ARG(ctx && grp && (n == 0 || ranks), "NULL argument");
    Ctx* c = static_cast<Ctx*>(ctx);
    *grp = nullptr;
    MM_CHECK_ARG(n >= 1 && n <= c->size, "group size %d outside [1,%d]", n, c->size);
    int my_pos = -1;
    for (int i = 0; i < n; ++i) {
        MM_CHECK_ARG(ranks[i] >= 0 && ranks[i] < c->size, "rank %d outside world", ranks[i]);
        MM_CHECK_ARG(i == 0 || ranks[i] > ranks[i - 1], "ranks must be strictly ascending");
        if (ranks[i] == c->rank) my_pos = i;
    }
    if (n == 1) return 0;  // singleton groups never communicate (syncsim.py:369-371)
    // every rank of the world takes part in the split; non-members opt out
    const int color = my_pos >= 0 ? 0 : NCCL_SPLIT_NOCOLOR;
    ncclComm_t sub = nullptr;
    MM_NCCL_TRY(ncclCommSplit(c->world, color, my_pos >= 0 ? my_pos : 0, &sub, nullptr));
    if (my_pos < 0) return 0;
    Group* g = new Group();
    g->comm = sub;
    g->size = n;
    *grp = g;
    return 0;
}

extern "C" int mm_group_destroy(void* grp) {
    if (!grp) return 0;
    Group* g = static_cast<Group*>(grp);
    int st = g->comm ? nccl_status(ncclCommDestroy(g->comm), "ncclCommDestroy") : 0;
    delete g;
    return st;
}

extern "C" int mm_ready_count(void* ctx, const int32_t* flags_dev, int32_t* n_dev, int n_modules,
                              void* stream) {
    MM_CHECK_ARG(ctx && flags_dev && n_dev && n_modules >= 0, "bad arguments");
    Ctx* c = static_cast<Ctx*>(ctx);
    if (n_modules == 0) return 0;
    MM_NCCL_TRY(ncclAllReduce(flags_dev, n_dev, (size_t)n_modules, ncclInt32, ncclSum, c->world,
                              mm::as_stream(stream)));
    return 0;
}

extern "C" int mm_reduce_modules(void* ctx, const mm_reduce_item* items, int n, void* stream) {
    MM_CHECK_ARG(ctx && (n == 0 || items), "bad arguments");
    MM_NCCL_TRY(ncclGroupStart());
    for (int i = 0; i < n; ++i) {
        const mm_reduce_item& it = items[i];
        if (!it.group || it.n_elems == 0) continue;
        Group* g = static_cast<Group*>(it.group);
        const ncclDataType_t dt = it.dtype == 1 ? ncclBfloat16 : ncclFloat32;
        if (it.root >= g->size) {
            ncclGroupEnd();
            mm::set_error("reduce item root %d outside a group of %d", it.root, g->size);
            return mm::kArg;
        }
        if (it.mode == 1 || it.mode == 2) {
            // partitioned: in-place reduce-scatter / all-gather over the padded
            // bucket of g * shard elements; group rank j owns [j*shard, (j+1)*shard)
            if (it.shard <= 0 || it.n_elems != int64_t(g->size) * it.shard) {
                ncclGroupEnd();
                mm::set_error("partitioned item: n_elems %lld != group %d x shard %lld",
                              (long long)it.n_elems, g->size, (long long)it.shard);
                return mm::kArg;
            }
            int me = 0;
            ncclCommUserRank(g->comm, &me);
            const size_t esz = it.dtype == 1 ? 2 : 4;
            char* base = static_cast<char*>(it.buf);
            char* mine = base + size_t(me) * size_t(it.shard) * esz;
            ncclResult_t r = it.mode == 1
                                 ? ncclReduceScatter(base, mine, (size_t)it.shard, dt, ncclSum, g->comm,
                                                     mm::as_stream(stream))
                                 : ncclAllGather(mine, base, (size_t)it.shard, dt, g->comm,
                                                 mm::as_stream(stream));
            if (r != ncclSuccess) {
                ncclGroupEnd();
                return nccl_status(r, it.mode == 1 ? "ncclReduceScatter" : "ncclAllGather");
            }
            continue;
        }
        // n = 1: the single ready member's buffer is the Algorithm-1 sum (the
        // others hold zeros), so a broadcast moves (g-1)/g of the allreduce's
        // 2(g-1)/g bytes and gives bit-identical results
        ncclResult_t r = it.root >= 0
                             ? ncclBroadcast(it.buf, it.buf, (size_t)it.n_elems, dt, it.root, g->comm,
                                             mm::as_stream(stream))
                             : ncclAllReduce(it.buf, it.buf, (size_t)it.n_elems, dt, ncclSum, g->comm,
                                             mm::as_stream(stream));
        if (r != ncclSuccess) {
            ncclGroupEnd();
            return nccl_status(r, it.root >= 0 ? "ncclBroadcast" : "ncclAllReduce");
        }
    }
    MM_NCCL_TRY(ncclGroupEnd());
    return 0;
}

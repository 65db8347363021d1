// dist.cu -- multi-GPU searches (north star (4)).
//
// The reference scans all m references for every query inside one process
// (src/bruteforce.cpp:24-29,81-96: one OpenMP thread per query row, the m axis
// never split).  Here that m axis is what is sharded across GPUs:
//
//   reference-sharded  device g holds R[lo_g, hi_g) (shard_bounds) and all of Q;
//                      it searches its shard (raw keys, global indices
//                      lo_g + j), the n x k lists of all devices are
//                      all-gathered over NCCL into [G][n][k] and merged on the
//                      device under the (key, index) order.  Every device's
//                      list is the exact top-k of a disjoint range, so the
//                      merged table is bitwise one search over all of R.
//   query-sharded      device g holds all of R and searches rows
//                      [lo_g, hi_g) of Q: independent rows, no collective.
//
// Two ways in: one process driving G devices (knn_b200_sharded_*:
// ncclCommInitAll + grouped collectives), or one process per GPU
// (knn_b200_comm_* + knn_b200_dist_search_device: the caller exchanges the
// NCCL unique id, e.g. with torch.distributed, and every rank calls the search
// on its own shard).  NCCL is loaded at first use (dlopen of libnccl.so.2,
// preferring a copy the process already loaded, e.g. PyTorch's), so the
// library has no link-time NCCL dependency.  NCCL failures map to
// KNN_B200_ENCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/knn_b200.h"
#include "common.cuh"
#include "engine.cuh"
#include "exact_kernel.cuh"

namespace knnb200 {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    std::string load_error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // 1. a copy already in the process (e.g. PyTorch's); 2. an explicit path
        // (the Python mirror points it at the pip NCCL that PyTorch links, so a
        // later `import torch` finds its own version under the same soname);
        // 3. the system library
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* path = std::getenv("KNN_B200_NCCL_LIB");
        if (!h && path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char* e = dlerror();
            api.load_error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && api.load_error.empty()) api.load_error = std::string("libnccl lacks ") + name;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommInitAll, "ncclCommInitAll");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.AllGather, "ncclAllGather");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
        sym(api.GetVersion, "ncclGetVersion");
    });
    if (!api.load_error.empty()) throw NcclError(api.load_error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw NcclError(std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

// Merge [parts][n][k] raw-key lists (rank-major, each sorted) into the
// finalized n x k table (merge_kernel.cu).
void merge_parts(DeviceContext& ctx, cudaStream_t s, const float* keys, const int64_t* idx,
                 int parts, int64_t n, int k, int metric, float* out_d, int64_t* out_i) {
    MergeArgs mg{};
    mg.part_key = keys;
    mg.part_idx = idx;
    mg.parts = parts;
    mg.n = n;
    mg.k = k;
    mg.metric = metric == kMahalanobis ? kL2 : metric;
    mg.finalize = 1;
    mg.out_key = out_d;
    mg.out_idx = out_i;
    if (k > 1024) {
        Sizer sz;
        sz.take<float>(static_cast<size_t>(n) * k);
        sz.take<int64_t>(static_cast<size_t>(n) * k);
        ctx.s->arena.reserve(sz.used + 256);
        Carver cv{static_cast<char*>(ctx.s->arena.base())};
        mg.glist_key = cv.take<float>(static_cast<size_t>(n) * k);
        mg.glist_idx = cv.take<int64_t>(static_cast<size_t>(n) * k);
    }
    launch_merge(mg, s);
}

}  // namespace knnb200

using namespace knnb200;

// one rank of a multi-process communicator
struct knn_b200_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = 0;
    ~knn_b200_comm() {
        if (comm) nccl().CommDestroy(comm);
    }
};

struct knn_b200_sharded {
    int mode = KNN_B200_SHARD_REFERENCES;
    int G = 0;
    int64_t m = 0;
    int d = 0;
    std::vector<int> devices;
    std::vector<knn_b200_index*> shards;  // per device (R mode: its range; Q mode: all of R)
    std::vector<int64_t> lo;              // R mode: global first row of each shard
    std::vector<ncclComm_t> comms;        // R mode, G > 1
    std::vector<cudaStream_t> streams;
    std::mutex mu;
    ~knn_b200_sharded() {
        for (auto* h : shards) knn_b200_index_destroy(h);
        for (auto c : comms)
            if (c) nccl().CommDestroy(c);
        for (size_t g = 0; g < streams.size(); ++g) {
            cudaSetDevice(devices[g]);
            cudaStreamDestroy(streams[g]);
        }
    }
};

namespace {
template <typename F>
knn_b200_status dist_guarded(F&& body) {
    return static_cast<knn_b200_status>(abi_guarded(std::forward<F>(body)));
}

// a status from another entry point of this library: re-raise with its message
void rethrow(knn_b200_status st) {
    if (st == KNN_B200_OK) return;
    const std::string msg = knn_b200_last_error();
    switch (st) {
        case KNN_B200_EINVAL: throw InvalidArgument(msg);
        case KNN_B200_ENOMEM: throw OutOfMemory(msg);
        case KNN_B200_ECUDA: throw CudaError(msg);
        case KNN_B200_ENCCL: throw NcclError(msg);
        default: throw std::runtime_error(msg);
    }
}

int64_t shard_lo(int64_t total, int G, int g) { return total * g / G; }
}  // namespace

extern "C" {

knn_b200_status knn_b200_nccl_unique_id(void* out, size_t len) {
    return dist_guarded([&] {
        if (!out || len < sizeof(ncclUniqueId))
            throw InvalidArgument("knn_b200_nccl_unique_id: buffer must hold " +
                                  std::to_string(sizeof(ncclUniqueId)) + " bytes");
        ncclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, &id, sizeof(id));
    });
}

int knn_b200_nccl_version(void) {
    try {
        int v = 0;
        nccl_check(nccl().GetVersion(&v), "ncclGetVersion");
        return v;
    } catch (...) {
        return -1;
    }
}

knn_b200_status knn_b200_comm_create(const void* unique_id, size_t len, int32_t nranks,
                                     int32_t rank, int32_t device, knn_b200_comm** out) {
    return dist_guarded([&] {
        if (!out || !unique_id || len < sizeof(ncclUniqueId))
            throw InvalidArgument("knn_b200_comm_create: null out or short unique id");
        if (nranks < 1 || rank < 0 || rank >= nranks)
            throw InvalidArgument("knn_b200_comm_create: rank out of range");
        KNN_CUDA_CHECK(cudaSetDevice(device));
        auto c = std::make_unique<knn_b200_comm>();
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        nccl_check(nccl().CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
        *out = c.release();
    });
}

void knn_b200_comm_destroy(knn_b200_comm* comm) { delete comm; }

knn_b200_status knn_b200_dist_search_device(knn_b200_comm* comm, knn_b200_index* local,
                                            const float* d_queries, int64_t n, int32_t k,
                                            int32_t metric, const knn_b200_options* opt,
                                            float* d_out_dist, int64_t* d_out_idx) {
    return dist_guarded([&] {
        if (!comm || !local) throw InvalidArgument("knn_b200_dist_search_device: null handle");
        knn_b200_options o;
        if (opt) o = *opt;
        else knn_b200_options_init(&o);
        DeviceContext& ctx = context_for(comm->device);
        KNN_CUDA_CHECK(cudaSetDevice(comm->device));
        cudaStream_t s = o.stream ? static_cast<cudaStream_t>(o.stream) : ctx.stream;
        const int G = comm->nranks;
        // this rank's shard: raw keys + global indices into rank-local scratch,
        // all-gathered rank-major, merged on every rank
        float* lk = nullptr;
        int64_t* li = nullptr;
        float* gk = nullptr;
        int64_t* gi = nullptr;
        {
            std::lock_guard<std::mutex> lock(ctx.mu);
            Scratch& sc = ctx.bind(s);
            Sizer sz;
            sz.take<float>(static_cast<size_t>(n) * k);
            sz.take<int64_t>(static_cast<size_t>(n) * k);
            sz.take<float>(static_cast<size_t>(G) * n * k);
            sz.take<int64_t>(static_cast<size_t>(G) * n * k);
            sc.coll.reserve(sz.used + 256);
            Carver cv{static_cast<char*>(sc.coll.base())};
            lk = cv.take<float>(static_cast<size_t>(n) * k);
            li = cv.take<int64_t>(static_cast<size_t>(n) * k);
            gk = cv.take<float>(static_cast<size_t>(G) * n * k);
            gi = cv.take<int64_t>(static_cast<size_t>(G) * n * k);
        }
        knn_b200_options lo = o;
        lo.raw_keys = 1;
        lo.stream = s;
        rethrow(knn_b200_index_search_device(local, d_queries, n, k, metric, &lo, lk, li));
        const size_t cnt = static_cast<size_t>(n) * k;
        nccl_check(nccl().GroupStart(), "ncclGroupStart");
        nccl_check(nccl().AllGather(lk, gk, cnt, ncclFloat32, comm->comm, s), "ncclAllGather");
        nccl_check(nccl().AllGather(li, gi, cnt, ncclInt64, comm->comm, s), "ncclAllGather");
        nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
        {
            std::lock_guard<std::mutex> lock(ctx.mu);
            ctx.bind(s);
            merge_parts(ctx, s, gk, gi, G, n, k, metric, d_out_dist, d_out_idx);
        }
        if (!o.stream) KNN_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

knn_b200_status knn_b200_sharded_create(const float* references, int64_t m, int32_t d,
                                        int32_t num_devices, const int32_t* devices,
                                        int32_t shard_mode, const knn_b200_options* opt,
                                        knn_b200_sharded** out) {
    return dist_guarded([&] {
        if (!out) throw InvalidArgument("knn_b200_sharded_create: null out");
        if (num_devices < 1) throw InvalidArgument("knn_b200_sharded_create: num_devices must be >= 1");
        if (shard_mode != KNN_B200_SHARD_REFERENCES && shard_mode != KNN_B200_SHARD_QUERIES)
            throw InvalidArgument("knn_b200_sharded_create: unknown shard mode");
        if (shard_mode == KNN_B200_SHARD_REFERENCES && m / num_devices < 1)
            throw InvalidArgument("knn_b200_sharded_create: fewer references than devices");
        auto h = std::make_unique<knn_b200_sharded>();
        h->mode = shard_mode;
        h->G = num_devices;
        h->m = m;
        h->d = d;
        for (int g = 0; g < num_devices; ++g) h->devices.push_back(devices ? devices[g] : g);
        knn_b200_options o;
        if (opt) o = *opt;
        else knn_b200_options_init(&o);
        for (int g = 0; g < num_devices; ++g) {
            const int dev = h->devices[g];
            KNN_CUDA_CHECK(cudaSetDevice(dev));
            cudaStream_t st = nullptr;
            KNN_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            h->streams.push_back(st);
            const int64_t lo = shard_mode == KNN_B200_SHARD_REFERENCES ? shard_lo(m, num_devices, g) : 0;
            const int64_t hi = shard_mode == KNN_B200_SHARD_REFERENCES ? shard_lo(m, num_devices, g + 1) : m;
            knn_b200_options io = o;
            io.device = dev;
            knn_b200_index* ix = nullptr;
            rethrow(knn_b200_index_create(references + lo * d, hi - lo, d, lo, &io, &ix));
            h->shards.push_back(ix);
            h->lo.push_back(lo);
        }
        if (shard_mode == KNN_B200_SHARD_REFERENCES && num_devices > 1) {
            h->comms.resize(num_devices);
            nccl_check(nccl().CommInitAll(h->comms.data(), num_devices, h->devices.data()),
                       "ncclCommInitAll");
        }
        *out = h.release();
    });
}

knn_b200_status knn_b200_sharded_search(knn_b200_sharded* h, const float* queries, int64_t n,
                                        int32_t k, int32_t metric, const knn_b200_options* opt,
                                        float* out_dist, int64_t* out_idx) {
    return dist_guarded([&] {
        if (!h) throw InvalidArgument("knn_b200_sharded_search: null handle");
        if (!queries || !out_dist || !out_idx)
            throw InvalidArgument("knn_b200_sharded_search: null buffer");
        std::lock_guard<std::mutex> hl(h->mu);
        knn_b200_options o;
        if (opt) o = *opt;
        else knn_b200_options_init(&o);
        const int G = h->G;
        const int d = h->d;
        if (h->mode == KNN_B200_SHARD_REFERENCES && h->m / G < k)
            throw InvalidArgument("bf_knn: k = " + std::to_string(k) +
                                  " exceeds the smallest reference shard (" +
                                  std::to_string(h->m / G) + ")");
        // per-device buffers: Q (R mode: all rows; Q mode: this device's rows),
        // local and gathered lists, final table
        struct Dev {
            float* q = nullptr;
            float* lk = nullptr;
            int64_t* li = nullptr;
            float* gk = nullptr;
            int64_t* gi = nullptr;
            float* od = nullptr;
            int64_t* oi = nullptr;
            int64_t q0 = 0, nq = 0;
        };
        std::vector<Dev> dv(G);
        auto cleanup = [&] {
            for (int g = 0; g < G; ++g) {
                cudaSetDevice(h->devices[g]);
                for (void* p : {static_cast<void*>(dv[g].q), static_cast<void*>(dv[g].lk),
                                static_cast<void*>(dv[g].li), static_cast<void*>(dv[g].gk),
                                static_cast<void*>(dv[g].gi), static_cast<void*>(dv[g].od),
                                static_cast<void*>(dv[g].oi)})
                    if (p) cudaFreeAsync(p, h->streams[g]);
            }
        };
        try {
            for (int g = 0; g < G; ++g) {
                Dev& D = dv[g];
                KNN_CUDA_CHECK(cudaSetDevice(h->devices[g]));
                cudaStream_t s = h->streams[g];
                D.q0 = h->mode == KNN_B200_SHARD_QUERIES ? shard_lo(n, G, g) : 0;
                D.nq = h->mode == KNN_B200_SHARD_QUERIES ? shard_lo(n, G, g + 1) - D.q0 : n;
                if (D.nq == 0) continue;
                const size_t nk = static_cast<size_t>(D.nq) * k;
                KNN_CUDA_CHECK(cudaMallocAsync(&D.q, sizeof(float) * D.nq * d, s));
                KNN_CUDA_CHECK(cudaMemcpyAsync(D.q, queries + D.q0 * d, sizeof(float) * D.nq * d,
                                               cudaMemcpyHostToDevice, s));
                knn_b200_options so = o;
                so.device = h->devices[g];
                so.stream = s;
                if (h->mode == KNN_B200_SHARD_QUERIES || G == 1) {
                    KNN_CUDA_CHECK(cudaMallocAsync(&D.od, sizeof(float) * nk, s));
                    KNN_CUDA_CHECK(cudaMallocAsync(&D.oi, sizeof(int64_t) * nk, s));
                    so.raw_keys = 0;
                    rethrow(knn_b200_index_search_device(h->shards[g], D.q, D.nq, k, metric, &so,
                                                         D.od, D.oi));
                } else {
                    KNN_CUDA_CHECK(cudaMallocAsync(&D.lk, sizeof(float) * nk, s));
                    KNN_CUDA_CHECK(cudaMallocAsync(&D.li, sizeof(int64_t) * nk, s));
                    KNN_CUDA_CHECK(cudaMallocAsync(&D.gk, sizeof(float) * G * nk, s));
                    KNN_CUDA_CHECK(cudaMallocAsync(&D.gi, sizeof(int64_t) * G * nk, s));
                    so.raw_keys = 1;
                    rethrow(knn_b200_index_search_device(h->shards[g], D.q, D.nq, k, metric, &so,
                                                         D.lk, D.li));
                }
            }
            if (h->mode == KNN_B200_SHARD_REFERENCES && G > 1) {
                const size_t cnt = static_cast<size_t>(n) * k;
                nccl_check(nccl().GroupStart(), "ncclGroupStart");
                for (int g = 0; g < G; ++g) {
                    nccl_check(nccl().AllGather(dv[g].lk, dv[g].gk, cnt, ncclFloat32, h->comms[g],
                                                h->streams[g]),
                               "ncclAllGather");
                    nccl_check(nccl().AllGather(dv[g].li, dv[g].gi, cnt, ncclInt64, h->comms[g],
                                                h->streams[g]),
                               "ncclAllGather");
                }
                nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
                // merge once, on the first device
                Dev& D = dv[0];
                KNN_CUDA_CHECK(cudaSetDevice(h->devices[0]));
                cudaStream_t s = h->streams[0];
                KNN_CUDA_CHECK(cudaMallocAsync(&D.od, sizeof(float) * cnt, s));
                KNN_CUDA_CHECK(cudaMallocAsync(&D.oi, sizeof(int64_t) * cnt, s));
                DeviceContext& ctx = context_for(h->devices[0]);
                {
                    std::lock_guard<std::mutex> lock(ctx.mu);
                    ctx.bind(s);
                    merge_parts(ctx, s, D.gk, D.gi, G, n, k, metric, D.od, D.oi);
                }
                KNN_CUDA_CHECK(cudaMemcpyAsync(out_dist, D.od, sizeof(float) * cnt,
                                               cudaMemcpyDeviceToHost, s));
                KNN_CUDA_CHECK(cudaMemcpyAsync(out_idx, D.oi, sizeof(int64_t) * cnt,
                                               cudaMemcpyDeviceToHost, s));
            } else {
                for (int g = 0; g < G; ++g) {
                    Dev& D = dv[g];
                    if (D.nq == 0) continue;
                    KNN_CUDA_CHECK(cudaSetDevice(h->devices[g]));
                    const size_t nk = static_cast<size_t>(D.nq) * k;
                    KNN_CUDA_CHECK(cudaMemcpyAsync(out_dist + D.q0 * k, D.od, sizeof(float) * nk,
                                                   cudaMemcpyDeviceToHost, h->streams[g]));
                    KNN_CUDA_CHECK(cudaMemcpyAsync(out_idx + D.q0 * k, D.oi, sizeof(int64_t) * nk,
                                                   cudaMemcpyDeviceToHost, h->streams[g]));
                }
            }
            for (int g = 0; g < G; ++g) {
                KNN_CUDA_CHECK(cudaSetDevice(h->devices[g]));
                KNN_CUDA_CHECK(cudaStreamSynchronize(h->streams[g]));
            }
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
        for (int g = 0; g < G; ++g) {
            KNN_CUDA_CHECK(cudaSetDevice(h->devices[g]));
            KNN_CUDA_CHECK(cudaStreamSynchronize(h->streams[g]));
        }
    });
}

void knn_b200_sharded_destroy(knn_b200_sharded* h) { delete h; }

}  // extern "C"

// profile.cu -- per-kernel CUDA-event timing (bench.py's roofline numbers) and
// the device-side synthetic input generator.
//
// When profiling is enabled on a thread, every engine launch on that thread is
// bracketed by a pair of CUDA events recorded on the launch stream, so the
// per-kernel durations come from the device clock of the very stream the
// kernel ran on.  knn_b200_profile_collect() synchronizes those events and
// returns per-kernel totals.
#include <cstring>
#include <string>
#include <vector>

#include "../../include/knn_b200.h"
#include "common.cuh"
#include "profile.cuh"

namespace knnb200 {

namespace {
struct Rec {
    const char* name;
    cudaEvent_t a, b;
};
thread_local bool g_profile = false;
thread_local std::string g_only;  // name prefix filter ("" = all)
thread_local std::vector<Rec> g_recs;
thread_local std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    KNN_CUDA_CHECK(cudaEventCreate(&e));
    return e;
}
}  // namespace

ProfileScope::ProfileScope(cudaStream_t s, const char* name) : stream_(s), name_(name) {
    if (!g_profile) return;
    if (!g_only.empty() && std::strncmp(name, g_only.c_str(), g_only.size()) != 0) return;
    a_ = take_event();
    b_ = take_event();
    KNN_CUDA_CHECK(cudaEventRecord(static_cast<cudaEvent_t>(a_), stream_));
}

ProfileScope::~ProfileScope() {
    if (!a_) return;
    cudaEventRecord(static_cast<cudaEvent_t>(b_), stream_);
    g_recs.push_back({name_, static_cast<cudaEvent_t>(a_), static_cast<cudaEvent_t>(b_)});
}

// counter-based uniform [0,1): splitmix64(seed + offset + i) >> 40, * 2^-24
// (oracle/knn_oracle.c ko_fill_counter_f32 reproduces it on the host)
__global__ void fill_uniform_kernel(float* out, int64_t count, uint64_t seed, int64_t offset) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += stride) {
        uint64_t z = seed + static_cast<uint64_t>(offset + i) + 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        out[i] = static_cast<float>(z >> 40) * 0x1.0p-24f;
    }
}

}  // namespace knnb200

using namespace knnb200;

extern "C" {

void knn_b200_profile_enable(int on) { g_profile = on != 0; }

void knn_b200_profile_only(const char* prefix) { g_only = prefix ? prefix : ""; }

int knn_b200_profile_collect(char* names, size_t names_len, double* ms, uint64_t* counts,
                             int max_kernels) {
    // aggregate by name, in first-seen order
    std::vector<std::string> order;
    std::vector<double> tot;
    std::vector<uint64_t> cnt;
    for (const Rec& r : g_recs) {
        float t = 0.f;
        if (cudaEventSynchronize(r.b) != cudaSuccess) return -1;
        cudaEventElapsedTime(&t, r.a, r.b);
        size_t j = 0;
        while (j < order.size() && order[j] != r.name) ++j;
        if (j == order.size()) {
            order.emplace_back(r.name);
            tot.push_back(0.0);
            cnt.push_back(0);
        }
        tot[j] += t;
        cnt[j] += 1;
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    std::string joined;
    const int nk = static_cast<int>(order.size());
    for (int j = 0; j < nk && j < max_kernels; ++j) {
        if (ms) ms[j] = tot[j];
        if (counts) counts[j] = cnt[j];
        joined += order[j];
        joined += '\n';
    }
    if (names && names_len) {
        std::strncpy(names, joined.c_str(), names_len - 1);
        names[names_len - 1] = '\0';
    }
    return nk;
}

knn_b200_status knn_b200_fill_uniform_device(float* d_out, int64_t count, uint64_t seed,
                                             int64_t offset, void* stream) {
    if (!d_out || count < 0) return KNN_B200_EINVAL;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    {
        ProfileScope ps(s, "fill_uniform_kernel");
        fill_uniform_kernel<<<kSmCount * 8, 256, 0, s>>>(d_out, count, seed, offset);
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? KNN_B200_OK : KNN_B200_ECUDA;
}

}  // extern "C"

// profile.cuh -- RAII event bracket around one kernel launch (no-op unless
// knn_b200_profile_enable(1) was called on this thread).
#pragma once

#include <cuda_runtime.h>

namespace knnb200 {

class ProfileScope {
public:
    ProfileScope(cudaStream_t s, const char* name);
    ~ProfileScope();
    ProfileScope(const ProfileScope&) = delete;
    ProfileScope& operator=(const ProfileScope&) = delete;

private:
    cudaStream_t stream_;
    const char* name_;
    void* a_ = nullptr;
    void* b_ = nullptr;
};

}  // namespace knnb200

// Shared device/host helpers for the B200 ADPSGD learner step (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "adpsgd_b200.h"

// L2 sector promotion of every tcgen05 operand / epilogue tensor map (A/B builds may override)
#ifndef ADPSGD_L2PROMO
#define ADPSGD_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

namespace ab {

// Status-carrying exception used inside the library; converted to adpsgd_status at the
// C ABI (errors.hpp:9-46 taxonomy).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define AB_CUDA(x)                                                                        \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess)                                                            \
            throw ::ab::Error(ADPSGD_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + \
                                                 " @" + __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

#define AB_CHECK(cond, code, msg)                      \
    do {                                               \
        if (!(cond)) throw ::ab::Error((code), (msg)); \
    } while (0)

using bf16 = __nv_bfloat16;

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }

// Counts this library's kernel launches (reported as gpu_launches by bench.py).
extern int64_t g_launch_count;
inline void count_launch(int64_t n = 1) { g_launch_count += n; }

// L2 persisting set-aside (reserved on first use; 0 when the device has none) and the largest
// access-policy window.
inline size_t l2_persist_bytes() {
    static long long v = -1;
    if (v < 0) {
        int dev = 0, mx = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
        size_t want = static_cast<size_t>(mx) < (size_t(64) << 20) ? static_cast<size_t>(mx) : (size_t(64) << 20);
        size_t got = 0;
        if (want && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess)
            cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
        cudaGetLastError();
        v = static_cast<long long>(got);
    }
    return static_cast<size_t>(v);
}
inline size_t l2_window_max() {
    static int v = -1;
    if (v < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        if (v < 0) v = 0;
    }
    return static_cast<size_t>(v);
}

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace ab

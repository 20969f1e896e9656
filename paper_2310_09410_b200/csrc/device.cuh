// Device helpers shared by the kernels of liblopf (resident.cu, kernels.cu, batch.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace lopf {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Warp sums of five doubles by a reduce-scatter butterfly (fixed order, deterministic): 18 shuffles and
// 9 adds instead of 50 and 25.  Returns the total of value (lane >> 2) on lanes with (lane >> 2) < 5.
__device__ __forceinline__ double warp_sum5(const double (&v)[5], const int lane) {
    const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
    double w[4];                                   // xor 16: lanes keep values 0-3 (b16 = 0) or 4-7
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double lo = v[i], hi = i == 0 ? v[4] : 0.0;
        const double send = b16 ? lo : hi, keep = b16 ? hi : lo;
        w[i] = keep + __shfl_xor_sync(kFull, send, 16);
    }
    double x[2];                                   // xor 8: keep 2 of the 4
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double send = b8 ? w[i] : w[i + 2], keep = b8 ? w[i + 2] : w[i];
        x[i] = keep + __shfl_xor_sync(kFull, send, 8);
    }
    double y;                                      // xor 4: keep 1 of the 2
    {
        const double send = b4 ? x[0] : x[1], keep = b4 ? x[1] : x[0];
        y = keep + __shfl_xor_sync(kFull, send, 4);
    }
    y += __shfl_xor_sync(kFull, y, 2);
    y += __shfl_xor_sync(kFull, y, 1);
    return y;                                      // value index 4 b16 + 2 b8 + b4 = lane >> 2
}

// Counter grid barrier of a cooperative launch: every CTA arrives once per call; `target` is the
// cumulative arrival count after this call (calls x gridDim.x).
__device__ __forceinline__ void grid_sync(unsigned long long* cnt, const unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1ULL);
        while (ld_acquire_u64(cnt) < target) {
        }
    }
    __syncthreads();
}

}  // namespace dev
}  // namespace lopf

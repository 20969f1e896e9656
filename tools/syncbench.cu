// Microbenchmark of inter-CTA synchronisation primitives on one GPU (diagnostics for DESIGN.md §4.2).
//   pingpong   : two CTAs bounce a flag (one-way latency = total / (2 * rounds))
//   fence      : cost of __threadfence() with / without outstanding stores
//   counter    : centralized counter barrier across G CTAs (red.add + ld.acquire poll)
//   counter_rlx: same with relaxed polling + one fence after
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o syncbench tools/syncbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_vol(const unsigned long long* p) {
    return *(volatile const unsigned long long*)p;
}
__device__ __forceinline__ void st_rlx(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// mode 0: relaxed st / relaxed poll; 1: release st / acquire poll; 2: fence+relaxed st / volatile poll
__global__ void pingpong(unsigned long long* f, int rounds, int mode, long long* out) {
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x, other = 1 - me;
    __syncwarp();
    long long t0 = clock64();
    for (int r = 1; r <= rounds; ++r) {
        if (me == 0) {
            if (mode == 0) st_rlx(f + 0, r); else if (mode == 1) st_rel(f + 0, r); else { __threadfence(); st_rlx(f + 0, r); }
            if (mode == 0) while (ld_rlx(f + 1) < (unsigned long long)r) {}
            else if (mode == 1) while (ld_acq(f + 1) < (unsigned long long)r) {}
            else while (ld_vol(f + 1) < (unsigned long long)r) {}
        } else {
            if (mode == 0) while (ld_rlx(f + 0) < (unsigned long long)r) {}
            else if (mode == 1) while (ld_acq(f + 0) < (unsigned long long)r) {}
            else while (ld_vol(f + 0) < (unsigned long long)r) {}
            if (mode == 0) st_rlx(f + 1, r); else if (mode == 1) st_rel(f + 1, r); else { __threadfence(); st_rlx(f + 1, r); }
        }
    }
    out[me] = clock64() - t0;
}

__global__ void fencecost(double* buf, int n, long long* out) {
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    for (int i = 0; i < 100; ++i) __threadfence();
    long long t1 = clock64();
    for (int i = 0; i < 100; ++i) { __stcg(buf + (i & 31), (double)i); __threadfence(); }
    long long t2 = clock64();
    out[0] = (t1 - t0) / 100;
    out[1] = (t2 - t1) / 100;
}

// counter barrier: mode 0 red.release + ld.acquire poll (thread 0); mode 1 atomicAdd + volatile poll + fence
__global__ void counter(unsigned long long* bar, int rounds, int mode, long long* out) {
    const int G = gridDim.x;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 1; r <= rounds; ++r) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long target = (unsigned long long)r * G;
            if (mode == 0) {
                __threadfence();
                asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
                while (ld_acq(bar) < target) {}
            } else {
                __threadfence();
                atomicAdd(bar, 1ULL);
                while (ld_vol(bar) < target) {}
                __threadfence();
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    unsigned long long* f;
    long long* out;
    double* buf;
    cudaMalloc(&f, 4096);
    cudaMalloc(&out, 8 * 4096);
    cudaMalloc(&buf, 4096);
    long long h[4096];
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("SMs %d clock %d kHz\n", sms, clk);
    const int R = 20000;
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(f, 0, 4096);
        pingpong<<<2, 32>>>(f, R, mode, out);
        cudaDeviceSynchronize();
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("pingpong mode %d: one-way %.0f cycles\n", mode, (double)h[0] / (2.0 * R));
    }
    fencecost<<<1, 32>>>(buf, 32, out);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("threadfence: %lld cycles idle, %lld cycles after a store\n", h[0], h[1]);
    for (int G : {2, 4, 16, 64, 145, 148}) {
        for (int mode = 0; mode < 2; ++mode) {
            cudaMemset(f, 0, 4096);
            void* args[] = {&f, (void*)&R, &mode, &out};
            int rr = 5000;
            args[1] = &rr;
            cudaLaunchCooperativeKernel((void*)counter, dim3(G), dim3(1024), args, 0, 0);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, out, 8 * G, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (int i = 0; i < G; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("counter barrier G=%3d mode %d: %.0f cycles/barrier %s\n", G, mode, mx / rr,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}

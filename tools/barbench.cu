// Microbenchmark: cost of a CTA-wide __syncthreads loop (empty sweep skeleton of the resident kernel)
// and of dependent SMEM load chains.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o barbench tools/barbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void bar_loop(int iters, long long* out) {
    __shared__ double red[32][5];
    __shared__ int s_stop[2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x < 2) s_stop[threadIdx.x] = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int t = 0; t < iters; ++t) {
        if (lane == 0) for (int k = 0; k < 5; ++k) red[wid][k] = (double)t;
        __syncthreads();
        if (wid == 0 && lane == 0) s_stop[t & 1] = t >= iters;
        __syncthreads();
        if (s_stop[t & 1]) break;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

__global__ void lds_chain(int iters, long long* out, int stride) {
    extern __shared__ int sm[];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (i * stride + 7) & 8191;
    __syncthreads();
    int p = threadIdx.x & 8191;
    long long t0 = clock64();
    for (int t = 0; t < iters; ++t) p = sm[p];
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    if (p == -1) out[1] = p;
}

__global__ void dfma_chain(int iters, long long* out, double a) {
    double x = threadIdx.x, y = 1.0 + threadIdx.x;
    long long t0 = clock64();
    for (int t = 0; t < iters; ++t) { x = fma(x, a, y); }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    if (x == -1.0) out[1] = 1;
}

int main() {
    long long* out;
    cudaMalloc(&out, 8 * 1024);
    long long h[4];
    const int N = 10000;
    for (int th : {1024, 768, 512, 256, 32}) {
        bar_loop<<<148, th>>>(N, out);
        cudaDeviceSynchronize();
        cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("bar_loop %4d threads: %.0f cycles / sweep (2 barriers)\n", th, (double)h[0] / N);
    }
    for (int th : {32, 1024}) {
        lds_chain<<<1, th, 32768>>>(N, out, 33);
        cudaDeviceSynchronize();
        cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("lds chain %4d threads: %.1f cycles / load\n", th, (double)h[0] / N);
        dfma_chain<<<1, th>>>(N, out, 0.999);
        cudaDeviceSynchronize();
        cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("dfma chain %4d threads: %.1f cycles / fma\n", th, (double)h[0] / N);
    }
    return 0;
}

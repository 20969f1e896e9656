// Fused ADMM sweep for sm_100a (B200): Algorithm 1 of arXiv 2310.09410.
//
// One persistent cooperative launch runs the whole loop.  Per sweep, every warp walks its
// tasks (packed subsystems, see pack.cpp) and, per row slot (one lane),
//   a4  consensus  x_g = clamp((sum_{k in seg(g)} u_k - c_g/rho) / nu_g, lo_g, hi_g)
//                  (closed_1 with rho restored; reading C1), recomputed by every
//                  copy from the ping-pong buffer u (identical bits for all copies of g)
//   a5  local      x_s = (1/rho) Abar_s d + bbar_s,  d = -rho v - lambda_s       (closed_2)
//                  Abar column loads coalesced, d exchanged by warp shuffles
//   a6  dual       lambda_s += rho (v - x_s) (ADMM-3);  u = x_s - lambda_s / rho
//   a7  residuals  five per-lane sums -> warp shuffle tree -> block -> per-block partial;
//                  the last CTA to arrive reduces the partials in block order (deterministic),
//                  evaluates (termination) and releases the grid.
// One grid barrier per sweep; no host synchronisation inside the loop.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"

namespace lopf {

namespace {

constexpr int kBlock = kStreamBlock;
constexpr int kWarps = kBlock / 32;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int R>
__device__ __forceinline__ void task_sweep(const DevProblem& P, const int4 tr, const double* __restrict__ ucur,
                                           double* __restrict__ unext, double (&acc)[5], const int lane,
                                           double* __restrict__ dsm) {
    double d[R], v[R], lam[R], xo[R], bb[R];
    int info[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        const int slot = tr.x + h * 32 + lane;
        info[h] = __ldg(P.s_info + slot);
        d[h] = 0.0; v[h] = 0.0; lam[h] = 0.0; xo[h] = 0.0; bb[h] = 0.0;
        if (info[h] & kInfoValid) {
            const int g = __ldg(P.s_g + slot);
            lam[h] = __ldcs(P.lam + slot);
            xo[h] = __ldcs(P.xl + slot);
            if (info[h] & kInfoBbar) bb[h] = __ldcs(P.s_bbar + slot);
            const double2 gp0 = __ldg(reinterpret_cast<const double2*>(P.gpar + g));       // {c/rho, 1/nu}
            const double2 gp1 = __ldg(reinterpret_cast<const double2*>(P.gpar + g) + 1);   // {lo, hi}
            double sigma;
            if (info[h] & kInfoInline) {                       // nu <= 4: neighbour slots inline
                const int4 nb = __ldg(P.s_nbr + slot);
                const int nu = (info[h] >> kInfoNuShift) & 0xFF;
                const double a0 = __ldcg(ucur + nb.x);
                const double a1 = nu > 1 ? __ldcg(ucur + nb.y) : 0.0;
                const double a2 = nu > 2 ? __ldcg(ucur + nb.z) : 0.0;
                const double a3 = nu > 3 ? __ldcg(ucur + nb.w) : 0.0;
                sigma = a0;                                    // ascending canonical copy order
                if (nu > 1) sigma += a1;
                if (nu > 2) sigma += a2;
                if (nu > 3) sigma += a3;
            } else {
                const int q0 = __ldg(P.seg_ptr + g), q1 = __ldg(P.seg_ptr + g + 1);
                sigma = 0.0;
                for (int q = q0; q < q1; ++q) sigma += __ldcg(ucur + __ldg(P.seg_slot + q));
            }
            const double xg = fmin(fmax((sigma - gp0.x) * gp0.y, gp1.x), gp1.y);   // IEEE +-inf = no clamp
            if (info[h] & kInfoFirst) P.x[g] = xg;
            v[h] = xg;
            d[h] = -P.rho * xg - lam[h];
        }
    }
    double ax[R];
#pragma unroll
    for (int h = 0; h < R; ++h) ax[h] = 0.0;
    const double* __restrict__ A = P.abar + tr.y;
    const int kmax = tr.z;
    int base[R];
#pragma unroll
    for (int h = 0; h < R; ++h) base[h] = info[h] & kInfoBaseMask;
    if (R > 1) {                                   // d staged in this warp's SMEM; row h*32+lane reads
#pragma unroll                                     // d[base + k] of its own subsystem
        for (int h = 0; h < R; ++h) dsm[h * 32 + lane] = d[h];
        __syncwarp();
#pragma unroll 2
        for (int k = 0; k < kmax; ++k) {
#pragma unroll
            for (int h = 0; h < R; ++h)
                ax[h] = fma(__ldcs(A + (size_t)k * (32 * R) + h * 32 + lane), dsm[base[h] + k], ax[h]);
        }
        __syncwarp();
    } else {
#pragma unroll 4
        for (int k = 0; k < kmax; ++k)
            ax[0] = fma(__ldcs(A + (size_t)k * 32 + lane), __shfl_sync(kFull, d[0], base[0] + k), ax[0]);
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {
        if (!(info[h] & kInfoValid)) continue;
        const int slot = tr.x + h * 32 + lane;
        const double xn = fma(ax[h], P.inv_rho, bb[h]);                 // (1/rho) Abar d + bbar
        const double ln = lam[h] + P.rho * (v[h] - xn);                  // ADMM-3
        __stcs(P.xl + slot, xn);
        __stcs(P.lam + slot, ln);
        unext[slot] = xn - ln * P.inv_rho;                               // next consensus input
        const double r = v[h] - xn, dx = xn - xo[h];
        acc[0] += r * r;
        acc[1] += dx * dx;
        acc[2] += v[h] * v[h];
        acc[3] += xn * xn;
        acc[4] += ln * ln;
    }
}

template <int RMAX>   // largest task width in the problem; RMAX <= 4 keeps 64 registers (2 CTAs / SM)
__global__ void __launch_bounds__(kBlock, RMAX <= 4 ? kStreamCtasPerSm : 1) admm_stream_kernel(DevProblem P) {
    __shared__ double red[kWarps][5];
    __shared__ double dstage[kWarps][256];
    __shared__ int s_stop;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarps + wid, nw = gridDim.x * kWarps;
    const long long total0 = *(volatile long long*)&P.ctrl->total;
    long long it = 0;
    while (it < P.max_iter) {
        const long long t = total0 + it;
        const double* ucur = (t & 1) ? P.u1 : P.u0;
        double* unext = (t & 1) ? P.u0 : P.u1;
        double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int task = gw; task < P.n_tasks; task += nw) {
            const int4 tr = __ldg(P.tasks + task);
            double* dsm = dstage[wid];
            switch (tr.w) {
                case 1: task_sweep<1>(P, tr, ucur, unext, acc, lane, dsm); break;
                case 2: task_sweep<2>(P, tr, ucur, unext, acc, lane, dsm); break;
                case 4: if constexpr (RMAX >= 4) task_sweep<4>(P, tr, ucur, unext, acc, lane, dsm); break;
                default: if constexpr (RMAX >= 8) task_sweep<8>(P, tr, ucur, unext, acc, lane, dsm); break;
            }
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_xor_sync(kFull, acc[k], off);
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 5; ++k) red[wid][k] = acc[k];
        }
        __syncthreads();
        ++it;
        if (wid == 0) {
            int last = 0;
            if (lane == 0) {
                double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                for (int w = 0; w < kWarps; ++w)
                    for (int k = 0; k < 5; ++k) s[k] += red[w][k];
                double* part = P.partial + (size_t)blockIdx.x * 8;
                for (int k = 0; k < 5; ++k) part[k] = s[k];
                __threadfence();
                const unsigned long long old = atomicAdd(&P.ctrl->arrive, 1ULL);
                last = (old + 1 == (unsigned long long)it * gridDim.x);
            }
            last = __shfl_sync(kFull, last, 0);
            if (last) {                                        // reduce partials in block order
                __threadfence();
                double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                for (int b = lane; b < (int)gridDim.x; b += 32)
                    for (int k = 0; k < 5; ++k) s[k] += __ldcg(P.partial + (size_t)b * 8 + k);
#pragma unroll
                for (int k = 0; k < 5; ++k) {
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) s[k] += __shfl_xor_sync(kFull, s[k], off);
                }
                if (lane == 0) {
                    const double pres = sqrt(s[0]), dres = P.rho * sqrt(s[1]);
                    const double ep = P.eps_rel * fmax(sqrt(s[2]), sqrt(s[3])), ed = P.eps_rel * sqrt(s[4]);
                    const int numeric = !(isfinite(s[0]) && isfinite(s[1]) && isfinite(s[2]) && isfinite(s[3]) && isfinite(s[4]));
                    const int conv = P.test && (pres <= ep) && (dres <= ed);
                    const int stop = conv || numeric;
                    DevCtrl* c = P.ctrl;
                    if (P.trace_every > 0 && (it % P.trace_every) == 0) {
                        const long long row = it / P.trace_every - 1;
                        if (row < P.trace_cap) {
                            double* tr = P.trace + row * 5;
                            tr[0] = (double)(total0 + it); tr[1] = pres; tr[2] = dres; tr[3] = ep; tr[4] = ed;
                            c->trace_rows = row + 1;
                        }
                    }
                    if (stop || it == P.max_iter) {                // final sweep of this launch
                        double obj = 0.0;
                        for (int j = 0; j < P.n_obj; ++j) obj += P.obj_c[j] * __ldcg(P.x + P.obj_idx[j]);
                        c->res[0] = pres; c->res[1] = dres; c->res[2] = ep; c->res[3] = ed;
                        c->objective = obj;
                        c->iters = it;
                        c->total = total0 + it;
                        c->outcome = conv ? LOPF_CONVERGED : LOPF_MAX_ITER;
                        c->numeric = numeric;
                    }
                    __threadfence();
                    st_release_u64(&c->flag, ((unsigned long long)it << 2) | ((unsigned long long)stop << 1) |
                                                 (unsigned long long)numeric);
                    s_stop = stop;
                }
            } else if (lane == 0) {
                unsigned long long f;
                while (((f = ld_acquire_u64(&P.ctrl->flag)) >> 2) < (unsigned long long)it) __nanosleep(32);
                s_stop = (int)((f >> 1) & 1);
                __threadfence();
            }
        }
        __syncthreads();
        if (s_stop) break;
    }
}

// a3: reset the iterate to the initial point: x_s = x0, lambda = 0, u = x0.
__global__ void reset_kernel(DevProblem P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P.n_slots) {
        const double x0 = P.x0[i];
        P.xl[i] = x0;
        P.lam[i] = 0.0;
        P.u0[i] = x0;
        P.u1[i] = 0.0;
    }
    if (i == 0) {
        P.ctrl->arrive = 0; P.ctrl->flag = 0; P.ctrl->total = 0; P.ctrl->iters = 0; P.ctrl->trace_rows = 0;
    }
}

}  // namespace

static const void* stream_kernel_for(int rmax) {
    return rmax <= 1 ? (const void*)admm_stream_kernel<1>
         : rmax <= 2 ? (const void*)admm_stream_kernel<2>
         : rmax <= 4 ? (const void*)admm_stream_kernel<4>
                     : (const void*)admm_stream_kernel<8>;
}

lopf_status query_grid(int rmax, int* grid, std::string& err) {
    int dev = 0, sms = 0, per = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, stream_kernel_for(rmax), kBlock, 0);
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    if (per < 1) { err = "streaming kernel cannot be resident (occupancy 0)"; return LOPF_E_CUDA; }
    *grid = sms * per;
    return LOPF_OK;
}

lopf_status launch_solve(const DevProblem& P, int grid, void* stream, std::string& err) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(P.ctrl, 0, 2 * sizeof(unsigned long long), s);   // arrive, flag
    if (e == cudaSuccess) e = cudaMemsetAsync(&P.ctrl->trace_rows, 0, sizeof(long long), s);
    if (e == cudaSuccess && P.max_iter > 0) {
        DevProblem Q = P;
        void* args[] = {&Q};
        e = cudaLaunchCooperativeKernel(stream_kernel_for(P.rmax), dim3(grid), dim3(kBlock), args, 0, s);
    }
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_reset(const DevProblem& P, void* stream, std::string& err) {
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = (P.n_slots + 255) / 256;
    reset_kernel<<<nb > 0 ? nb : 1, 256, 0, s>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

}  // namespace lopf

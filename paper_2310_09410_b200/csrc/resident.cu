// SMEM-resident ADMM kernel for sm_100a: Algorithm 1 of arXiv 2310.09410
// with every CTA owning a connected chunk of the feeder.
//
// At launch each CTA copies its blob (operators Abar_s / bbar_s, maps, iterate) into shared
// memory; the iterate then stays on chip for the whole solve.  Per sweep:
//   G-phase   x_g for every global with a copy in the chunk (closed_1, rho restored):
//             the segment is summed in canonical copy order from SMEM u (own copies) and from the
//             global exchange buffer (boundary copies owned by other CTAs, one L2 round trip);
//             meanwhile warp 0 reduces the previous sweep's residual partials (fixed order) and takes
//             the (termination) decision — identical in every CTA.
//   L-phase   per warp task: d = -rho v - lambda, x_s = (1/rho) Abar d + bbar (closed_2), lambda += rho (v - x_s)
//             (ADMM-3) in SMEM; u = x_s - lambda/rho of boundary copies -> exchange buffer; residual sums.
//             (u of a CTA's own copies is re-formed from x_s and lambda in the next G-phase.)
//   barrier   one grid barrier (release/acquire counter) per sweep.
// x^t is double-buffered so that the sweep after the stopping one can be abandoned without loss.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"

namespace lopf {

namespace {

constexpr int RB = kResBlock;
constexpr int RW = RB / 32;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_sync(unsigned long long* bar, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_acq(bar) < target) {
        }
    }
    __syncthreads();
}

template <int R>
__device__ __forceinline__ void res_task(const int4 tr, const int32_t* __restrict__ sinfo,
                                         const int32_t* __restrict__ saoff, const double* __restrict__ sabar,
                                         const double* __restrict__ sbbar, double* __restrict__ sxl,
                                         double* __restrict__ slam, const double* __restrict__ xg, const double rho,
                                         const double inv_rho, double (&acc)[5], const int lane) {
    double d[R], v[R], lam[R], xo[R], bb[R];
    int info[R], ao[R], ns[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        const int slot = tr.x + h * 32 + lane;
        info[h] = sinfo[slot];
        const bool valid = info[h] & kResValid;
        ns[h] = (info[h] >> kResNsShift) & 0x7F;              // 0 for unused lanes
        ao[h] = saoff[slot];
        v[h] = valid ? xg[info[h] >> kResGlShift] : 0.0;      // B_s x
        lam[h] = slam[slot];
        xo[h] = sxl[slot];
        bb[h] = sbbar[slot];
        d[h] = valid ? (-rho * v[h] - lam[h]) : 0.0;          // d = -rho B_s x - lambda_s
    }
    double ax[R];
#pragma unroll
    for (int h = 0; h < R; ++h) ax[h] = 0.0;
    const int kmax = tr.y;
    const int base = info[0] & 0x3F;
#pragma unroll 2
    for (int k = 0; k < kmax; ++k) {
        double dk;
        if (R == 1) {
            dk = __shfl_sync(kFull, d[0], base + k);           // src >= 32 only when k >= n_s (masked below)
        } else {
            const double e0 = __shfl_sync(kFull, d[0], k & 31);
            const double e1 = __shfl_sync(kFull, d[R - 1], k & 31);
            dk = (k >> 5) ? e1 : e0;
        }
#pragma unroll
        for (int h = 0; h < R; ++h)
            if (k < ns[h]) ax[h] = fma(sabar[ao[h] + k * ns[h]], dk, ax[h]);   // Abar_s[r][k] d_k
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {
        if (!(info[h] & kResValid)) continue;
        const int slot = tr.x + h * 32 + lane;
        const double xn = fma(ax[h], inv_rho, bb[h]);        // (1/rho) Abar d + bbar      (closed_2)
        const double ln = lam[h] + rho * (v[h] - xn);         // lambda + rho (B x - x_s)   (ADMM-3)
        sxl[slot] = xn;
        slam[slot] = ln;
        const double r = v[h] - xn, dx = xn - xo[h];
        acc[0] += r * r;
        acc[1] += dx * dx;
        acc[2] += v[h] * v[h];
        acc[3] += xn * xn;
        acc[4] += ln * ln;
    }
}

// next consensus input u = x_s - lambda / rho (the same rounding wherever it is formed)
__device__ __forceinline__ double u_of(const double x, const double l, const double inv_rho) {
    return __fma_rn(-l, inv_rho, x);
}

__global__ void __launch_bounds__(RB, 1) admm_resident_kernel(ResProblem P) {
    extern __shared__ __align__(16) uint8_t sm[];
    __shared__ CtaHdr H;
    __shared__ double red[RW][5];
    __shared__ double s_res[4];
    __shared__ int s_stop, s_conv, s_num;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x;
    if (tid < (int)(sizeof(CtaHdr) / 4)) ((int*)&H)[tid] = ((const int*)(P.hdr + blockIdx.x))[tid];
    __syncthreads();
    uint8_t* blob = P.blobs + H.blob_off;
    {
        const int4* src = (const int4*)blob;
        int4* dst = (int4*)sm;
        const int n16 = H.blob_bytes / 16;
        for (int i = tid; i < n16; i += RB) dst[i] = __ldcg(src + i);
    }
    __syncthreads();
    const int NG = H.n_glob, NT = H.n_tasks, NX = H.n_expl;
    const double* sabar = (const double*)(sm + H.off_abar);
    const double* sbbar = (const double*)(sm + H.off_bbar);
    double* sxl = (double*)(sm + H.off_xl);
    double* slam = (double*)(sm + H.off_lam);
    const double4* gpar = (const double4*)(sm + H.off_gpar);
    const int4* stasks = (const int4*)(sm + H.off_tasks);
    const int32_t* sinfo = (const int32_t*)(sm + H.off_sinfo);
    const int32_t* saoff = (const int32_t*)(sm + H.off_aoff);
    const int32_t* gsegoff = (const int32_t*)(sm + H.off_gsegoff);
    const int32_t* gseg = (const int32_t*)(sm + H.off_gseg);
    const int32_t* gown = (const int32_t*)(sm + H.off_gown);
    const int2* expl = (const int2*)(sm + H.off_expl);
    double* sxg = (double*)(sm + H.off_xg);                  // [2][NG]
    unsigned long long* bar = &P.ctrl->arrive;
    const long long total0 = *(volatile long long*)&P.ctrl->total;
    const double rho = P.rho, inv_rho = P.inv_rho;
    unsigned long long target = 0;
    int cur = (int)(total0 & 1);

    // publish the boundary copies of the current u so the exchange buffer matches the iterate
    for (int i = tid; i < NX; i += RB) {
        const int2 e = expl[i];
        __stcg(P.xchg + (size_t)cur * P.n_exp + e.y, u_of(sxl[e.x], slam[e.x], inv_rho));
    }
    if (G > 1) { target += G; grid_sync(bar, target); } else __syncthreads();

    long long t = 0;
    for (;;) {
        const int nxt = cur ^ 1;
        const double* xc = P.xchg + (size_t)cur * P.n_exp;
        double* xgn = sxg + (((t + 1) & 1) ? NG : 0);
        // warp 0: issue the loads of sweep t's residual partials before its share of the G-phase
        double ps[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if (t > 0 && wid == 0) {
            const double* part = P.partial + (size_t)(t & 1) * G * 8;
            for (int b = lane; b < G; b += 32) {
#pragma unroll
                for (int k = 0; k < 5; ++k) ps[k] += __ldcg(part + (size_t)b * 8 + k);
            }
        }
        // G-phase: x_g = clamp((sum_seg u - c/rho) / nu, lo, hi), segment in canonical copy order
        for (int j = tid; j < NG; j += RB) {
            const int q0 = gsegoff[j], q1 = gsegoff[j + 1];
            double sigma = 0.0;
            for (int q = q0; q < q1; ++q) {
                const int e = gseg[q];
                sigma += e >= 0 ? u_of(sxl[e], slam[e], inv_rho) : __ldcg(xc + (-e - 1));
            }
            const double4 gp = gpar[j];
            xgn[j] = fmin(fmax((sigma - gp.x) * gp.y, gp.z), gp.w);
        }
        if (t > 0 && wid == 0) {
#pragma unroll
            for (int k = 0; k < 5; ++k) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) ps[k] += __shfl_xor_sync(kFull, ps[k], off);
            }
            if (lane == 0) {
                const double pres = sqrt(ps[0]), dres = rho * sqrt(ps[1]);
                const double ep = P.eps_rel * fmax(sqrt(ps[2]), sqrt(ps[3])), ed = P.eps_rel * sqrt(ps[4]);
                const int num = !(isfinite(ps[0]) && isfinite(ps[1]) && isfinite(ps[2]) && isfinite(ps[3]) &&
                                  isfinite(ps[4]));
                const int conv = P.test && pres <= ep && dres <= ed;
                s_res[0] = pres; s_res[1] = dres; s_res[2] = ep; s_res[3] = ed;
                s_conv = conv; s_num = num;
                s_stop = conv || num || t >= P.max_iter;
                if (blockIdx.x == 0 && P.trace_every > 0 && (t % P.trace_every) == 0) {
                    const long long row = t / P.trace_every - 1;
                    if (row < P.trace_cap) {
                        double* tr = P.trace + row * 5;
                        tr[0] = (double)(total0 + t); tr[1] = pres; tr[2] = dres; tr[3] = ep; tr[4] = ed;
                        P.ctrl->trace_rows = row + 1;
                    }
                }
            }
        }
        __syncthreads();
        if (t > 0 && s_stop) break;
        // L-phase
        double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int task = wid; task < NT; task += RW) {
            const int4 tr = stasks[task];
            if (tr.z == 1) res_task<1>(tr, sinfo, saoff, sabar, sbbar, sxl, slam, xgn, rho, inv_rho, acc, lane);
            else res_task<2>(tr, sinfo, saoff, sabar, sbbar, sxl, slam, xgn, rho, inv_rho, acc, lane);
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
        double* xn_ex = P.xchg + (size_t)nxt * P.n_exp;       // boundary copies -> exchange buffer
        for (int i = tid; i < NX; i += RB) {
            const int2 e = expl[i];
            __stcg(xn_ex + e.y, u_of(sxl[e.x], slam[e.x], inv_rho));
        }
        if (tid == 0) {
            double* part = P.partial + (size_t)((t + 1) & 1) * G * 8 + (size_t)blockIdx.x * 8;
            for (int k = 0; k < 5; ++k) {
                double s = 0.0;
                for (int w = 0; w < RW; ++w) s += red[w][k];
                __stcg(part + k, s);
            }
        }
        ++t;
        cur = nxt;
        if (G > 1) { target += G; grid_sync(bar, target); } else __syncthreads();
    }

    // write the iterate back (x_s and lambda are one contiguous region) and this chunk's x
    {
        const int4* src = (const int4*)(sm + H.off_xl);
        int4* dst = (int4*)(blob + H.off_xl);
        const int n16 = (H.off_gpar - H.off_xl) / 16;
        for (int i = tid; i < n16; i += RB) __stcg(dst + i, src[i]);
    }
    const double* xfin = sxg + ((t & 1) ? NG : 0);
    for (int j = tid; j < NG; j += RB) {
        const int g = gown[j];
        if (g >= 0) __stcg(P.x + g, xfin[j]);
    }
    if (G > 1) { target += G; grid_sync(bar, target); } else __syncthreads();
    if (blockIdx.x == 0 && tid == 0) {
        double obj = 0.0;
        for (int j = 0; j < P.n_obj; ++j) obj += P.obj_c[j] * __ldcg(P.x + P.obj_idx[j]);
        DevCtrl* c = P.ctrl;
        c->res[0] = s_res[0]; c->res[1] = s_res[1]; c->res[2] = s_res[2]; c->res[3] = s_res[3];
        c->objective = obj;
        c->iters = t;
        c->total = total0 + t;
        c->outcome = s_conv ? LOPF_CONVERGED : LOPF_MAX_ITER;
        c->numeric = s_num;
    }
}

// a3 for the resident layout: x_s = x0, lambda = 0, u = x0 in every blob; sweep counter 0.
__global__ void reset_resident_kernel(ResProblem P) {
    const CtaHdr& H = P.hdr[blockIdx.x];
    uint8_t* blob = P.blobs + H.blob_off;
    double* xl = (double*)(blob + H.off_xl);
    double* lam = (double*)(blob + H.off_lam);
    const double* x0 = P.x0 + H.slot_base;
    for (int i = threadIdx.x; i < H.n_slots; i += blockDim.x) {
        xl[i] = x0[i];
        lam[i] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.ctrl->arrive = 0; P.ctrl->flag = 0; P.ctrl->total = 0; P.ctrl->iters = 0; P.ctrl->trace_rows = 0;
    }
}

}  // namespace

lopf_status resident_capacity(int* sms, int* smem_optin, std::string& err) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_resident(const ResProblem& P, void* stream, std::string& err) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaFuncSetAttribute(admm_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P.max_smem);
    if (e == cudaSuccess) e = cudaMemsetAsync(P.ctrl, 0, 2 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(&P.ctrl->trace_rows, 0, sizeof(long long), s);
    if (e == cudaSuccess && P.max_iter > 0) {
        ResProblem Q = P;
        void* args[] = {&Q};
        e = cudaLaunchCooperativeKernel((const void*)admm_resident_kernel, dim3(P.G), dim3(RB), args, P.max_smem, s);
    }
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_reset_resident(const ResProblem& P, void* stream, std::string& err) {
    reset_resident_kernel<<<P.G, 256, 0, (cudaStream_t)stream>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

}  // namespace lopf

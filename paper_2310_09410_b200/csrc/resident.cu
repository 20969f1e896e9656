// SMEM-resident ADMM kernel for sm_100a: Algorithm 1 of arXiv 2310.09410
// with every CTA owning a connected, DFS-contiguous chunk of the feeder.
//
// At launch each CTA copies its blob (operators Abar_s / bbar_s, maps, iterate) into shared memory;
// the iterate then stays on chip for the whole solve, ping-ponged by sweep parity.  Per sweep t+1:
//   workers (31 warps), one lane per row slot of a packed task:
//     a4  x_g = clamp((sum_{k in seg(g)} u_k - c_g/rho) / nu_g, lo_g, hi_g)   (closed_1, rho restored;
//         PAPER.md:305-310, reading C1) in canonical copy order; u_k = x_k - lambda_k/rho is formed from
//         SMEM for this CTA's copies and read from the L2 exchange buffer for boundary copies
//     a5  d = -rho v - lambda, x_s = (1/rho) Abar_s d + bbar_s                  (closed_2)
//     a6  lambda_s += rho (v - x_s)                                            (ADMM-3)
//         boundary copies publish u to the exchange buffer; five residual sums per lane
//   reducer (1 warp), concurrently: waits until every CTA has published sweep t, reduces the residual
//     partials of sweep t in CTA order and takes the (termination) decision;
//     identical in every CTA.  A stop at t discards the speculative sweep t+1 (state t is the other
//     ping-pong buffer).
//   publish: CTA partials, then flag[c] = t+2 (release); wait for the neighbour CTAs' flags only.
// No grid-wide barrier inside the loop; one at exit.  Diagnostics: optional per-CTA cycle counters.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"

namespace lopf {

namespace {

constexpr int RB = kResBlock;
constexpr int RW = RB / 32;
constexpr int NWORK = RW - 1;              // worker warps 0 .. RW-2
constexpr int RED = RW - 1;                // reducer warp
constexpr unsigned kFull = 0xffffffffu;

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
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// consensus input u = x_s - lambda / rho, formed with the same rounding wherever it is needed
__device__ __forceinline__ double u_of(const double x, const double l, const double inv_rho) {
    return __fma_rn(-l, inv_rho, x);
}

struct Ctx {
    const int32_t* sinfo;
    const int32_t* saoff;
    const int32_t* sexp;
    const double* sabar;
    const double* sbbar;
    const int32_t* gsegoff;
    const int32_t* gseg;
    const double4* gpar;
    const double* xl_c;
    const double* lam_c;
    double* xl_n;
    double* lam_n;
    double* xout_n;
    const double* xch_c;
    double* xch_n;
    double rho, inv_rho;
};

template <int R>
__device__ __forceinline__ void task_sweep(const Ctx& C, const int4 tr, double* __restrict__ dst, double (&acc)[5],
                                           const int lane) {
    double v[R], lam[R], xo[R];
    int info[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        const int slot = tr.x + h * 32 + lane;
        info[h] = C.sinfo[slot];
        double d = 0.0;
        v[h] = lam[h] = xo[h] = 0.0;
        if (info[h] & kResValid) {
            const int gl = info[h] >> kResGlShift;
            const int q0 = C.gsegoff[gl], q1 = C.gsegoff[gl + 1];
            double sigma = 0.0;                                          // canonical copy order
            for (int q = q0; q < q1; ++q) {
                const int e = C.gseg[q];
                sigma += e >= 0 ? u_of(C.xl_c[e], C.lam_c[e], C.inv_rho) : __ldcg(C.xch_c + (-e - 1));
            }
            const double4 gp = C.gpar[gl];
            const double xg = fmin(fmax((sigma - gp.x) * gp.y, gp.z), gp.w);   // IEEE +-inf = no clamp
            if (info[h] & kResFirst) C.xout_n[gl] = xg;
            v[h] = xg;
            lam[h] = C.lam_c[slot];
            xo[h] = C.xl_c[slot];
            d = -C.rho * xg - lam[h];
        }
        dst[h * 32 + lane] = d;
    }
    __syncwarp();
    double ax[R];
    int ns[R], ao[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        ax[h] = 0.0;
        ns[h] = (info[h] >> kResNsShift) & 0x7F;                        // 0 for unused lanes
        ao[h] = C.saoff[tr.x + h * 32 + lane];
    }
    const double* __restrict__ db = dst + (R == 1 ? (info[0] & 0x3F) : 0);
    const int kmax = tr.y;
#pragma unroll 4
    for (int k = 0; k < kmax; ++k) {
#pragma unroll
        for (int h = 0; h < R; ++h)
            if (k < ns[h]) ax[h] = fma(C.sabar[ao[h] + k * ns[h]], db[k], ax[h]);   // sum_k Abar_s[r][k] d_k
    }
    __syncwarp();                                                        // dst is reused by the next task
#pragma unroll
    for (int h = 0; h < R; ++h) {
        if (!(info[h] & kResValid)) continue;
        const int slot = tr.x + h * 32 + lane;
        const double xn = fma(ax[h], C.inv_rho, C.sbbar[slot]);          // (1/rho) Abar d + bbar  (closed_2)
        const double ln = lam[h] + C.rho * (v[h] - xn);                  // ADMM-3
        C.xl_n[slot] = xn;
        C.lam_n[slot] = ln;
        const int e = C.sexp[slot];
        if (e >= 0) __stcg(C.xch_n + e, u_of(xn, ln, C.inv_rho));        // boundary copy -> exchange
        const double r = v[h] - xn, dx = xn - xo[h];
        acc[0] += r * r;
        acc[1] += dx * dx;
        acc[2] += v[h] * v[h];
        acc[3] += xn * xn;
        acc[4] += ln * ln;
    }
}

__global__ void __launch_bounds__(RB, 1) admm_resident_kernel(ResProblem P) {
    extern __shared__ __align__(16) uint8_t sm[];
    __shared__ CtaHdr H;
    __shared__ double red[RW][5];
    __shared__ double s_res[4];
    __shared__ int s_stop, s_conv, s_num;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    if (tid < (int)(sizeof(CtaHdr) / 4)) ((int*)&H)[tid] = ((const int*)(P.hdr + cta))[tid];
    if (tid == 0) { s_stop = 0; s_conv = 0; s_num = 0; s_res[0] = s_res[1] = s_res[2] = s_res[3] = 0.0; }
    __syncthreads();
    uint8_t* blob = P.blobs + H.blob_off;
    {
        const int4* src = (const int4*)blob;
        int4* d16 = (int4*)sm;
        const int n16 = H.blob_bytes / 16;
        for (int i = tid; i < n16; i += RB) d16[i] = __ldcg(src + i);
    }
    __syncthreads();
    const int NS = H.n_slots, NG = H.n_glob, NT = H.n_tasks, NNB = H.n_nbr;
    double* xl[2] = {(double*)(sm + H.off_xl0), (double*)(sm + H.off_xl1)};
    double* lm[2] = {(double*)(sm + H.off_lam0), (double*)(sm + H.off_lam1)};
    double* xout = (double*)(sm + H.off_xout);                   // [2][NG]
    const int32_t* sexp = (const int32_t*)(sm + H.off_sexp);
    const int32_t* gown = (const int32_t*)(sm + H.off_gown);
    const int32_t* nbr = (const int32_t*)(sm + H.off_nbr);
    const int4* stasks = (const int4*)(sm + H.off_tasks);
    const int dst_stride = (H.smem_bytes - H.off_dst) / (8 * RW);      // 32 or 64 doubles per warp
    double* dst = (double*)(sm + H.off_dst) + wid * dst_stride;
    Ctx C;
    C.sinfo = (const int32_t*)(sm + H.off_sinfo);
    C.saoff = (const int32_t*)(sm + H.off_aoff);
    C.sexp = sexp;
    C.sabar = (const double*)(sm + H.off_abar);
    C.sbbar = (const double*)(sm + H.off_bbar);
    C.gsegoff = (const int32_t*)(sm + H.off_gsegoff);
    C.gseg = (const int32_t*)(sm + H.off_gseg);
    C.gpar = (const double4*)(sm + H.off_gpar);
    C.rho = P.rho;
    C.inv_rho = P.inv_rho;
    const long long total0 = *(volatile long long*)&P.ctrl->total;
    const bool prof = P.prof != nullptr;
    long long c_w = 0, c_p = 0, c0 = 0;

    // initial publication: boundary u of the state into exchange slot 0; flag = 1
    for (int i = tid; i < NS; i += RB) {
        const int e = sexp[i];
        if (e >= 0) __stcg(P.xchg + e, u_of(xl[0][i], lm[0][i], P.inv_rho));
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        st_rel(P.flags + cta, 1ULL);
        for (int i = 0; i < NNB; ++i)
            while (ld_acq(P.flags + nbr[i]) < 1ULL) {
            }
    }
    __syncthreads();

    long long t = 0;                                   // sweeps completed; state t in buffer t & 1
    for (;;) {
        const int cur = (int)(t & 1), nxt = cur ^ 1;
        if (prof && tid == 0) c0 = clock64();
        if (wid == RED) {
            if (t >= 1) {                              // decision for sweep t
                const unsigned long long need = (unsigned long long)t + 1ULL;
                for (;;) {
                    bool ok = true;
                    for (int b = lane; b < G; b += 32) ok &= ld_rlx(P.flags + b) >= need;
                    if (__all_sync(kFull, ok)) break;
                    __nanosleep(32);
                }
                fence_acq_rel();
                double ps[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                const double* part = P.partial + (size_t)(t & 1) * G * 8;
                for (int b = lane; b < G; b += 32) {
#pragma unroll
                    for (int k = 0; k < 5; ++k) ps[k] += __ldcg(part + (size_t)b * 8 + k);
                }
#pragma unroll
                for (int k = 0; k < 5; ++k) {
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) ps[k] += __shfl_xor_sync(kFull, ps[k], off);
                }
                if (lane == 0) {
                    const double pres = sqrt(ps[0]), dres = P.rho * sqrt(ps[1]);
                    const double ep = P.eps_rel * fmax(sqrt(ps[2]), sqrt(ps[3])), ed = P.eps_rel * sqrt(ps[4]);
                    const int num = !(isfinite(ps[0]) && isfinite(ps[1]) && isfinite(ps[2]) && isfinite(ps[3]) &&
                                      isfinite(ps[4]));
                    const int conv = P.test && pres <= ep && dres <= ed;
                    s_res[0] = pres; s_res[1] = dres; s_res[2] = ep; s_res[3] = ed;
                    s_conv = conv; s_num = num;
                    s_stop = conv || num || t >= P.max_iter;
                    if (cta == 0 && P.trace_every > 0 && (t % P.trace_every) == 0) {
                        const long long row = t / P.trace_every - 1;
                        if (row < P.trace_cap) {
                            double* tr = P.trace + row * 5;
                            tr[0] = (double)(total0 + t); tr[1] = pres; tr[2] = dres; tr[3] = ep; tr[4] = ed;
                            P.ctrl->trace_rows = row + 1;
                        }
                    }
                }
            }
        } else {                                       // workers: sweep t+1 (speculative until decided)
            double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            if (t < P.max_iter && !(P.skip & 2)) {
                C.xl_c = xl[cur]; C.lam_c = lm[cur]; C.xl_n = xl[nxt]; C.lam_n = lm[nxt];
                C.xout_n = xout + nxt * NG;
                C.xch_c = P.xchg + (size_t)cur * P.n_exp;
                C.xch_n = P.xchg + (size_t)nxt * P.n_exp;
                for (int task = wid; task < NT; task += NWORK) {
                    const int4 tr = stasks[task];
                    if (tr.z == 1) task_sweep<1>(C, tr, dst, acc, lane);
                    else task_sweep<2>(C, tr, dst, acc, lane);
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
        }
        __syncthreads();                               // [A]
        if (prof && tid == 0) { const long long c1 = clock64(); c_w += c1 - c0; c0 = c1; }
        if (s_stop) break;                             // state t (buffer cur); x^t in xout[cur]
        if (wid == 0) {                                // publish sweep t+1, then wait for the neighbours
            double s[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                s[k] = lane < NWORK ? red[lane][k] : 0.0;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) s[k] += __shfl_xor_sync(kFull, s[k], off);
            }
            if (lane == 0) {
                double* part = P.partial + (size_t)((t + 1) & 1) * G * 8 + (size_t)cta * 8;
#pragma unroll
                for (int k = 0; k < 5; ++k) __stcg(part + k, s[k]);
                __threadfence();
                st_rel(P.flags + cta, (unsigned long long)t + 2ULL);
            }
            const unsigned long long need = (unsigned long long)t + 2ULL;
            for (int i = lane; i < NNB; i += 32)
                while (ld_acq(P.flags + nbr[i]) < need) {
                }
            __syncwarp();
        }
        __syncthreads();                               // [B]
        if (prof && tid == 0) c_p += clock64() - c0;
        ++t;
    }

    // exit: state t (buffer t & 1) back to the blob, this CTA's x, then one grid barrier for the result
    const int fin = (int)(t & 1);
    {
        double* gx = (double*)(blob + H.off_xl0);
        double* gl = (double*)(blob + H.off_lam0);
        for (int i = tid; i < NS; i += RB) {
            __stcg(gx + i, xl[fin][i]);
            __stcg(gl + i, lm[fin][i]);
        }
    }
    for (int j = tid; j < NG; j += RB) {
        const int g = gown[j];
        if (g >= 0) __stcg(P.x + g, xout[fin * NG + j]);
    }
    if (prof && tid == 0) {
        long long* pr = P.prof + 4 * cta;
        pr[0] = c_w; pr[1] = c_p; pr[2] = 0; pr[3] = t;
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        atomicAdd(&P.ctrl->arrive, 1ULL);
        if (cta == 0) {
            while (ld_acq(&P.ctrl->arrive) < (unsigned long long)G) {
            }
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
}

// a3 for the resident layout: x_s = x0, lambda = 0 in every blob; sweep counter 0.
__global__ void reset_resident_kernel(ResProblem P) {
    const CtaHdr& H = P.hdr[blockIdx.x];
    uint8_t* blob = P.blobs + H.blob_off;
    double* xl = (double*)(blob + H.off_xl0);
    double* lam = (double*)(blob + H.off_lam0);
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
    if (e == cudaSuccess) e = cudaMemsetAsync(P.flags, 0, sizeof(unsigned long long) * P.G, s);
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

// Batch kernel for sm_100a (config 4): many load scenarios of one feeder, each an
// independent run of Algorithm 1 with its own termination test.
//
// Lane = scenario: a CTA owns a group of 32 scenarios and its 8 warps split the subsystems.  All
// per-scenario arrays are scenario-fastest, so for every copy / operator entry a warp touches one
// 256-byte line; operators of subsystems without a load are the same for every scenario (uniform
// addresses: broadcast loads served by L1/L2).  Per sweep and subsystem:
//   phase 1  consensus (closed_1, rho restored) for each row's global from the ping-pong iterate,
//            d = -rho v - lambda staged in SMEM per warp
//   phase 2  x_s = (1/rho) Abar_s d + bbar_s (closed_2), lambda += rho (v - x_s) (ADMM-3), residual sums
// then the five per-scenario sums are reduced across warps in fixed order and each scenario takes its
// own stop decision; converged scenarios freeze (their lanes stop writing).  No inter-CTA
// synchronisation at all: groups are independent problems.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"

namespace lopf {

namespace {

constexpr int BB = kBatchBlock;
constexpr int BW = kBatchWarps;

__device__ __forceinline__ double u_of(const double x, const double l, const double inv_rho) {
    return __fma_rn(-l, inv_rho, x);
}

__global__ void __launch_bounds__(BB, 1) admm_batch_kernel(BatchProblem P) {
    extern __shared__ double dsh[];                 // [BW][2][ns_max][32]: staged d and v
    __shared__ double red[BW][5][32];
    __shared__ int s_act[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    double* dst = dsh + (size_t)w * 2 * P.ns_max * 32;
    double* vst = dst + (size_t)P.ns_max * 32;
    const int s0 = P.warp_sub[w], s1 = P.warp_sub[w + 1];
    const size_t buf = (size_t)P.n_grp * P.nc * 32;      // doubles per ping-pong buffer
    for (int grp = blockIdx.x; grp < P.n_grp; grp += gridDim.x) {
        const int sc = grp * 32 + lane;
        const bool valid = sc < P.n_scen;
        const long long tot0 = valid ? P.res[sc].total : 0;
        if (w == 0) s_act[lane] = valid;
        double last[4] = {0.0, 0.0, 0.0, 0.0};
        long long t = 0;
        __syncthreads();
        const size_t gofs = (size_t)grp * P.nc * 32 + lane;
        for (; t < P.max_iter; ++t) {
            const bool act = s_act[lane];
            if (!__syncthreads_or(act)) break;
            const int cur = (int)((tot0 + t) & 1);               // per-lane parity (scenarios may differ)
            const double* xl_c = P.xl + (size_t)cur * buf + gofs;
            const double* lm_c = P.lam + (size_t)cur * buf + gofs;
            double* xl_n = P.xl + (size_t)(cur ^ 1) * buf + gofs;
            double* lm_n = P.lam + (size_t)(cur ^ 1) * buf + gofs;
            double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            for (int s = s0; s < s1; ++s) {
                const int ns = P.sub_ns[s], o = P.sub_ptr[s], op = P.sub_op[s];
                for (int r = 0; r < ns; ++r) {                     // phase 1: consensus, d
                    const int2 ci = P.copy_info[o + r];
                    const int q0 = P.seg_ptr[ci.x], q1 = P.seg_ptr[ci.x + 1];
                    double sigma = 0.0;                            // canonical copy order
                    for (int q = q0; q < q1; ++q) {
                        const size_t k = (size_t)P.seg_copy[q] * 32;
                        sigma += u_of(xl_c[k], lm_c[k], P.inv_rho);
                    }
                    const double4 gp = P.gpar[ci.x];
                    const double xg = fmin(fmax((sigma - gp.x) * gp.y, gp.z), gp.w);
                    if (act && ci.y) P.xout[((size_t)grp * P.n + ci.x) * 32 + lane] = xg;
                    const double l = lm_c[(size_t)(o + r) * 32];
                    dst[r * 32 + lane] = -P.rho * xg - l;
                    vst[r * 32 + lane] = xg;
                }
                __syncwarp();
                const double* Ash = P.shared_abar + (op >= 0 ? op : 0);
                const int vi = op >= 0 ? 0 : -op - 1;
                const double* Avar = P.var_abar + ((size_t)grp * P.VA + (op >= 0 ? 0 : P.vsub_a[vi])) * 32 + lane;
                const double* Bvar = P.var_bbar + ((size_t)grp * P.VB + (op >= 0 ? 0 : P.vsub_b[vi])) * 32 + lane;
                for (int r = 0; r < ns; ++r) {                     // phase 2: local + dual update
                    double y = 0.0;
                    if (op >= 0) {
#pragma unroll 4
                        for (int k = 0; k < ns; ++k) y = fma(Ash[r * ns + k], dst[k * 32 + lane], y);
                    } else {
#pragma unroll 4
                        for (int k = 0; k < ns; ++k) y = fma(Avar[(size_t)(r * ns + k) * 32], dst[k * 32 + lane], y);
                    }
                    const double bb = op >= 0 ? 0.0 : Bvar[(size_t)r * 32];
                    const double xn = fma(y, P.inv_rho, bb);         // (1/rho) Abar d + bbar
                    const double v = vst[r * 32 + lane];
                    const size_t k = (size_t)(o + r) * 32;
                    const double l = lm_c[k], xo = xl_c[k];
                    const double ln = l + P.rho * (v - xn);          // ADMM-3
                    if (act) {
                        xl_n[k] = xn;
                        lm_n[k] = ln;
                        const double rr = v - xn, dx = xn - xo;
                        acc[0] += rr * rr;
                        acc[1] += dx * dx;
                        acc[2] += v * v;
                        acc[3] += xn * xn;
                        acc[4] += ln * ln;
                    }
                }
                __syncwarp();
            }
#pragma unroll
            for (int q = 0; q < 5; ++q) red[w][q][lane] = acc[q];
            __syncthreads();
            if (w == 0 && act) {                                   // per-scenario (termination)
                double sm5[5];
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    double a = 0.0;
                    for (int ww = 0; ww < BW; ++ww) a += red[ww][q][lane];
                    sm5[q] = a;
                }
                const double pres = sqrt(sm5[0]), dres = P.rho * sqrt(sm5[1]);
                const double ep = P.eps_rel * fmax(sqrt(sm5[2]), sqrt(sm5[3])), ed = P.eps_rel * sqrt(sm5[4]);
                last[0] = pres; last[1] = dres; last[2] = ep; last[3] = ed;
                const bool num = !(isfinite(sm5[0]) && isfinite(sm5[1]) && isfinite(sm5[2]) && isfinite(sm5[3]) &&
                                   isfinite(sm5[4]));
                const bool conv = P.test && pres <= ep && dres <= ed;
                if (conv || num) {
                    ScenResult& R = P.res[sc];
                    R.iters = t + 1;
                    R.total = tot0 + t + 1;
                    R.status = num ? 3 : 1;
                    R.res[0] = pres; R.res[1] = dres; R.res[2] = ep; R.res[3] = ed;
                    s_act[lane] = 0;
                }
            }
            __syncthreads();
        }
        if (w == 0 && valid) {
            ScenResult& R = P.res[sc];
            if (s_act[lane]) {                                     // ran out of sweeps in this launch
                R.iters = t;
                R.total = tot0 + t;
                R.status = 2;
                R.res[0] = last[0]; R.res[1] = last[1]; R.res[2] = last[2]; R.res[3] = last[3];
            }
            double obj = 0.0;
            for (int j = 0; j < P.n_obj; ++j) obj += P.obj_c[j] * P.xout[((size_t)grp * P.n + P.obj_idx[j]) * 32 + lane];
            R.objective = obj;
        }
        __syncthreads();
    }
}

// a3 for every scenario: buffer 0 = x0, lambda = 0, counters cleared.
__global__ void reset_batch_kernel(BatchProblem P, const double* __restrict__ x0) {
    const size_t n = (size_t)P.n_grp * P.nc * 32;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t k = (i / 32) % P.nc;
        P.xl[i] = x0[k];
        P.lam[i] = 0.0;
    }
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (size_t)P.n_grp * 32; i += (size_t)gridDim.x * blockDim.x) {
        ScenResult& R = P.res[i];
        R.iters = 0; R.total = 0; R.status = 0; R.objective = 0.0;
        R.res[0] = R.res[1] = R.res[2] = R.res[3] = 0.0;
    }
}

}  // namespace

lopf_status launch_batch(const BatchProblem& P, void* stream, std::string& err) {
    cudaStream_t s = (cudaStream_t)stream;
    const int smem = (int)(sizeof(double) * BW * 2 * P.ns_max * 32);
    cudaError_t e = cudaFuncSetAttribute(admm_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0, sms = 0, per = 0;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, admm_batch_kernel, BB, smem);
    if (e == cudaSuccess && per < 1) { err = "batch kernel cannot be resident"; return LOPF_E_CUDA; }
    const int grid = P.n_grp < sms * per ? P.n_grp : sms * per;
    if (e == cudaSuccess && P.max_iter > 0) {
        admm_batch_kernel<<<grid, BB, smem, s>>>(P);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_reset_batch(const BatchProblem& P, const double* x0, void* stream, std::string& err) {
    reset_batch_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(P, x0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

}  // namespace lopf

// Batch kernel for sm_100a (config 4): many load scenarios of one feeder, each an
// independent run of Algorithm 1 with its own (termination) test.
//
// Lane = scenario.  Scenarios form groups of 32 and every per-scenario array is [group][entry][32], so a
// warp instruction moves one 256-byte line for 32 scenarios while everything structural -- rows, segment
// lists, bounds, the operators of subsystems without a load -- is the same address for all 32 lanes
// (uniform loads).  A work item is (group, task), a task a depth-first run of subsystems; per item and
// subsystem s the warp computes, for its 32 scenarios at once,
//   a4  x_g = clamp((sum_{k in seg(g)} u_k - c_g/rho) / nu_g, lo_g, hi_g) for each row (closed_1, rho
//       restored, reading C1), canonical copy order; d = -rho v - lambda staged in SMEM [row][lane]
//   a5  y = Abar_s d, one row quad at a time (k ascending, FMA); Abar_s from the shared pool (row quads
//       [k][4], one 4-wide uniform load per column) or, for a load subsystem, the scenario's quad-block
//       upper layout ([entry][lane], coalesced, every operand at an immediate offset of one block pointer)
//   a6  x_s = y / rho + bbar_s, lambda += rho (v - x_s), u = x_s - lambda / rho     (closed_2, ADMM-3)
//   a7  five residual sums per lane (scenario), written per item
// The ACTIVE items of a sweep (groups with a scenario still running, times tasks) are handed out one at a
// time from an atomic counter, costliest tasks first.  Grid barrier; one warp per active group then sums
// each scenario's item partials in task order (deterministic whichever warp ran an item) and takes its
// decision; converged scenarios freeze (their lanes stop storing), a group leaves the item list when all
// 32 have; grid barrier.
#include <cuda_runtime.h>

#include <cmath>

#include "device.cuh"
#include "internal.h"

namespace lopf {

namespace {

using dev::grid_sync;
using dev::kFull;

#ifndef LOPF_BATCH_CROWS
#define LOPF_BATCH_CROWS 4                    // consensus rows whose gathers are issued together
#endif
#ifndef LOPF_BATCH_L2PF
#define LOPF_BATCH_L2PF 1                     // per-subsystem lane-parallel L2 prefetch (fp64 only: fp32 A/B 291 ->
                                              // 235 us without it): 1 x_s, 2 the operator, 4 lambda, 8 own u rows
#endif
constexpr int BW = kBatchWarps;
constexpr int CR = LOPF_BATCH_CROWS;
constexpr int BB = 32 * BW;

template <class T> struct V2;                 // {c/rho, lo}, {hi, 1/nu} per global
template <> struct V2<double> { using type = double2; };
template <> struct V2<float> { using type = float2; };

#ifndef LOPF_BATCH_EVICT
#define LOPF_BATCH_EVICT 1                    // L2 evict_first on last-use loads and on every state store: 1 fp32
#endif                                        // only (fp64 A/B: DRAM 1.54 -> 1.44 GB per sweep, time +0.5%), 2 both

// L2 eviction hints: a line's last use in a sweep (and every store of the state, read again only a sweep
// = ~1 GB of traffic later) is marked evict_first, so the L2 keeps the lines a sweep re-reads soon
// (lambda and the parked v of the current subsystem, neighbouring u, the shared operators).
__device__ __forceinline__ unsigned long long pol_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_last(const double* p, unsigned long long pol) {
    if (LOPF_BATCH_EVICT != 2) return __ldcg(p);
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_last(const float* p, unsigned long long pol) {
    if (!LOPF_BATCH_EVICT) return __ldcg(p);
    float v;
    asm volatile("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_op(const double* p, unsigned long long pol) {
    if (LOPF_BATCH_EVICT != 2) return __ldg(p);
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_op(const float* p, unsigned long long pol) {
    if (!LOPF_BATCH_EVICT) return __ldg(p);
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_first(double* p, double v, unsigned long long pol) {
    if (LOPF_BATCH_EVICT != 2) { __stcg(p, v); return; }
    asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_first(float* p, float v, unsigned long long pol) {
    if (!LOPF_BATCH_EVICT) { __stcg(p, v); return; }
    asm volatile("st.global.cg.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}

// four consecutive T of a 4-aligned address, same for every lane (uniform 16-byte loads)
__device__ __forceinline__ void ld4_uniform(const double* p, double (&a)[4]) {
    const double2 lo = __ldg(reinterpret_cast<const double2*>(p)), hi = __ldg(reinterpret_cast<const double2*>(p) + 1);
    a[0] = lo.x; a[1] = lo.y; a[2] = hi.x; a[3] = hi.y;
}
__device__ __forceinline__ void ld4_uniform(const float* p, float (&a)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
}

__device__ __forceinline__ void prefetch_l2_line(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Per-warp shared memory: d of the current subsystem [kBatchDMax][32] (a subsystem with more rows keeps
// its d in the global scratch `dscr` instead, an L2-resident [group][row][32] array), and the records of
// up to 32 rows ({g, info, n0..n3} and {c/rho, lo, hi, 1/nu}) staged by one coalesced load per lane, so
// the row loop reads its uniform metadata with shared-memory broadcasts instead of dependent global loads.
template <class T>
struct WarpSmem {
    T* d;                                      // [kBatchDMax][32]
    int* mi;                                   // [32][6]
    T* mp;                                     // [32][4]
};
template <class T>
__host__ __device__ constexpr int warp_smem_bytes() {
    return kBatchDMax * 32 * (int)sizeof(T) + 32 * 6 * 4 + 32 * 4 * (int)sizeof(T);
}

// One subsystem of a (group, task) item for the 32 scenarios of the group (lane = scenario; `act`: the
// lane's scenario is running -- frozen or padding lanes compute but store nothing and add nothing).  Every
// loop keeps many independent loads in flight: four rows' gathers at a time, the mat-vec's operator loads
// of four rows x four columns, the four rows' finish loads.  BIG: d in the global scratch.
template <class T, bool BIG>
__device__ __forceinline__ void batch_sub(const BatchProblem& B, const int4 sm, const size_t gb,
                                          const T* __restrict__ ucur, T* __restrict__ unext, const WarpSmem<T>& W,
                                          const int lane, const bool act, double (&acc)[5], const size_t grp) {
    using T2 = typename V2<T>::type;
    const T rho = (T)B.rho, inv_rho = (T)B.inv_rho;
    const unsigned long long pf = pol_first();
    // this group's lane views: element (row r) at [32 r] (32-bit indices on 64-bit bases)
    const T* __restrict__ ug = ucur + gb * 32 + lane;
    T* __restrict__ ung = unext + gb * 32 + lane;
    T* __restrict__ xlg = reinterpret_cast<T*>(B.xl) + gb * 32 + lane;
    T* __restrict__ lmg = reinterpret_cast<T*>(B.lam) + gb * 32 + lane;
    T* __restrict__ xg = reinterpret_cast<T*>(B.x) + grp * B.n * 32 + lane;
    const T2* __restrict__ gpar = reinterpret_cast<const T2*>(B.gpar);
    const int2* __restrict__ rows = reinterpret_cast<const int2*>(B.rows);
    const int row0 = sm.x, ns = sm.y;
    T* __restrict__ dd = BIG ? reinterpret_cast<T*>(B.dscr) + (gb + row0) * 32 + lane : W.d + lane;   // d_r at dd[32 r]
    const bool var = sm.w & kBVar;
    const T* __restrict__ V = reinterpret_cast<const T*>(B.vpool) + (grp * B.ve + (var ? sm.z : 0)) * 32 + lane;
    if (LOPF_BATCH_L2PF && sizeof(T) == 8) {
        // lane-parallel L2 prefetch of the lines this subsystem streams from HBM (x_s read in the finish, the
        // per-scenario operator in the mat-vec), issued before the consensus so they arrive while it runs
        const char* xb = reinterpret_cast<const char*>(xlg - lane);
        const int xlines = (int)(ns * 32 * sizeof(T) / 128);
        if (LOPF_BATCH_L2PF & 1)
            for (int e = lane; e < xlines; e += 32) prefetch_l2_line(xb + (size_t)(32 * row0) * sizeof(T) + 128 * e);
        if (LOPF_BATCH_L2PF & 4) {
            const char* lb = reinterpret_cast<const char*>(lmg - lane);
            for (int e = lane; e < xlines; e += 32) prefetch_l2_line(lb + (size_t)(32 * row0) * sizeof(T) + 128 * e);
        }
        if (LOPF_BATCH_L2PF & 8) {
            const char* ub = reinterpret_cast<const char*>(ug - lane);
            for (int e = lane; e < xlines; e += 32) prefetch_l2_line(ub + (size_t)(32 * row0) * sizeof(T) + 128 * e);
        }
        if ((LOPF_BATCH_L2PF & 2) && var) {
            const char* vb = reinterpret_cast<const char*>(V - lane);
            const int nl = (batch_var_entries(ns) + ns) * (int)(32 * sizeof(T) / 128);
            for (int e = lane; e < nl; e += 32) prefetch_l2_line(vb + 128 * e);
        }
    }
    // a4: consensus of every row's global, 32 rows per chunk; v parked in unext (replaced by u below)
    for (int c0 = 0; c0 < ns; c0 += 32) {
        const int nrow = min(32, ns - c0);
        if (lane < nrow) {                                              // lane l stages row c0 + l's records
            const int row = row0 + c0 + lane;
            const int2 a = __ldg(rows + 3 * row), b = __ldg(rows + 3 * row + 1), c = __ldg(rows + 3 * row + 2);
            int* mi = W.mi + lane * 6;
            mi[0] = a.x; mi[1] = a.y; mi[2] = b.x; mi[3] = b.y; mi[4] = c.x; mi[5] = c.y;
            const T2 p0 = __ldg(gpar + 2 * a.x), p1 = __ldg(gpar + 2 * a.x + 1);
            T* mp = W.mp + lane * 4;
            mp[0] = p0.x; mp[1] = p0.y; mp[2] = p1.x; mp[3] = p1.y;
        }
        __syncwarp();
        for (int r = 0; r < nrow; r += CR) {
            T ua[CR][4], lm[CR];
#pragma unroll
            for (int i = 0; i < CR; ++i) {                              // every load of CR rows first
                const int rr = min(r + i, nrow - 1);
                const int* mi = W.mi + rr * 6;
                const int inf = mi[1];
                const bool inl = inf & kBInline;
                const int nu = inl ? (inf >> kBNuShift) & 0xFF : 0;
                const int self = row0 + c0 + rr;
                ua[i][0] = __ldcg(ug + 32 * (inl ? mi[2] : self));
                ua[i][1] = nu > 1 ? __ldcg(ug + 32 * mi[3]) : T(0);
                ua[i][2] = nu > 2 ? __ldcg(ug + 32 * mi[4]) : T(0);
                ua[i][3] = nu > 3 ? __ldcg(ug + 32 * mi[5]) : T(0);
                lm[i] = __ldcg(lmg + 32 * self);
            }
#pragma unroll
            for (int i = 0; i < CR; ++i) {
                if (r + i >= nrow) break;
                const int* mi = W.mi + (r + i) * 6;
                const T* mp = W.mp + (r + i) * 4;
                const int g = mi[0], inf = mi[1];
                T sig = ((ua[i][0] + ua[i][1]) + ua[i][2]) + ua[i][3];   // ascending canonical copy order
                if (!(inf & kBInline)) {                                // nu > 4 (rare): the segment list
                    sig = T(0);
                    for (int q = 0; q < mi[3]; ++q) sig += __ldcg(ug + 32 * __ldg(B.seg_rows + mi[2] + q));
                }
                const T v = fmin(fmax((sig - mp[0]) * mp[3], mp[1]), mp[2]);   // IEEE +-inf = no clamp
                const int at = 32 * (row0 + c0 + r + i);
                if (act && (inf & kBFirst)) st_first(xg + 32 * g, v, pf);
                const T d = -rho * v - lm[i];
                if (BIG) __stcg(dd + (c0 + r + i) * 32, d);
                else dd[(c0 + r + i) * 32] = d;
                if (act) __stcg(ung + at, v);
            }
        }
        __syncwarp();                                                   // the row records are restaged
    }
    // a5-a7, one row quad at a time: y_r = sum_k Abar[r][k] d_k with k ascending (zero entries past n_s add
    // nothing; d past n_s reads a finite value: staged zeros, or the clamped last row for BIG)
    const int nq = (ns + 3) >> 2, nsp = nq << 2;
    const T* __restrict__ A = reinterpret_cast<const T*>(B.spool) + (var ? 0 : sm.z);
    if (!BIG) {
        __syncwarp();
        for (int k = ns; k < nsp; ++k) dd[k * 32] = T(0);
        __syncwarp();
    }
    auto dk_at = [&](const int k) -> T {
        if (BIG) return __ldcg(dd + min(k, ns - 1) * 32);
        return dd[k * 32];
    };
    for (int q = 0; q < nq; ++q) {
        T y[4] = {T(0), T(0), T(0), T(0)};
        if (var && !LOPF_BATCH_VQB) {
            // packed upper triangle, row-major: (i, j >= i) at i n - i (i - 1) / 2 + j - i; row r reads
            // (min(r, k), max(r, k)): the walk steps by n - k - 1 while k < r, then by 1
            int p[4], rq[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) p[i] = rq[i] = min(4 * q + i, ns - 1);
#pragma unroll 4
            for (int k = 0; k < ns; ++k) {
                const T dk = dk_at(k);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    y[i] = fma(ld_op(V + 32 * p[i], pf), dk, y[i]);
                    p[i] += k < rq[i] ? ns - k - 1 : 1;
                }
            }
        } else if (var) {
            // quad-block upper layout: block q' at Q(q') = sum_{p < q'} 4 (nsp - 4p) entries; for k < 4q the
            // entry (r = 4q + i, k = 4q' + j) is the stored (k, r): block q', column 4q + i, row j
            int Q = 0;
            for (int qp = 0; qp < q; ++qp) {
                const T* __restrict__ Bp = V + 32 * (Q + 16 * (q - qp));
                T dj[4], a[4][4];
#pragma unroll
                for (int j = 0; j < 4; ++j) dj[j] = dk_at(4 * qp + j);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) a[i][j] = ld_op(Bp + 32 * (4 * i + j), pf);
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) y[i] = fma(a[i][j], dj[j], y[i]);
                Q += 4 * (nsp - 4 * qp);
            }
            const T* __restrict__ Bq = V + 32 * Q;                          // block q: column k at 4 (k - 4q)
            for (int k = 4 * q; k < nsp; k += 4, Bq += 32 * 16) {
                T dj[4], a[4][4];
#pragma unroll
                for (int j = 0; j < 4; ++j) dj[j] = dk_at(k + j);
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[i][j] = ld_op(Bq + 32 * (4 * j + i), pf);
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) y[i] = fma(a[i][j], dj[j], y[i]);
            }
        } else {
            // row quad q: [k][4] over the padded width, one 4-wide uniform load per column
            const T* __restrict__ Aq = A + q * nsp * 4;
            for (int k = 0; k < nsp; k += 4, Aq += 16) {
                T dj[4], a[4][4];
#pragma unroll
                for (int j = 0; j < 4; ++j) dj[j] = dk_at(k + j);
#pragma unroll
                for (int j = 0; j < 4; ++j) ld4_uniform(Aq + 4 * j, a[j]);
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) y[i] = fma(a[j][i], dj[j], y[i]);
            }
        }
        const int r0 = 4 * q;
        int rr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) rr[i] = min(r0 + i, ns - 1);        // rows past n_s: discarded
        T vv[4], lam[4], xo[4], bb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {                                   // the four rows' loads first
            const int at = 32 * (row0 + rr[i]);
            vv[i] = ld_last(ung + at, pf);
            lam[i] = ld_last(lmg + at, pf);
            xo[i] = ld_last(xlg + at, pf);
            bb[i] = (sm.w & kBBbar) ? ld_op(V + 32 * (batch_var_entries(ns) + rr[i]), pf) : T(0);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (r0 + i >= ns) break;
            const int at = 32 * (row0 + r0 + i);
            const T xn = fma(y[i], inv_rho, bb[i]);                     // (1/rho) Abar d + bbar
            const T v = vv[i];
            const T ln = lam[i] + rho * (v - xn);                       // ADMM-3
            const T un = xn - ln * inv_rho;                             // next consensus input
            if (act) {
                st_first(xlg + at, xn, pf);
                st_first(lmg + at, ln, pf);
                st_first(ung + at, un, pf);
                const T rs = v - xn, dx = xn - xo[i];                   // terms in T, sums in fp64 (F1)
                acc[0] += (double)(rs * rs);
                acc[1] += (double)(dx * dx);
                acc[2] += (double)(v * v);
                acc[3] += (double)(xn * xn);
                acc[4] += (double)(ln * ln);
            }
        }
    }
    __syncwarp();                                                       // d is reused by the next subsystem
}

template <class T>
__device__ __forceinline__ void batch_item(const BatchProblem& B, const int grp, const int task,
                                           const T* __restrict__ ucur, T* __restrict__ unext, const WarpSmem<T>& W,
                                           const int lane, const bool act, double (&acc)[5]) {
    const int4 tk = __ldg(reinterpret_cast<const int4*>(B.tasks) + 2 * task);
    const size_t gb = (size_t)grp * B.n_rows;                        // first row of this group
    for (int s = tk.x; s < tk.y; ++s) {
        const int4 sm = __ldg(reinterpret_cast<const int4*>(B.subs) + s);   // {row0, ns, op, flags}
        if (sm.y <= kBatchDMax) batch_sub<T, false>(B, sm, gb, ucur, unext, W, lane, act, acc, grp);
        else batch_sub<T, true>(B, sm, gb, ucur, unext, W, lane, act, acc, grp);
    }
}

template <class T>
__global__ void __launch_bounds__(BB, 1) admm_batch_kernel(BatchProblem B) {
    extern __shared__ __align__(16) unsigned char bsm[];
    __shared__ int s_gl[kBatchMaxGrp];                  // active groups of this sweep, ascending
    __shared__ int s_na;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gw = blockIdx.x * BW + wid, nw = gridDim.x * BW;
    WarpSmem<T> W;
    {
        unsigned char* base = bsm + (size_t)wid * warp_smem_bytes<T>();
        W.d = reinterpret_cast<T*>(base);
        unsigned char* meta = base + kBatchDMax * 32 * sizeof(T);
        W.mp = reinterpret_cast<T*>(meta);
        W.mi = reinterpret_cast<int*>(meta + 32 * 4 * sizeof(T));
    }
    const long long total0 = *(volatile long long*)&B.ctrl->total;
    const int NT = B.n_tasks, NG = B.n_grp;
    unsigned long long bars = 0;
    long long it = 0;
    while (it < B.max_iter) {
        const long long t = total0 + it;
        const T* ucur = reinterpret_cast<const T*>((t & 1) ? B.u1 : B.u0);
        T* unext = reinterpret_cast<T*>((t & 1) ? B.u0 : B.u1);
        const uint32_t* gcur = B.gact + (size_t)(it & 1) * NG;
        if (wid == 0) {
            int run = 0;
            for (int g0 = 0; g0 < NG; g0 += 32) {
                const int g = g0 + lane;
                const bool a = g < NG && __ldcg(gcur + g) != 0u;
                const unsigned m = __ballot_sync(kFull, a);
                if (a) s_gl[run + __popc(m & ((1u << lane) - 1u))] = g;
                run += __popc(m);
            }
            if (lane == 0) s_na = run;
        }
        if (blockIdx.x == 0)
            for (int g = threadIdx.x; g < NG; g += blockDim.x) B.gact[(size_t)((it + 1) & 1) * NG + g] = 0u;
        __syncthreads();
        const int NA = s_na;
        if (NA == 0) break;                             // every scenario has stopped (same view in every CTA)
        const long long NI = (long long)NA * NT;
        // dynamic hand-out: item i = (task torder[i / NA], active group i % NA), costliest tasks first; lane 0
        // claims the next item while the warp computes the current one.  The partials land per (group, task),
        // so the result does not depend on which warp ran an item.
        unsigned long long* ictr = B.cnt + 1 + (it & 1);
        long long a = 0;
        if (lane == 0) a = (long long)atomicAdd(ictr, 1ULL);
        a = __shfl_sync(kFull, a, 0);
        while (a < NI) {
            long long nxt = 0;
            if (lane == 0) nxt = (long long)atomicAdd(ictr, 1ULL);
            const long long tq = a / NA;
            const int grp = s_gl[(int)(a - tq * NA)], task = __ldg(B.torder + tq);
            const int sc = grp * 32 + lane;
            const bool act = sc < B.n_scen && __ldcg(B.stopped + sc) == 0;
            double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            batch_item<T>(B, grp, task, ucur, unext, W, lane, act, acc);
            double* pp = B.partial + ((size_t)grp * NT + task) * 5 * 32 + lane;
#pragma unroll
            for (int k = 0; k < 5; ++k) __stcg(pp + k * 32, acc[k]);
            a = __shfl_sync(kFull, nxt, 0);
        }
        grid_sync(B.cnt, (++bars) * gridDim.x);
        if (blockIdx.x == 0 && threadIdx.x == 0) B.cnt[1 + ((it + 1) & 1)] = 0ULL;   // next sweep's counter (seen
                                                                                    // after the second barrier)
        // per-scenario (termination): warp per active group, lane = scenario
        uint32_t* gnext = B.gact + (size_t)((it + 1) & 1) * NG;
        for (int ag = gw; ag < NA; ag += nw) {
            const int grp = s_gl[ag], sc = grp * 32 + lane;
            const bool act = sc < B.n_scen && __ldcg(B.stopped + sc) == 0;
            double s5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            const double* pp = B.partial + (size_t)grp * NT * 160 + lane;
#pragma unroll 8
            for (int k2 = 0; k2 < NT; ++k2)                      // task order: fixed (loads run 8 tasks ahead)
#pragma unroll
                for (int k = 0; k < 5; ++k) s5[k] += __ldcg(pp + (size_t)k2 * 160 + k * 32);
            const double pres = sqrt(s5[0]), dres = B.rho * sqrt(s5[1]);
            const double ep = B.eps_rel * fmax(sqrt(s5[2]), sqrt(s5[3])), ed = B.eps_rel * sqrt(s5[4]);
            const int num = !(isfinite(s5[0]) && isfinite(s5[1]) && isfinite(s5[2]) && isfinite(s5[3]) && isfinite(s5[4]));
            const int conv = B.test && pres <= ep && dres <= ed;
            const bool fin = conv || num || it + 1 == B.max_iter;
            if (act) {
                ScenResult& R = B.res[sc];
                R.iters = it + 1;
                R.total = t + 1;
                R.res[0] = pres; R.res[1] = dres; R.res[2] = ep; R.res[3] = ed;
                R.status = conv ? 1 : num ? 3 : (fin ? 2 : 0);
                if (fin) {
                    double obj = 0.0;
                    const T* xs = reinterpret_cast<const T*>(B.x) + (size_t)grp * B.n * 32 + lane;
                    for (int j = 0; j < B.n_obj; ++j) obj += B.obj_c[j] * (double)__ldcg(xs + (size_t)B.obj_idx[j] * 32);
                    R.objective = obj;
                }
                if (conv || num) B.stopped[sc] = 1;
            }
            if (__any_sync(kFull, act && !(conv || num)) && lane == 0) gnext[grp] = 1u;
        }
        grid_sync(B.cnt, (++bars) * gridDim.x);
        ++it;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        B.ctrl->total = total0 + it;
        B.ctrl->iters = it;
    }
}

// Before each launch: the first sweep's active groups from the stopped flags (scenarios stopped in an
// earlier launch stay frozen); the other parity cleared.
__global__ void batch_gact_kernel(BatchProblem B) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < B.n_grp; g += gridDim.x * blockDim.x) {
        uint32_t any = 0u;
        for (int l = 0; l < 32; ++l) {
            const int sc = g * 32 + l;
            if (sc < B.n_scen && !B.stopped[sc]) any = 1u;
        }
        B.gact[g] = any;
        B.gact[B.n_grp + g] = 0u;
    }
}

// a3 for every scenario: x_s = x0, lambda = 0, u = x0; x = 0; results cleared.
template <class T>
__global__ void reset_batch_kernel(BatchProblem B) {
    const T* x0 = reinterpret_cast<const T*>(B.x0);
    const size_t nr = (size_t)B.n_grp * B.n_rows * 32, nx = (size_t)B.n_grp * B.n * 32;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += stride) {
        const T v = x0[(i >> 5) % B.n_rows];
        reinterpret_cast<T*>(B.xl)[i] = v;
        reinterpret_cast<T*>(B.lam)[i] = T(0);
        reinterpret_cast<T*>(B.u0)[i] = v;
        reinterpret_cast<T*>(B.u1)[i] = T(0);
    }
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nx; i += stride) reinterpret_cast<T*>(B.x)[i] = T(0);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (size_t)B.n_scen; i += stride) {
        ScenResult& R = B.res[i];
        R.iters = 0; R.total = 0; R.status = 0; R.pad = 0; R.objective = 0.0;
        R.res[0] = R.res[1] = R.res[2] = R.res[3] = 0.0;
        B.stopped[i] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        B.ctrl->total = 0;
        B.ctrl->iters = 0;
    }
}

// Scenario scen's x_s, lambda (rows) and x (globals) widened to fp64 into the staging area:
// stage[0 .. n_rows) = x_s, [n_rows .. 2 n_rows) = lambda, [2 n_rows .. 2 n_rows + n) = x.
template <class T>
__global__ void gather_scen_kernel(BatchProblem B, int32_t scen) {
    const int grp = scen >> 5, lane = scen & 31;
    const size_t gb = (size_t)grp * B.n_rows;
    const int stride = gridDim.x * blockDim.x;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < B.n_rows; r += stride) {
        B.stage[r] = (double)reinterpret_cast<const T*>(B.xl)[(gb + r) * 32 + lane];
        B.stage[B.n_rows + r] = (double)reinterpret_cast<const T*>(B.lam)[(gb + r) * 32 + lane];
    }
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < B.n; g += stride)
        B.stage[2 * (size_t)B.n_rows + g] = (double)reinterpret_cast<const T*>(B.x)[((size_t)grp * B.n + g) * 32 + lane];
}

const void* batch_kernel_for(int esz) {
    return esz == 4 ? (const void*)admm_batch_kernel<float> : (const void*)admm_batch_kernel<double>;
}

}  // namespace

int batch_block() { return BB; }

int batch_smem(int ns_max, int esz) {
    (void)ns_max;
    return BW * (esz == 4 ? warp_smem_bytes<float>() : warp_smem_bytes<double>());
}

lopf_status query_batch_grid(int ns_max, int esz, int* grid, std::string& err) {
    int dev = 0, sms = 0, per = 0;
    const void* k = batch_kernel_for(esz);
    const int smem = batch_smem(ns_max, esz);
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, BB, smem);
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    if (per < 1) { err = "batch kernel cannot be resident (occupancy 0)"; return LOPF_E_CUDA; }
    *grid = sms * per;
    return LOPF_OK;
}

lopf_status launch_batch(const BatchProblem& B, int grid, void* stream, std::string& err) {
    cudaStream_t s = (cudaStream_t)stream;
    const void* k = batch_kernel_for(B.esz);
    const int smem = batch_smem(B.ns_max, B.esz);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaMemsetAsync(B.cnt, 0, 3 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) {
        batch_gact_kernel<<<(B.n_grp + 255) / 256, 256, 0, s>>>(B);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && B.max_iter > 0) {
        BatchProblem C = B;
        void* args[] = {&C};
        e = cudaLaunchCooperativeKernel(k, dim3(grid), dim3(BB), args, smem, s);
    }
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_reset_batch(const BatchProblem& B, void* stream, std::string& err) {
    if (B.esz == 4) reset_batch_kernel<float><<<1184, 256, 0, (cudaStream_t)stream>>>(B);
    else reset_batch_kernel<double><<<1184, 256, 0, (cudaStream_t)stream>>>(B);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_gather_scen(const BatchProblem& B, int32_t scen, void* stream, std::string& err) {
    if (B.esz == 4) gather_scen_kernel<float><<<64, 256, 0, (cudaStream_t)stream>>>(B, scen);
    else gather_scen_kernel<double><<<64, 256, 0, (cudaStream_t)stream>>>(B, scen);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

}  // namespace lopf

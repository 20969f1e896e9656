// Batch kernel for sm_100a (config 4): many load scenarios of one feeder, each an
// independent run of Algorithm 1 with its own (termination) test.
//
// Lane = scenario.  Scenarios form groups of 32 and every per-scenario array is [group][entry][32], so a
// warp instruction moves one 256-byte line for 32 scenarios while everything structural -- rows, segment
// lists, bounds, the operators of subsystems without a load -- is the same address for all 32 lanes
// (uniform loads).  A work item is (group, task), a task a depth-first run of subsystems, run by a team of
// kTeamWarps warps (see the kernel below); per item and subsystem s the team computes, for its 32
// scenarios at once,
//   a4  x_g = clamp((sum_{k in seg(g)} u_k - c_g/rho) / nu_g, lo_g, hi_g) for each row (closed_1, rho
//       restored, reading C1), canonical copy order; d = -rho v - lambda staged in team SMEM [row][lane]
//   a5  y = Abar_s d, one row quad at a time (k ascending, FMA); Abar_s from the shared pool (row quads
//       [k][4], one 4-wide uniform load per column) or, for a load subsystem, the scenario's quad-block
//       upper layout ([entry][lane], coalesced, every operand at an immediate offset of one block pointer)
//   a6  x_s = y / rho + bbar_s, lambda += rho (v - x_s), u = x_s - lambda / rho     (closed_2, ADMM-3)
//   a7  five residual sums per lane (scenario), written per item
// The ACTIVE items of a sweep (groups with a scenario still running, times tasks) are handed out one at a
// time from an atomic counter, costliest tasks first, to the teams.  Grid barrier; one warp per active group then sums
// each scenario's item partials in task order (deterministic whichever warp ran an item) and takes its
// decision; converged scenarios freeze (their lanes stop storing), a group leaves the item list when all
// 32 have; grid barrier.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "device.cuh"
#include "internal.h"

namespace lopf {

namespace {

using dev::grid_sync;
using dev::kFull;

#ifndef LOPF_BATCH_TEAMS
#define LOPF_BATCH_TEAMS 6                    // most teams per CTA (fewer when the task rows need more SMEM)
#endif
#ifndef LOPF_BATCH_VPARK
#define LOPF_BATCH_VPARK 1                    // team kernel: 1 parks v in u-next (L2), 0 in team SMEM
#endif
#ifndef LOPF_BATCH_BPF
#define LOPF_BATCH_BPF 15                     // team kernel bulk L2 prefetch at item start, of the current item: 1
#endif                                        // operators, 2 x_s rows, 4 lambda rows, 8 u rows; bits 4-7 the same
                                              // of the next item
#ifndef LOPF_BATCH_JH
#define LOPF_BATCH_JH 4                       // operator columns per load batch of the per-scenario mat-vec (4 or 2)
#endif
constexpr int CR = 4;                         // consensus rows per group (gathers issued together); the team
                                              // splits a task's rows in groups of exactly CR
static_assert(CR == 4, "the team kernel stages and splits rows in four-row groups");
constexpr int JH = LOPF_BATCH_JH;
constexpr int kTeamWarps = kBatchTeamWarps;
constexpr int kTeamMax = LOPF_BATCH_TEAMS;
constexpr int kSmemBudget = 232448 - 2048;    // opt-in dynamic SMEM per block minus the static arrays

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

// ---- per-row / per-quad arithmetic ---------------------------------------------------------------

// Consensus (a4, closed_1 with rho restored, reading C1) of up to CR rows whose records sit at mi + 6 i,
// mp + 4 i (i < cnt) and whose own rows are self0 + i: every gather of the CR rows is issued first, then
// x_g = clamp((sum_k u_k - c/rho) / nu, lo, hi) in ascending canonical copy order; x stored by the first
// copy; put(i, v, d) receives v = x_g and d = -rho v - lambda of row i.
template <class T, class Put>
__device__ __forceinline__ void consensus_group(const BatchProblem& B, const int* mi0, const T* mp0, const int cnt,
                                                const int self0, const T* __restrict__ ug, const T* __restrict__ lmg,
                                                T* __restrict__ xg, const bool act, const unsigned long long pf, Put put) {
    const T rho = (T)B.rho;
    T ua[CR][4], lm[CR];
#pragma unroll
    for (int i = 0; i < CR; ++i) {                                      // every load of CR rows first
        const int rr = min(i, cnt - 1);
        const int* mi = mi0 + rr * 6;
        const int inf = mi[1];
        const bool inl = inf & kBInline;
        const int nu = inl ? (inf >> kBNuShift) & 0xFF : 0;
        const int self = self0 + rr;
        ua[i][0] = __ldcg(ug + 32 * (inl ? mi[2] : self));
        ua[i][1] = nu > 1 ? __ldcg(ug + 32 * mi[3]) : T(0);
        ua[i][2] = nu > 2 ? __ldcg(ug + 32 * mi[4]) : T(0);
        ua[i][3] = nu > 3 ? __ldcg(ug + 32 * mi[5]) : T(0);
        lm[i] = __ldcg(lmg + 32 * self);
    }
#pragma unroll
    for (int i = 0; i < CR; ++i) {
        if (i >= cnt) break;
        const int* mi = mi0 + i * 6;
        const T* mp = mp0 + i * 4;
        const int g = mi[0], inf = mi[1];
        T sig = ((ua[i][0] + ua[i][1]) + ua[i][2]) + ua[i][3];           // ascending canonical copy order
        if (!(inf & kBInline)) {                                        // nu > 4 (rare): the segment list
            sig = T(0);
            for (int q = 0; q < mi[3]; ++q) sig += __ldcg(ug + 32 * __ldg(B.seg_rows + mi[2] + q));
        }
        const T v = fmin(fmax((sig - mp[0]) * mp[3], mp[1]), mp[2]);       // IEEE +-inf = no clamp
        if (act && (inf & kBFirst)) st_first(xg + 32 * g, v, pf);
        put(i, v, -rho * v - lm[i]);
    }
}

// a5 for row quad q of subsystem sm: y_i = sum_k Abar[4q + i][k] d_k, k ascending (zero entries past n_s
// add nothing; dk(k) for k in [n_s, 4 nq) must return a finite value).  V: the group's per-scenario pool
// at the subsystem (lane view), A: the shared pool.
template <class T, class DK>
__device__ __forceinline__ void matvec_quad(const int4 sm, const T* __restrict__ V, const T* __restrict__ A,
                                            const int q, const unsigned long long pf, DK dk, T (&y)[4]) {
    const int ns = sm.y, nq = (ns + 3) >> 2, nsp = nq << 2;
    const bool var = sm.w & kBVar;
#pragma unroll
    for (int i = 0; i < 4; ++i) y[i] = T(0);
    if (var && !batch_vqb((int)sizeof(T))) {
        // packed upper triangle, row-major: (i, j >= i) at i n - i (i - 1) / 2 + j - i; row r reads
        // (min(r, k), max(r, k)): the walk steps by n - k - 1 while k < r, then by 1
        int p[4], rq[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = rq[i] = min(4 * q + i, ns - 1);
#pragma unroll 4
        for (int k = 0; k < ns; ++k) {
            const T dkv = dk(k);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                y[i] = fma(ld_op(V + 32 * p[i], pf), dkv, y[i]);
                p[i] += k < rq[i] ? ns - k - 1 : 1;
            }
        }
    } else if (var) {
        // quad-block upper layout: block q' at Q(q') = sum_{p < q'} 4 (nsp - 4p) entries; for k < 4q the
        // entry (r = 4q + i, k = 4q' + j) is the stored (k, r): block q', column 4q + i, row j.  The 16
        // operands of a 4 x 4 block are loaded JH columns at a time (JH = 4: all at once; 2: fewer registers)
        int Q = 0;
        for (int qp = 0; qp < q; ++qp) {
            const T* __restrict__ Bp = V + 32 * (Q + 16 * (q - qp));
#pragma unroll
            for (int j0 = 0; j0 < 4; j0 += JH) {
                T dj[JH], a[4][JH];
#pragma unroll
                for (int j = 0; j < JH; ++j) dj[j] = dk(4 * qp + j0 + j);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < JH; ++j) a[i][j] = ld_op(Bp + 32 * (4 * i + j0 + j), pf);
#pragma unroll
                for (int j = 0; j < JH; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) y[i] = fma(a[i][j], dj[j], y[i]);
            }
            Q += 4 * (nsp - 4 * qp);
        }
        const T* __restrict__ Bq = V + 32 * Q;                          // block q: column k at 4 (k - 4q)
        for (int k = 4 * q; k < nsp; k += 4, Bq += 32 * 16) {
#pragma unroll
            for (int j0 = 0; j0 < 4; j0 += JH) {
                T dj[JH], a[4][JH];
#pragma unroll
                for (int j = 0; j < JH; ++j) dj[j] = dk(k + j0 + j);
#pragma unroll
                for (int j = 0; j < JH; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[i][j] = ld_op(Bq + 32 * (4 * (j0 + j) + i), pf);
#pragma unroll
                for (int j = 0; j < JH; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) y[i] = fma(a[i][j], dj[j], y[i]);
            }
        }
    } else {
        // row quad q: [k][4] over the padded width, one 4-wide uniform load per column
        const T* __restrict__ Aq = A + q * nsp * 4;
        for (int k = 0; k < nsp; k += 4, Aq += 16) {
            T dj[4], a[4][4];
#pragma unroll
            for (int j = 0; j < 4; ++j) dj[j] = dk(k + j);
#pragma unroll
            for (int j = 0; j < 4; ++j) ld4_uniform(Aq + 4 * j, a[j]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) y[i] = fma(a[j][i], dj[j], y[i]);
        }
    }
}

// a6-a7 for row quad q of subsystem sm (rows past n_s discarded): x_s = y / rho + bbar, lambda += rho (v -
// x_s) (ADMM-3), u = x_s - lambda / rho; five residual sums per lane (terms in T, sums in fp64, F1).  vof(r)
// returns the row's consensus value v (parked in u-next or staged in SMEM).
template <class T, class VOF>
__device__ __forceinline__ void finish_quad(const BatchProblem& B, const int4 sm, const T* __restrict__ V, const int q,
                                            const T (&y)[4], T* __restrict__ ung, T* __restrict__ lmg,
                                            T* __restrict__ xlg, const bool act, const unsigned long long pf, VOF vof,
                                            double (&acc)[5]) {
    const T rho = (T)B.rho, inv_rho = (T)B.inv_rho;
    const int row0 = sm.x, ns = sm.y, r0 = 4 * q;
    int rr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) rr[i] = min(r0 + i, ns - 1);
    T vv[4], lam[4], xo[4], bb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {                                       // the four rows' loads first
        const int at = 32 * (row0 + rr[i]);
        vv[i] = vof(rr[i]);
        lam[i] = ld_last(lmg + at, pf);
        xo[i] = ld_last(xlg + at, pf);
        bb[i] = (sm.w & kBBbar) ? ld_op(V + 32 * (batch_var_entries(ns, batch_vqb((int)sizeof(T))) + rr[i]), pf) : T(0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (r0 + i >= ns) break;
        const int at = 32 * (row0 + r0 + i);
        const T xn = fma(y[i], inv_rho, bb[i]);                         // (1/rho) Abar d + bbar
        const T v = vv[i];
        const T ln = lam[i] + rho * (v - xn);                           // ADMM-3
        const T un = xn - ln * inv_rho;                                 // next consensus input
        if (act) {
            st_first(xlg + at, xn, pf);
            st_first(lmg + at, ln, pf);
            st_first(ung + at, un, pf);
            const T rs = v - xn, dx = xn - xo[i];
            acc[0] += (double)(rs * rs);
            acc[1] += (double)(dx * dx);
            acc[2] += (double)(v * v);
            acc[3] += (double)(xn * xn);
            acc[4] += (double)(ln * ln);
        }
    }
}

// Stage the records of row `row` ({g, info, n0..n3} and {c/rho, lo, hi, 1/nu}) at mi[6], mp[4].
template <class T>
__device__ __forceinline__ void stage_record(const BatchProblem& B, const int row, int* mi, T* mp) {
    using T2 = typename V2<T>::type;
    const int2* __restrict__ rows = reinterpret_cast<const int2*>(B.rows);
    const T2* __restrict__ gpar = reinterpret_cast<const T2*>(B.gpar);
    const int2 a = __ldg(rows + 3 * row), b = __ldg(rows + 3 * row + 1), c = __ldg(rows + 3 * row + 2);
    mi[0] = a.x; mi[1] = a.y; mi[2] = b.x; mi[3] = b.y; mi[4] = c.x; mi[5] = c.y;
    const T2 p0 = __ldg(gpar + 2 * a.x), p1 = __ldg(gpar + 2 * a.x + 1);
    mp[0] = p0.x; mp[1] = p0.y; mp[2] = p1.x; mp[3] = p1.y;
}

// The lane views of group grp: element (row r) at [32 r] (32-bit indices on 64-bit bases).
template <class T>
struct LaneViews {
    const T* ug;
    T *ung, *xlg, *lmg, *xg;
    const T* V;                                        // per-scenario pool of the group
    __device__ __forceinline__ LaneViews(const BatchProblem& B, const T* ucur, T* unext, const int grp, const int lane) {
        const size_t gb = (size_t)grp * B.n_rows;
        ug = ucur + gb * 32 + lane;
        ung = unext + gb * 32 + lane;
        xlg = reinterpret_cast<T*>(B.xl) + gb * 32 + lane;
        lmg = reinterpret_cast<T*>(B.lam) + gb * 32 + lane;
        xg = reinterpret_cast<T*>(B.x) + (size_t)grp * B.n * 32 + lane;
        V = reinterpret_cast<const T*>(B.vpool) + (size_t)grp * B.ve * 32 + lane;
    }
};

// Sweep prologue (every CTA): the active groups of this sweep into s_gl (ascending), their count into
// s_na; CTA 0 clears the next sweep's flags.
__device__ __forceinline__ int batch_active_groups(const BatchProblem& B, const long long it, int* s_gl, int* s_na) {
    const int lane = threadIdx.x & 31, NG = B.n_grp;
    const uint32_t* gcur = B.gact + (size_t)(it & 1) * NG;
    if (threadIdx.x < 32) {
        int run = 0;
        for (int g0 = 0; g0 < NG; g0 += 32) {
            const int g = g0 + lane;
            const bool a = g < NG && __ldcg(gcur + g) != 0u;
            const unsigned m = __ballot_sync(kFull, a);
            if (a) s_gl[run + __popc(m & ((1u << lane) - 1u))] = g;
            run += __popc(m);
        }
        if (lane == 0) *s_na = run;
    }
    if (blockIdx.x == 0)
        for (int g = threadIdx.x; g < NG; g += blockDim.x) B.gact[(size_t)((it + 1) & 1) * NG + g] = 0u;
    __syncthreads();
    return *s_na;
}

// Per-scenario (termination), after the sweep's grid barrier: warp gw (of nw) per active
// group, lane = scenario; the item partials summed in task order (fixed whichever warp ran an item).
template <class T>
__device__ __forceinline__ void batch_decide(const BatchProblem& B, const int* s_gl, const int NA, const long long it,
                                             const long long t, const int gw, const int nw) {
    const int lane = threadIdx.x & 31, NT = B.n_tasks;
    uint32_t* gnext = B.gact + (size_t)((it + 1) & 1) * B.n_grp;
    for (int ag = gw; ag < NA; ag += nw) {
        const int grp = s_gl[ag], sc = grp * 32 + lane;
        const bool act = sc < B.n_scen && __ldcg(B.stopped + sc) == 0;
        double s5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const double* pp = B.partial + (size_t)grp * NT * 160 + lane;
#pragma unroll 8
        for (int k2 = 0; k2 < NT; ++k2)                          // task order: fixed (loads run 8 tasks ahead)
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
}

// ---- the batch kernel -----------------------------------------------------------------------------
// A (group, task) item is run by a TEAM of kTeamWarps warps that share its rows through SMEM: the team
// stages the task's row records, splits the consensus rows (four-row groups round robin over its warps;
// d of every row of the task into team SMEM, v parked in u-next), then splits the mat-vec + finish units (subsystem,
// row quad) as the packer assigned them (longest first onto the least-loaded warp).  An item therefore
// completes ~kTeamWarps times sooner than with one warp per item, and the L2 lines it touches twice
// (lambda, the parked v, the u it gathers) are re-read moments later instead of after ~2 L2 turnovers.
// When the item is claimed one lane issues bulk L2 prefetches of its contiguous per-scenario inputs (the
// task's operators, x_s, lambda and u rows).
// Residual sums: per warp over its units in order, then warp 0 + 1 + ... in order (deterministic whichever
// team ran the item).
constexpr int TW = kTeamWarps;
constexpr int kTeamThreads = 32 * TW;

constexpr bool kVPark = LOPF_BATCH_VPARK;        // v parked in u-next (L2) instead of team SMEM
// named barriers: 1 + team (the team), 1 + kTeamMax + team (the residual hand-over, when ids remain)
constexpr bool kRedArrive = 2 * kTeamMax + 1 <= 16;

// rows per team buffer: the task's rows + 4 zero rows (d past the last row)
__host__ __device__ constexpr int team_rows_alloc(int trmax) { return trmax + 4; }
__host__ __device__ constexpr int team_smem_bytes(int trmax, int esz) {
    // D (and Vv) [TRA][32] T, the residual area [TW - 1][5][32] double, mp [TRA][4] T, mi [TRA][6] int
    return team_rows_alloc(trmax) * ((kVPark ? 1 : 2) * 32 * esz + 4 * esz + 24) + (TW - 1) * 5 * 32 * 8;
}

__device__ __forceinline__ void team_bar(const int team) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(kTeamThreads) : "memory");
}
__device__ __forceinline__ void red_arrive(const int team) {
    if (kRedArrive) asm volatile("bar.arrive %0, %1;" ::"r"(1 + kTeamMax + team), "r"(kTeamThreads) : "memory");
    else team_bar(team);
}
__device__ __forceinline__ void red_wait(const int team) {
    if (kRedArrive) asm volatile("bar.sync %0, %1;" ::"r"(1 + kTeamMax + team), "r"(kTeamThreads) : "memory");
    else team_bar(team);
}
__device__ __forceinline__ void prefetch_bulk_l2(const void* p, const unsigned bytes) {
    if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Bulk L2 prefetch of item (grp, task)'s contiguous per-scenario inputs: `what` bits 1 the task's
// operators, 2 x_s rows, 4 lambda rows, 8 u rows (the gathers' own rows).
template <class T>
__device__ __forceinline__ void team_prefetch(const BatchProblem& B, const T* ucur, const int grp, const int task,
                                              const int what) {
    const int4 tk = __ldg(reinterpret_cast<const int4*>(B.tasks) + 2 * task);
    const int4 tv = __ldg(reinterpret_cast<const int4*>(B.tasks) + 2 * task + 1);
    const size_t gb = (size_t)grp * B.n_rows, rb = (size_t)(tk.w - tk.z) * 32 * sizeof(T);
    if (what & 1)
        prefetch_bulk_l2(reinterpret_cast<const T*>(B.vpool) + ((size_t)grp * B.ve + tv.x) * 32,
                         (unsigned)((size_t)(tv.y - tv.x) * 32 * sizeof(T)));
    if (what & 2) prefetch_bulk_l2(reinterpret_cast<const T*>(B.xl) + (gb + tk.z) * 32, (unsigned)rb);
    if (what & 4) prefetch_bulk_l2(reinterpret_cast<const T*>(B.lam) + (gb + tk.z) * 32, (unsigned)rb);
    if (what & 8) prefetch_bulk_l2(ucur + (gb + tk.z) * 32, (unsigned)rb);
}

template <class T>
__global__ void __launch_bounds__(kTeamThreads * kTeamMax, 1) admm_batch_team_kernel(BatchProblem B) {
    extern __shared__ __align__(16) unsigned char bsm[];
    __shared__ int s_gl[kBatchMaxGrp];                  // active groups of this sweep, ascending
    __shared__ int s_na;
    __shared__ long long s_item[kTeamMax][2];           // a team's current / next item (claim double buffer)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int team = wid / TW, wt = wid - team * TW, tid = wt * 32 + lane;
    const int nwarp = blockDim.x >> 5;
    const int gw = blockIdx.x * nwarp + wid, nw = gridDim.x * nwarp;
    const int TRA = team_rows_alloc(B.trmax);
    T *D, *Vv, *mp;
    int* mi;
    double* red;
    {
        unsigned char* base = bsm + (size_t)team * team_smem_bytes(B.trmax, (int)sizeof(T));
        D = reinterpret_cast<T*>(base);
        Vv = D + (kVPark ? 0 : TRA * 32);
        red = reinterpret_cast<double*>(Vv + TRA * 32);  // [TW - 1][5][32]
        mp = reinterpret_cast<T*>(red + (TW - 1) * 5 * 32);
        mi = reinterpret_cast<int*>(mp + TRA * 4);
    }
    const unsigned long long pf = pol_first();
    const long long total0 = *(volatile long long*)&B.ctrl->total;
    const int NT = B.n_tasks;
    unsigned long long bars = 0;
    long long it = 0;
    while (it < B.max_iter) {
        const long long t = total0 + it;
        const T* ucur = reinterpret_cast<const T*>((t & 1) ? B.u1 : B.u0);
        T* unext = reinterpret_cast<T*>((t & 1) ? B.u0 : B.u1);
        const int NA = batch_active_groups(B, it, s_gl, &s_na);
        if (NA == 0) break;                             // every scenario has stopped (same view in every CTA)
        const long long NI = (long long)NA * NT;
        // dynamic hand-out as in the warp kernel, per team: item i = (task torder[i / NA], active group
        // i % NA), costliest tasks first; the leader claims the next item while the team runs the current one
        unsigned long long* ictr = B.cnt + 1 + (it & 1);
        if (tid == 0) s_item[team][0] = (long long)atomicAdd(ictr, 1ULL);
        team_bar(team);
        long long a = s_item[team][0];
        int par = 0;
        while (a < NI) {
            const long long tq = a / NA;
            const int grp = s_gl[(int)(a - tq * NA)], task = __ldg(B.torder + tq);
            if (tid == 0) {
                const long long nx = (long long)atomicAdd(ictr, 1ULL);
                s_item[team][par ^ 1] = nx;
                team_prefetch<T>(B, ucur, grp, task, LOPF_BATCH_BPF & 15);
                if ((LOPF_BATCH_BPF >> 4) && nx < NI) {
                    const long long nq = nx / NA;
                    team_prefetch<T>(B, ucur, s_gl[(int)(nx - nq * NA)], __ldg(B.torder + nq), LOPF_BATCH_BPF >> 4);
                }
            }
            const int sc = grp * 32 + lane;
            const bool act = sc < B.n_scen && __ldcg(B.stopped + sc) == 0;
            const LaneViews<T> L(B, ucur, unext, grp, lane);
            const int4 tk = __ldg(reinterpret_cast<const int4*>(B.tasks) + 2 * task);   // {sub0, sub1, row0, row1}
            const int R0 = tk.z, nr = tk.w - tk.z;
            // each warp stages the records of its own consensus rows (row r on warp (r / 4) mod TW), so the
            // slots a warp writes are only ever read by that warp: no team barrier before the consensus
            for (int k = lane; ; k += 32) {
                const int r = 4 * (wt + TW * (k >> 2)) + (k & 3);
                if (r >= nr + 3) break;
                if (r < nr) stage_record<T>(B, R0 + r, mi + 6 * r, mp + 4 * r);
            }
            if (wt == 0)
                for (int e = lane; e < 4 * 32; e += 32) D[nr * 32 + e] = T(0);   // d past the last row: 0
            __syncwarp();
            // a4: four-row groups round robin over the team's warps; d (and v) of every row into SMEM
            for (int c = CR * wt; c < nr; c += CR * TW) {
                consensus_group<T>(B, mi + 6 * c, mp + 4 * c, min(CR, nr - c), R0 + c, L.ug, L.lmg, L.xg, act, pf,
                                   [&](const int i, const T v, const T d) {
                                       D[(c + i) * 32 + lane] = d;
                                       if (kVPark) {
                                           if (act) __stcg(L.ung + 32 * (R0 + c + i), v);
                                       } else {
                                           Vv[(c + i) * 32 + lane] = v;
                                       }
                                   });
            }
            team_bar(team);
            // a5-a7: the units (subsystem, row quad) the packer gave this warp (cost-balanced), ascending
            double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            const int u1 = __ldg(B.tunit_ptr + task * TW + wt + 1);
            for (int u = __ldg(B.tunit_ptr + task * TW + wt); u < u1; ++u) {
                const int code = __ldg(B.tunits + u), q = code & 0xFF;
                const int4 sm = __ldg(reinterpret_cast<const int4*>(B.subs) + tk.x + (code >> 8));   // {row0, ns, op, flags}
                const int l0 = sm.x - R0;
                const bool var = sm.w & kBVar;
                const T* __restrict__ V = L.V + (var ? 32 * (size_t)sm.z : 0);
                const T* __restrict__ A = reinterpret_cast<const T*>(B.spool) + (var ? 0 : sm.z);
                const T* Ds = D + l0 * 32 + lane;
                const T* Vs = Vv + l0 * 32 + lane;
                T y[4];
                matvec_quad<T>(sm, V, A, q, pf, [&](const int k) { return Ds[k * 32]; }, y);
                finish_quad<T>(B, sm, V, q, y, L.ung, L.lmg, L.xlg, act, pf,
                               [&](const int r) {
                                   return kVPark ? ld_last(L.ung + 32 * (sm.x + r), pf) : Vs[r * 32];
                               },
                               acc);
            }
            team_bar(team);                              // every unit done: D and Vv are free for the next item
            if (wt > 0) {
#pragma unroll
                for (int k = 0; k < 5; ++k) red[((wt - 1) * 5 + k) * 32 + lane] = acc[k];
                red_arrive(team);
            } else {
                red_wait(team);
                double* pp = B.partial + ((size_t)grp * NT + task) * 5 * 32 + lane;
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    double s = acc[k];
                    for (int w = 1; w < TW; ++w) s += red[((w - 1) * 5 + k) * 32 + lane];
                    __stcg(pp + k * 32, s);
                }
            }
            a = s_item[team][par ^ 1];
            par ^= 1;
        }
        grid_sync(B.cnt, (++bars) * gridDim.x);
        if (blockIdx.x == 0 && threadIdx.x == 0) B.cnt[1 + ((it + 1) & 1)] = 0ULL;   // next sweep's counter (seen
                                                                                    // after the second barrier)
        batch_decide<T>(B, s_gl, NA, it, t, gw, nw);
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
    return esz == 4 ? (const void*)admm_batch_team_kernel<float> : (const void*)admm_batch_team_kernel<double>;
}

}  // namespace

static int batch_teams(int trmax, int esz) {
    const int per = team_smem_bytes(trmax, esz);
    return std::max(1, std::min(kTeamMax, kSmemBudget / per));
}
int batch_block(int trmax, int esz) { return kTeamThreads * batch_teams(trmax, esz); }
int batch_smem(int trmax, int esz) { return batch_teams(trmax, esz) * team_smem_bytes(trmax, esz); }

static cudaError_t set_smem_attrs(const void* k, int smem) {
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

lopf_status query_batch_grid(int trmax, int esz, int* grid, std::string& err) {
    int dev = 0, sms = 0, per = 0;
    const void* k = batch_kernel_for(esz);
    const int smem = batch_smem(trmax, esz);
    if (smem > kSmemBudget) { err = "batch kernel: the largest task needs more shared memory than a CTA has"; return LOPF_E_ARG; }
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = set_smem_attrs(k, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, batch_block(trmax, esz), smem);
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    if (per < 1) { err = "batch kernel cannot be resident (occupancy 0)"; return LOPF_E_CUDA; }
    *grid = sms * per;
    return LOPF_OK;
}

lopf_status launch_batch(const BatchProblem& B, int grid, void* stream, std::string& err) {
    cudaStream_t s = (cudaStream_t)stream;
    const void* k = batch_kernel_for(B.esz);
    const int smem = batch_smem(B.trmax, B.esz);
    cudaError_t e = set_smem_attrs(k, smem);
    if (e == cudaSuccess) e = cudaMemsetAsync(B.cnt, 0, 3 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) {
        batch_gact_kernel<<<(B.n_grp + 255) / 256, 256, 0, s>>>(B);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && B.max_iter > 0) {
        BatchProblem C = B;
        void* args[] = {&C};
        e = cudaLaunchCooperativeKernel(k, dim3(grid), dim3(batch_block(B.trmax, B.esz)), args, smem, s);
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

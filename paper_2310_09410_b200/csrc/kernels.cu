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

#include <algorithm>
#include <cmath>

#include "device.cuh"
#include "internal.h"

namespace lopf {

namespace {

using dev::kFull;
using dev::ld_acquire_u64;
using dev::st_release_u64;
using dev::warp_sum5;

#ifndef LOPF_STREAM_UNROLL
#define LOPF_STREAM_UNROLL 4
#endif
constexpr int kStreamUnroll = LOPF_STREAM_UNROLL;   // packed-task column loop unroll
constexpr int kInvNu = 64;                 // SMEM table of 1 / nu (the host's 1.0 / nu, bit for bit)

// ---- bulk-copy (TMA) staging ---------------------------------------------------------------------
// A packed task's inputs are contiguous byte ranges: its operator block (upper-triangular Abar of
// each subsystem, then b-bar if nonzero) in the pool, and 32*R entries of each per-slot array.  One
// elected lane copies them into one of the warp's two SMEM stages with cp.async.bulk, completing
// on that stage's mbarrier, one task ahead of the compute.
// T = double (the parity path) or float (the paper's GPU precision; reading F1): the
// operator block holds kPackBudget entries of T, then the per-slot inputs of 64 slots.
// Compile-time variants of the sweep (template M): the device-initiated exchange, residual balancing.
constexpr int kModeP2P = 1, kModeAdapt = 2;

template <class T> struct Stg {
    static constexpr int kOffMeta = (int)sizeof(T) * kPackBudget;
    static constexpr int kOffLam = kOffMeta + (int)sizeof(SlotMeta) * 64;
    static constexpr int kOffXl = kOffLam + (int)sizeof(T) * 64;
    static constexpr int kBytes = kOffXl + (int)sizeof(T) * 64;
    static_assert(kOffMeta % 16 == 0 && kBytes % 16 == 0, "bulk copies need 16-byte alignment");
};
template <class T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };
template <class T> using vec2_t = typename Vec2<T>::type;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
}
#ifndef LOPF_STREAM_EVICT
#define LOPF_STREAM_EVICT 1              // L2 evict_first on the staged task inputs (read once per sweep), fp32 only
#endif                                   // (16 x 8500 A/B: fp32 50.7 -> 48.5 us/sweep, fp64 69.8 -> 70.6)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m, bool hint = false) {
    if (hint) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)), "l"(pol) : "memory");
    } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
    }
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 ::"r"(smem_u32(m)), "r"(parity) : "memory");
}

struct Stage {                   // per-warp pipeline: the j-th staged task of this warp uses stage j & 1
    char* buf;                   // [2][kStageBytes]
    uint64_t* bar;               // [2]
    uint32_t issued, consumed;
};

// `full_fence`: the copies read lambda / x_s this warp stored in the same sweep (the next-sweep
// prefetch); otherwise only the stage's SMEM (read by this warp's previous task) needs ordering.
template <class T>
__device__ __forceinline__ void issue_task(const DevProblem& P, Stage& st, const int4 tr, const int lane,
                                           const bool full_fence) {
    constexpr int kStageBytes = Stg<T>::kBytes;
    if (!(tr.w & kTaskPacked)) return;                          // full tasks read HBM directly
    const int b = st.issued & 1;
    ++st.issued;
    if (lane == 0) {
        char* sb = st.buf + b * kStageBytes;
        const uint32_t n = (uint32_t)(tr.w >> kTaskUsedShift) & 0xFFu;
        const bool ablk = !(tr.w & kTaskDirect);
        constexpr uint32_t E = sizeof(T);
        const uint32_t bytes = ((uint32_t)sizeof(SlotMeta) + 2u * E) * n + (ablk ? E * (uint32_t)tr.z : 0u);
        uint64_t* m = st.bar + b;
        if (full_fence) asm volatile("fence.proxy.async;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
        constexpr bool H = LOPF_STREAM_EVICT && sizeof(T) == 4;
        if (ablk) bulk_g2s(sb, reinterpret_cast<const T*>(P.abar) + tr.y, E * (uint32_t)tr.z, m, H);
        bulk_g2s(sb + Stg<T>::kOffMeta, P.s_meta + tr.x, (uint32_t)sizeof(SlotMeta) * n, m, H);
        bulk_g2s(sb + Stg<T>::kOffLam, reinterpret_cast<const T*>(P.lam) + tr.x, E * n, m, H);
        bulk_g2s(sb + Stg<T>::kOffXl, reinterpret_cast<const T*>(P.xl) + tr.x, E * n, m, H);
    }
}

// A {value, tag} exchange entry, written and read as ONE 128-bit access at system scope (single-copy
// atomic): a reader that sees the tag of sweep t also sees that sweep's value -- no fences, no flags.
__device__ __forceinline__ void st_entry_sys(double2* p, const double v, const unsigned long long tag) {
    asm volatile("{\n .reg .b128 x;\n mov.b128 x, {%1, %2};\n st.relaxed.sys.global.b128 [%0], x;\n}"
                 ::"l"(p), "l"(__double_as_longlong(v)), "l"(tag) : "memory");
}
__device__ __forceinline__ double ld_entry_sys(const double2* p, const unsigned long long tag) {
    unsigned long long lo, hi;
    do {
        asm volatile("{\n .reg .b128 x;\n ld.relaxed.sys.global.b128 x, [%2];\n mov.b128 {%0, %1}, x;\n}"
                     : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
    } while (hi != tag);
    return __longlong_as_double(lo);
}

// a4 for one slot: the global's consensus value from the ping-pong copies (closed_1, rho restored)
template <class T, int M>
__device__ __forceinline__ T consensus(const DevProblem& P, const int inf, const int g, const int4 nb,
                                       const T* __restrict__ ucur, const T* __restrict__ inv_nu, const T rho) {
    const vec2_t<T> bd = __ldg(reinterpret_cast<const vec2_t<T>*>(P.gbnd) + g);        // {lo, hi}
    T cr = (inf & kInfoCost) ? __ldg(reinterpret_cast<const T*>(P.gcost) + g) : T(0);   // c / rho
    if constexpr ((M & kModeAdapt) != 0) cr = cr / rho;                // adaptive rho: gcost holds c
    T sigma, inv;
    if (inf & kInfoInline) {                               // nu <= 4: neighbour slots inline
        const int nu = (inf >> kInfoNuShift) & 0xF;
        const T a0 = __ldcg(ucur + nb.x);
        const T a1 = nu > 1 ? __ldcg(ucur + nb.y) : T(0);
        const T a2 = nu > 2 ? __ldcg(ucur + nb.z) : T(0);
        const T a3 = nu > 3 ? __ldcg(ucur + nb.w) : T(0);
        sigma = a0;                                        // ascending canonical copy order
        if (nu > 1) sigma += a1;
        if (nu > 2) sigma += a2;
        if (nu > 3) sigma += a3;
        inv = inv_nu[nu];
    } else {
        const int q0 = __ldg(P.seg_ptr + g), q1 = __ldg(P.seg_ptr + g + 1);
        sigma = T(0);
        for (int q = q0; q < q1; ++q) sigma += __ldcg(ucur + __ldg(P.seg_slot + q));
        inv = q1 - q0 < kInvNu ? inv_nu[q1 - q0] : T(1) / (T)(q1 - q0);
    }
    const T xg = fmin(fmax((sigma - cr) * inv, bd.x), bd.y);            // IEEE +-inf = no clamp
    if (inf & kInfoFirst) reinterpret_cast<T*>(P.x)[g] = xg;
    return xg;
}

// a6 + a7 for one slot.  The five residual terms are formed in T and summed in fp64 (reading F1).
template <class T, int M>
__device__ __forceinline__ void finish_slot(const DevProblem& P, const int inf, const int slot, const T ax, const T bb,
                                            const T v, const T lam, const T xo, T* __restrict__ unext,
                                            double (&acc)[5], const T rho, const T inv_rho, const bool val = true,
                                            const unsigned long long xtag = 0) {
    const T xn = fma(ax, inv_rho, bb);                                 // (1/rho) Abar d + bbar
    const T ln = lam + rho * (v - xn);                                 // ADMM-3
    const T un = xn - ln * inv_rho;                                    // next consensus input
    if (val) {
        __stcs(reinterpret_cast<T*>(P.xl) + slot, xn);
        __stcs(reinterpret_cast<T*>(P.lam) + slot, ln);
        unext[slot] = un;
    }
    if (inf & kInfoExport) {                                           // partitioned: to the other ranks
        const int e = __ldg(P.s_exp + slot);
        if constexpr ((M & kModeP2P) != 0) {                           // device-initiated: a tagged entry into
            const size_t xo = unext == reinterpret_cast<T*>(P.u0) ? (size_t)P.xstride : 0;   // every rank's buffer
            for (int q = 0; q < P.world; ++q)                          // of this sweep's parity (t & 1)
                st_entry_sys(P.peer_xe[q] + xo + e, (double)un, xtag);
        } else {
            __stcg(P.xbuf + e, (double)un);
        }
    }
    const T rr = v - xn, dx = xn - xo;
    acc[0] += (double)(rr * rr);
    acc[1] += (double)(dx * dx);
    acc[2] += (double)(v * v);
    acc[3] += (double)(xn * xn);
    acc[4] += (double)(ln * ln);
}

// Packed task (R <= 2 halves): inputs from the SMEM stage; operator block from the stage or, for a
// lone large subsystem (kTaskDirect), straight from the pool.
// SRC: where the operator block is read -- 1 the pool (direct task), 2 the SMEM stage (shared-space
// loads), 0 decided per task at run time (one code path: the batch kernel, whose registers are tighter)
template <int R, class T, int SRC, int M>
__device__ __forceinline__ void task_packed(const DevProblem& P, const int4 tr, const T* __restrict__ ucur,
                                            T* __restrict__ unext, double (&acc)[5], const int lane,
                                            T* __restrict__ dsm, Stage& st, const T* __restrict__ inv_nu,
                                            const T rho, const T inv_rho, const unsigned long long xtag) {
    constexpr int kStageBytes = Stg<T>::kBytes;
    const int b = st.consumed & 1;
    mbar_wait(st.bar + b, (st.consumed >> 1) & 1);
    ++st.consumed;
    const char* sb = st.buf + b * kStageBytes;
    const SlotMeta* s_meta = reinterpret_cast<const SlotMeta*>(sb + Stg<T>::kOffMeta);
    const T* s_lam = reinterpret_cast<const T*>(sb + Stg<T>::kOffLam);
    const T* s_xl = reinterpret_cast<const T*>(sb + Stg<T>::kOffXl);
    const bool direct = SRC == 1 || (SRC == 0 && (tr.w & kTaskDirect));
    const T* S = direct ? reinterpret_cast<const T*>(P.abar) + tr.y : reinterpret_cast<const T*>(sb);
    const int used = (tr.w >> kTaskUsedShift) & 0xFF;       // stage entries past `used` are stale
    T v[R], ax[R];
    int info[R];
    // a4, split so that every gather of both halves is in flight before the first is consumed
    T ua[R][4], lo[R], hi[R], cr[R];
    int g[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        const int j = h * 32 + lane;
        info[h] = j < used ? s_meta[j].info : 0;
        const bool val = info[h] & kInfoValid, inl = val && (info[h] & kInfoInline);
        const int nu = (info[h] >> kInfoNuShift) & 0xF;
        g[h] = s_meta[j].g;
        const int2 n01 = s_meta[j].n01, n23 = s_meta[j].n23;
        const int4 nb = make_int4(n01.x, n01.y, n23.x, n23.y);
        ua[h][0] = inl ? __ldcg(ucur + nb.x) : T(0);
        ua[h][1] = inl && nu > 1 ? __ldcg(ucur + nb.y) : T(0);
        ua[h][2] = inl && nu > 2 ? __ldcg(ucur + nb.z) : T(0);
        ua[h][3] = inl && nu > 3 ? __ldcg(ucur + nb.w) : T(0);
        vec2_t<T> bd;
        bd.x = T(0), bd.y = T(0);
        if (val) bd = __ldg(reinterpret_cast<const vec2_t<T>*>(P.gbnd) + g[h]);
        lo[h] = bd.x;
        hi[h] = bd.y;
        cr[h] = val && (info[h] & kInfoCost) ? __ldg(reinterpret_cast<const T*>(P.gcost) + g[h]) : T(0);
        if constexpr ((M & kModeAdapt) != 0) cr[h] = cr[h] / rho;   // adaptive rho: gcost holds c
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {      // branch-free for the inline case (absent entries are exact zeros)
        const int j = h * 32 + lane;
        const bool val = info[h] & kInfoValid;
        const int nu = (info[h] >> kInfoNuShift) & 0xF;
        T sigma = ((ua[h][0] + ua[h][1]) + ua[h][2]) + ua[h][3];      // ascending canonical copy order
        T inv = inv_nu[nu];
        if (val && !(info[h] & kInfoInline)) {                         // nu > 4: the CSR segment
            const int q0 = __ldg(P.seg_ptr + g[h]), q1 = __ldg(P.seg_ptr + g[h] + 1);
            sigma = T(0);
            for (int q = q0; q < q1; ++q) sigma += __ldcg(ucur + __ldg(P.seg_slot + q));
            inv = q1 - q0 < kInvNu ? inv_nu[q1 - q0] : T(1) / (T)(q1 - q0);
        }
        v[h] = fmin(fmax((sigma - cr[h]) * inv, lo[h]), hi[h]);       // closed_1; IEEE +-inf = no clamp
        if (val && (info[h] & kInfoFirst)) reinterpret_cast<T*>(P.x)[g[h]] = v[h];
        dsm[j] = val ? -rho * v[h] - s_lam[j] : T(0);
        ax[h] = T(0);
    }
    __syncwarp();
    // Row r of subsystem s: sum_k Abar[r][k] d[k], k ascending, from the upper-triangular block
    // (row-major, (i, j >= i) at i*n - i(i-1)/2 + j - i): entry (min(r,k), max(r,k)); the walk p(k)
    // steps by n - k - 1 while k < r (down column r) and by 1 after (along row r).
    int ns[R], r[R], p[R], base[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        base[h] = info[h] & kInfoBaseMask;
        ns[h] = (info[h] & kInfoValid) ? (info[h] >> kInfoNsShift) & 0x3F : 0;
        r[h] = h * 32 + lane - base[h];
        p[h] = ((unsigned)info[h] >> kInfoPoffShift) + r[h];
    }
    const int kmax = (tr.w >> kTaskKmaxShift) & 0xFF;
#pragma unroll kStreamUnroll
    for (int k = 0; k < kmax; ++k) {
#pragma unroll
        for (int h = 0; h < R; ++h) {
            if (k < ns[h]) {
                ax[h] = fma(S[p[h]], dsm[base[h] + k], ax[h]);
                p[h] += k < r[h] ? ns[h] - k - 1 : 1;
            }
        }
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {      // an empty slot has ax = b-bar = v = lambda = 0: exact zeros, no stores
        const int j = h * 32 + lane;
        const bool val = info[h] & kInfoValid;
        // b-bar follows the subsystem's triangle in the block when nonzero
        const T bb = (info[h] & kInfoBbar)
                         ? S[((unsigned)info[h] >> kInfoPoffShift) + ns[h] * (ns[h] + 1) / 2 + r[h]] : T(0);
        finish_slot<T, M>(P, info[h], tr.x + j, ax[h], bb, v[h], val ? s_lam[j] : T(0), val ? s_xl[j] : T(0), unext,
                       acc, rho, inv_rho, val, xtag);
    }
    __syncwarp();
}

// Full task (one subsystem of n_s > 63, R = 2, 4 or 8): Abar as kmax columns of 32*R entries and the
// per-slot inputs read straight from HBM.
template <int R, class T, int M>
__device__ __forceinline__ void task_full(const DevProblem& P, const int4 tr, const T* __restrict__ ucur,
                                          T* __restrict__ unext, double (&acc)[5], const int lane,
                                          T* __restrict__ dsm, const T* __restrict__ inv_nu, const T rho,
                                          const T inv_rho, const unsigned long long xtag) {
    const T* lamp = reinterpret_cast<const T*>(P.lam);
    T v[R], ax[R];
    int info[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        const int slot = tr.x + h * 32 + lane;
        info[h] = __ldg(&P.s_meta[slot].info);
        v[h] = T(0);
        T d = T(0);
        if (info[h] & kInfoValid) {
            const int2 n01 = __ldg(&P.s_meta[slot].n01), n23 = __ldg(&P.s_meta[slot].n23);
            v[h] = consensus<T, M>(P, info[h], __ldg(&P.s_meta[slot].g), make_int4(n01.x, n01.y, n23.x, n23.y), ucur,
                                inv_nu, rho);
            d = -rho * v[h] - lamp[slot];
        }
        dsm[h * 32 + lane] = d;
        ax[h] = T(0);
    }
    __syncwarp();
    const T* __restrict__ A = reinterpret_cast<const T*>(P.abar) + tr.y;
    for (int k = 0; k < tr.z; ++k) {
        const T dk = dsm[k];                                   // one subsystem per full task: base 0
#pragma unroll
        for (int h = 0; h < R; ++h) ax[h] = fma(__ldcs(A + (size_t)k * (32 * R) + h * 32 + lane), dk, ax[h]);
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {
        if (!(info[h] & kInfoValid)) continue;
        const int slot = tr.x + h * 32 + lane;
        const T bb = (info[h] & kInfoBbar) ? __ldg(reinterpret_cast<const T*>(P.s_bbar) + slot) : T(0);
        finish_slot<T, M>(P, info[h], slot, ax[h], bb, v[h], lamp[slot], reinterpret_cast<const T*>(P.xl)[slot], unext, acc,
                       rho, inv_rho, true, xtag);
    }
    __syncwarp();
}

template <int RMAX, class T>
struct StreamWarps {
    static constexpr int value = RMAX > 2 ? kStreamWarpsWide : sizeof(T) == 8 ? kStreamWarpsF64 : kStreamWarpsF32;
};

// The persistent sweep loop of the streaming kernel for CTA `cta` of `ncta` (one rank's grid).  P2P: the
// partitioned mode with a device-initiated exchange: boundary copies' u go
// straight into every rank's entry buffer as tagged 128-bit entries (peer memory over NVLink, or local
// memory when the ranks are emulated on one GPU); the last CTA of each rank publishes the rank's residual
// sums the same way, reads every rank's sums and its own ghosts when their tags say "this sweep", and
// takes the (termination) decision on the rank-ordered sums -- one launch per solve, no host, no NCCL.
template <int RMAX, class T, int M>
__device__ __forceinline__ void stream_body(const DevProblem& P, const int cta, const int ncta) {
    constexpr bool P2P = (M & kModeP2P) != 0, ADAPT = (M & kModeAdapt) != 0;
    constexpr int kWarps = StreamWarps<RMAX, T>::value;
    constexpr int kStageBytes = Stg<T>::kBytes;
    extern __shared__ __align__(128) char sdyn[];      // [kWarps][2][kStageBytes] stages, [kWarps][32*RMAX] d
    __shared__ double red[kWarps][5];
    __shared__ uint64_t sbar[kWarps][2];
    __shared__ T inv_nu[kInvNu];
    __shared__ int s_stop, s_chg;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gw = cta * kWarps + wid, nw = ncta * kWarps;
    Stage st{sdyn + (size_t)wid * 2 * kStageBytes, sbar[wid], 0u, 0u};
    T* dsm = reinterpret_cast<T*>(sdyn + (size_t)kWarps * 2 * kStageBytes) + (size_t)wid * 32 * RMAX;
    for (int i = threadIdx.x; i < kInvNu; i += blockDim.x) inv_nu[i] = i > 0 ? T(1) / (T)i : T(0);
    if (lane == 0) {
        mbar_init(st.bar);
        mbar_init(st.bar + 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (!P2P && P.part && *(volatile long long*)&P.ctrl->stopped) return;   // partitioned: decided, no more sweeps
    const long long total0 = *(volatile long long*)&P.ctrl->total;
    const int4 tr0 = gw < P.n_tasks ? __ldg(P.tasks + gw) : make_int4(0, 0, 0, 0);
    // the penalty in force: fixed (kernel parameters: no loop-carried registers under the 128-register
    // cap), or (residual balancing, F2) the device copy in the control block
    double rho_d = ADAPT ? *(volatile double*)&P.ctrl->rho_cur : P.rho;
    T rho = (T)rho_d, inv_rho = ADAPT ? (T)(1.0 / rho_d) : (T)P.inv_rho;
    unsigned long long bars2 = 0;
    long long it = 0;
    if (P.max_iter > 0) issue_task<T>(P, st, tr0, lane, false);
    while (it < P.max_iter) {
        const long long t = total0 + it;
        const T* ucur = reinterpret_cast<const T*>((t & 1) ? P.u1 : P.u0);
        T* unext = reinterpret_cast<T*>((t & 1) ? P.u0 : P.u1);
        double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const unsigned long long xtag = (unsigned long long)(t + 1);     // p2p exchange tag of this sweep
        int4 tr = tr0;
        int4 tr1 = gw + nw < P.n_tasks ? __ldg(P.tasks + gw + nw) : make_int4(0, 0, 0, 0);
        for (int task = gw; task < P.n_tasks; task += nw) {
            const int4 tr2 = task + 2 * nw < P.n_tasks ? __ldg(P.tasks + task + 2 * nw) : make_int4(0, 0, 0, 0);
            if (task + nw < P.n_tasks) issue_task<T>(P, st, tr1, lane, false);   // one task ahead
            if (tr.w & kTaskPacked) {
                const bool dir = tr.w & kTaskDirect;
                if ((tr.w & 0xF) == 1) {
                    if (dir) task_packed<1, T, 1, M>(P, tr, ucur, unext, acc, lane, dsm, st, inv_nu, rho, inv_rho, xtag);
                    else task_packed<1, T, 2, M>(P, tr, ucur, unext, acc, lane, dsm, st, inv_nu, rho, inv_rho, xtag);
                } else if constexpr (RMAX >= 2) {
                    if (dir) task_packed<2, T, 1, M>(P, tr, ucur, unext, acc, lane, dsm, st, inv_nu, rho, inv_rho, xtag);
                    else task_packed<2, T, 2, M>(P, tr, ucur, unext, acc, lane, dsm, st, inv_nu, rho, inv_rho, xtag);
                }
            } else {
                switch (tr.w & 0xF) {
                    case 2: if constexpr (RMAX >= 2) task_full<2, T, M>(P, tr, ucur, unext, acc, lane, dsm, inv_nu, rho, inv_rho, xtag); break;
                    case 4: if constexpr (RMAX >= 4) task_full<4, T, M>(P, tr, ucur, unext, acc, lane, dsm, inv_nu, rho, inv_rho, xtag); break;
                    default: if constexpr (RMAX >= 8) task_full<8, T, M>(P, tr, ucur, unext, acc, lane, dsm, inv_nu, rho, inv_rho, xtag); break;
                }
            }
            tr = tr1;
            tr1 = tr2;
        }
        // this warp's first task of the next sweep, staged across the grid barrier: its operators are
        // constant and its lambda / x_s were written by this warp only (all lanes, before __syncwarp)
        if (it + 1 < P.max_iter && gw < P.n_tasks) issue_task<T>(P, st, tr0, lane, true);
        {
            const double ws = warp_sum5(acc, lane);
            if ((lane & 3) == 0 && (lane >> 2) < 5) red[wid][lane >> 2] = ws;
        }
        __syncthreads();
        ++it;
        if (wid == 0) {
            int last = 0;
            if (lane == 0) {
                double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                for (int w = 0; w < kWarps; ++w)
                    for (int k = 0; k < 5; ++k) s[k] += red[w][k];
                double* part = P.partial + (size_t)cta * 8;
                for (int k = 0; k < 5; ++k) part[k] = s[k];
                __threadfence();
                const unsigned long long old = atomicAdd(&P.ctrl->arrive, 1ULL);
                last = (old + 1 == (unsigned long long)it * ncta);
            }
            last = __shfl_sync(kFull, last, 0);
            if (last) {                                        // reduce partials in block order
                __threadfence();
                double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                for (int b = lane; b < ncta; b += 32)
                    for (int k = 0; k < 5; ++k) s[k] += __ldcg(P.partial + (size_t)b * 8 + k);
#pragma unroll
                for (int k = 0; k < 5; ++k) {
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) s[k] += __shfl_xor_sync(kFull, s[k], off);
                }
                if (P2P && P.world > 1) {
                    // this rank's five sums as tagged entries into every rank's buffer; then every rank's sums
                    // and this rank's ghosts, each read when its tag says "sweep t" -- the rank-ordered sums
                    // are then identical everywhere.  No flags, no fences: each entry is one 128-bit access.
                    const size_t xo = (size_t)(t & 1) * P.xstride;
                    if (lane < 5)
                        for (int q = 0; q < P.world; ++q)
                            st_entry_sys(P.peer_xe[q] + xo + P.n_bnd + (size_t)P.rank * 8 + lane, s[lane], xtag);
                    const double2* xe = P.xent + xo;                 // this rank's buffer
                    for (int i = lane; i < P.n_imp; i += 32) unext[P.ghost0 + i] = (T)ld_entry_sys(xe + __ldg(P.imp + i), xtag);
                    for (int k = 0; k < 5; ++k) s[k] = 0.0;
                    for (int r = 0; r < P.world; ++r)
                        for (int k = 0; k < 5; ++k) s[k] += ld_entry_sys(xe + P.n_bnd + (size_t)r * 8 + k, xtag);
                    __syncwarp();
                    __threadfence();                                 // ghosts before the local release below
                }
                if (lane == 0 && P.part && !P2P) {             // partitioned: this rank's sums go to the exchange;
                    double* rs = P.xbuf + P.n_bnd + (size_t)P.rank * 8;   // the import kernel decides
                    for (int k = 0; k < 5; ++k) rs[k] = s[k];
                    __threadfence();
                    st_release_u64(&P.ctrl->flag, ((unsigned long long)it << 3));
                    s_stop = 0;
                    s_chg = 0;
                } else if (lane == 0) {
                    const double pres = sqrt(s[0]), dres = rho_d * sqrt(s[1]);
                    const double ep = P.eps_rel * fmax(sqrt(s[2]), sqrt(s[3])), ed = P.eps_rel * sqrt(s[4]);
                    const int numeric = !(isfinite(s[0]) && isfinite(s[1]) && isfinite(s[2]) && isfinite(s[3]) && isfinite(s[4]));
                    const int conv = P.test && (pres <= ep) && (dres <= ed);
                    const int stop = conv || numeric;
                    DevCtrl* c = P.ctrl;
                    int chg = 0;                               // residual balancing (F2): rho of the next sweep
                    if (ADAPT && !stop && ((total0 + it) % P.adapt_every) == 0) {
                        double rn = rho_d;
                        if (pres > P.adapt_mu * dres) rn = P.adapt_tau * rho_d;
                        else if (dres > P.adapt_mu * pres) rn = rho_d / P.adapt_tau;
                        if (rn != rho_d) {
                            c->rho_cur = rn;
                            c->rho_changes = c->rho_changes + 1;
                            chg = 1;
                        }
                    }
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
                        const T* xg = reinterpret_cast<const T*>(P.x);
                        for (int j = 0; j < P.n_obj; ++j) obj += P.obj_c[j] * (double)__ldcg(xg + P.obj_idx[j]);
                        c->res[0] = pres; c->res[1] = dres; c->res[2] = ep; c->res[3] = ed;
                        c->objective = obj;
                        c->iters = it;
                        c->total = total0 + it;
                        c->outcome = conv ? LOPF_CONVERGED : LOPF_MAX_ITER;
                        c->numeric = numeric;
                    }
                    __threadfence();
                    st_release_u64(&c->flag, ((unsigned long long)it << 3) | ((unsigned long long)chg << 2) |
                                                 ((unsigned long long)stop << 1) | (unsigned long long)numeric);
                    s_stop = stop;
                    s_chg = chg;
                }
            } else if (lane == 0) {
                unsigned long long f;
                while (((f = ld_acquire_u64(&P.ctrl->flag)) >> 3) < (unsigned long long)it) __nanosleep(32);
                s_stop = (int)((f >> 1) & 1);
                s_chg = (int)((f >> 2) & 1);
                __threadfence();
            }
        }
        __syncthreads();
        if (s_stop) break;
        if (ADAPT && s_chg) {   // rho changed: every u of the next sweep's buffer re-formed with it, then a barrier
            rho_d = *(volatile double*)&P.ctrl->rho_cur;
            rho = (T)rho_d;
            inv_rho = (T)(1.0 / rho_d);
            const T* xlp = reinterpret_cast<const T*>(P.xl);
            const T* lmp = reinterpret_cast<const T*>(P.lam);
            for (int i = cta * blockDim.x + threadIdx.x; i < P.n_slots; i += ncta * blockDim.x)
                unext[i] = __ldcg(xlp + i) - __ldcg(lmp + i) * inv_rho;
            dev::grid_sync(&P.ctrl->arrive2, (++bars2) * ncta);
        }
    }
    while (st.consumed < st.issued) {                          // drain the prefetch of a sweep not run
        mbar_wait(st.bar + (st.consumed & 1), (st.consumed >> 1) & 1);
        ++st.consumed;
    }
}

// RMAX: largest task width in the problem (RMAX > 2 only with n_s > 64: the S = 1 path); ADAPT: residual balancing
template <int RMAX, class T, bool ADAPT>
__global__ void __launch_bounds__(32 * StreamWarps<RMAX, T>::value, 1) admm_stream_kernel(DevProblem P) {
    stream_body<RMAX, T, ADAPT ? kModeAdapt : 0>(P, blockIdx.x, gridDim.x);
}

// Partitioned mode with the device-initiated exchange, one rank per GPU (one launch per rank).
template <int RMAX, class T>
__global__ void __launch_bounds__(32 * StreamWarps<RMAX, T>::value, 1) admm_p2p_kernel(DevProblem P) {
    stream_body<RMAX, T, kModeP2P>(P, blockIdx.x, gridDim.x);
}

// ... every rank of an emulation on one GPU in one cooperative launch: CTA b runs rank (b / gsize)'s share
// from a shared-memory copy of that rank's argument.
template <int RMAX, class T>
__global__ void __launch_bounds__(32 * StreamWarps<RMAX, T>::value, 1) admm_p2p_emu_kernel(const DevProblem* parr, int gsize) {
    __shared__ __align__(16) DevProblem sP;
    {
        const int* src = reinterpret_cast<const int*>(parr + blockIdx.x / gsize);
        int* dst = reinterpret_cast<int*>(&sP);
        for (int i = threadIdx.x; i < (int)(sizeof(DevProblem) / 4); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    stream_body<RMAX, T, kModeP2P>(sP, blockIdx.x % gsize, gsize);
}

// Partitioned mode, after the exchange-buffer allreduce of sweep t: the other ranks' boundary u into
// this rank's ghost slots of the buffer sweep t+1 reads.  One CTA per 256 ghosts.  It only READS the
// control block (sweep count, stop flag); the decision that changes them is a separate one-thread launch
// after it (part_decide_kernel), so no block of a large import can see a half-updated control block.
template <class T>
__global__ void part_import_kernel(DevProblem P) {
    const DevCtrl* c = P.ctrl;
    if (*(volatile const long long*)&c->stopped) return;
    const long long t = *(volatile const long long*)&c->total;
    T* dst = reinterpret_cast<T*>((t & 1) ? P.u0 : P.u1);               // = unext of sweep t
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n_imp; i += gridDim.x * blockDim.x)
        dst[P.ghost0 + i] = (T)__ldcg(P.xbuf + P.imp[i]);
}

// ... then the termination test of sweep t on the residual sums added in rank order (identical on every
// rank) and the sweep count / stop flag of the next sweep.
template <class T>
__global__ void part_decide_kernel(DevProblem P) {
    DevCtrl* c = P.ctrl;
    if (*(volatile long long*)&c->stopped) return;
    const long long t = *(volatile long long*)&c->total;
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int r = 0; r < P.world; ++r)
        for (int k = 0; k < 5; ++k) s[k] += __ldcg(P.xbuf + P.n_bnd + (size_t)r * 8 + k);
    const double pres = sqrt(s[0]), dres = P.rho * sqrt(s[1]);
    const double ep = P.eps_rel * fmax(sqrt(s[2]), sqrt(s[3])), ed = P.eps_rel * sqrt(s[4]);
    const int numeric = !(isfinite(s[0]) && isfinite(s[1]) && isfinite(s[2]) && isfinite(s[3]) && isfinite(s[4]));
    const int conv = P.test && (pres <= ep) && (dres <= ed);
    double obj = 0.0;                                              // this rank's share of c^T x
    const T* xg = reinterpret_cast<const T*>(P.x);
    for (int j = 0; j < P.n_obj; ++j) obj += P.obj_c[j] * (double)__ldcg(xg + P.obj_idx[j]);
    c->res[0] = pres; c->res[1] = dres; c->res[2] = ep; c->res[3] = ed;
    c->objective = obj;
    c->iters = c->iters + 1;
    c->total = t + 1;
    c->outcome = conv ? LOPF_CONVERGED : LOPF_MAX_ITER;
    c->numeric = numeric;
    if (conv || numeric) c->stopped = 1;
}

// a3: reset the iterate to the initial point: x_s = x0, lambda = 0, u = x0.
template <class T>
__global__ void reset_kernel(DevProblem P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P.n_slots) {
        const T x0 = reinterpret_cast<const T*>(P.x0)[i];
        reinterpret_cast<T*>(P.xl)[i] = x0;
        reinterpret_cast<T*>(P.lam)[i] = T(0);
        reinterpret_cast<T*>(P.u0)[i] = x0;
        reinterpret_cast<T*>(P.u1)[i] = T(0);
    }
    if (i == 0) {
        P.ctrl->arrive = 0; P.ctrl->flag = 0; P.ctrl->total = 0; P.ctrl->iters = 0; P.ctrl->trace_rows = 0;
        P.ctrl->stopped = 0;
        P.ctrl->rho_cur = P.rho;
        P.ctrl->rho_changes = 0;
    }
}

// lopf_fetch_async: the result record (lopf_result layout, solve_ms = 0) and x widened to fp64 into the
// staging area: stage[0 .. 8) = the record (64 bytes), stage[8 .. 8 + n) = x.
template <class T>
__global__ void fetch_kernel(const DevCtrl* c, const T* x, int64_t n, double* stage) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        lopf_result r;
        r.outcome = c->outcome;
        r.reserved0 = c->numeric;
        r.iters = c->iters;
        r.pres = c->res[0]; r.dres = c->res[1]; r.eps_prim = c->res[2]; r.eps_dual = c->res[3];
        r.objective = c->objective;
        r.solve_ms = 0.0;
        *reinterpret_cast<lopf_result*>(stage) = r;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        stage[8 + i] = (double)__ldcg(x + i);
}

}  // namespace

lopf_status launch_fetch(const DevCtrl* ctrl, const void* x, int64_t n, int esz, void* stage, void* stream, std::string& err) {
    const int nb = (int)std::min<int64_t>(148, (n + 255) / 256 + 1);
    if (esz == 4) fetch_kernel<float><<<nb, 256, 0, (cudaStream_t)stream>>>(ctrl, (const float*)x, n, (double*)stage);
    else fetch_kernel<double><<<nb, 256, 0, (cudaStream_t)stream>>>(ctrl, (const double*)x, n, (double*)stage);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

template <class T, bool ADAPT>
static const void* stream_kernel_t(int rmax) {
    return rmax <= 1 ? (const void*)admm_stream_kernel<1, T, ADAPT>
         : rmax <= 2 ? (const void*)admm_stream_kernel<2, T, ADAPT>
         : rmax <= 4 ? (const void*)admm_stream_kernel<4, T, ADAPT>
                     : (const void*)admm_stream_kernel<8, T, ADAPT>;
}
static const void* stream_kernel_for(int rmax, int esz, bool adapt) {
    if (adapt) return esz == 4 ? stream_kernel_t<float, true>(rmax) : stream_kernel_t<double, true>(rmax);
    return esz == 4 ? stream_kernel_t<float, false>(rmax) : stream_kernel_t<double, false>(rmax);
}

static int stream_smem(int rmax, int esz) {
    const int r = rmax <= 1 ? 1 : rmax <= 2 ? 2 : rmax <= 4 ? 4 : 8;
    const int stage = esz == 4 ? Stg<float>::kBytes : Stg<double>::kBytes;
    return stream_block(rmax, esz) / 32 * (2 * stage + esz * 32 * r);
}

int stream_block(int rmax, int esz) {
    return 32 * (rmax > 2 ? kStreamWarpsWide : esz == 8 ? kStreamWarpsF64 : kStreamWarpsF32);
}

lopf_status query_grid(int rmax, int esz, int* grid, std::string& err) {
    int dev = 0, sms = 0, per = 0;
    const void* k = stream_kernel_for(rmax, esz, false);
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, stream_smem(rmax, esz));
    if (e == cudaSuccess)          // the residual-balancing variant launches with the same block and SMEM
        e = cudaFuncSetAttribute(stream_kernel_for(rmax, esz, true), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 stream_smem(rmax, esz));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, stream_block(rmax, esz), stream_smem(rmax, esz));
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    if (per < 1) { err = "streaming kernel cannot be resident (occupancy 0)"; return LOPF_E_CUDA; }
    *grid = sms * per;
    return LOPF_OK;
}

lopf_status launch_solve(const DevProblem& P, int grid, void* stream, std::string& err) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(P.ctrl, 0, 2 * sizeof(unsigned long long), s);   // arrive, flag
    if (e == cudaSuccess) e = cudaMemsetAsync(&P.ctrl->arrive2, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(&P.ctrl->trace_rows, 0, sizeof(long long), s);
    if (e == cudaSuccess && P.max_iter > 0) {
        DevProblem Q = P;
        void* args[] = {&Q};
        e = cudaLaunchCooperativeKernel(stream_kernel_for(P.rmax, P.esz, P.adapt_every > 0), dim3(grid), dim3(stream_block(P.rmax, P.esz)), args,
                                        stream_smem(P.rmax, P.esz), s);
    }
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}


template <class T>
static const void* p2p_kernel_t(int rmax, bool emu) {
    if (emu)
        return rmax <= 1 ? (const void*)admm_p2p_emu_kernel<1, T>
             : rmax <= 2 ? (const void*)admm_p2p_emu_kernel<2, T>
             : rmax <= 4 ? (const void*)admm_p2p_emu_kernel<4, T>
                         : (const void*)admm_p2p_emu_kernel<8, T>;
    return rmax <= 1 ? (const void*)admm_p2p_kernel<1, T>
         : rmax <= 2 ? (const void*)admm_p2p_kernel<2, T>
         : rmax <= 4 ? (const void*)admm_p2p_kernel<4, T>
                     : (const void*)admm_p2p_kernel<8, T>;
}

// CTAs per rank of a p2p launch with `world_here` ranks on this GPU: every CTA of the launch co-resident
int p2p_max_group(int rmax, int esz, int world_here) {
    int dev = 0, sms = 0, per = 0;
    const void* k = esz == 4 ? p2p_kernel_t<float>(rmax, world_here > 1) : p2p_kernel_t<double>(rmax, world_here > 1);
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, stream_smem(rmax, esz)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, stream_block(rmax, esz), stream_smem(rmax, esz)) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return sms * per / world_here;
}

lopf_status launch_p2p(const DevProblem* parr_dev, const DevProblem* one, int world_here, int gsize, int rmax, int esz,
                       void* stream, std::string& err) {
    const bool emu = world_here > 1;
    const void* k = esz == 4 ? p2p_kernel_t<float>(rmax, emu) : p2p_kernel_t<double>(rmax, emu);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, stream_smem(rmax, esz));
    if (e == cudaSuccess) {
        const DevProblem* a0 = parr_dev;
        int g = gsize;
        DevProblem P = one ? *one : DevProblem{};
        void* args_emu[] = {&a0, &g};
        void* args_one[] = {&P};
        e = cudaLaunchCooperativeKernel(k, dim3(world_here * gsize), dim3(stream_block(rmax, esz)), emu ? args_emu : args_one,
                                        stream_smem(rmax, esz), (cudaStream_t)stream);
    }
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_part_import(const DevProblem& P, void* stream, std::string& err) {
    const int nb = P.n_imp > 0 ? (P.n_imp + 255) / 256 : 1;
    cudaStream_t s = (cudaStream_t)stream;
    if (P.esz == 4) {
        part_import_kernel<float><<<nb < 148 ? nb : 148, 256, 0, s>>>(P);
        part_decide_kernel<float><<<1, 1, 0, s>>>(P);
    } else {
        part_import_kernel<double><<<nb < 148 ? nb : 148, 256, 0, s>>>(P);
        part_decide_kernel<double><<<1, 1, 0, s>>>(P);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_reset(const DevProblem& P, void* stream, std::string& err) {
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = (P.n_slots + 255) / 256;
    if (P.esz == 4) reset_kernel<float><<<nb > 0 ? nb : 1, 256, 0, s>>>(P);
    else reset_kernel<double><<<nb > 0 ? nb : 1, 256, 0, s>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

}  // namespace lopf

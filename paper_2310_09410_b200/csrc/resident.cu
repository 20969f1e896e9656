// SMEM-resident ADMM kernel for sm_100a: Algorithm 1 of arXiv 2310.09410
// with every CTA owning a connected, DFS-contiguous chunk of the feeder.
//
// At launch each CTA copies its blob (operators Abar_s / bbar_s, maps, iterate) into shared memory;
// the iterate then stays on chip for the whole solve, ping-ponged by sweep parity.  Iteration t
// (state t known) computes sweep t+1:
//   workers (all warps but one), one lane per row slot of a packed task:
//     import: the u of every copy owned by another CTA that the task reads, from the exchange buffer
//         (16-byte {u, tag} entries, spinning until the tag says "state t") into the CTA's ghost slots
//     a4  x_g = clamp((sum_{k in seg(g)} u_k - c_g/rho) / nu_g, lo_g, hi_g)   (closed_1, rho restored;
//         PAPER.md:305-310, reading C1) in canonical copy order, u_k = x_k - lambda_k/rho from SMEM
//     a5  d = -rho v - lambda, x_s = (1/rho) Abar_s d + bbar_s                  (closed_2)
//     a6  lambda_s += rho (v - x_s)                                            (ADMM-3)
//         each exported copy's u goes out at once as {u, tag of state t+1}; five residual sums per lane
//   reducer (1 warp), concurrently: publishes this CTA's residual partials of sweep t (summed by the
//     workers in iteration t-1) as parity-signed 16-byte entries; CTA 0's reducer gathers them all,
//     reduces them in CTA order, takes the (termination) decision for sweep t and
//     publishes it as one tagged entry, which every other reducer waits for.
//   one CTA barrier; a stop at t discards the speculative sweep t+1 (state t is the other buffer).
// No flags, fences or grid barrier inside the loop: a CTA waits only for the values it reads, each
// entry written by one 128-bit store (value and tag travel together).  Two parity slots suffice:
// the copy of a shared global that a CTA writes for state t+2 depends on every copy of that global at
// state t+1, and those are written only after their owners have read the state-t entries.  Tags
// carry the launch number, so entries from earlier launches never match.
#include <cuda_runtime.h>

#include <cmath>

#include "device.cuh"
#include "internal.h"

namespace lopf {

namespace {

constexpr int RB = kResBlock;
constexpr int RW = RB / 32;
constexpr int NWORK = RW - 1;              // worker warps 0 .. RW-2
constexpr int RED = RW - 1;                // reducer warp
constexpr unsigned kFull = 0xffffffffu;
#ifndef LOPF_RES_UNROLL
#define LOPF_RES_UNROLL 8                  // mat-vec column loop unroll (A/B: 1 4.83, 2 4.63, 4 4.59, 8 4.54 us)
#endif
#ifndef LOPF_DIAG_SKIP
#define LOPF_DIAG_SKIP 0                   // diagnostics builds only: bit 1 skips the update work (sync cost alone)
#endif
#ifndef LOPF_RES_CLAMP_SEL
#define LOPF_RES_CLAMP_SEL 1
#endif
#ifndef LOPF_RES_SLEEP
#define LOPF_RES_SLEEP 20                  // reducer poll back-off (ns)
#endif
constexpr int kUnroll = LOPF_RES_UNROLL;
constexpr int kPer = 5;                    // flags / partials per reducer lane per round (G <= 160 in one round)

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) { return dev::ld_acquire_u64(p); }
using dev::warp_sum5;

// consensus input u = x_s - lambda / rho, formed with the same rounding wherever it is needed
template <class T>
__device__ __forceinline__ T u_of(const T x, const T l, const T inv_rho) {
    return fma(-l, inv_rho, x);
}

extern __shared__ __align__(16) uint8_t sm[];

// SMEM accessors on 32-bit byte offsets (LDS/STS with 32-bit addresses, no 64-bit generic pointers)
template <class T> __device__ __forceinline__ T& Dt(int off, int i) { return reinterpret_cast<T*>(sm + off)[i]; }
template <class T> struct V2;                      // {x, y} pair of T (global parameters in SMEM)
template <> struct V2<double> { using type = double2; };
template <> struct V2<float> { using type = float2; };
__device__ __forceinline__ int Ii(int off, int i) { return reinterpret_cast<const int*>(sm + off)[i]; }

template <class T>                                 // T: element type of the SMEM state (fp64, or fp32: reading F1)
struct Ctx {                                       // byte offsets into SMEM + the two exchange slots
    int sinfo, sexp, sabar, sbbar, grec, gxb, gseg, gimp, gpar;
    int xl_c, lam_c, xl_n, lam_n, xout_n, dst;
    const double2* xch_c;                          // {u, tag} entries of state t / t+1 (u widened to fp64)
    double2* xch_n;
    unsigned long long tag_c, tag_n;
    T rho, inv_rho;
};

__device__ __forceinline__ void st_entry(double2* p, const double u, const unsigned long long tag) {
    asm volatile("{\n .reg .b128 v;\n mov.b128 v, {%1, %2};\n st.relaxed.gpu.global.b128 [%0], v;\n}"
                 ::"l"(p), "l"(__double_as_longlong(u)), "l"(tag) : "memory");
}
__device__ __forceinline__ double ld_entry(const double2* p, const unsigned long long tag) {
    unsigned long long lo, hi;
    do {
        asm volatile("{\n .reg .b128 v;\n ld.relaxed.gpu.global.b128 v, [%2];\n mov.b128 {%0, %1}, v;\n}"
                     : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
    } while (hi != tag);
    return __longlong_as_double(lo);
}

// raw 128-bit entry access (single-copy atomic at gpu scope)
__device__ __forceinline__ void st_pair(double2* p, const unsigned long long lo, const unsigned long long hi) {
    asm volatile("{\n .reg .b128 v;\n mov.b128 v, {%1, %2};\n st.relaxed.gpu.global.b128 [%0], v;\n}"
                 ::"l"(p), "l"(lo), "l"(hi) : "memory");
}
__device__ __forceinline__ void ld_pair(const double2* p, unsigned long long& lo, unsigned long long& hi) {
    asm volatile("{\n .reg .b128 v;\n ld.relaxed.gpu.global.b128 v, [%2];\n mov.b128 {%0, %1}, v;\n}"
                 : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
}
// residual partial (>= 0 or NaN) with the sweep parity bit in its sign bit, and back
__device__ __forceinline__ unsigned long long enc_par(const double v, const unsigned long long par) {
    return ((unsigned long long)__double_as_longlong(v) & ~(1ull << 63)) | par;
}
__device__ __forceinline__ double dec_par(const unsigned long long b) {
    return __longlong_as_double((long long)(b & ~(1ull << 63)));
}

__device__ __forceinline__ void ld_entry_once(const double2* p, unsigned long long& lo, unsigned long long& hi) {
    asm volatile("{\n .reg .b128 v;\n ld.relaxed.gpu.global.b128 v, [%2];\n mov.b128 {%0, %1}, v;\n}"
                 : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
}

// u of the copy in SMEM slot e (own, ghost or zero slot)
template <class T>
__device__ __forceinline__ T u_at(const Ctx<T>& C, const int e) {
    return u_of<T>(Dt<T>(C.xl_c, e), Dt<T>(C.lam_c, e), C.inv_rho);
}

// one task of 32R rows (tr.w = R | imports << 4 | first import << 12): lane l owns rows l (and l + 32 when R = 2: two dependency chains)
template <int R, class T>
__device__ __forceinline__ void task_sweep(const Ctx<T>& C, const int4 tr, double (&acc)[5], const int lane) {
    constexpr int E = sizeof(T);
    using T2 = typename V2<T>::type;
    // boundary values first: the u of every copy owned by another CTA that this task's rows read, from the
    // exchange buffer into the CTA's ghost slots (x = u, lambda = 0).  All entries of the task are requested
    // before any is waited on (one L2 round trip), each lane spinning until its entry's tag says "state t".
    {
        const int nimp = (tr.w >> 4) & 0xFF, i0 = tr.w >> 12;
        if (nimp > 0) {
            const int2* im = reinterpret_cast<const int2*>(sm + C.gimp) + i0;
            const int2 a = lane < nimp ? im[lane] : make_int2(0, 0);
            const int2 b = lane + 32 < nimp ? im[lane + 32] : make_int2(0, 0);
            unsigned long long alo = 0, ahi = C.tag_c, blo = 0, bhi = C.tag_c;
            if (lane < nimp) ld_entry_once(C.xch_c + a.x, alo, ahi);
            if (lane + 32 < nimp) ld_entry_once(C.xch_c + b.x, blo, bhi);
            for (int i = lane + 64; i < nimp; i += 32) {              // (> 64 imports: rare)
                const int2 c = im[i];
                Dt<T>(C.xl_c, c.y) = (T)ld_entry(C.xch_c + c.x, C.tag_c);
            }
            while (ahi != C.tag_c) ld_entry_once(C.xch_c + a.x, alo, ahi);
            while (bhi != C.tag_c) ld_entry_once(C.xch_c + b.x, blo, bhi);
            if (lane < nimp) Dt<T>(C.xl_c, a.y) = (T)__longlong_as_double((long long)alo);
            if (lane + 32 < nimp) Dt<T>(C.xl_c, b.y) = (T)__longlong_as_double((long long)blo);
            __syncwarp();
        }
    }
    T v[2], lam[2], xo[2];
    int info[2], gl[2];
    // a4 for both rows, straight-line from SMEM: the four entries of the global's record (own, ghost or zero
    // slots) summed in canonical copy order; nu > 4 walks the global's slot list
    T sig[2];
#pragma unroll
    for (int h = 0; h < R; ++h) {
        info[h] = Ii(C.sinfo, tr.x + h * 32 + lane);
        gl[h] = info[h] >> kResGlShift;                                  // an empty row: global 0, discarded
        const int4 rc = reinterpret_cast<const int4*>(sm + C.grec)[gl[h]];
        sig[h] = ((u_at<T>(C, rc.x) + u_at<T>(C, rc.y)) + u_at<T>(C, rc.z)) + u_at<T>(C, rc.w);
        if (info[h] & kResSlow) {
            const int2 sl = reinterpret_cast<const int2*>(sm + C.gxb)[gl[h]];   // {first entry, nu}
            sig[h] = T(0);
            for (int q = 0; q < sl.y; ++q) sig[h] += u_at<T>(C, Ii(C.gseg, sl.x + q));
        }
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {
        const int slot = tr.x + h * 32 + lane;
        const T2 g0 = reinterpret_cast<const T2*>(sm + C.gpar)[2 * gl[h]];       // {c/rho, 1/nu}
        const T2 g1 = reinterpret_cast<const T2*>(sm + C.gpar)[2 * gl[h] + 1];   // {lo, hi}
        // clamp to [lo, hi] with the semantics of fmin(fmax(y, lo), hi) (a NaN y gives lo; IEEE +-inf = no
        // clamp) in two compare-selects
        const T y = (sig[h] - g0.x) * g0.y;
#if LOPF_RES_CLAMP_SEL
        const T ylo = y > g1.x ? y : g1.x;
        const T xg = ylo < g1.y ? ylo : g1.y;
#else
        const T xg = fmin(fmax(y, g1.x), g1.y);
#endif
        const bool val = info[h] & kResValid;
        if (val && (info[h] & kResFirst)) Dt<T>(C.xout_n, gl[h]) = xg;
        v[h] = val ? xg : T(0);
        lam[h] = val ? Dt<T>(C.lam_c, slot) : T(0);
        xo[h] = val ? Dt<T>(C.xl_c, slot) : T(0);
        Dt<T>(C.dst, h * 32 + lane) = val ? -C.rho * xg - lam[h] : T(0);
    }
    __syncwarp();
    // local update: x_s = (1/rho) Abar_s d + bbar_s.  The task tile is zero-padded (tile[k][row] = 0 for
    // k >= n_s of the row's subsystem), so the loop has no masks: 2 tile loads + 2 staged-d loads + 2 FMA
    // per column; d indices beyond the subsystem land on finite d values or the zeroed staging tail.
    const int kmax = tr.y;
    const int at = C.sabar + E * (tr.z + lane);                          // byte offset of tile[0][lane]
    const int d0 = C.dst + E * (info[0] & 0x3F), d1 = C.dst + E * (info[R - 1] & 0x3F);
    T ax0 = T(0), ax1 = T(0);
    if (R == 2) {
#pragma unroll kUnroll
        for (int k = 0; k < kmax; ++k) {
            ax0 = fma(Dt<T>(at, 64 * k), Dt<T>(d0, k), ax0);
            ax1 = fma(Dt<T>(at, 64 * k + 32), Dt<T>(d1, k), ax1);
        }
    } else {
#pragma unroll kUnroll
        for (int k = 0; k < kmax; ++k) ax0 = fma(Dt<T>(at, 32 * k), Dt<T>(d0, k), ax0);
    }
    const T axr[2] = {ax0, ax1};
    __syncwarp();                                                        // dst is reused by the next task
#pragma unroll
    for (int h = 0; h < R; ++h) {      // no branch on validity: an empty row has a zero tile row, b-bar and d,
        const int slot = tr.x + h * 32 + lane;   // so it stores zeros and adds exact zeros to the sums
        const T xn = fma(axr[h], C.inv_rho, Dt<T>(C.sbbar, slot));       // (1/rho) Abar d + bbar
        const T ln = lam[h] + C.rho * (v[h] - xn);                       // ADMM-3
        Dt<T>(C.xl_n, slot) = xn;
        Dt<T>(C.lam_n, slot) = ln;
        const int e = Ii(C.sexp, slot);
        if (e >= 0) st_entry(C.xch_n + e, (double)u_of<T>(xn, ln, C.inv_rho), C.tag_n);   // boundary copy -> exchange
        const T r = v[h] - xn, dx = xn - xo[h];                          // terms in T, sums in fp64 (F1)
        acc[0] += (double)(r * r);
        acc[1] += (double)(dx * dx);
        acc[2] += (double)(v[h] * v[h]);
        acc[3] += (double)(xn * xn);
        acc[4] += (double)(ln * ln);
    }
}


#if LOPF_RES_TIMELINE == 1   // diagnostics build: per-warp clock64 events of CTA G/2, sweeps 500..502, into P.prof
#ifndef LOPF_RES_TL_CTA
#define LOPF_RES_TL_CTA (G / 2)
#endif
#define TL(e) do { if (P.prof && cta == LOPF_RES_TL_CTA && t >= 500 && t < 503 && lane == 0) \
    P.prof[((t - 500) * RW + wid) * 8 + (e)] = clock64(); } while (0)
#elif LOPF_RES_TIMELINE == 2  // every CTA, sweeps 500..503: cycles from each warp's loop top to its work end
                              // (event 1; slot = warp) and, for warp 0, to the end-of-iteration barrier (slot 31)
#define TL(e) do { if (P.prof && t >= 500 && t < 504 && lane == 0) { \
    if ((e) == 0) tl_top = clock64(); \
    else if ((e) == 1) P.prof[4 * G + ((t - 500) * G + cta) * 32 + wid] = clock64() - tl_top; \
    else if ((e) == 7 && wid == 0) P.prof[4 * G + ((t - 500) * G + cta) * 32 + 31] = clock64() - tl_top; } } while (0)
#else
#define TL(e) do { } while (0)
#endif

template <class T>
__global__ void __launch_bounds__(RB, 1) admm_resident_kernel(ResProblem P) {
    constexpr int E = sizeof(T);
    __shared__ CtaHdr H;
    __shared__ double red[2][RW][5];               // worker sums by sweep parity (reducer reads the older)
    __shared__ double s_res[2][4];                 // decision records double-buffered by sweep parity: the
    __shared__ int s_stop[2], s_conv[2], s_num[2]; // reducer writes t+1's while slow warps still read t's
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    if (tid < (int)(sizeof(CtaHdr) / 4)) ((int*)&H)[tid] = ((const int*)(P.hdr + cta))[tid];
    if (tid < 2) {
        s_stop[tid] = 0; s_conv[tid] = 0; s_num[tid] = 0;
        s_res[tid][0] = s_res[tid][1] = s_res[tid][2] = s_res[tid][3] = 0.0;
    }
    __syncthreads();
    uint8_t* blob = P.blobs + H.blob_off;
    {
        const int4* src = (const int4*)blob;
        int4* d16 = (int4*)sm;
        const int n16 = H.blob_bytes / 16;
        for (int i = tid; i < n16; i += RB) d16[i] = __ldcg(src + i);
    }
    __syncthreads();
    const int NS = H.n_slots, NG = H.n_glob, NT = H.n_tasks;
    const int dst_stride = H.dst_stride;                              // 64 + largest task width, doubles
    for (int i = tid; i < RW * dst_stride; i += RB) Dt<T>(H.off_dst, i) = T(0);   // zero tail of the d staging
    for (int i = NS + tid; i <= NS + H.n_ghost; i += RB) {       // zero and ghost slots of parity 1
        Dt<T>(H.off_xl1, i) = T(0);
        Dt<T>(H.off_lam1, i) = T(0);
    }
    Ctx<T> C;
    C.sinfo = H.off_sinfo; C.sexp = H.off_sexp; C.sabar = H.off_abar; C.sbbar = H.off_bbar;
    C.grec = H.off_grec; C.gxb = H.off_gxb; C.gseg = H.off_gseg; C.gimp = H.off_gimp; C.gpar = H.off_gpar;
    C.dst = H.off_dst + E * wid * dst_stride;
    C.rho = (T)P.rho;
    C.inv_rho = (T)P.inv_rho;
    double2* dec = reinterpret_cast<double2*>(P.flags);                  // {decision bits, tag of sweep t}
    const long long total0 = *(volatile long long*)&P.ctrl->total;
#ifndef LOPF_RES_PROF
#define LOPF_RES_PROF 0                           // 1: per-CTA phase counters (lopf_get_profile, diagnostics builds)
#endif
#ifdef LOPF_RES_TIMELINE
    const bool prof = P.prof != nullptr;
#else
    const bool prof = LOPF_RES_PROF && P.prof != nullptr;
#endif
    __shared__ long long s_prof[3];
    if (tid == 0) s_prof[0] = s_prof[1] = s_prof[2] = 0;

    double2* xchg = reinterpret_cast<double2*>(P.xchg);
    // tag of state t in this launch (0 = never written; the epoch keeps earlier launches' entries out)
    auto tag_of = [&](long long tt) { return ((unsigned long long)P.epoch << 32) | (unsigned long long)(tt + 1); };
    // state 0: boundary u into exchange slot 0
    for (int i = tid; i < NS; i += RB) {
        const int e = Ii(H.off_sexp, i);
        if (e >= 0) st_entry(xchg + e, (double)u_of<T>(Dt<T>(H.off_xl0, i), Dt<T>(H.off_lam0, i), C.inv_rho), tag_of(0));
    }
    __syncthreads();

    long long t = 0;                                   // sweeps completed; state t in buffer t & 1
#if LOPF_RES_TIMELINE == 2
    long long tl_top = 0;
#endif
    for (;;) {
        const int cur = (int)(t & 1);
        if (prof && tid == 0) s_prof[2] = clock64();
        TL(0);
        if (wid == RED) {
            if (t >= 1) {
                // this CTA's residual partials of sweep t (the workers' sums of iteration t-1), published as
                // three 16-byte entries {s0, s1} {s2, s3} {s4, s4} in slot u & 3 (u = t - 1: publications are
                // numbered from 0 in each launch); the sign bit of each (non-negative) value carries (u >> 2) & 1,
                // so the reader tells this publication from the one four earlier with no flag and no fence (each
                // entry is one 128-bit access).  The launch fills the slots with sign bit 1: u = 0..3 never match
                // them, and u >= 4 finds its slot written at least once before (per-location coherence).
                const long long u = t - 1;
                const int slot = (int)(u & 3);
                const unsigned long long par = (unsigned long long)((u >> 2) & 1) << 63;
                double2* part = reinterpret_cast<double2*>(P.partial) + (size_t)slot * G * 4;
                {
                    double sk = 0.0;                   // four interleaved chains, combined in a fixed order
                    if (lane < 5) {
                        double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                        for (int w = 0; w < NWORK; ++w) q4[w & 3] += red[cur][w][lane];
                        sk = (q4[0] + q4[1]) + (q4[2] + q4[3]);
                    }
                    const double a = __shfl_sync(kFull, sk, 2 * lane < 5 ? 2 * lane : 4);
                    const double b = __shfl_sync(kFull, sk, 2 * lane + 1 < 5 ? 2 * lane + 1 : 4);
                    if (lane < 3) st_pair(part + (size_t)cta * 4 + lane, enc_par(a, par), enc_par(b, par));
                }
                TL(3);
                // the decision: CTA 0's reducer gathers every CTA's entries (lane l: CTAs l, l + 32, ...), sums
                // them in CTA order per lane then across lanes (fixed order), decides and publishes one tagged
                // entry; every other CTA's reducer waits for that entry
                double ps[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                if (cta == 0) {
                    unsigned long long ev[kPer][3][2];
                    unsigned pend = 0;                 // entries of this lane still to be (re)read
#pragma unroll
                    for (int j = 0; j < kPer; ++j)
                        if (j * 32 + lane < G) pend |= 7u << (3 * j);
#pragma unroll
                    for (int j = 0; j < kPer; ++j)
#pragma unroll
                        for (int e = 0; e < 3; ++e) { ev[j][e][0] = par; ev[j][e][1] = par; }
                    while (pend) {                     // every stale entry re-requested together: one round trip
#pragma unroll
                        for (int j = 0; j < kPer; ++j)
#pragma unroll
                            for (int e = 0; e < 3; ++e)
                                if (pend >> (3 * j + e) & 1) ld_pair(part + (size_t)(j * 32 + lane) * 4 + e, ev[j][e][0], ev[j][e][1]);
#pragma unroll
                        for (int j = 0; j < kPer; ++j)
#pragma unroll
                            for (int e = 0; e < 3; ++e)
                                if (!(((ev[j][e][0] ^ par) | (ev[j][e][1] ^ par)) >> 63)) pend &= ~(1u << (3 * j + e));
                    }
                    TL(4);
#pragma unroll
                    for (int j = 0; j < kPer; ++j)
#pragma unroll
                        for (int k = 0; k < 5; ++k) ps[k] += dec_par(ev[j][k >> 1][k & 1]);   // CTA order per lane
#pragma unroll
                    for (int k = 0; k < 5; ++k) {
#pragma unroll
                        for (int off = 16; off > 0; off >>= 1) ps[k] += __shfl_xor_sync(kFull, ps[k], off);
                    }
                }
                // the five square roots one per lane (every lane holds all five sums after the butterfly)
                double rt = 0.0;
                bool fin = true;
                if (cta == 0) {
                    const double mine = lane == 0 ? ps[0] : lane == 1 ? ps[1] : lane == 2 ? ps[2] : lane == 3 ? ps[3] : ps[4];
                    rt = sqrt(mine);
                    fin = __all_sync(kFull, lane >= 5 || isfinite(mine));
                }
                const double r1 = __shfl_sync(kFull, rt, 1), r2 = __shfl_sync(kFull, rt, 2);
                const double r3 = __shfl_sync(kFull, rt, 3), r4 = __shfl_sync(kFull, rt, 4);
                if (lane == 0 && cta == 0) {
                    const double pres = rt, dres = P.rho * r1;
                    const double ep = P.eps_rel * fmax(r2, r3), ed = P.eps_rel * r4;
                    const int num = !fin;
                    const int conv = P.test && pres <= ep && dres <= ed;
                    const int q = (int)(t & 1);
                    s_res[q][0] = pres; s_res[q][1] = dres; s_res[q][2] = ep; s_res[q][3] = ed;
                    s_conv[q] = conv; s_num[q] = num;
                    s_stop[q] = conv || num || t >= P.max_iter;
                    TL(5);
                    st_pair(dec, (unsigned long long)(s_stop[q] | (conv << 1) | (num << 2)), tag_of(t));   // decision of t
                    if (P.trace_every > 0 && (t % P.trace_every) == 0) {
                        const long long row = t / P.trace_every - 1;
                        if (row < P.trace_cap) {
                            double* tr = P.trace + row * 5;
                            tr[0] = (double)(total0 + t); tr[1] = pres; tr[2] = dres; tr[3] = ep; tr[4] = ed;
                            P.ctrl->trace_rows = row + 1;
                        }
                    }
                } else if (lane == 0 && cta != 0) {
                    unsigned long long bits, tg;
                    ld_pair(dec, bits, tg);
                    while (tg != tag_of(t)) {
                        if (LOPF_RES_SLEEP > 0) __nanosleep(LOPF_RES_SLEEP);
                        ld_pair(dec, bits, tg);
                    }
                    TL(5);
                    const int q = (int)(t & 1);
                    s_stop[q] = (int)(bits & 1);
                    s_conv[q] = (int)((bits >> 1) & 1);
                    s_num[q] = (int)((bits >> 2) & 1);
                }
            }
            TL(1);
        } else {                                       // workers: sweep t+1 (speculative until decided)
            double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            const bool busy = t < P.max_iter && !(LOPF_DIAG_SKIP & 2) && wid < NT;
            if (busy) {
                C.xl_c = cur ? H.off_xl1 : H.off_xl0;
                C.lam_c = cur ? H.off_lam1 : H.off_lam0;
                C.xl_n = cur ? H.off_xl0 : H.off_xl1;
                C.lam_n = cur ? H.off_lam0 : H.off_lam1;
                C.xout_n = H.off_xout + (cur ? 0 : E * NG);
                C.xch_c = xchg + (size_t)cur * P.n_exp;
                C.xch_n = xchg + (size_t)(cur ^ 1) * P.n_exp;
                C.tag_c = tag_of(t);
                C.tag_n = tag_of(t + 1);
                for (int task = wid; task < NT; task += NWORK) {
                    const int4 tr = reinterpret_cast<const int4*>(sm + H.off_tasks)[task];
                    if ((tr.w & 0xF) == 1) task_sweep<1, T>(C, tr, acc, lane);
                    else task_sweep<2, T>(C, tr, acc, lane);
                }
#if LOPF_RES_TIMELINE == 2
                if (P.prof && t == 500) {   // task signature of this warp: kmax | tasks << 8 | rows << 16 | xreads << 32
                    long long sig = 0, rows = 0, xr = 0, km = 0, nt = 0;
                    for (int task = wid; task < NT; task += NWORK) {
                        const int4 tr = reinterpret_cast<const int4*>(sm + H.off_tasks)[task];
                        km = km > tr.y ? km : tr.y;
                        ++nt;
                        for (int h = 0; h < ((tr.w & 0xF) == 1 ? 1 : 2); ++h) {
                            const int inf = Ii(C.sinfo, tr.x + h * 32 + lane);
                            if (!(inf & kResValid)) continue;
                            ++rows;
                            xr += (inf & kResSlow) != 0;
                        }
                    }
                    for (int off = 16; off > 0; off >>= 1) {
                        rows += __shfl_xor_sync(kFull, rows, off);
                        xr += __shfl_xor_sync(kFull, xr, off);
                    }
                    sig = km | (nt << 8) | (rows << 16) | (xr << 32);
                    if (lane == 0) P.prof[4 * G + 128 * G + cta * 32 + wid] = sig;
                }
#endif
            }
            TL(1);
            // the five warp sums of sweep t+1 (idle warps contribute exact zeros without shuffling)
            const double wsum = busy ? warp_sum5(acc, lane) : 0.0;
            if ((lane & 3) == 0 && (lane >> 2) < 5) red[cur ^ 1][wid][lane >> 2] = wsum;
            TL(2);
        }
        __syncthreads();                               // sweep t+1 computed; decision for sweep t known
        if (prof && tid == 0) { const long long c1 = clock64(); s_prof[0] += c1 - s_prof[2]; s_prof[2] = c1; }
        TL(7);
        if (s_stop[t & 1]) break;                      // state t (buffer t & 1); x^t in xout[t & 1]
        ++t;
    }

    // exit: state t (buffer t & 1) back to the blob, this CTA's x, then one grid barrier for the result
    const int fin = (int)(t & 1);
    {
        T* gx = (T*)(blob + H.off_xl0);
        T* gl = (T*)(blob + H.off_lam0);
        const int oxl = fin ? H.off_xl1 : H.off_xl0, olm = fin ? H.off_lam1 : H.off_lam0;
        for (int i = tid; i < NS; i += RB) {
            __stcg(gx + i, Dt<T>(oxl, i));
            __stcg(gl + i, Dt<T>(olm, i));
        }
    }
    const int* gown = reinterpret_cast<const int*>(blob + H.off_gown);  // global memory (not staged in SMEM)
    for (int j = tid; j < NG; j += RB) {
        const int g = __ldg(gown + j);
        if (g >= 0) __stcg(reinterpret_cast<T*>(P.x) + g, Dt<T>(H.off_xout, fin * NG + j));
    }
#if !LOPF_RES_TIMELINE
    if (prof && tid == 0) {
        long long* pr = P.prof + 4 * cta;
        pr[0] = s_prof[0]; pr[1] = s_prof[1]; pr[2] = 0; pr[3] = t;
    }
#endif
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        atomicAdd(&P.ctrl->arrive, 1ULL);
        if (cta == 0) {
            while (ld_acq(&P.ctrl->arrive) < (unsigned long long)G) {
            }
            double obj = 0.0;
            for (int j = 0; j < P.n_obj; ++j) obj += P.obj_c[j] * (double)__ldcg(reinterpret_cast<const T*>(P.x) + P.obj_idx[j]);
            DevCtrl* c = P.ctrl;
            const int q = (int)(t & 1);
            c->res[0] = s_res[q][0]; c->res[1] = s_res[q][1]; c->res[2] = s_res[q][2]; c->res[3] = s_res[q][3];
            c->objective = obj;
            c->iters = t;
            c->total = total0 + t;
            c->outcome = s_conv[q] ? LOPF_CONVERGED : LOPF_MAX_ITER;
            c->numeric = s_num[q];
        }
    }
}

// a3 for the resident layout: x_s = x0, lambda = 0 in every blob; sweep counter 0.
template <class T>
__global__ void reset_resident_kernel(ResProblem P) {
    const CtaHdr& H = P.hdr[blockIdx.x];
    uint8_t* blob = P.blobs + H.blob_off;
    T* xl = (T*)(blob + H.off_xl0);
    T* lam = (T*)(blob + H.off_lam0);
    const T* x0 = reinterpret_cast<const T*>(P.x0) + H.slot_base;
    for (int i = threadIdx.x; i < H.n_slots; i += blockDim.x) {
        xl[i] = x0[i];
        lam[i] = T(0);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.ctrl->arrive = 0; P.ctrl->flag = 0; P.ctrl->total = 0; P.ctrl->iters = 0; P.ctrl->trace_rows = 0;
    }
}

// lopf_get_state on the resident layout: every CTA blob's x_s and lambda (state at the last exit) widened
// to fp64 into the staging area in global slot order: stage[slot] = x_s, stage[total + slot] = lambda.
template <class T>
__global__ void gather_resident_kernel(ResProblem P, double* stage) {
    const CtaHdr& H = P.hdr[blockIdx.x];
    const uint8_t* blob = P.blobs + H.blob_off;
    const T* xl = reinterpret_cast<const T*>(blob + H.off_xl0);
    const T* lam = reinterpret_cast<const T*>(blob + H.off_lam0);
    for (int i = threadIdx.x; i < H.n_slots; i += blockDim.x) {
        stage[H.slot_base + i] = (double)xl[i];
        stage[(size_t)P.total_slots + H.slot_base + i] = (double)lam[i];
    }
}

}  // namespace

lopf_status launch_gather_resident(const ResProblem& P, void* stage, void* stream, std::string& err) {
    if (P.esz == 4) gather_resident_kernel<float><<<P.G, 256, 0, (cudaStream_t)stream>>>(P, (double*)stage);
    else gather_resident_kernel<double><<<P.G, 256, 0, (cudaStream_t)stream>>>(P, (double*)stage);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

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
    const void* k = P.esz == 4 ? (const void*)admm_resident_kernel<float> : (const void*)admm_resident_kernel<double>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, P.max_smem);
    if (e == cudaSuccess) e = cudaMemsetAsync(P.ctrl, 0, 2 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(&P.ctrl->trace_rows, 0, sizeof(long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P.flags, 0, sizeof(unsigned long long) * 32 * (P.G + 1), s);
    // partial entries: all sign bits set, i.e. "sweep parity 1", which the first sweeps (parity 0) never match
    // and later sweeps only meet after their slot was written at parity 0 (per-location coherence)
    if (e == cudaSuccess) e = cudaMemsetAsync(P.partial, 0xFF, sizeof(double) * 8 * 4 * P.G, s);
    if (e == cudaSuccess && P.max_iter > 0) {
        ResProblem Q = P;
        void* args[] = {&Q};
        e = cudaLaunchCooperativeKernel(k, dim3(P.G), dim3(RB), args, P.max_smem, s);
    }
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

lopf_status launch_reset_resident(const ResProblem& P, void* stream, std::string& err) {
    if (P.esz == 4) reset_resident_kernel<float><<<P.G, 256, 0, (cudaStream_t)stream>>>(P);
    else reset_resident_kernel<double><<<P.G, 256, 0, (cudaStream_t)stream>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("CUDA: ") + cudaGetErrorString(e); return LOPF_E_CUDA; }
    return LOPF_OK;
}

}  // namespace lopf

// Device layout of the batch kernel (config 4): scenario-fastest arrays so that one
// warp (lane = scenario) reads one 256-byte line per copy / operator entry, and operators of the
// subsystems without a load are shared by all scenarios (broadcast loads from L1/L2).
#include <algorithm>
#include <cstring>

#include <vector_functions.h>

#include "internal.h"

namespace lopf {

static size_t a256b(size_t x) { return (x + 255) & ~(size_t)255; }

lopf_status pack_batch(const Canon& P, const BatchOps& bo, const lopf_options& opt, Layout& L, std::string& err) {
    L = Layout();
    L.kernel = 3;
    L.n_scen = bo.n_scen;
    L.n_grp = (bo.n_scen + 31) / 32;
    const int64_t S = P.S, NC = P.nc, N = P.n, G = L.n_grp, V = (int64_t)bo.vsub.size();
    if (NC > INT32_MAX / 64 || bo.VA > INT32_MAX) { err = "batch: problem too large"; return LOPF_E_ARG; }
    for (int64_t s = 0; s < S; ++s) L.ns_max = std::max(L.ns_max, P.n_s[s]);
    if (L.ns_max > 64) { err = "batch kernel supports n_s <= 64"; return LOPF_E_ARG; }
    // subsystem ranges per warp, balanced by n_s^2 + 8 n_s (mat-vec + consensus)
    std::vector<int32_t> warp_sub(kBatchWarps + 1, 0);
    {
        double tot = 0;
        for (int64_t s = 0; s < S; ++s) tot += (double)P.n_s[s] * P.n_s[s] + 8.0 * P.n_s[s];
        double acc = 0;
        int w = 1;
        for (int64_t s = 0; s < S; ++s) {
            acc += (double)P.n_s[s] * P.n_s[s] + 8.0 * P.n_s[s];
            while (w < kBatchWarps && acc >= tot * w / kBatchWarps) warp_sub[w++] = (int32_t)s + 1;
        }
        while (w <= kBatchWarps) warp_sub[w++] = (int32_t)S;
    }
    std::vector<int32_t> sub_op(S), vsub_a(std::max<int64_t>(V, 1)), vsub_b(std::max<int64_t>(V, 1));
    std::vector<double> shared;
    for (int64_t s = 0; s < S; ++s) {
        if (bo.vidx[s] >= 0) { sub_op[s] = -(1 + bo.vidx[s]); continue; }
        sub_op[s] = (int32_t)shared.size();
        shared.insert(shared.end(), P.abar.begin() + P.abar_ptr[s], P.abar.begin() + P.abar_ptr[s + 1]);
        for (int64_t r = P.sub_ptr[s]; r < P.sub_ptr[s + 1]; ++r)
            if (P.bbar[r] != 0.0) { err = "batch: a subsystem without a load has bbar != 0"; return LOPF_E_ARG; }
    }
    for (int64_t v = 0; v < V; ++v) { vsub_a[v] = (int32_t)bo.va_off[v]; vsub_b[v] = (int32_t)bo.vb_off[v]; }
    std::vector<int2> copy_info(NC);
    for (int64_t k = 0; k < NC; ++k) {
        const int32_t g = P.copy_global[k];
        copy_info[k] = make_int2(g, P.seg_copy[P.seg_ptr[g]] == k ? 1 : 0);
    }
    std::vector<int32_t> obj_idx;
    std::vector<double> obj_c;
    for (int64_t i = 0; i < N; ++i)
        if (P.c[i] != 0.0) { obj_idx.push_back((int32_t)i); obj_c.push_back(P.c[i]); }
    L.n_obj = (int64_t)obj_idx.size();

    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = a256b(o + std::max<size_t>(bytes, 1)); return r; };
    L.off_bwarp = take(4 * warp_sub.size());
    L.off_bsubptr = take(4 * (S + 1));
    L.off_bns = take(4 * S);
    L.off_bop = take(4 * S);
    L.off_bva = take(4 * vsub_a.size());
    L.off_bvb = take(4 * vsub_b.size());
    L.off_bcopy = take(8 * NC);
    L.off_gpar = take(32 * N);
    L.off_segptr = take(4 * (N + 1));
    L.off_segslot = take(4 * NC);
    L.off_bshared = take(8 * shared.size());
    L.off_bvabar = take(8 * (size_t)G * bo.VA * 32);
    L.off_bvbbar = take(8 * (size_t)G * bo.VB * 32);
    L.off_bxl = take(8 * 2 * (size_t)G * NC * 32);
    L.off_blam = take(8 * 2 * (size_t)G * NC * 32);
    L.off_bxout = take(8 * (size_t)G * N * 32);
    L.off_bres = take(sizeof(ScenResult) * (size_t)G * 32);
    L.off_x0 = take(8 * NC);
    L.off_objidx = take(4 * obj_idx.size());
    L.off_objc = take(8 * obj_c.size());
    L.off_ctrl = take(sizeof(DevCtrl));
    L.bytes = o;
    L.image.assign(L.bytes, 0);
    uint8_t* img = L.image.data();
    std::memcpy(img + L.off_bwarp, warp_sub.data(), 4 * warp_sub.size());
    int32_t* sp = (int32_t*)(img + L.off_bsubptr);
    for (int64_t s = 0; s <= S; ++s) sp[s] = (int32_t)P.sub_ptr[s];
    std::memcpy(img + L.off_bns, P.n_s.data(), 4 * S);
    std::memcpy(img + L.off_bop, sub_op.data(), 4 * S);
    std::memcpy(img + L.off_bva, vsub_a.data(), 4 * vsub_a.size());
    std::memcpy(img + L.off_bvb, vsub_b.data(), 4 * vsub_b.size());
    std::memcpy(img + L.off_bcopy, copy_info.data(), 8 * NC);
    double4* gpar = (double4*)(img + L.off_gpar);
    for (int64_t i = 0; i < N; ++i) {
        const double nu = (double)(P.seg_ptr[i + 1] - P.seg_ptr[i]);
        gpar[i] = make_double4(P.c[i] / opt.rho, 1.0 / nu, P.lo[i], P.hi[i]);
    }
    int32_t* segp = (int32_t*)(img + L.off_segptr);
    for (int64_t i = 0; i <= N; ++i) segp[i] = (int32_t)P.seg_ptr[i];
    std::memcpy(img + L.off_segslot, P.seg_copy.data(), 4 * NC);
    std::memcpy(img + L.off_bshared, shared.data(), 8 * shared.size());
    double* va = (double*)(img + L.off_bvabar);
    double* vb = (double*)(img + L.off_bvbbar);
    for (int32_t sc = 0; sc < bo.n_scen; ++sc) {           // scenario-fastest (lane = sc % 32)
        const int64_t g = sc / 32, ln = sc % 32;
        for (int64_t q = 0; q < bo.VA; ++q) va[((size_t)g * bo.VA + q) * 32 + ln] = bo.abar[(size_t)sc * bo.VA + q];
        for (int64_t q = 0; q < bo.VB; ++q) vb[((size_t)g * bo.VB + q) * 32 + ln] = bo.bbar[(size_t)sc * bo.VB + q];
    }
    std::memcpy(img + L.off_x0, P.x0.data(), 8 * NC);
    std::memcpy(img + L.off_objidx, obj_idx.data(), 4 * obj_idx.size());
    std::memcpy(img + L.off_objc, obj_c.data(), 8 * obj_c.size());
    // initial state in buffer 0 for every scenario
    double* xl = (double*)(img + L.off_bxl);
    for (int64_t g = 0; g < G; ++g)
        for (int64_t k = 0; k < NC; ++k)
            for (int ln = 0; ln < 32; ++ln) xl[((size_t)g * NC + k) * 32 + ln] = P.x0[k];
    return LOPF_OK;
}

}  // namespace lopf

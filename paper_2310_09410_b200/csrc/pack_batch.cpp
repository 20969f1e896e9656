// Device layout of the batch mode (config 4): the streaming layout of ONE scenario
// (pack_streaming: DFS-ordered tasks, packed operator blocks, per-slot metadata) is the template; every
// scenario gets its own iterate arrays ([scenario][slot]) and solution ([scenario][global]), and the
// tasks that hold a load subsystem -- whose A_s depends on the load level (VDLM-1/2)
// -- get a per-scenario operator block in `var_pool` ([scenario][VP]).  Metadata and the operators of
// every other task are shared by all scenarios (they stay in L2).
#include <algorithm>
#include <cstring>

#include <vector_functions.h>

#include "internal.h"

namespace lopf {

static size_t a256b(size_t x) { return (x + 255) & ~(size_t)255; }

lopf_status pack_batch(const Net& N, const Canon& P, const BatchOps& bo, const lopf_options& opt, Layout& L,
                       std::string& err) {
    Layout T;
    lopf_status st = pack_streaming(N, P, opt, 4096, T, err);
    if (st != LOPF_OK) return st;
    for (const int4& tr : T.trec)
        if (!(tr.w & kTaskPacked)) { err = "batch mode supports n_s <= 63"; return LOPF_E_ARG; }
    const int64_t NT = T.n_tasks, NS = T.n_slots, NG = P.n, NSC = bo.n_scen;
    // per-scenario blocks: tasks holding at least one varying (load) subsystem
    std::vector<int4> trec = T.trec;
    std::vector<int64_t> var_off(NT, -1);
    int64_t VP = 0;
    for (int64_t t = 0; t < NT; ++t) {
        bool var = false;
        for (int32_t j = T.tsub_ptr[t]; j < T.tsub_ptr[t + 1]; ++j) var |= bo.vidx[T.tsub_s[j]] >= 0;
        if (!var) continue;
        var_off[t] = VP;
        trec[t].y = (int)VP;
        trec[t].w |= kTaskVar;
        VP += trec[t].z;                                     // block length (entries, 16-byte multiple)
    }
    if (VP * NSC > ((int64_t)1 << 40)) { err = "batch: per-scenario operators too large"; return LOPF_E_ARG; }

    L = Layout();
    L.kernel = 3;
    const size_t e = (size_t)T.esz;                          // (T) element size (fp32 variant: reading F1)
    L.esz = T.esz;
    L.n_scen = (int32_t)NSC;
    L.n_tasks = NT;
    L.n_slots = NS;
    L.rmax = T.rmax;
    L.staged = 1;
    for (const int4& tr : trec)
        if (tr.w & kTaskDirect) L.staged = 0;
    L.VP = VP;
    L.n_obj = T.n_obj;
    L.slot_of_copy = T.slot_of_copy;
    L.max_grid = 4096;
    L.trace_cap = 1;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = a256b(o + std::max<size_t>(bytes, 1)); return r; };
    L.off_tasks = take(16 * NT);
    L.off_meta = take(sizeof(SlotMeta) * NS);
    L.off_bbar = take(e * NS);
    L.off_x0 = take(e * NS);
    L.off_gpar = take(2 * e * NG);
    L.off_gcost = take(e * NG);
    L.off_segptr = take(4 * (NG + 1));
    L.off_segslot = take(4 * P.nc);
    L.off_abar = take(e * (size_t)T.abar_doubles);
    L.off_objidx = take(4 * (size_t)T.n_obj);
    L.off_objc = take(8 * (size_t)T.n_obj);
    L.off_bvar = take(e * (size_t)VP * NSC);
    L.off_xl = take(e * (size_t)NS * NSC);
    L.off_lam = take(e * (size_t)NS * NSC);
    L.off_u0 = take(e * (size_t)NS * NSC);
    L.off_u1 = take(e * (size_t)NS * NSC);
    L.off_x = take(e * (size_t)NG * NSC);
    L.off_bres = take(sizeof(ScenResult) * (size_t)NSC);
    L.off_bstop = take(4 * (size_t)NSC);
    L.off_bpart = take(8 * 8 * (size_t)NT * NSC);
    L.off_bcnt = take(8 * 4);
    L.off_bmask = take(4 * 2 * (((size_t)NSC + 31) / 32));
    L.off_bwpre = take(8 * ((size_t)NT + 1));
    L.off_partial = take(8 * 8 * 4096);
    L.off_ctrl = take(sizeof(DevCtrl));
    L.off_trace = take(8 * 5);
    L.bytes = o;
    L.image.assign(L.bytes, 0);
    uint8_t* img = L.image.data();
    const uint8_t* ti = T.image.data();
    std::memcpy(img + L.off_tasks, trec.data(), 16 * NT);
    {   // work-split weights: a fixed per-item cost plus the mat-vec columns x halves (kmax * R)
        long long* wp = reinterpret_cast<long long*>(img + L.off_bwpre);
        wp[0] = 0;
        for (int64_t t = 0; t < NT; ++t)
            wp[t + 1] = wp[t] + LOPF_BATCH_WBASE + (long long)((trec[t].w >> kTaskKmaxShift) & 0xFF) * (trec[t].w & 0xF);
    }
    std::memcpy(img + L.off_meta, ti + T.off_meta, sizeof(SlotMeta) * NS);
    std::memcpy(img + L.off_bbar, ti + T.off_bbar, e * NS);
    std::memcpy(img + L.off_x0, ti + T.off_x0, e * NS);
    std::memcpy(img + L.off_gpar, ti + T.off_gpar, 2 * e * NG);
    std::memcpy(img + L.off_gcost, ti + T.off_gcost, e * NG);
    std::memcpy(img + L.off_segptr, ti + T.off_segptr, 4 * (NG + 1));
    std::memcpy(img + L.off_segslot, ti + T.off_segslot, 4 * P.nc);
    std::memcpy(img + L.off_abar, ti + T.off_abar, e * (size_t)T.abar_doubles);
    std::memcpy(img + L.off_objidx, ti + T.off_objidx, 4 * (size_t)T.n_obj);
    std::memcpy(img + L.off_objc, ti + T.off_objc, 8 * (size_t)T.n_obj);
    // per-scenario operator blocks: the template block with each load subsystem's triangle and b-bar
    // replaced by the scenario's (same packing, so the per-slot metadata stays valid)
    const uint8_t* tpool = ti + T.off_abar;
    uint8_t* vpool = img + L.off_bvar;
    auto put = [e](uint8_t* base, size_t i, double v) {
        if (e == 8) reinterpret_cast<double*>(base)[i] = v;
        else reinterpret_cast<float*>(base)[i] = (float)v;
    };
    for (int64_t t = 0; t < NT; ++t) {
        if (var_off[t] < 0) continue;
        const int4 tr = T.trec[t];
        for (int64_t sc = 0; sc < NSC; ++sc) {
            const size_t dst = (size_t)sc * VP + var_off[t];
            std::memcpy(vpool + e * dst, tpool + e * (size_t)tr.y, e * (size_t)tr.z);
            for (int32_t j = T.tsub_ptr[t]; j < T.tsub_ptr[t + 1]; ++j) {
                const int64_t s = T.tsub_s[j];
                const int32_t v = bo.vidx[s];
                if (v < 0) continue;
                const int ns = P.n_s[s];
                const double* A = &bo.abar[(size_t)sc * bo.VA + bo.va_off[v]];
                const double* b = &bo.bbar[(size_t)sc * bo.VB + bo.vb_off[v]];
                const size_t blk = dst + T.tsub_poff[j];
                bool has_b = false;
                for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) has_b |= P.bbar[k] != 0.0;
                for (int r = 0; r < ns; ++r)
                    for (int k = r; k < ns; ++k) put(vpool, blk + r * ns - r * (r - 1) / 2 + (k - r), A[(size_t)r * ns + k]);
                if (has_b)
                    for (int r = 0; r < ns; ++r) put(vpool, blk + ns * (ns + 1) / 2 + r, b[r]);
            }
        }
    }
    (void)opt;
    return LOPF_OK;
}

}  // namespace lopf

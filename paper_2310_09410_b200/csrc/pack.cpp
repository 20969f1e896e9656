// Device layout of the streaming kernel.
//
// Subsystems are packed into warp TASKS: a task owns 32*R row SLOTS (lane l handles slots
// l, l+32, ...).  Tasks follow the depth-first order of the feeder (gather locality, see
// pack_streaming) and are homogeneous in n_s, so a task's column loop has no padding.  The operator
// pool stores, per task, Abar columns k = 0..kmax-1 as 32*R consecutive doubles (slot-major inside
// a column), so every column read of a warp is one coalesced 256-byte request per half.  Per-slot
// metadata, b-bar and the iterate (x_s, lambda, u ping-pong) are slot-indexed arrays; globals keep
// {c/rho, 1/nu, lo, hi} as one 32-byte record.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

#include <vector_functions.h>

#include "internal.h"

namespace lopf {

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

lopf_status pack_streaming(const Net& N, const Canon& P, const lopf_options& opt, int max_grid, Layout& L,
                           std::string& err, const PartSpec* part, int32_t rank) {
    L = Layout();
    L.kernel = 1;
    // element size of operators / iterate / globals (fp32 variant: reading F1); a stage holds kPackBudget
    // operator entries of either type; bulk copies stay 16-byte aligned
    const int esz = opt.precision == 32 ? 4 : 8;
    const int budget = kPackBudget, al = 16 / esz;
    L.esz = esz;
    // partitioned mode: only this rank's subsystems; remote copies its globals read become ghost slots
    auto local_sub = [&](int64_t s) { return !part || part->sub_owner[s] == rank; };
    // ---- tasks ---------------------------------------------------------------------------------
    // Subsystems are taken in depth-first order of the feeder (neighbouring subsystems share
    // globals, so the u values a task gathers were fetched into L2 by a task that ran moments
    // earlier) and packed greedily into PACKED tasks of up to 32 * kTaskHalves slots whose operator
    // blocks (upper-triangular Abar of each subsystem, then its b-bar if nonzero), concatenated, fit
    // the per-warp SMEM stage (kPackBudget doubles): the kernel bulk-copies (TMA) the block and the
    // task's per-slot inputs into SMEM one task ahead.  A subsystem whose block alone exceeds the
    // stage is a DIRECT packed task of its own (block read from HBM); n_s > 63 (the S = 1 path) gets
    // a FULL task: Abar as kmax columns of 32*R doubles.
    struct T { int R, kmax, plen, used; bool packed, direct; std::vector<int64_t> subs; std::vector<int> base, poff; };
    std::vector<T> tasks;
    for (int64_t s = 0; s < P.S; ++s)
        if (P.n_s[s] > 256) {
            err = "subsystem " + std::to_string(s) + " has n_s = " + std::to_string(P.n_s[s]) +
                  " > 256 (unsupported by the warp-task layout; the S = 1 path is for small feeders)";
            return LOPF_E_ARG;
        }
    auto has_bbar = [&](int64_t s) {
        for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k)
            if (P.bbar[k] != 0.0) return true;
        return false;
    };
    {
        T cur{1, 0, 0, 0, true, false, {}, {}, {}};
        int fill = 0;
        auto close = [&] {
            if (!cur.subs.empty()) {
                cur.R = fill > 32 ? 2 : 1;
                cur.used = (fill + 3) & ~3;                      // slots the bulk copies move (16-byte multiples)
                cur.plen = (cur.plen + al - 1) & ~(al - 1);
                tasks.push_back(std::move(cur));
            }
            cur = T{1, 0, 0, 0, true, false, {}, {}, {}};
            fill = 0;
        };
        for (int64_t s : dfs_order(N, P)) {
            const int ns = P.n_s[s];
            if (ns == 0 || !local_sub(s)) continue;
            const int ps = ns * (ns + 1) / 2 + (has_bbar(s) ? ns : 0);   // triangle (+ b-bar)
            if (ns > 63) {                                       // full task (S = 1 path)
                close();
                const int R = ns <= 64 ? 2 : ns <= 128 ? 4 : 8;
                tasks.push_back(T{R, ns, 0, 32 * R, false, false, {s}, {0}, {0}});
                continue;
            }
            if (ps > budget) {                                   // block read from HBM, task of its own
                close();
                tasks.push_back(T{ns <= 32 ? 1 : 2, ns, (ps + al - 1) & ~(al - 1), (ns + 3) & ~3, true, true, {s}, {0}, {0}});
                continue;
            }
            if (fill + ns > 32 * kTaskHalves || cur.plen + ps > budget) close();
            cur.subs.push_back(s);
            cur.base.push_back(fill);                            // rows may straddle the two halves
            cur.poff.push_back(cur.plen);
            cur.kmax = std::max(cur.kmax, ns);
            cur.plen += ps;
            fill += ns;
        }
        close();
    }
    L.n_tasks = (int64_t)tasks.size();
    std::vector<int4> trec(L.n_tasks);
    int64_t slots = 0, pool = 0;
    for (int64_t t = 0; t < L.n_tasks; ++t) {
        const T& k = tasks[t];
        trec[t] = k.packed ? make_int4((int)slots, (int)pool, k.plen,
                                       k.R | kTaskPacked | (k.direct ? kTaskDirect : 0) | (k.kmax << kTaskKmaxShift) |
                                           (k.used << kTaskUsedShift))
                           : make_int4((int)slots, (int)pool, k.kmax, k.R);
        L.rmax = std::max(L.rmax, k.R);
        slots += 32 * k.R;
        pool += k.packed ? (int64_t)k.plen : (int64_t)k.kmax * 32 * k.R;
    }
    // ghost slots (partitioned mode): remote copies of the globals this rank's copies belong to, in
    // canonical (global, copy) order; their u arrives through the exchange buffer every sweep
    std::vector<int64_t> ghosts;
    if (part) {
        std::vector<char> seen(P.n, 0);
        std::vector<int32_t> gl;
        for (int64_t s = 0; s < P.S; ++s)
            if (local_sub(s))
                for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k)
                    if (!seen[P.copy_global[k]]) { seen[P.copy_global[k]] = 1; gl.push_back(P.copy_global[k]); }
        std::sort(gl.begin(), gl.end());
        for (int32_t g : gl)
            for (int64_t q = P.seg_ptr[g]; q < P.seg_ptr[g + 1]; ++q)
                if (part->copy_owner[P.seg_copy[q]] != rank) ghosts.push_back(P.seg_copy[q]);
        L.part = 1;
        L.rank = rank;
        L.world = part->world;
        L.n_bnd = part->n_bnd;
        L.n_imp = (int32_t)ghosts.size();
        L.ghost0 = (int32_t)slots;
        slots += (int64_t)ghosts.size();
    }
    if (slots > INT32_MAX || pool > INT32_MAX) { err = "problem too large for 32-bit slot / pool offsets"; return LOPF_E_ARG; }
    L.n_slots = slots;
    L.abar_doubles = pool;
    L.max_grid = max_grid;
    L.trace_cap = opt.trace_cap > 0 ? opt.trace_cap : 4096;

    // ---- objective terms (c != 0) -----------------------------------------------------------------
    std::vector<int32_t> obj_idx;
    std::vector<double> obj_c;
    for (int64_t i = 0; i < P.n; ++i)          // partitioned: the globals whose first copy is local
        if (P.c[i] != 0.0 && (!part || part->copy_owner[P.seg_copy[P.seg_ptr[i]]] == rank)) {
            obj_idx.push_back((int32_t)i);
            obj_c.push_back(P.c[i]);
        }
    L.n_obj = (int64_t)obj_idx.size();

    // ---- arena offsets --------------------------------------------------------------------------------
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align256(o + std::max<size_t>(bytes, 1)); return r; };
    const size_t NS = (size_t)slots, NG = (size_t)P.n, NC = (size_t)P.nc;
    L.off_tasks = take(sizeof(int4) * L.n_tasks);
    L.off_meta = take(sizeof(SlotMeta) * NS);
    L.off_bbar = take(esz * NS);
    L.off_xl = take(esz * NS);
    L.off_lam = take(esz * NS);
    L.off_u0 = take(esz * NS);
    L.off_u1 = take(esz * NS);
    L.off_x0 = take(esz * NS);
    L.off_gpar = take(2 * esz * NG);
    L.off_gcost = take(esz * NG);
    L.off_segptr = take(4 * (NG + 1));
    L.off_segslot = take(4 * NC);
    L.off_x = take(esz * NG);
    L.off_abar = take(esz * (size_t)pool);
    L.off_partial = take(8 * 8 * (size_t)max_grid);
    L.off_ctrl = take(sizeof(DevCtrl));
    L.off_trace = take(8 * 5 * (size_t)L.trace_cap);
    L.off_objidx = take(4 * obj_idx.size());
    L.off_objc = take(8 * obj_c.size());
    if (part) {
        L.off_sexp = take(4 * NS);
        L.off_imp = take(4 * ghosts.size());
        L.off_xbuf = take(8 * ((size_t)part->n_bnd + 8 * (size_t)part->world));       // host-driven (NCCL) exchange
        L.off_xent = take(16 * 2 * ((size_t)part->n_bnd + 8 * (size_t)part->world));  // p2p tagged entries [2 parities]
        L.off_peer = take(8 * (size_t)part->world);                                   // p2p: every rank's entry buffer
        L.off_parr = take(sizeof(DevProblem) * (size_t)part->world);                  // p2p launch argument(s)
    }
    L.bytes = o;
    L.image.assign(L.bytes, 0);
    uint8_t* img = L.image.data();
    auto at = [&](size_t off) { return img + off; };

    std::memcpy(at(L.off_tasks), trec.data(), sizeof(int4) * trec.size());
    SlotMeta* meta = (SlotMeta*)at(L.off_meta);
    std::vector<int32_t> info(NS, 0), gs(NS, -1);
    std::vector<int4> nbr(NS, make_int4(0, 0, 0, 0));
    // (T) arrays: values computed in fp64, stored as T (fp32: each rounded once to nearest)
    auto put = [esz](uint8_t* base, size_t i, double v) {
        if (esz == 8) reinterpret_cast<double*>(base)[i] = v;
        else reinterpret_cast<float*>(base)[i] = (float)v;
    };
    uint8_t* bbar = at(L.off_bbar);
    uint8_t* abar = at(L.off_abar);

    L.slot_of_copy.assign(NC, -1);
    L.trec = trec;
    L.tsub_ptr.assign(1, 0);
    for (int64_t t = 0; t < L.n_tasks; ++t) {
        for (size_t j = 0; j < tasks[t].subs.size(); ++j) {
            L.tsub_s.push_back((int32_t)tasks[t].subs[j]);
            L.tsub_poff.push_back(tasks[t].poff[j]);
        }
        L.tsub_ptr.push_back((int32_t)L.tsub_s.size());
    }
    for (int64_t t = 0; t < L.n_tasks; ++t) {
        const T& tk = tasks[t];
        const int P32 = 32 * tk.R;
        for (size_t j = 0; j < tk.subs.size(); ++j) {
            const int64_t s = tk.subs[j];
            const int ns = P.n_s[s], base = tk.base[j];
            const double* Ab = &P.abar[P.abar_ptr[s]];
            const bool has_b = has_bbar(s);
            for (int r = 0; r < ns; ++r) {
                const int64_t slot = trec[t].x + base + r;
                const int64_t copy = P.sub_ptr[s] + r;
                L.slot_of_copy[copy] = (int32_t)slot;
                info[slot] = base | kInfoValid | (has_b ? kInfoBbar : 0) | (ns << kInfoNsShift) |
                             (tk.packed ? tk.poff[j] << kInfoPoffShift : 0);
                gs[slot] = P.copy_global[copy];
                put(bbar, slot, P.bbar[copy]);
                if (tk.packed) {                  // upper triangle, row-major: (r, k >= r); then b-bar
                    const size_t dst = (size_t)trec[t].y + tk.poff[j];
                    for (int k = r; k < ns; ++k) put(abar, dst + r * ns - r * (r - 1) / 2 + (k - r), Ab[(size_t)r * ns + k]);
                    if (has_b) put(abar, dst + ns * (ns + 1) / 2 + r, P.bbar[copy]);
                } else {                          // lane (slot) r computes row r: sum_k Abar[r][k] d[k]
                    for (int k = 0; k < ns; ++k)
                        put(abar, (size_t)trec[t].y + (size_t)k * P32 + base + r, Ab[(size_t)r * ns + k]);
                }
            }
        }
    }
    for (size_t i = 0; i < ghosts.size(); ++i) L.slot_of_copy[ghosts[i]] = L.ghost0 + (int32_t)i;
    if (part) {
        int32_t* sexp = (int32_t*)at(L.off_sexp);
        int32_t* imp = (int32_t*)at(L.off_imp);
        for (size_t i = 0; i < NS; ++i) sexp[i] = -1;
        for (size_t i = 0; i < ghosts.size(); ++i) imp[i] = part->bidx[ghosts[i]];
        for (int64_t k = 0; k < P.nc; ++k)
            if (part->copy_owner[k] == rank && part->bidx[k] >= 0) {
                info[L.slot_of_copy[k]] |= kInfoExport;
                sexp[L.slot_of_copy[k]] = part->bidx[k];
            }
    }
    // segments: inline neighbour slots (nu <= 4) + CSR fallback; first-copy flag
    int32_t* segptr = (int32_t*)at(L.off_segptr);
    int32_t* segslot = (int32_t*)at(L.off_segslot);
    for (int64_t i = 0; i <= P.n; ++i) segptr[i] = (int32_t)P.seg_ptr[i];
    for (int64_t q = 0; q < P.nc; ++q) segslot[q] = L.slot_of_copy[P.seg_copy[q]];
    for (int64_t k = 0; k < P.nc; ++k) {
        const int32_t slot = L.slot_of_copy[k];
        if (slot < 0 || (part && part->copy_owner[k] != rank)) continue;   // not computed here
        const int32_t g = P.copy_global[k];
        const int64_t s0 = P.seg_ptr[g], nu = P.seg_ptr[g + 1] - s0;
        info[slot] |= (int)(std::min<int64_t>(nu, 15) << kInfoNuShift);
        if (P.seg_copy[s0] == k) info[slot] |= kInfoFirst;
        if (P.c[g] != 0.0) info[slot] |= kInfoCost;
        if (nu <= 4) {
            info[slot] |= kInfoInline;
            int v[4] = {0, 0, 0, 0};
            for (int64_t j = 0; j < nu; ++j) v[j] = segslot[s0 + j];
            nbr[slot] = make_int4(v[0], v[1], v[2], v[3]);
        }
    }
    for (size_t i = 0; i < NS; ++i)
        meta[i] = SlotMeta{make_int2(nbr[i].x, nbr[i].y), make_int2(nbr[i].z, nbr[i].w), info[i], gs[i]};
    uint8_t* gbnd = at(L.off_gpar);                   // {lo, hi} pairs (IEEE +-inf kept in fp32 too)
    uint8_t* gcost = at(L.off_gcost);
    for (int64_t i = 0; i < P.n; ++i) {
        put(gbnd, 2 * i, P.lo[i]);
        put(gbnd, 2 * i + 1, P.hi[i]);
        put(gcost, i, opt.adapt_every > 0 ? P.c[i] : P.c[i] / opt.rho);   // adaptive rho: c, divided on device
    }
    std::memcpy(at(L.off_objidx), obj_idx.data(), 4 * obj_idx.size());
    std::memcpy(at(L.off_objc), obj_c.data(), 8 * obj_c.size());
    init_state_image(P, L);
    reinterpret_cast<DevCtrl*>(L.image.data() + L.off_ctrl)->rho_cur = opt.rho;   // the penalty in force at bind
    return LOPF_OK;
}

// Initial iterate (Algorithm 1 line 1): x_s = x0, lambda = 0, u = x_s - lambda/rho = x0.
void init_state_image(const Canon& P, Layout& L) {
    uint8_t* img = L.image.data();
    const size_t e = (size_t)L.esz;
    for (size_t off : {L.off_xl, L.off_lam, L.off_u0, L.off_u1, L.off_x0}) std::memset(img + off, 0, e * L.n_slots);
    for (int64_t k = 0; k < P.nc; ++k) {
        const int32_t s = L.slot_of_copy[k];
        if (s < 0) continue;                                   // (partitioned: own copies and ghosts)
        for (size_t off : {L.off_xl, L.off_u0, L.off_x0}) {
            if (e == 8) reinterpret_cast<double*>(img + off)[s] = P.x0[k];
            else reinterpret_cast<float*>(img + off)[s] = (float)P.x0[k];
        }
    }
    std::memset(img + L.off_ctrl, 0, sizeof(DevCtrl));
}

}  // namespace lopf

// Device layout of the batch mode (config 4; kernel in batch.cu).
//
// Lane = scenario: scenarios form groups of 32 and every per-scenario array is [group][entry][32].
// Rows are the copies in depth-first subsystem order (neighbouring subsystems share globals, so the
// u lines a subsystem gathers were touched moments earlier).  Shared by all scenarios: per-row records
// (global, first-copy flag, the segment's rows in canonical copy order), per-subsystem records, the
// {c/rho, lo, hi, 1/nu} of every global and the dense Abar of every subsystem without a load.  Per
// scenario: the packed upper triangle and b-bar of every subsystem that holds a load (its A_s depends on
// the load level through VDLM-1/2), and the iterate.  Tasks are depth-first runs of
// whole subsystems of about kBatchTaskRows (fp32: kBatchTaskRows32) rows; a work item is (group, task).
#include <algorithm>
#include <cstring>

#include "internal.h"

namespace lopf {

static size_t a256b(size_t x) { return (x + 255) & ~(size_t)255; }

lopf_status pack_batch(const Net& N, const Canon& P, const BatchOps& bo, const lopf_options& opt, Layout& L,
                       std::string& err) {
    L = Layout();
    L.kernel = 3;
    const int64_t E = opt.precision == 32 ? 4 : 8;            // (T) element size (fp32 variant: reading F1)
    L.esz = (int32_t)E;
    const bool vqb = batch_vqb((int)E);                        // per-scenario operator layout (internal.h)
    int ns_max = 1;
    for (int64_t s = 0; s < P.S; ++s) ns_max = std::max(ns_max, P.n_s[s]);
    if (ns_max > 255) { err = "batch mode supports n_s <= 255"; return LOPF_E_ARG; }
    const int32_t NSC = bo.n_scen, NG = (NSC + 31) / 32;
    const std::vector<int64_t> order = dfs_order(N, P);

    // ---- rows (copies in DFS subsystem order), subsystems, segments ---------------------------------
    std::vector<int32_t> row_of_copy(P.nc, -1);
    int32_t nr = 0;
    for (int64_t s : order)
        for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) row_of_copy[k] = nr++;
    std::vector<BRow> rows(nr);
    std::vector<int32_t> seg_rows;
    for (int64_t k = 0; k < P.nc; ++k) {
        const int32_t g = P.copy_global[k];
        const int64_t q0 = P.seg_ptr[g], q1 = P.seg_ptr[g + 1], nu = q1 - q0;
        BRow& R = rows[row_of_copy[k]];
        R.g = g;
        R.info = (P.seg_copy[q0] == k ? kBFirst : 0);
        R.n0 = R.n1 = R.n2 = R.n3 = 0;
        if (nu <= 4) {
            R.info |= kBInline | (int32_t)(nu << kBNuShift);
            int32_t* n = &R.n0;
            for (int64_t q = q0; q < q1; ++q) n[q - q0] = row_of_copy[P.seg_copy[q]];
        } else {
            R.n0 = (int32_t)seg_rows.size();
            R.n1 = (int32_t)nu;
            for (int64_t q = q0; q < q1; ++q) seg_rows.push_back(row_of_copy[P.seg_copy[q]]);
        }
    }
    std::vector<BSub> subs;
    std::vector<double> spool;                                     // dense Abar of shared subsystems
    std::vector<int64_t> var_op(P.S, -1);
    int64_t ve = 0;
    std::vector<char> has_b(P.S, 0);
    for (int64_t s = 0; s < P.S; ++s)
        for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) has_b[s] |= P.bbar[k] != 0.0;
    int32_t r0 = 0;
    for (int64_t s : order) {
        const int ns = P.n_s[s];
        BSub b{r0, ns, 0, 0};
        const int nq = (ns + 3) / 4, nsp = 4 * nq;
        if (bo.vidx[s] >= 0) {
            b.flags = kBVar | kBBbar;
            b.op = (int32_t)ve;
            var_op[s] = ve;
            ve += batch_var_entries(ns, vqb) + ns;
        } else {
            if (has_b[s]) { err = "batch mode: a subsystem without a load has a nonzero b-bar"; return LOPF_E_ARG; }
            // row quads, each [k][4] over the padded width (zero rows and columns past n_s): the four rows'
            // entries of one column are one 4-wide uniform load
            b.op = (int32_t)spool.size();
            const double* A = &P.abar[P.abar_ptr[s]];
            for (int q = 0; q < nq; ++q)
                for (int k = 0; k < nsp; ++k)
                    for (int i = 0; i < 4; ++i) {
                        const int r = 4 * q + i;
                        spool.push_back(r < ns && k < ns ? A[(size_t)r * ns + k] : 0.0);
                    }
        }
        subs.push_back(b);
        r0 += ns;
    }
    if ((int64_t)NG * ve * 32 * E > ((int64_t)1 << 40)) { err = "batch: per-scenario operators too large"; return LOPF_E_ARG; }
    // tasks: DFS runs of whole subsystems of ~trows rows; cost weight = consensus rows + the
    // mat-vec entries (a per-scenario operator entry is a coalesced line, a shared one a uniform load)
    std::vector<BTask> tasks;
    const int trows = E == 8 ? kBatchTaskRows : kBatchTaskRows32;
    std::vector<long long> wpre(1, 0);
    for (size_t i = 0; i < subs.size();) {
        BTask t{(int32_t)i, (int32_t)i, subs[i].row0, subs[i].row0, -1, -1, {0, 0}};
        long long w = 0;
        while (i < subs.size() && (t.row1 - t.row0 < trows || t.sub1 == t.sub0)) {
            const long long ns = subs[i].ns;
            w += 16 + 12 * ns + ns * ns * ((subs[i].flags & kBVar) ? 2 : 1);
            t.row1 += subs[i].ns;
            if (subs[i].flags & kBVar) {                           // var entries are assigned in DFS order
                const int32_t e1 = subs[i].op + (int32_t)(batch_var_entries((int)ns, vqb) + ns);
                if (t.vop0 < 0) t.vop0 = subs[i].op;
                t.vop1 = e1;
            }
            t.sub1 = (int32_t)++i;
        }
        if (t.vop0 < 0) t.vop0 = t.vop1 = 0;
        tasks.push_back(t);
        wpre.push_back(wpre.back() + w);
    }
    const int64_t NT = (int64_t)tasks.size();
    int32_t trmax = 1;
    for (const BTask& t : tasks) trmax = std::max(trmax, t.row1 - t.row0);
    std::vector<int32_t> torder(NT);
    for (int64_t t = 0; t < NT; ++t) torder[t] = (int32_t)t;
    std::stable_sort(torder.begin(), torder.end(),
                     [&](int32_t a, int32_t b) { return wpre[a + 1] - wpre[a] > wpre[b + 1] - wpre[b]; });

    // unit (subsystem, row quad) -> team warp: longest processing time first on a cost model of the loads
    // a unit issues (a per-scenario operator row quad reads nq 4 x 4 blocks of coalesced lines, a shared one
    // nq 4 x 4 uniform loads) plus its finish; each warp then runs its units in ascending order
    const int TW = kBatchTeamWarps;
    std::vector<int32_t> tunp(1, 0), tun;
    for (const BTask& t : tasks) {
        std::vector<std::pair<long long, int32_t>> units;             // (cost, code)
        for (int32_t s = t.sub0; s < t.sub1; ++s) {
            const int nq = (subs[s].ns + 3) / 4;
            const long long c = ((subs[s].flags & kBVar) ? 16LL : 4LL) * nq + 12;
            for (int q = 0; q < nq; ++q) units.push_back({c, ((s - t.sub0) << 8) | q});
        }
        std::vector<std::vector<int32_t>> per(TW);
        std::vector<long long> load(TW, 0);
        std::vector<size_t> ord(units.size());
        for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
        if (LOPF_BATCH_LPT)
            std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return units[a].first > units[b].first; });
        for (size_t k = 0; k < ord.size(); ++k) {
            int w = (int)(k % TW);                                     // round robin (LOPF_BATCH_LPT = 0)
            if (LOPF_BATCH_LPT) w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
            per[w].push_back(units[ord[k]].second);
            load[w] += units[ord[k]].first;
        }
        for (int w = 0; w < TW; ++w) {
            std::sort(per[w].begin(), per[w].end());
            tun.insert(tun.end(), per[w].begin(), per[w].end());
            tunp.push_back((int32_t)tun.size());
        }
    }

    // ---- arena -----------------------------------------------------------------------------------
    std::vector<int32_t> obj_idx;
    std::vector<double> obj_c;
    for (int64_t i = 0; i < P.n; ++i)
        if (P.c[i] != 0.0) { obj_idx.push_back((int32_t)i); obj_c.push_back(P.c[i]); }
    L.n_scen = NSC;
    L.n_grp = NG;
    L.ns_max = ns_max;
    L.task_rows_max = trmax;
    L.n_rows = nr;
    L.n_bsub = (int32_t)subs.size();
    L.ve = (int32_t)ve;
    L.n_tasks = NT;
    L.n_slots = nr;
    L.n_obj = (int64_t)obj_idx.size();
    L.abar_doubles = (int64_t)spool.size() + ve;
    L.slot_of_copy = row_of_copy;
    L.max_grid = 4096;
    L.trace_cap = 1;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = a256b(o + std::max<size_t>(bytes, 1)); return r; };
    // inputs (uploaded by bind)
    L.off_brow = take(sizeof(BRow) * (size_t)nr);
    L.off_bsub = take(sizeof(BSub) * subs.size());
    L.off_btask = take(sizeof(BTask) * (size_t)NT);
    L.off_bseg = take(4 * seg_rows.size());
    L.off_gpar = take(4 * E * (size_t)P.n);
    L.off_bspool = take(E * spool.size());
    L.off_x0 = take(E * (size_t)nr);
    L.off_bwpre = take(8 * (size_t)(NT + 1));
    L.off_btorder = take(4 * (size_t)NT);
    L.off_btunp = take(4 * tunp.size());
    L.off_btun = take(4 * tun.size());
    L.off_objidx = take(4 * obj_idx.size());
    L.off_objc = take(8 * obj_c.size());
    L.off_bvpool = take(E * (size_t)NG * ve * 32);
    L.image_bytes = o;
    // device state (initialised by the reset kernel)
    const size_t per = E * (size_t)NG * nr * 32;
    L.off_xl = take(per);
    L.off_lam = take(per);
    L.off_u0 = take(per);
    L.off_u1 = take(per);
    L.off_x = take(E * (size_t)NG * P.n * 32);
    L.off_bpart = take(8 * 160 * (size_t)NG * NT);
    L.off_bres = take(sizeof(ScenResult) * (size_t)NSC);
    L.off_bstop = take(4 * (size_t)NSC);
    L.off_bgact = take(4 * 2 * (size_t)NG);
    L.off_bcnt = take(8 * 4);
    L.off_ctrl = take(sizeof(DevCtrl));
    L.off_bstage = take(8 * (2 * (size_t)nr + (size_t)P.n));
    L.off_trace = take(8 * 5);
    L.bytes = o;
    L.image.assign(L.image_bytes, 0);
    uint8_t* img = L.image.data();
    auto put = [E](uint8_t* base, size_t i, double v) {
        if (E == 8) reinterpret_cast<double*>(base)[i] = v;
        else reinterpret_cast<float*>(base)[i] = (float)v;
    };
    std::memcpy(img + L.off_brow, rows.data(), sizeof(BRow) * (size_t)nr);
    std::memcpy(img + L.off_bsub, subs.data(), sizeof(BSub) * subs.size());
    std::memcpy(img + L.off_btask, tasks.data(), sizeof(BTask) * (size_t)NT);
    std::memcpy(img + L.off_bseg, seg_rows.data(), 4 * seg_rows.size());
    for (int64_t g = 0; g < P.n; ++g) {
        const double nu = (double)(P.seg_ptr[g + 1] - P.seg_ptr[g]);
        put(img + L.off_gpar, 4 * g, P.c[g] / opt.rho);
        put(img + L.off_gpar, 4 * g + 1, P.lo[g]);
        put(img + L.off_gpar, 4 * g + 2, P.hi[g]);
        put(img + L.off_gpar, 4 * g + 3, 1.0 / nu);
    }
    for (size_t i = 0; i < spool.size(); ++i) put(img + L.off_bspool, i, spool[i]);
    for (int64_t k = 0; k < P.nc; ++k) put(img + L.off_x0, row_of_copy[k], P.x0[k]);
    std::memcpy(img + L.off_bwpre, wpre.data(), 8 * wpre.size());
    std::memcpy(img + L.off_btorder, torder.data(), 4 * torder.size());
    std::memcpy(img + L.off_btunp, tunp.data(), 4 * tunp.size());
    std::memcpy(img + L.off_btun, tun.data(), 4 * tun.size());
    std::memcpy(img + L.off_objidx, obj_idx.data(), 4 * obj_idx.size());
    std::memcpy(img + L.off_objc, obj_c.data(), 8 * obj_c.size());
    // per-scenario operators: [group][entry][lane]; padding lanes of the last group stay zero
    uint8_t* vp = img + L.off_bvpool;
    for (int64_t v = 0; v < (int64_t)bo.vsub.size(); ++v) {
        const int64_t s = bo.vsub[v];
        const int ns = P.n_s[s];
        const int64_t op = var_op[s];
        for (int32_t sc = 0; sc < NSC; ++sc) {
            const double* A = &bo.abar[(size_t)sc * bo.VA + bo.va_off[v]];
            const double* b = &bo.bbar[(size_t)sc * bo.VB + bo.vb_off[v]];
            const size_t base = ((size_t)(sc >> 5) * ve + op) * 32 + (sc & 31);
            // quad-block upper layout: block q holds, for each column k in [4q, nsp), the entries of rows
            // 4q..4q+3 (zero past n_s); then b-bar
            const int nq = (ns + 3) / 4, nsp = 4 * nq;
            int64_t e = 0;
            if (!vqb)
                for (int i = 0; i < ns; ++i)
                    for (int j = i; j < ns; ++j, ++e) put(vp, base + 32 * (size_t)e, A[(size_t)i * ns + j]);
            else
            for (int q = 0; q < nq; ++q)
                for (int k = 4 * q; k < nsp; ++k)
                    for (int i = 0; i < 4; ++i, ++e) {
                        const int r = 4 * q + i;
                        put(vp, base + 32 * (size_t)e, r < ns && k < ns ? A[(size_t)r * ns + k] : 0.0);
                    }
            for (int i = 0; i < ns; ++i, ++e) put(vp, base + 32 * (size_t)e, b[i]);
        }
    }
    return LOPF_OK;
}

}  // namespace lopf

// Device layout of the SMEM-resident kernel.
//
// 1. Subsystems are ordered by a depth-first walk of the feeder from the root (a bus, then each of
//    its lines followed by the subtree behind it), so a contiguous run of that order is a
//    connected piece of the network.
// 2. The order is cut into G chunks of balanced shared-memory footprint (<= kResSmemBudget each);
//    chunk c is owned by CTA c for the whole solve.
// 3. Inside a chunk, subsystems are bin-packed (first fit decreasing) into 32-row warp tasks
//    (n_s > 32: one subsystem per 64-row task); each Abar_s is stored compactly (n_s x n_s, exactly
//    sum n_s^2 doubles per chunk) and lane r of subsystem s reads Abar_s[k][r] at base_s + k n_s + r.
// 4. Every global variable with a copy in the chunk gets a local index and a segment list in
//    canonical copy order whose entries are local slots (u in SMEM) or, for copies owned by other
//    CTAs, indices into the global exchange buffer (only boundary copies are exchanged).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>

#include <vector_functions.h>

#include "internal.h"

namespace lopf {

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }
static int32_t a16(int64_t x) { return (int32_t)((x + 15) & ~(int64_t)15); }

// depth-first order of the subsystems from the root bus
std::vector<int64_t> dfs_order(const Net& N, const Canon& P) {
    std::vector<int64_t> order;
    order.reserve(P.S);
    if (P.S == 1) { order.push_back(0); return order; }
    std::vector<int64_t> sub_of_bus(N.n_bus, -1), sub_of_line(N.n_line, -1);
    for (int64_t s = 0; s < P.S; ++s) {
        if (P.kind[s] == BUS) sub_of_bus[P.comp[s]] = s;
        else {
            sub_of_line[P.comp[s]] = s;
            if (P.kind[s] == LEAF) sub_of_bus[P.leaf[s]] = s;
        }
    }
    std::vector<std::vector<int32_t>> adj(N.n_bus);
    for (int e = 0; e < N.n_line; ++e) { adj[N.line_from[e]].push_back(e); adj[N.line_to[e]].push_back(e); }
    for (auto& a : adj) std::sort(a.begin(), a.end());
    std::vector<char> emitted(P.S, 0), seen(N.n_bus, 0);
    auto emit = [&](int64_t s) { if (s >= 0 && !emitted[s]) { emitted[s] = 1; order.push_back(s); } };
    auto walk = [&](int root) {
        std::vector<std::pair<int, size_t>> st;
        st.push_back({root, 0});
        seen[root] = 1;
        emit(sub_of_bus[root]);
        while (!st.empty()) {
            auto& [b, k] = st.back();
            if (k >= adj[b].size()) { st.pop_back(); continue; }
            const int e = adj[b][k++];
            const int o = N.line_from[e] == b ? N.line_to[e] : N.line_from[e];
            emit(sub_of_line[e]);
            if (!seen[o]) {
                seen[o] = 1;
                emit(sub_of_bus[o]);
                st.push_back({o, 0});
            }
        }
    };
    if (N.n_bus > 0) walk(N.root);
    for (int b = 0; b < N.n_bus; ++b)
        if (!seen[b]) walk(b);
    for (int64_t s = 0; s < P.S; ++s) emit(s);
    return order;
}

namespace {
struct Chunk {
    std::vector<int64_t> subs;
};
struct TaskR {
    int R, kmax;
    std::vector<int64_t> subs;
};

// 64-row tasks (R = 2: lane l handles rows l and l + 32), subsystems first-fit-decreasing by n_s
std::vector<TaskR> make_tasks(const Canon& P, const std::vector<int64_t>& subs) {
    std::vector<int64_t> v;
    for (int64_t s : subs)
        if (P.n_s[s] > 0) v.push_back(s);
    std::stable_sort(v.begin(), v.end(), [&](int64_t a, int64_t b) { return P.n_s[a] > P.n_s[b]; });
    std::vector<TaskR> tasks;
    std::vector<int> room;
    for (int64_t s : v) {
        const int ns = P.n_s[s];
        size_t t = 0;
        for (; t < tasks.size(); ++t)
            if (room[t] >= ns) break;
        if (t == tasks.size()) { tasks.push_back({2, 0, {}}); room.push_back(64); }
        tasks[t].subs.push_back(s);
        tasks[t].kmax = std::max(tasks[t].kmax, ns);
        room[t] -= ns;
    }
    return tasks;
}

// Use the chunk's idle worker warps: the most expensive 64-row tasks whose subsystems fit two 32-row
// halves become two R = 1 tasks (lane l: row l only) run by two warps.  The period of the kernel is set by
// the slowest warp of the slowest CTA (tools/res_timeline2.py: a warp's cycles ~ 45 per tile column + 90
// per boundary read, issue-bound), so halving the longest tasks shortens the critical path.  The split
// never grows the SMEM footprint (same slots, tiles of 32 x kmax_half <= 64 x kmax).
// A task's subsystems are re-packed first-fit-decreasing into as many 32-row tasks as the idle warps and
// the SMEM margin allow.  Measured (profiles/r01_ab_resident_split*.log): the 123 shape (G = 4) gains
// 3.43 -> 3.31 us/sweep, the 8500 shape (G = 145) loses 4.53 -> 4.73 (the extra active warps raise the
// issue contention of every warp), so it is applied to small feeders (G <= 16) only.
#ifndef LOPF_RES_SPLIT_TASKS
#define LOPF_RES_SPLIT_TASKS 1
#endif
void split_tasks(const Canon& P, std::vector<TaskR>& tasks, const std::vector<int32_t>& copy_chunk, int c,
                 int workers, int64_t smem_room, int64_t E) {
    if (!LOPF_RES_SPLIT_TASKS) return;
    auto cost = [&](const TaskR& t) {
        int64_t xr = 0;
        for (int64_t s : t.subs)
            for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) {
                const int32_t g = P.copy_global[k];
                for (int64_t q = P.seg_ptr[g]; q < P.seg_ptr[g + 1]; ++q) xr += copy_chunk[P.seg_copy[q]] != c;
            }
        return 45.0 * t.kmax + 90.0 * (double)xr;
    };
    std::vector<int> idx(tasks.size());
    std::vector<double> cs(tasks.size());
    for (size_t i = 0; i < tasks.size(); ++i) { idx[i] = (int)i; cs[i] = cost(tasks[i]); }
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return cs[a] > cs[b]; });
    int idle = workers - (int)tasks.size();
    const int64_t per_slot = 5 * E + 8;                  // bbar, x_s and lambda (two parities), sinfo, sexp
    std::vector<std::vector<TaskR>> parts(tasks.size());
    for (int i : idx) {
        if (idle <= 0) break;
        const TaskR& t = tasks[i];
        if (t.R != 2) continue;
        std::vector<TaskR> bins;                          // first fit decreasing into 32-row R = 1 tasks
        std::vector<int> room;
        bool ok = true;
        for (int64_t s : t.subs) {                        // (subs are in decreasing n_s order)
            const int ns = P.n_s[s];
            if (ns > 32) { ok = false; break; }
            size_t b = 0;
            while (b < bins.size() && room[b] < ns) ++b;
            if (b == bins.size()) { bins.push_back(TaskR{1, 0, {}}); room.push_back(32); }
            bins[b].subs.push_back(s);
            bins[b].kmax = std::max(bins[b].kmax, ns);
            room[b] -= ns;
        }
        const int extra = (int)bins.size() - 1;
        if (!ok || extra > idle) continue;
        int64_t xr_t = 0;                                 // remote-copy reads of the task: bounds the extra
        for (int64_t s : t.subs)                          // import entries of each new bin
            for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) {
                const int32_t g = P.copy_global[k];
                for (int64_t q = P.seg_ptr[g]; q < P.seg_ptr[g + 1]; ++q) xr_t += copy_chunk[P.seg_copy[q]] != c;
            }
        int64_t grow = 32 * per_slot * ((int64_t)bins.size() - 2) + 8 * xr_t * extra;   // 32 slots per R = 1 task
        for (auto& b : bins) grow += E * 32 * b.kmax;
        grow -= E * 64 * t.kmax;
        if (grow > smem_room) continue;
        smem_room -= grow;
        parts[i] = bins;
        idle -= extra;
    }
    std::vector<TaskR> out;
    for (size_t i = 0; i < tasks.size(); ++i) {
        if (parts[i].empty()) { out.push_back(tasks[i]); continue; }
        for (auto& b : parts[i]) out.push_back(b);
    }
    tasks.swap(out);
}

// exact SMEM bytes of a chunk; mirrors the blob layout built below.  Ghost slots: one per copy owned by
// another chunk of a global this chunk touches (nu - copies here); import entries: per task, the remote
// copies of the globals of its rows.
int64_t chunk_bytes(const Canon& P, const std::vector<int64_t>& subs, std::vector<int32_t>& cnt, const int64_t E) {
    auto tasks = make_tasks(P, subs);
    int64_t NS = 0, pool = 0, NG = 0, NSEG = 0, NGH = 0, NIMP = 0;
    int kpad = 0;
    for (auto& t : tasks) { NS += 64; pool += (int64_t)t.kmax * 64; kpad = std::max(kpad, t.kmax); }
    std::vector<int32_t> touched;
    for (int64_t s : subs)
        for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) {
            const int32_t g = P.copy_global[k];
            if (cnt[g]++ == 0) { ++NG; touched.push_back(g); }
        }
    for (int32_t g : touched) {
        const int64_t nu = P.seg_ptr[g + 1] - P.seg_ptr[g];
        NGH += nu - cnt[g];
        if (nu > 4) NSEG += nu;
    }
    for (auto& t : tasks) {                                      // distinct globals per task (cnt < 0: seen)
        std::vector<int32_t> seen;
        for (int64_t s : t.subs)
            for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) {
                const int32_t g = P.copy_global[k];
                if (cnt[g] < 0) continue;
                NIMP += (P.seg_ptr[g + 1] - P.seg_ptr[g]) - cnt[g];
                cnt[g] = -cnt[g];
                seen.push_back(g);
            }
        for (int32_t g : seen) cnt[g] = -cnt[g];
    }
    for (int32_t g : touched) cnt[g] = 0;
    const int64_t NT = (int64_t)tasks.size(), NX = NS + 1 + NGH;
    int64_t b = 0;
    for (int64_t sz : {E * pool, E * NS, 4 * E * NG, 16 * NT, 4 * NS, 4 * NS, 16 * NG, 8 * NG, 4 * NSEG, 8 * NIMP,
                       E * NX, E * NX, E * NX, E * NX, 2 * E * NG, E * (64 + kpad) * (kResBlock / 32)})
        b = a16(b + sz);
    return b;
}
}  // namespace

lopf_status pack_resident(const Net& N, const Canon& P, const lopf_options& opt, Layout& L, std::string& err) {
    L = Layout();
    L.kernel = 2;
    const int64_t E = opt.precision == 32 ? 4 : 8;           // element size of the SMEM state (reading F1)
    L.esz = (int32_t)E;
    const int max_ctas = opt.max_ctas > 0 ? opt.max_ctas : 148;
    for (int64_t s = 0; s < P.S; ++s)
        if (P.n_s[s] > 64) { err = "resident kernel supports n_s <= 64 (use the streaming kernel)"; return LOPF_E_ARG; }
    const std::vector<int64_t> order = dfs_order(N, P);
    std::vector<int32_t> cnt(P.n, 0);

    // ---- choose G and cut the DFS order into chunks of balanced SMEM footprint -----------------------
    std::vector<int64_t> est(P.S);
    int64_t total = 0;
    for (int64_t s = 0; s < P.S; ++s) {
        est[s] = E * P.n_s[s] * P.n_s[s] + (40 + 4 * E) * P.n_s[s];
        total += est[s];
    }
    const int warps = kResBlock / 32;
    int G = (int)std::max<int64_t>(1, (total + (kResSmemBudget * 8 / 10) - 1) / (kResSmemBudget * 8 / 10));
    {   // work heuristic: ~3 warp tasks per warp per sweep before adding CTAs is worth a bigger barrier
        int64_t approx_tasks = 0;
        std::map<int, int64_t> cnt;
        for (int64_t s = 0; s < P.S; ++s) cnt[P.n_s[s]]++;
        int64_t rows = 0;
        for (auto& [ns, c] : cnt) rows += (int64_t)ns * c;
        approx_tasks = (rows + 31) / 32;
        G = std::max<int>(G, (int)((approx_tasks + 3 * warps - 1) / (3 * warps)));
    }
    if (G > max_ctas / (E == 8 ? 2 : 4)) G = max_ctas;   // large problems: use every SM
    std::vector<Chunk> chunks;
    // span[p]: globals whose copies lie on both sides of a cut placed before DFS position p (each becomes a
    // boundary global whose copies are exchanged through L2 every sweep).  A chunk ends where span is
    // smallest within +-LOPF_RES_CUT_WINDOW of the balanced target, so cuts fall between weakly coupled
    // subsystems (a 1-phase lateral) rather than inside the 3-phase primary.
    std::vector<int64_t> span(P.S + 1, 0);
    {
        std::vector<int64_t> pos(P.S), first(P.n, P.S), last(P.n, -1);
        for (int64_t i = 0; i < P.S; ++i) pos[order[i]] = i;
        for (int64_t s = 0; s < P.S; ++s)
            for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) {
                const int32_t g = P.copy_global[k];
                first[g] = std::min(first[g], pos[s]);
                last[g] = std::max(last[g], pos[s]);
            }
        std::vector<int64_t> diff(P.S + 2, 0);
        for (int64_t g = 0; g < P.n; ++g)
            if (last[g] > first[g]) { diff[first[g] + 1] += 1; diff[last[g] + 1] -= 1; }
        int64_t run = 0;
        for (int64_t p = 0; p <= P.S; ++p) { run += diff[p]; span[p] = run; }
    }
#ifndef LOPF_RES_CUT_WINDOW
#define LOPF_RES_CUT_WINDOW 0.0           // A/B (profiles/r02_ab_resident_cut.log): 0 4.55, 0.05 4.78, 0.08 4.70, 0.15 5.18 us/sweep
#endif
    const double win = LOPF_RES_CUT_WINDOW;
    auto cut = [&](int64_t T, int64_t cap) {
        chunks.assign(1, Chunk{});
        int64_t acc = 0;
        size_t i = 0;
        while (i < order.size()) {
            // the end of this chunk: scan while the footprint stays within the window / cap
            const int64_t lo = (int64_t)(T * (1.0 - win)), hi = std::min<int64_t>((int64_t)(T * (1.0 + win)), cap);
            size_t j = i, best = i;
            int64_t a = acc, best_span = -1;
            while (j < order.size() && (a == 0 || a + est[order[j]] <= hi)) {
                a += est[order[j]];
                ++j;
                if (a >= lo && (best_span < 0 || span[j] < best_span)) { best_span = span[j]; best = j; }
            }
            if (best_span < 0 || win <= 0) best = j;           // window empty (or off): greedy end
            for (size_t q = i; q < best; ++q) chunks.back().subs.push_back(order[q]);
            if (best >= order.size()) break;
            chunks.push_back(Chunk{});
            acc = 0;
            i = best;
        }
    };
    bool done = false;
    double margin = 0.95;
    while (!done) {
        if (G > max_ctas) {
            err = "problem does not fit in the shared memory of " + std::to_string(max_ctas) + " CTAs";
            return LOPF_E_ARG;
        }
        const int64_t cap = (int64_t)(kResSmemBudget * margin);
        bool grew = false;
        for (int64_t T = (total + G - 1) / G;; T = T + T / 32 + 1) {    // smallest balanced target that fits G
            cut(T, cap);
            if ((int)chunks.size() <= G) break;
            if (T > cap) { ++G; grew = true; break; }
        }
        if (grew) continue;
        bool ok = true;
        for (auto& c : chunks)
            if (chunk_bytes(P, c.subs, cnt, E) > kResSmemBudget) { ok = false; break; }
        if (ok) done = true;
        else if (margin > 0.5) margin *= 0.95;
        else ++G;
    }
    L.G = (int32_t)chunks.size();

    // ---- copy -> chunk, exported copies -------------------------------------------------------------
    std::vector<int32_t> copy_chunk(P.nc, -1);
    for (int c = 0; c < L.G; ++c)
        for (int64_t s : chunks[c].subs)
            for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) copy_chunk[k] = c;
    std::vector<int32_t> xidx(P.nc, -1);
    int32_t n_exp = 0;
    for (int64_t g = 0; g < P.n; ++g) {
        bool multi = false;
        for (int64_t q = P.seg_ptr[g] + 1; q < P.seg_ptr[g + 1]; ++q)
            if (copy_chunk[P.seg_copy[q]] != copy_chunk[P.seg_copy[P.seg_ptr[g]]]) multi = true;
        if (multi)
            for (int64_t q = P.seg_ptr[g]; q < P.seg_ptr[g + 1]; ++q) xidx[P.seg_copy[q]] = n_exp++;
    }
    L.n_exp = n_exp;

    // ---- per-chunk blobs ------------------------------------------------------------------------------------
    struct Built {
        CtaHdr h;
        std::vector<uint8_t> blob;
        std::vector<double> x0;
    };
    std::vector<Built> B(L.G);
    L.slot_of_copy.assign(P.nc, -1);
    int32_t slot_base = 0;
    int max_smem = 0;
    std::vector<int32_t> gl_of(P.n, -1);
    for (int c = 0; c < L.G; ++c) {
        auto tasks = make_tasks(P, chunks[c].subs);
#ifndef LOPF_RES_SPLIT_MAXG
#define LOPF_RES_SPLIT_MAXG 16
#endif
        if (L.G <= LOPF_RES_SPLIT_MAXG)   // round 1: 123 shape 3.43 -> 3.31 us/sweep, 8500 shape 4.53 -> 4.73
            split_tasks(P, tasks, copy_chunk, c, kResBlock / 32 - 1,
                        kResSmemBudget - 512 - chunk_bytes(P, chunks[c].subs, cnt, E), E);
        CtaHdr& h = B[c].h;
        std::memset(&h, 0, sizeof(h));
        int64_t NS = 0, pool = 0;
        std::vector<int4> trec;
        int kpad = 0;
        for (auto& t : tasks) {                              // task tile: kmax columns x 32R rows, zero padded
            trec.push_back(make_int4((int)NS, t.kmax, (int)pool, t.R));
            NS += 32 * t.R;
            pool += (int64_t)t.kmax * 32 * t.R;
            kpad = std::max(kpad, t.kmax);
        }
        std::vector<int32_t> gl_list;
        for (size_t t = 0; t < tasks.size(); ++t)
            for (int64_t s : tasks[t].subs) {
                for (int r = 0; r < P.n_s[s]; ++r) {
                    const int32_t g = P.copy_global[P.sub_ptr[s] + r];
                    if (gl_of[g] < 0) { gl_of[g] = (int32_t)gl_list.size(); gl_list.push_back(g); }
                }
            }
        const int64_t NG = (int64_t)gl_list.size();
        if (NG >= (1 << (31 - kResGlShift))) { err = "too many globals in one CTA chunk"; return LOPF_E_ARG; }
        // own slots [0, NS), the zero slot NS, ghost slots NS + 1 + i: one per copy owned by another chunk
        // (its u imported from the exchange buffer by every task that reads it, x = u and lambda = 0)
        std::map<int32_t, int32_t> ghost;                            // remote copy -> ghost slot
        int64_t NSEG = 0;
        for (int64_t j = 0; j < NG; ++j) {
            const int32_t g = gl_list[j];
            const int64_t nu = P.seg_ptr[g + 1] - P.seg_ptr[g];
            if (nu > 255) { err = "a global with more than 255 copies (resident kernel)"; return LOPF_E_ARG; }
            if (nu > 4) NSEG += nu;
            for (int64_t p = P.seg_ptr[g]; p < P.seg_ptr[g + 1]; ++p) {
                const int32_t k = P.seg_copy[p];
                if (copy_chunk[k] != c) ghost.emplace(k, (int32_t)(NS + 1 + (int64_t)ghost.size()));
            }
        }
        const int64_t NGH = (int64_t)ghost.size(), NX = NS + 1 + NGH;
        // per task: the remote copies of the globals its rows read (each imported once per task)
        std::vector<int2> imp;
        for (size_t t = 0; t < tasks.size(); ++t) {
            const int32_t i0 = (int32_t)imp.size();
            std::vector<int32_t> seen;
            for (int64_t s : tasks[t].subs)
                for (int r = 0; r < P.n_s[s]; ++r) {
                    const int32_t g = P.copy_global[P.sub_ptr[s] + r];
                    if (std::find(seen.begin(), seen.end(), g) != seen.end()) continue;
                    seen.push_back(g);
                    for (int64_t p = P.seg_ptr[g]; p < P.seg_ptr[g + 1]; ++p) {
                        const int32_t k = P.seg_copy[p];
                        if (copy_chunk[k] != c) imp.push_back(make_int2(xidx[k], ghost.at(k)));
                    }
                }
            const int32_t n = (int32_t)imp.size() - i0;
            if (n > 255 || i0 >= (1 << 19)) { err = "too many boundary imports in one resident task"; return LOPF_E_ARG; }
            trec[t].w = tasks[t].R | (n << 4) | (i0 << 12);
        }
        const int64_t NIMP = (int64_t)imp.size();
        const int64_t NT = (int64_t)tasks.size();
        int32_t o = 0;
        h.off_abar = o;     o = a16(o + E * pool);
        h.off_bbar = o;     o = a16(o + E * NS);
        h.off_gpar = o;     o = a16(o + 4 * E * NG);
        h.off_tasks = o;    o = a16(o + 16 * NT);
        h.off_sinfo = o;    o = a16(o + 4 * NS);
        h.off_sexp = o;     o = a16(o + 4 * NS);
        h.off_grec = o;     o = a16(o + 16 * NG);                    // int4 per global: SMEM slots of 4 copies
        h.off_gxb = o;      o = a16(o + 8 * NG);                     // int2 per global: {first entry, nu} if nu > 4
        h.off_gseg = o;     o = a16(o + 4 * NSEG);
        h.off_gimp = o;     o = a16(o + 8 * NIMP);                   // int2 per import: {exchange index, ghost slot}
        h.off_xl0 = o;      o = a16(o + E * NX);
        h.off_lam0 = o;     o = a16(o + E * NX);
        h.blob_bytes = o;
        h.off_gown = o;                                              // blob only (not copied to SMEM)
        const int32_t blob_alloc = a16(o + 4 * NG);
        h.off_xl1 = o;      o = a16(o + E * NX);
        h.off_lam1 = o;     o = a16(o + E * NX);
        h.off_xout = o;     o = a16(o + 2 * E * NG);
        h.off_dst = o;      o = a16(o + E * (64 + kpad) * (kResBlock / 32));   // d staging; tail stays 0
        h.dst_stride = 64 + kpad;
        h.smem_bytes = o;
        if (h.smem_bytes > kResSmemBudget) { err = "internal: chunk exceeds the SMEM budget"; return LOPF_E_ARG; }
        h.n_tasks = (int32_t)NT; h.n_slots = (int32_t)NS; h.n_glob = (int32_t)NG; h.n_seg = (int32_t)NSEG;
        h.n_ghost = (int32_t)NGH;
        h.slot_base = slot_base;
        max_smem = std::max(max_smem, h.smem_bytes);
        std::vector<uint8_t>& blob = B[c].blob;
        blob.assign(blob_alloc, 0);
        auto put = [&](int32_t off, size_t i, double v) {          // (T) arrays: fp64, or rounded once to fp32
            if (E == 8) reinterpret_cast<double*>(blob.data() + off)[i] = v;
            else reinterpret_cast<float*>(blob.data() + off)[i] = (float)v;
        };
        auto I = [&](int32_t off) { return (int32_t*)(blob.data() + off); };
        std::memcpy(blob.data() + h.off_tasks, trec.data(), 16 * NT);
        std::memcpy(blob.data() + h.off_gimp, imp.data(), 8 * NIMP);

        int32_t* sinfo = I(h.off_sinfo);
        int32_t* sexp = I(h.off_sexp);
        B[c].x0.assign(NS, 0.0);
        for (int64_t i = 0; i < NS; ++i) sexp[i] = -1;
        for (size_t t = 0; t < tasks.size(); ++t) {
            int base = 0;
            for (int64_t s : tasks[t].subs) {
                const int ns = P.n_s[s];
                const double* Ab = &P.abar[P.abar_ptr[s]];
                const int rows = 32 * tasks[t].R;
                for (int r = 0; r < ns; ++r)             // row base+r of the tile: tile[k][base + r] = Abar_s[r][k]
                    for (int k = 0; k < ns; ++k) put(h.off_abar, (size_t)trec[t].z + (size_t)k * rows + base + r, Ab[(size_t)r * ns + k]);
                for (int r = 0; r < ns; ++r) {
                    const int64_t slot = trec[t].x + base + r;
                    const int64_t copy = P.sub_ptr[s] + r;
                    const int32_t g = P.copy_global[copy];
                    const bool first = P.seg_copy[P.seg_ptr[g]] == copy;     // canonical first copy: writes x_g
                    const int64_t nu = P.seg_ptr[g + 1] - P.seg_ptr[g];
                    sinfo[slot] = (base & 0x3F) | kResValid | (first ? kResFirst : 0) | (nu > 4 ? kResSlow : 0) |
                                  (gl_of[g] << kResGlShift);
                    sexp[slot] = xidx[copy];
                    put(h.off_bbar, slot, P.bbar[copy]);
                    put(h.off_xl0, slot, P.x0[copy]);
                    B[c].x0[slot] = P.x0[copy];
                    L.slot_of_copy[copy] = slot_base + (int32_t)slot;
                }
                base += ns;
            }
        }

        int32_t* grec = I(h.off_grec);
        int32_t* gxb = I(h.off_gxb);
        int32_t* seg = I(h.off_gseg);
        int32_t* gown = I(h.off_gown);
        int32_t q = 0;
        for (int64_t j = 0; j < NG; ++j) {
            const int32_t g = gl_list[j];
            const int64_t nu = P.seg_ptr[g + 1] - P.seg_ptr[g];
            put(h.off_gpar, 4 * j, P.c[g] / opt.rho);
            put(h.off_gpar, 4 * j + 1, 1.0 / (double)nu);
            put(h.off_gpar, 4 * j + 2, P.lo[g]);
            put(h.off_gpar, 4 * j + 3, P.hi[g]);
            auto smem_slot = [&](int32_t k) { return copy_chunk[k] == c ? L.slot_of_copy[k] - slot_base : ghost.at(k); };
            for (int k = 0; k < 4; ++k) grec[4 * j + k] = (int32_t)NS;           // the zero slot
            gxb[2 * j] = gxb[2 * j + 1] = 0;
            if (nu > 4) {                                        // the whole list, canonical order
                gxb[2 * j] = q;
                gxb[2 * j + 1] = (int32_t)nu;
                for (int64_t p = P.seg_ptr[g]; p < P.seg_ptr[g + 1]; ++p) seg[q++] = smem_slot(P.seg_copy[p]);
            } else {
                for (int64_t p = P.seg_ptr[g]; p < P.seg_ptr[g + 1]; ++p)      // canonical ascending copy order
                    grec[4 * j + (p - P.seg_ptr[g])] = smem_slot(P.seg_copy[p]);
            }
            gown[j] = copy_chunk[P.seg_copy[P.seg_ptr[g]]] == c ? g : -1;
        }
        if (std::getenv("LOPF_PACK_DEBUG")) {           // diagnostics: one line per CTA chunk
            int nsl = 0, nexp = 0, kmx = 0, imx = 0;
            for (int64_t i = 0; i < NS; ++i) { nsl += (sinfo[i] & kResSlow) != 0; nexp += sexp[i] >= 0; }
            for (size_t t = 0; t < tasks.size(); ++t) { kmx = std::max(kmx, tasks[t].kmax); imx = std::max(imx, (trec[t].w >> 4) & 0xFF); }
            std::fprintf(stderr, "cta %d tasks %d slots %d glob %d smem %d ghost %d imp %d impmax %d slow %d exp %d kmax %d margin %.3f\n",
                         c, (int)NT, (int)NS, (int)NG, h.smem_bytes, (int)NGH, (int)NIMP, imx, nsl, nexp, kmx, margin);
        }
        for (int32_t g : gl_list) gl_of[g] = -1;
        slot_base += (int32_t)NS;
    }
    L.total_slots = slot_base;
    L.max_smem = max_smem;
    L.n_slots = slot_base;
    for (auto& b : B) L.n_tasks += b.h.n_tasks;
    int64_t pool_all = 0;
    for (int c = 0; c < L.G; ++c) pool_all += (B[c].h.off_bbar - B[c].h.off_abar) / E;
    L.abar_doubles = pool_all;

    // ---- objective, arena ---------------------------------------------------------------------------
    std::vector<int32_t> obj_idx;
    std::vector<double> obj_c;
    for (int64_t i = 0; i < P.n; ++i)
        if (P.c[i] != 0.0) { obj_idx.push_back((int32_t)i); obj_c.push_back(P.c[i]); }
    L.n_obj = (int64_t)obj_idx.size();
    L.trace_cap = opt.trace_cap > 0 ? opt.trace_cap : 4096;
    L.max_grid = L.G;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t r = off; off = a256(off + std::max<size_t>(bytes, 1)); return r; };
    L.off_hdr = take(sizeof(CtaHdr) * L.G);
    size_t blobs_total = 0;
    for (auto& b : B) { b.h.blob_off = (long long)blobs_total; blobs_total = a256(blobs_total + b.blob.size()); }
    L.off_blobs = take(blobs_total);
    L.off_xchg = take(16 * 2 * (size_t)std::max(n_exp, 1));   // {u, tag} per boundary copy and parity
    L.off_flags = take(8 * 32 * (size_t)(L.G + 1));   // one flag per 256-byte line + the published count
    L.off_x0r = take(E * (size_t)L.total_slots);
    L.off_x = take(E * (size_t)P.n);
    L.off_partial = take(8 * 8 * 4 * (size_t)L.G);     // 4 sweep slots (lagged decision, see resident.cu)
    L.off_ctrl = take(sizeof(DevCtrl));
    L.off_trace = take(8 * 5 * (size_t)L.trace_cap);
    L.off_prof = take(8 * 4 * (size_t)L.G + 8 * 5 * 32 * (size_t)L.G);   // counters + LOPF_RES_TIMELINE=2 events
    L.off_objidx = take(4 * obj_idx.size());
    L.off_objc = take(8 * obj_c.size());
    L.bytes = off;
    L.image.assign(L.bytes, 0);
    uint8_t* img = L.image.data();
    L.hdr.resize(L.G);
    L.slot_cta.assign(L.total_slots, 0);
    for (int c = 0; c < L.G; ++c) {
        L.hdr[c] = B[c].h;
        std::memcpy(img + L.off_blobs + B[c].h.blob_off, B[c].blob.data(), B[c].blob.size());
        for (size_t i = 0; i < B[c].x0.size(); ++i) {
            const size_t at = L.off_x0r + (size_t)E * ((size_t)B[c].h.slot_base + i);
            if (E == 8) *reinterpret_cast<double*>(img + at) = B[c].x0[i];
            else *reinterpret_cast<float*>(img + at) = (float)B[c].x0[i];
        }
        for (int i = 0; i < B[c].h.n_slots; ++i) L.slot_cta[B[c].h.slot_base + i] = c;
    }
    std::memcpy(img + L.off_hdr, L.hdr.data(), sizeof(CtaHdr) * L.G);
    std::memcpy(img + L.off_objidx, obj_idx.data(), 4 * obj_idx.size());
    std::memcpy(img + L.off_objc, obj_c.data(), 8 * obj_c.size());
    return LOPF_OK;
}

}  // namespace lopf

// Host setup of liblopf: network validation, LP assembly, component decomposition and the
// Cholesky precompute of the local-update operators.  Independent of oracle/ by construction
// (different language, different factorisation, structural column rule).
//
//   assembly       PAPER.md:109-227 — operational bounds (2) :111-121, balance (3) :128-129,
//                  voltage-dependent loads (4) :140-161 with w-hat substituted (VDLM-3/4),
//                  linearized flow (5) :171-174 with M^p, M^q of :180-191, objective :200.
//   decomposition  PAPER.md:441-445 (leaf + its line merged; readings C10-C12),
//                  B_s as index lists, I_si / nu_i.
//   precompute     PAPER.md:342-346: with G = A_s A_s^T = L L^T and W = L^-1 A_s,
//                  Abar_s = W^T W - I (exactly symmetric) and bbar_s = W^T L^-1 b_s.
//                  Rank-deficient A_s are row-reduced first.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>

#include "internal.h"

namespace lopf {

static inline int popc3(uint8_t m) { return ((m >> 0) & 1) + ((m >> 1) & 1) + ((m >> 2) & 1); }
static inline bool has(uint8_t m, int ph) { return (m >> ph) & 1; }
static inline int rank_of(uint8_t m, int ph) {  // position of phase ph among the present phases
    int r = 0;
    for (int p = 0; p < ph; ++p) r += (m >> p) & 1;
    return r;
}

template <class T>
static void cp(std::vector<T>& dst, const T* src, size_t n) {
    dst.assign(src, src + n);
}

lopf_status copy_network(const lopf_network* s, Net& d, std::string& err) {
    if (!s) { err = "network is NULL"; return LOPF_E_ARG; }
    if (s->n_bus < 0 || s->n_line < 0 || s->n_gen < 0 || s->n_load < 0) { err = "negative component count"; return LOPF_E_ARG; }
    d.n_bus = s->n_bus; d.n_line = s->n_line; d.n_gen = s->n_gen; d.n_load = s->n_load; d.root = s->root_bus;
    const size_t B = (size_t)d.n_bus, L = (size_t)d.n_line, G = (size_t)d.n_gen, D = (size_t)d.n_load;
    auto need = [&](const void* p, size_t cnt, const char* name) {
        if (cnt && !p) { err = std::string("network array ") + name + " is NULL"; return false; }
        return true;
    };
    if (!need(s->bus_phases, B, "bus_phases") || !need(s->bus_wmin, B, "bus_wmin") || !need(s->bus_wmax, B, "bus_wmax") ||
        !need(s->bus_gsh, B, "bus_gsh") || !need(s->bus_bsh, B, "bus_bsh") || !need(s->line_from, L, "line_from") ||
        !need(s->line_to, L, "line_to") || !need(s->line_phases, L, "line_phases") || !need(s->line_r, L, "line_r") ||
        !need(s->line_x, L, "line_x") || !need(s->line_gs_from, L, "line_gs_from") || !need(s->line_bs_from, L, "line_bs_from") ||
        !need(s->line_gs_to, L, "line_gs_to") || !need(s->line_bs_to, L, "line_bs_to") || !need(s->line_tau, L, "line_tau") ||
        !need(s->line_pmin, L, "line_pmin") || !need(s->line_pmax, L, "line_pmax") || !need(s->line_qmin, L, "line_qmin") ||
        !need(s->line_qmax, L, "line_qmax") || !need(s->gen_bus, G, "gen_bus") || !need(s->gen_phases, G, "gen_phases") ||
        !need(s->gen_pmin, G, "gen_pmin") || !need(s->gen_pmax, G, "gen_pmax") || !need(s->gen_qmin, G, "gen_qmin") ||
        !need(s->gen_qmax, G, "gen_qmax") || !need(s->load_bus, D, "load_bus") || !need(s->load_phases, D, "load_phases") ||
        !need(s->load_conn, D, "load_conn") || !need(s->load_alpha, D, "load_alpha") || !need(s->load_beta, D, "load_beta") ||
        !need(s->load_a, D, "load_a") || !need(s->load_b, D, "load_b"))
        return LOPF_E_ARG;
    cp(d.bus_ph, s->bus_phases, B); cp(d.bus_wmin, s->bus_wmin, 3 * B); cp(d.bus_wmax, s->bus_wmax, 3 * B);
    cp(d.bus_gsh, s->bus_gsh, 3 * B); cp(d.bus_bsh, s->bus_bsh, 3 * B);
    cp(d.line_from, s->line_from, L); cp(d.line_to, s->line_to, L); cp(d.line_ph, s->line_phases, L);
    cp(d.line_r, s->line_r, 9 * L); cp(d.line_x, s->line_x, 9 * L);
    cp(d.line_gsf, s->line_gs_from, 3 * L); cp(d.line_bsf, s->line_bs_from, 3 * L);
    cp(d.line_gst, s->line_gs_to, 3 * L); cp(d.line_bst, s->line_bs_to, 3 * L); cp(d.line_tau, s->line_tau, 3 * L);
    cp(d.line_pmin, s->line_pmin, 3 * L); cp(d.line_pmax, s->line_pmax, 3 * L);
    cp(d.line_qmin, s->line_qmin, 3 * L); cp(d.line_qmax, s->line_qmax, 3 * L);
    cp(d.gen_bus, s->gen_bus, G); cp(d.gen_ph, s->gen_phases, G);
    cp(d.gen_pmin, s->gen_pmin, 3 * G); cp(d.gen_pmax, s->gen_pmax, 3 * G);
    cp(d.gen_qmin, s->gen_qmin, 3 * G); cp(d.gen_qmax, s->gen_qmax, 3 * G);
    cp(d.load_bus, s->load_bus, D); cp(d.load_ph, s->load_phases, D); cp(d.load_conn, s->load_conn, D);
    cp(d.load_alpha, s->load_alpha, 3 * D); cp(d.load_beta, s->load_beta, 3 * D);
    cp(d.load_a, s->load_a, 3 * D); cp(d.load_b, s->load_b, 3 * D);
    return LOPF_OK;
}

// Validation: SPEC.md:28-31 invariants + what the method needs (connected radial-or-meshed graph
// with no line joining two leaves, every phase set non-empty).
static lopf_status validate(const Net& n, std::string& err) {
    auto bad = [&](const std::string& m) { err = m; return LOPF_E_NETWORK; };
    if (n.n_bus > 0 && (n.root < 0 || n.root >= n.n_bus)) return bad("root_bus out of range");
    for (int i = 0; i < n.n_bus; ++i) {
        if ((n.bus_ph[i] & 7) == 0 || (n.bus_ph[i] & ~7)) return bad("bus " + std::to_string(i) + ": invalid phase set");
        for (int p = 0; p < 3; ++p)
            if (has(n.bus_ph[i], p) && !(n.bus_wmin[3 * i + p] <= n.bus_wmax[3 * i + p]))
                return bad("bus " + std::to_string(i) + ": wmin > wmax");
    }
    for (int e = 0; e < n.n_line; ++e) {
        int f = n.line_from[e], t = n.line_to[e];
        std::string nm = "line " + std::to_string(e);
        if (f < 0 || f >= n.n_bus || t < 0 || t >= n.n_bus) return bad(nm + ": dangling bus reference");
        if (f == t) return bad(nm + ": from == to");
        uint8_t m = n.line_ph[e];
        if ((m & 7) == 0 || (m & ~7)) return bad(nm + ": invalid phase set");
        if ((m & n.bus_ph[f]) != m || (m & n.bus_ph[t]) != m) return bad(nm + ": phases not a subset of its buses' phases");
        for (int p = 0; p < 3; ++p) {
            if (!has(m, p)) continue;
            if (!(n.line_tau[3 * e + p] > 0)) return bad(nm + ": tap ratio tau <= 0");
            if (!(n.line_pmin[3 * e + p] <= n.line_pmax[3 * e + p]) || !(n.line_qmin[3 * e + p] <= n.line_qmax[3 * e + p]))
                return bad(nm + ": flow lower bound > upper bound");
        }
    }
    for (int k = 0; k < n.n_gen; ++k) {
        std::string nm = "generator " + std::to_string(k);
        int b = n.gen_bus[k];
        if (b < 0 || b >= n.n_bus) return bad(nm + ": dangling bus reference");
        uint8_t m = n.gen_ph[k];
        if ((m & 7) == 0 || (m & n.bus_ph[b]) != m) return bad(nm + ": phases not a subset of its bus's phases");
        for (int p = 0; p < 3; ++p)
            if (has(m, p) && (!(n.gen_pmin[3 * k + p] <= n.gen_pmax[3 * k + p]) || !(n.gen_qmin[3 * k + p] <= n.gen_qmax[3 * k + p])))
                return bad(nm + ": lower bound > upper bound");
    }
    for (int l = 0; l < n.n_load; ++l) {
        std::string nm = "load " + std::to_string(l);
        int b = n.load_bus[l];
        if (b < 0 || b >= n.n_bus) return bad(nm + ": dangling bus reference");
        uint8_t m = n.load_ph[l];
        if ((m & 7) == 0 || (m & n.bus_ph[b]) != m) return bad(nm + ": phases not a subset of its bus's phases");
        if (n.load_conn[l] > 1) return bad(nm + ": connection must be 0 (wye) or 1 (delta)");
        if (n.load_conn[l] == 1 && m != 7) return bad(nm + ": delta loads must be 3-phase (SPEC.md:91)");
        for (int p = 0; p < 3; ++p)
            if (has(m, p) && (!(n.load_alpha[3 * l + p] >= 0) || !(n.load_beta[3 * l + p] >= 0)))
                return bad(nm + ": alpha, beta must be >= 0");
    }
    return LOPF_OK;
}

namespace {

struct Cols {  // global column numbering (canonical order, C12)
    std::vector<int64_t> gen, bus, load, line;
    int64_t n = 0;
};

struct Term {
    int64_t col;
    double v;
};
struct RowB {
    std::vector<Term> t;
    double rhs = 0;
    void add(int64_t c, double v) {
        for (auto& x : t)
            if (x.col == c) { x.v += v; return; }
        t.push_back({c, v});
    }
};

struct Builder {
    const Net& N;
    Cols C;
    std::vector<std::vector<int32_t>> lines_at, loads_at, gens_at;
    explicit Builder(const Net& n) : N(n) {
        lines_at.resize(N.n_bus); loads_at.resize(N.n_bus); gens_at.resize(N.n_bus);
        for (int e = 0; e < N.n_line; ++e) { lines_at[N.line_from[e]].push_back(e); lines_at[N.line_to[e]].push_back(e); }
        for (int l = 0; l < N.n_load; ++l) loads_at[N.load_bus[l]].push_back(l);
        for (int k = 0; k < N.n_gen; ++k) gens_at[N.gen_bus[k]].push_back(k);
        for (auto& v : lines_at) std::sort(v.begin(), v.end());
        int64_t o = 0;
        C.gen.resize(N.n_gen); C.bus.resize(N.n_bus); C.load.resize(N.n_load); C.line.resize(N.n_line);
        for (int k = 0; k < N.n_gen; ++k) { C.gen[k] = o; o += 2 * popc3(N.gen_ph[k]); }
        for (int i = 0; i < N.n_bus; ++i) { C.bus[i] = o; o += popc3(N.bus_ph[i]); }
        for (int l = 0; l < N.n_load; ++l) { C.load[l] = o; o += 4 * popc3(N.load_ph[l]); }
        for (int e = 0; e < N.n_line; ++e) { C.line[e] = o; o += 4 * popc3(N.line_ph[e]); }
        C.n = o;
    }
    // column of (role, component, phase): component-major, then role, then phase (C12)
    int64_t pg(int k, int p, int q) const { return C.gen[k] + q * popc3(N.gen_ph[k]) + rank_of(N.gen_ph[k], p); }  // q: 0 pg 1 qg
    int64_t w(int i, int p) const { return C.bus[i] + rank_of(N.bus_ph[i], p); }
    int64_t ld(int l, int role, int p) const { return C.load[l] + role * popc3(N.load_ph[l]) + rank_of(N.load_ph[l], p); }  // 0 pb 1 qb 2 pd 3 qd
    int64_t fl(int e, int role, int p) const { return C.line[e] + role * popc3(N.line_ph[e]) + rank_of(N.line_ph[e], p); }  // 0 pf 1 qf 2 pt 3 qt

    // rows of bus i: balance (3) then its loads (4)
    void bus_rows(int i, std::vector<RowB>& rows) const {
        uint8_t m = N.bus_ph[i];
        for (int kind = 0; kind < 2; ++kind) {          // 0: p-balance, 1: q-balance
            for (int p = 0; p < 3; ++p) {
                if (!has(m, p)) continue;
                RowB r;
                for (int e : lines_at[i]) {
                    if (!has(N.line_ph[e], p)) continue;
                    bool from = N.line_from[e] == i;     // p_eij leaves i: pf at the from end, pt at the to end
                    r.add(fl(e, (from ? 0 : 2) + kind, p), 1.0);
                }
                for (int l : loads_at[i])
                    if (has(N.load_ph[l], p)) r.add(ld(l, kind, p), 1.0);
                double sh = kind == 0 ? N.bus_gsh[3 * i + p] : -N.bus_bsh[3 * i + p];
                if (sh != 0.0) r.add(w(i, p), sh);
                for (int k : gens_at[i])
                    if (has(N.gen_ph[k], p)) r.add(pg(k, p, kind), -1.0);
                rows.push_back(std::move(r));
            }
        }
        for (int l : loads_at[i]) {
            uint8_t lm = N.load_ph[l];
            const double kap = N.load_conn[l] == 1 ? 3.0 : 1.0;    // VDLM-4 (delta) / VDLM-3 (wye)
            for (int p = 0; p < 3; ++p) {                            // VDLM-1
                if (!has(lm, p)) continue;
                double a = N.load_a[3 * l + p], al = N.load_alpha[3 * l + p];
                RowB r; r.add(ld(l, 2, p), 1.0);
                double cw = -(a * al / 2.0) * kap;
                if (cw != 0.0) r.add(w(i, p), cw);
                r.rhs = a * (1.0 - al / 2.0);
                rows.push_back(std::move(r));
            }
            for (int p = 0; p < 3; ++p) {                            // VDLM-2
                if (!has(lm, p)) continue;
                double b = N.load_b[3 * l + p], be = N.load_beta[3 * l + p];
                RowB r; r.add(ld(l, 3, p), 1.0);
                double cw = -(b * be / 2.0) * kap;
                if (cw != 0.0) r.add(w(i, p), cw);
                r.rhs = b * (1.0 - be / 2.0);
                rows.push_back(std::move(r));
            }
            if (N.load_conn[l] == 0) {                               // VDLM-5: pb = pd, qb = qd
                for (int q = 0; q < 2; ++q)
                    for (int p = 0; p < 3; ++p) {
                        if (!has(lm, p)) continue;
                        RowB r; r.add(ld(l, q, p), 1.0); r.add(ld(l, 2 + q, p), -1.0);
                        rows.push_back(std::move(r));
                    }
            } else {                                                 // VDLM-6..10 (phases 1,2,3 = a,b,c)
                const double s3 = std::sqrt(3.0), h3 = s3 / 2.0;
                auto PB = [&](int ph) { return ld(l, 0, ph - 1); };
                auto QB = [&](int ph) { return ld(l, 1, ph - 1); };
                auto PD = [&](int ph) { return ld(l, 2, ph - 1); };
                auto QD = [&](int ph) { return ld(l, 3, ph - 1); };
                RowB r6p, r6q, r7, r8, r9, r10;
                for (int ph = 1; ph <= 3; ++ph) { r6p.add(PB(ph), 1.0); r6q.add(QB(ph), 1.0); }
                for (int ph = 1; ph <= 3; ++ph) { r6p.add(PD(ph), -1.0); r6q.add(QD(ph), -1.0); }
                // (3/2) pb2 - (s3/2) qb2 - pd2 - (1/2) pd1 + (s3/2) qd1 = 0
                r7.add(PB(2), 1.5); r7.add(QB(2), -h3); r7.add(PD(2), -1.0); r7.add(PD(1), -0.5); r7.add(QD(1), h3);
                // (s3/2) pb2 + (3/2) qb2 - (s3/2) pd1 - (1/2) qd1 - qd2 = 0
                r8.add(PB(2), h3); r8.add(QB(2), 1.5); r8.add(PD(1), -h3); r8.add(QD(1), -0.5); r8.add(QD(2), -1.0);
                // s3 qb2 + (3/2) pb3 - (s3/2) qb3 - (1/2) pd1 - (s3/2) qd1 - pd3 = 0
                r9.add(QB(2), s3); r9.add(PB(3), 1.5); r9.add(QB(3), -h3); r9.add(PD(1), -0.5); r9.add(QD(1), -h3); r9.add(PD(3), -1.0);
                // -s3 pb2 + (s3/2) pb3 + (3/2) qb3 + (s3/2) pd1 - (1/2) qd1 - qd3 = 0
                r10.add(PB(2), -s3); r10.add(PB(3), h3); r10.add(QB(3), 1.5); r10.add(PD(1), h3); r10.add(QD(1), -0.5); r10.add(QD(3), -1.0);
                rows.push_back(std::move(r6p)); rows.push_back(std::move(r6q)); rows.push_back(std::move(r7));
                rows.push_back(std::move(r8)); rows.push_back(std::move(r9)); rows.push_back(std::move(r10));
            }
        }
    }

    // rows of line e: loss-p, loss-q, volt-drop (5a)-(5c)
    void line_rows(int e, std::vector<RowB>& rows) const {
        const int i = N.line_from[e], j = N.line_to[e];
        const uint8_t m = N.line_ph[e];
        const double* r = &N.line_r[9 * e];
        const double* x = &N.line_x[9 * e];
        const double s3 = std::sqrt(3.0);
        // M^p, M^q: diagonal -2r / -2x; off-diagonal r +- s3 x, x -+ s3 r with the
        // printed sign pattern sgn(phi, psi) = -1 for (1,2), (2,3), (3,1) and +1 for (1,3), (2,1), (3,2).
        auto sgn = [](int a, int b) { return ((b - a + 3) % 3 == 1) ? -1.0 : 1.0; };
        double Mp[3][3], Mq[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                if (a == b) { Mp[a][b] = -2.0 * r[3 * a + b]; Mq[a][b] = -2.0 * x[3 * a + b]; }
                else {
                    Mp[a][b] = r[3 * a + b] + sgn(a, b) * s3 * x[3 * a + b];
                    Mq[a][b] = x[3 * a + b] - sgn(a, b) * s3 * r[3 * a + b];
                }
            }
        for (int p = 0; p < 3; ++p) {                       // (5a) p_eij + p_eji - g^s_eij w_i - g^s_eji w_j = 0
            if (!has(m, p)) continue;
            RowB rw; rw.add(fl(e, 0, p), 1.0); rw.add(fl(e, 2, p), 1.0);
            if (N.line_gsf[3 * e + p] != 0.0) rw.add(w(i, p), -N.line_gsf[3 * e + p]);
            if (N.line_gst[3 * e + p] != 0.0) rw.add(w(j, p), -N.line_gst[3 * e + p]);
            rows.push_back(std::move(rw));
        }
        for (int p = 0; p < 3; ++p) {                       // (5b) q_eij + q_eji + b^s_eij w_i + b^s_eji w_j = 0
            if (!has(m, p)) continue;
            RowB rw; rw.add(fl(e, 1, p), 1.0); rw.add(fl(e, 3, p), 1.0);
            if (N.line_bsf[3 * e + p] != 0.0) rw.add(w(i, p), N.line_bsf[3 * e + p]);
            if (N.line_bst[3 * e + p] != 0.0) rw.add(w(j, p), N.line_bst[3 * e + p]);
            rows.push_back(std::move(rw));
        }
        for (int p = 0; p < 3; ++p) {                       // (5c) w_i - tau w_j + Mp (p - g^s w_i) + Mq (q + b^s w_i) = 0
            if (!has(m, p)) continue;
            RowB rw;
            rw.add(w(i, p), 1.0);
            rw.add(w(j, p), -N.line_tau[3 * e + p]);
            for (int q = 0; q < 3; ++q) {
                if (!has(m, q)) continue;
                rw.add(fl(e, 0, q), Mp[p][q]);
                rw.add(w(i, q), -Mp[p][q] * N.line_gsf[3 * e + q]);
                rw.add(fl(e, 1, q), Mq[p][q]);
                rw.add(w(i, q), Mq[p][q] * N.line_bsf[3 * e + q]);
            }
            rows.push_back(std::move(rw));
        }
    }

    // structural column sets (reading C11)
    void bus_cols(int i, std::vector<int64_t>& cols) const {
        uint8_t m = N.bus_ph[i];
        for (int e : lines_at[i]) {
            bool from = N.line_from[e] == i;
            for (int p = 0; p < 3; ++p)
                if (has(N.line_ph[e], p)) { cols.push_back(fl(e, from ? 0 : 2, p)); cols.push_back(fl(e, from ? 1 : 3, p)); }
        }
        for (int l : loads_at[i])
            for (int role = 0; role < 4; ++role)
                for (int p = 0; p < 3; ++p)
                    if (has(N.load_ph[l], p)) cols.push_back(ld(l, role, p));
        for (int k : gens_at[i])
            for (int q = 0; q < 2; ++q)
                for (int p = 0; p < 3; ++p)
                    if (has(N.gen_ph[k], p)) cols.push_back(pg(k, p, q));
        for (int p = 0; p < 3; ++p) {
            if (!has(m, p)) continue;
            bool inc = N.bus_gsh[3 * i + p] != 0.0 || N.bus_bsh[3 * i + p] != 0.0;
            for (int l : loads_at[i]) {
                if (!has(N.load_ph[l], p)) continue;
                if ((N.load_a[3 * l + p] != 0.0 && N.load_alpha[3 * l + p] != 0.0) ||
                    (N.load_b[3 * l + p] != 0.0 && N.load_beta[3 * l + p] != 0.0))
                    inc = true;
            }
            if (inc) cols.push_back(w(i, p));
        }
    }
    void line_cols(int e, std::vector<int64_t>& cols) const {
        for (int role = 0; role < 4; ++role)
            for (int p = 0; p < 3; ++p)
                if (has(N.line_ph[e], p)) cols.push_back(fl(e, role, p));
        for (int p = 0; p < 3; ++p)
            if (has(N.line_ph[e], p)) { cols.push_back(w(N.line_from[e], p)); cols.push_back(w(N.line_to[e], p)); }
    }
};

// --- dense linear algebra for one subsystem ----------------------------------------------------
// Cholesky of the m x m SPD matrix G (lower, in place).  Returns false on a non-positive pivot.
static bool cholesky(std::vector<double>& G, int m) {
    double dmax = 0;
    for (int i = 0; i < m; ++i) dmax = std::max(dmax, G[(size_t)i * m + i]);
    const double tol = 1e-13 * std::max(dmax, 1e-300);
    for (int j = 0; j < m; ++j) {
        double s = G[(size_t)j * m + j];
        for (int k = 0; k < j; ++k) s -= G[(size_t)j * m + k] * G[(size_t)j * m + k];
        if (!(s > tol)) return false;
        double ljj = std::sqrt(s);
        G[(size_t)j * m + j] = ljj;
        for (int i = j + 1; i < m; ++i) {
            double t = G[(size_t)i * m + j];
            for (int k = 0; k < j; ++k) t -= G[(size_t)i * m + k] * G[(size_t)j * m + k];
            G[(size_t)i * m + j] = t / ljj;
        }
    }
    return true;
}

// Keep the rows of A (m x n) that are independent of the kept rows before them (modified
// Gram-Schmidt, relative tolerance 1e-10); returns kept row indices.
static std::vector<int> independent_rows(const std::vector<double>& A, int m, int n) {
    std::vector<std::vector<double>> Q;
    std::vector<int> keep;
    for (int r = 0; r < m; ++r) {
        std::vector<double> v(A.begin() + (size_t)r * n, A.begin() + (size_t)(r + 1) * n);
        double n0 = 0;
        for (double t : v) n0 += t * t;
        n0 = std::sqrt(n0);
        for (auto& q : Q) {
            double d = 0;
            for (int k = 0; k < n; ++k) d += q[k] * v[k];
            for (int k = 0; k < n; ++k) v[k] -= d * q[k];
        }
        double nv = 0;
        for (double t : v) nv += t * t;
        nv = std::sqrt(nv);
        if (nv > 1e-10 * std::max(n0, 1e-300)) {
            for (auto& t : v) t /= nv;
            Q.push_back(std::move(v));
            keep.push_back(r);
        }
    }
    return keep;
}

struct SubOut {
    int status = 0;  // 0 ok, LOPF_E_RANK, LOPF_E_INFEASIBLE_SUB
    std::vector<double> A, b, abar, bbar;
    int m = 0;
};

// Precompute for one subsystem: A (m x n row-major), b.
static void precompute_one(std::vector<double> A, std::vector<double> b, int m, int n, SubOut& o) {
    o.abar.assign((size_t)n * n, 0.0);
    o.bbar.assign(n, 0.0);
    const std::vector<double> A0 = A, b0 = b;
    const int m0 = m;
    if (m > 0) {
        std::vector<double> G((size_t)m * m);
        auto form = [&]() {
            G.assign((size_t)m * m, 0.0);
            for (int i = 0; i < m; ++i)
                for (int j = 0; j <= i; ++j) {
                    double s = 0;
                    for (int k = 0; k < n; ++k) s += A[(size_t)i * n + k] * A[(size_t)j * n + k];
                    G[(size_t)i * m + j] = G[(size_t)j * m + i] = s;
                }
        };
        form();
        if (!cholesky(G, m)) {                        // row reduction, then retry
            std::vector<int> keep = independent_rows(A, m, n);
            std::vector<double> A2, b2;
            for (int r : keep) {
                A2.insert(A2.end(), A.begin() + (size_t)r * n, A.begin() + (size_t)(r + 1) * n);
                b2.push_back(b[r]);
            }
            A.swap(A2); b.swap(b2); m = (int)keep.size();
            form();
            if (m > 0 && !cholesky(G, m)) { o.status = LOPF_E_RANK; return; }
        }
        if (m > 0) {
            // W = L^-1 A (forward substitution, column by column), y = L^-1 b
            std::vector<double> W = A, y = b;
            for (int i = 0; i < m; ++i) {
                const double lii = G[(size_t)i * m + i];
                for (int k = 0; k < i; ++k) {
                    const double lik = G[(size_t)i * m + k];
                    for (int c = 0; c < n; ++c) W[(size_t)i * n + c] -= lik * W[(size_t)k * n + c];
                    y[i] -= lik * y[k];
                }
                for (int c = 0; c < n; ++c) W[(size_t)i * n + c] /= lii;
                y[i] /= lii;
            }
            for (int r = 0; r < n; ++r)
                for (int c = r; c < n; ++c) {
                    double s = 0;
                    for (int i = 0; i < m; ++i) s += W[(size_t)i * n + r] * W[(size_t)i * n + c];
                    o.abar[(size_t)r * n + c] = s;
                    o.abar[(size_t)c * n + r] = s;
                }
            for (int r = 0; r < n; ++r) {
                double s = 0;
                for (int i = 0; i < m; ++i) s += W[(size_t)i * n + r] * y[i];
                o.bbar[r] = s;
            }
        }
    }
    for (int r = 0; r < n; ++r) o.abar[(size_t)r * n + r] -= 1.0;
    // consistency of every original row with the min-norm solution bbar
    for (int r = 0; r < m0; ++r) {
        double s = 0, sc = std::fabs(b0[r]);
        for (int k = 0; k < n; ++k) { s += A0[(size_t)r * n + k] * o.bbar[k]; sc = std::max(sc, std::fabs(A0[(size_t)r * n + k])); }
        if (std::fabs(s - b0[r]) > 1e-8 * std::max(1.0, sc)) { o.status = LOPF_E_INFEASIBLE_SUB; return; }
    }
    o.A.swap(A); o.b.swap(b); o.m = m;
}

}  // namespace

static const char* kRoleName[] = {"pg", "qg", "w", "pb", "qb", "pd", "qd", "p_eij", "q_eij", "p_eji", "q_eji"};

lopf_status build_canon(const Net& N, const lopf_options& opt, Canon& P, std::string& err) {
    lopf_status st = validate(N, err);
    if (st != LOPF_OK) return st;
    Builder B(N);
    P = Canon();
    P.n = B.C.n;
    // ---- globals: catalog, objective, bounds (2) ------------------------------------------------
    P.var.resize(P.n);
    P.c.assign(P.n, 0.0);
    P.lo.assign(P.n, -std::numeric_limits<double>::infinity());
    P.hi.assign(P.n, std::numeric_limits<double>::infinity());
    for (int k = 0; k < N.n_gen; ++k)
        for (int q = 0; q < 2; ++q)
            for (int p = 0; p < 3; ++p) {
                if (!has(N.gen_ph[k], p)) continue;
                int64_t j = B.pg(k, p, q);
                P.var[j] = {(int8_t)(q == 0 ? PG : QG), (int8_t)p, k};
                P.lo[j] = q == 0 ? N.gen_pmin[3 * k + p] : N.gen_qmin[3 * k + p];
                P.hi[j] = q == 0 ? N.gen_pmax[3 * k + p] : N.gen_qmax[3 * k + p];
                if (q == 0) P.c[j] = 1.0;                          // objective sum p^g
            }
    for (int i = 0; i < N.n_bus; ++i)
        for (int p = 0; p < 3; ++p) {
            if (!has(N.bus_ph[i], p)) continue;
            int64_t j = B.w(i, p);
            P.var[j] = {(int8_t)W, (int8_t)p, i};
            P.lo[j] = N.bus_wmin[3 * i + p];
            P.hi[j] = N.bus_wmax[3 * i + p];
        }
    for (int l = 0; l < N.n_load; ++l)
        for (int role = 0; role < 4; ++role)
            for (int p = 0; p < 3; ++p)
                if (has(N.load_ph[l], p)) P.var[B.ld(l, role, p)] = {(int8_t)(PB + role), (int8_t)p, l};
    for (int e = 0; e < N.n_line; ++e)
        for (int role = 0; role < 4; ++role)
            for (int p = 0; p < 3; ++p) {
                if (!has(N.line_ph[e], p)) continue;
                int64_t j = B.fl(e, role, p);
                P.var[j] = {(int8_t)(PF + role), (int8_t)p, e};
                bool isp = role == 0 || role == 2;
                P.lo[j] = isp ? N.line_pmin[3 * e + p] : N.line_qmin[3 * e + p];
                P.hi[j] = isp ? N.line_pmax[3 * e + p] : N.line_qmax[3 * e + p];
            }

    // ---- decomposition (C10): leaves = degree-1 non-root buses, merged with their line -------
    std::vector<int> deg(N.n_bus, 0);
    for (int e = 0; e < N.n_line; ++e) { deg[N.line_from[e]]++; deg[N.line_to[e]]++; }
    std::vector<char> leaf(N.n_bus, 0);
    for (int i = 0; i < N.n_bus; ++i) leaf[i] = (deg[i] == 1 && i != N.root) ? 1 : 0;
    std::vector<int> leaf_of_line(N.n_line, -1);
    for (int e = 0; e < N.n_line; ++e) {
        int a = N.line_from[e], b = N.line_to[e];
        if (leaf[a] && leaf[b]) { err = "line " + std::to_string(e) + " joins two leaves (disconnected network)"; return LOPF_E_NETWORK; }
        if (leaf[a]) leaf_of_line[e] = a;
        if (leaf[b]) leaf_of_line[e] = b;
    }
    if (opt.single) {
        P.kind = {BUS}; P.comp = {-1}; P.leaf = {-1};
    } else {
        for (int i = 0; i < N.n_bus; ++i)
            if (!leaf[i]) { P.kind.push_back(BUS); P.comp.push_back(i); P.leaf.push_back(-1); }
        for (int e = 0; e < N.n_line; ++e) {
            P.kind.push_back(leaf_of_line[e] >= 0 ? LEAF : LINE);
            P.comp.push_back(e);
            P.leaf.push_back(leaf_of_line[e]);
        }
    }
    P.S = (int64_t)P.kind.size();
    // coarse partition (reading C25): consecutive runs of opt.coarse component
    // subsystems in depth-first order become one subsystem holding their rows in that order
    std::vector<std::vector<int64_t>> members;
    std::vector<int32_t> ckind = P.kind, ccomp = P.comp, cleaf = P.leaf;
    if (!opt.single && opt.coarse > 1) {
        const std::vector<int64_t> order = dfs_order(N, P);
        for (size_t i = 0; i < order.size(); i += (size_t)opt.coarse)
            members.emplace_back(order.begin() + i, order.begin() + std::min(order.size(), i + (size_t)opt.coarse));
        const int64_t S2 = (int64_t)members.size();
        P.kind.assign(S2, COARSE);
        P.comp.resize(S2);
        for (int64_t s = 0; s < S2; ++s) P.comp[s] = (int32_t)s;
        P.leaf.assign(S2, -1);
        P.S = S2;
    } else {
        for (int64_t s = 0; s < P.S; ++s) members.push_back({s});
    }

    // ---- per subsystem: rows, structural columns, dense A_s, b_s -----------------------------------
    std::vector<std::vector<RowB>> rows(P.S);
    std::vector<std::vector<int64_t>> cols(P.S);
    for (int64_t s = 0; s < P.S; ++s) {
        auto& R = rows[s];
        auto& Cs = cols[s];
        if (opt.single) {
            for (int i = 0; i < N.n_bus; ++i) B.bus_rows(i, R);
            for (int e = 0; e < N.n_line; ++e) B.line_rows(e, R);
            for (int i = 0; i < N.n_bus; ++i) B.bus_cols(i, Cs);
            for (int e = 0; e < N.n_line; ++e) B.line_cols(e, Cs);
        } else {
            for (int64_t c : members[s]) {
                if (ckind[c] == BUS) {
                    B.bus_rows(ccomp[c], R); B.bus_cols(ccomp[c], Cs);
                } else {
                    B.line_rows(ccomp[c], R); B.line_cols(ccomp[c], Cs);
                    if (ckind[c] == LEAF) { B.bus_rows(cleaf[c], R); B.bus_cols(cleaf[c], Cs); }
                }
            }
        }
        std::sort(Cs.begin(), Cs.end());
        Cs.erase(std::unique(Cs.begin(), Cs.end()), Cs.end());
    }
    P.m = 0;
    P.sub_ptr.assign(P.S + 1, 0);
    for (int64_t s = 0; s < P.S; ++s) {
        P.sub_ptr[s + 1] = P.sub_ptr[s] + (int64_t)cols[s].size();
        P.m += (int64_t)rows[s].size();
    }
    P.nc = P.sub_ptr[P.S];
    if (P.nc > INT32_MAX) { err = "more than 2^31 local copies"; return LOPF_E_ARG; }
    P.copy_global.resize(P.nc);
    for (int64_t s = 0; s < P.S; ++s)
        for (size_t k = 0; k < cols[s].size(); ++k) P.copy_global[P.sub_ptr[s] + k] = (int32_t)cols[s][k];

    // consensus CSR + orphan check
    std::vector<int64_t> nu(P.n, 0);
    for (int64_t k = 0; k < P.nc; ++k) nu[P.copy_global[k]]++;
    for (int64_t i = 0; i < P.n; ++i)
        if (nu[i] == 0) {
            const Var& v = P.var[i];
            err = "orphan global variable " + std::to_string(i) + " (" + kRoleName[v.role] + ", component " +
                  std::to_string(v.comp) + ", phase " + "abc"[v.phase] + "): nu = 0";
            return LOPF_E_ORPHAN;
        }
    P.seg_ptr.assign(P.n + 1, 0);
    for (int64_t i = 0; i < P.n; ++i) P.seg_ptr[i + 1] = P.seg_ptr[i] + nu[i];
    P.seg_copy.resize(P.nc);
    {
        std::vector<int64_t> fill(P.seg_ptr.begin(), P.seg_ptr.end() - 1);
        for (int64_t k = 0; k < P.nc; ++k) P.seg_copy[fill[P.copy_global[k]]++] = (int32_t)k;
    }

    // ---- precompute (parallel over subsystems; each one deterministic) -------------------------
    std::vector<SubOut> outs(P.S);
    auto work = [&](int64_t s0, int64_t s1) {
        for (int64_t s = s0; s < s1; ++s) {
            const auto& Cs = cols[s];
            const int n = (int)Cs.size(), m = (int)rows[s].size();
            std::vector<double> A((size_t)m * n, 0.0), b(m, 0.0);
            bool ok = true;
            for (int r = 0; r < m; ++r) {
                for (const Term& t : rows[s][r].t) {
                    if (t.v == 0.0) continue;
                    auto it = std::lower_bound(Cs.begin(), Cs.end(), t.col);
                    if (it == Cs.end() || *it != t.col) { ok = false; break; }
                    A[(size_t)r * n + (it - Cs.begin())] += t.v;
                }
                b[r] = rows[s][r].rhs;
            }
            if (!ok) { outs[s].status = -1; continue; }
            precompute_one(std::move(A), std::move(b), m, n, outs[s]);
        }
    };
    unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (P.S < 256) nt = 1;
    std::vector<std::thread> th;
    int64_t chunk = (P.S + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        int64_t s0 = (int64_t)t * chunk, s1 = std::min(P.S, s0 + chunk);
        if (s0 < s1) th.emplace_back(work, s0, s1);
    }
    for (auto& t : th) t.join();

    P.m_s.resize(P.S); P.m_raw.resize(P.S); P.n_s.resize(P.S);
    P.a_ptr.assign(P.S + 1, 0); P.b_ptr.assign(P.S + 1, 0); P.abar_ptr.assign(P.S + 1, 0);
    for (int64_t s = 0; s < P.S; ++s) {
        if (outs[s].status != 0) {
            std::string who = "subsystem " + std::to_string(s) + " (" +
                              (P.kind[s] == BUS ? "bus " : P.kind[s] == LINE ? "line " : P.kind[s] == LEAF ? "leaf line "
                                                                                                       : "coarse run ") +
                              std::to_string(P.comp[s]) + ")";
            if (outs[s].status == -1) { err = who + ": row references a column outside its structural set"; return LOPF_E_NETWORK; }
            err = who + (outs[s].status == LOPF_E_RANK ? ": A_s A_s^T is singular after row reduction"
                                                       : ": equality rows are inconsistent");
            return (lopf_status)outs[s].status;
        }
        const int n = (int)cols[s].size();
        P.m_raw[s] = (int32_t)rows[s].size();
        P.m_s[s] = outs[s].m;
        P.n_s[s] = n;
        P.a_ptr[s + 1] = P.a_ptr[s] + (int64_t)outs[s].m * n;
        P.b_ptr[s + 1] = P.b_ptr[s] + outs[s].m;
        P.abar_ptr[s + 1] = P.abar_ptr[s] + (int64_t)n * n;
    }
    P.A.resize(P.a_ptr[P.S]); P.b.resize(P.b_ptr[P.S]); P.abar.resize(P.abar_ptr[P.S]); P.bbar.resize(P.nc);
    for (int64_t s = 0; s < P.S; ++s) {
        std::copy(outs[s].A.begin(), outs[s].A.end(), P.A.begin() + P.a_ptr[s]);
        std::copy(outs[s].b.begin(), outs[s].b.end(), P.b.begin() + P.b_ptr[s]);
        std::copy(outs[s].abar.begin(), outs[s].abar.end(), P.abar.begin() + P.abar_ptr[s]);
        std::copy(outs[s].bbar.begin(), outs[s].bbar.end(), P.bbar.begin() + P.sub_ptr[s]);
    }
    // ---- initial point (reading C7) ------------------------------------------------
    P.x0.resize(P.nc);
    for (int64_t k = 0; k < P.nc; ++k) {
        int32_t g = P.copy_global[k];
        if (P.var[g].role == W) P.x0[k] = 1.0;
        else if (std::isfinite(P.lo[g]) && std::isfinite(P.hi[g])) P.x0[k] = 0.5 * (P.lo[g] + P.hi[g]);
        else P.x0[k] = 0.0;
    }
    return LOPF_OK;
}

// Per-scenario operators for config 4 (BASELINE.json configs[3]): scenario sigma scales every load's
// (a, b) by scale[sigma * n_load + l] (> 0, so the structural column sets are unchanged).  Only the
// subsystems holding a load see a different A_s / b_s; their Abar, bbar are recomputed per scenario.
lopf_status build_batch_ops(const Net& base, const Canon& P, int32_t n_scen, const double* scale, BatchOps& out,
                            std::string& err) {
    out = BatchOps();
    out.n_scen = n_scen;
    if (n_scen <= 0 || !scale) { err = "batch: n_scen must be > 0 with a load_scale array"; return LOPF_E_ARG; }
    for (int64_t q = 0; q < (int64_t)n_scen * base.n_load; ++q)
        if (!(scale[q] > 0) || !std::isfinite(scale[q])) { err = "batch: load scales must be finite and > 0"; return LOPF_E_ARG; }
    std::vector<char> has_load(base.n_bus, 0);
    for (int l = 0; l < base.n_load; ++l) has_load[base.load_bus[l]] = 1;
    out.vidx.assign(P.S, -1);
    for (int64_t s = 0; s < P.S; ++s) {
        bool v = false;
        if (P.S == 1) v = base.n_load > 0;
        else if (P.kind[s] == BUS) v = has_load[P.comp[s]];
        else if (P.kind[s] == LEAF) v = has_load[P.leaf[s]];
        if (v) { out.vidx[s] = (int32_t)out.vsub.size(); out.vsub.push_back(s); }
    }
    const int64_t V = (int64_t)out.vsub.size();
    out.va_off.assign(V + 1, 0);
    out.vb_off.assign(V + 1, 0);
    for (int64_t v = 0; v < V; ++v) {
        const int ns = P.n_s[out.vsub[v]];
        out.va_off[v + 1] = out.va_off[v] + (int64_t)ns * ns;
        out.vb_off[v + 1] = out.vb_off[v] + ns;
    }
    out.VA = out.va_off[V];
    out.VB = out.vb_off[V];
    out.abar.assign((size_t)n_scen * out.VA, 0.0);
    out.bbar.assign((size_t)n_scen * out.VB, 0.0);
    std::vector<int> status(n_scen, 0);
    auto work_body = [&](int32_t s0, int32_t s1) {
        Net N = base;                                  // this thread's scaled copy
        Builder B(N);
        for (int32_t sc = s0; sc < s1; ++sc) {
            for (int l = 0; l < base.n_load; ++l)
                for (int p = 0; p < 3; ++p) {
                    const double k = scale[(int64_t)sc * base.n_load + l];
                    N.load_a[3 * l + p] = base.load_a[3 * l + p] * k;
                    N.load_b[3 * l + p] = base.load_b[3 * l + p] * k;
                }
            for (int64_t v = 0; v < V && !status[sc]; ++v) {
                const int64_t s = out.vsub[v];
                std::vector<RowB> rows;
                if (P.S == 1) {
                    for (int i = 0; i < N.n_bus; ++i) B.bus_rows(i, rows);
                    for (int e = 0; e < N.n_line; ++e) B.line_rows(e, rows);
                } else if (P.kind[s] == BUS) {
                    B.bus_rows(P.comp[s], rows);
                } else {
                    B.line_rows(P.comp[s], rows);
                    B.bus_rows(P.leaf[s], rows);
                }
                const int n = P.n_s[s], m = (int)rows.size();
                const int32_t* cols = &P.copy_global[P.sub_ptr[s]];
                std::vector<double> A((size_t)m * n, 0.0), b(m, 0.0);
                for (int r = 0; r < m; ++r) {
                    for (const Term& t : rows[r].t) {
                        if (t.v == 0.0) continue;
                        const int32_t* it = std::lower_bound(cols, cols + n, (int32_t)t.col);
                        if (it == cols + n || *it != t.col) { status[sc] = -1; break; }
                        A[(size_t)r * n + (it - cols)] += t.v;
                    }
                    b[r] = rows[r].rhs;
                }
                if (status[sc]) break;
                SubOut o;
                precompute_one(std::move(A), std::move(b), m, n, o);
                if (o.status) { status[sc] = o.status; break; }
                std::copy(o.abar.begin(), o.abar.end(), out.abar.begin() + (size_t)sc * out.VA + out.va_off[v]);
                std::copy(o.bbar.begin(), o.bbar.end(), out.bbar.begin() + (size_t)sc * out.VB + out.vb_off[v]);
            }
        }
    };
    // no exception may leave a worker thread (it would terminate the process): a failure marks the
    // thread's scenarios with -2 and is reported after the join
    auto work = [&](int32_t s0, int32_t s1) {
        try {
            work_body(s0, s1);
        } catch (...) {
            for (int32_t sc = s0; sc < s1; ++sc)
                if (!status[sc]) status[sc] = -2;
        }
    };
    unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    nt = (unsigned)std::min<int64_t>(nt, n_scen);
    std::vector<std::thread> th;
    const int32_t chunk = (n_scen + (int32_t)nt - 1) / (int32_t)nt;
    int32_t ran = 0;                                   // scenarios handed to threads; the rest run here
    try {
        for (unsigned t = 0; t < nt; ++t) {
            const int32_t s0 = (int32_t)t * chunk, s1 = std::min(n_scen, s0 + chunk);
            if (s0 < s1) { th.emplace_back(work, s0, s1); ran = s1; }
        }
    } catch (...) {                                    // thread creation failed: finish on this thread
    }
    for (auto& t : th) t.join();
    if (ran < n_scen) work(ran, n_scen);
    for (int32_t sc = 0; sc < n_scen; ++sc)
        if (status[sc]) {
            err = "batch scenario " + std::to_string(sc) + ": " +
                  (status[sc] == -2 ? std::string("host failure (out of memory?) in the precompute")
                   : status[sc] == -1 ? std::string("row outside the structural column set")
                                    : status[sc] == LOPF_E_RANK ? std::string("A_s A_s^T singular")
                                                                : std::string("inconsistent equality rows"));
            return status[sc] == -2 ? LOPF_E_ARG : status[sc] == -1 ? LOPF_E_NETWORK : (lopf_status)status[sc];
        }
    return LOPF_OK;
}

}  // namespace lopf

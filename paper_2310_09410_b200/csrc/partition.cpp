// Feeder partition for the multi-GPU partitioned mode (config 5).
//
// Buses are split into `world` contiguous intervals of the depth-first preorder from the substation,
// balanced by subtree work (copies of the subsystems each bus anchors), so every part is a union of
// whole subtrees plus one path to them.  Subsystems follow their anchor bus: BUS(i) -> bus i,
// LINE(e) -> the end of e farther from the root, LEAF -> the merged leaf bus.  A global whose copies
// land on two or more ranks is a BOUNDARY global; every copy of it gets a slot in the exchange
// buffer, numbered in canonical (global, copy) order, identical on every rank because every rank
// builds the same canonical problem.
#include <algorithm>

#include "internal.h"

namespace lopf {

static void dfs_buses(const Net& N, std::vector<int32_t>& order, std::vector<int32_t>& parent_line) {
    std::vector<std::vector<int32_t>> adj(N.n_bus);
    for (int e = 0; e < N.n_line; ++e) { adj[N.line_from[e]].push_back(e); adj[N.line_to[e]].push_back(e); }
    for (auto& a : adj) std::sort(a.begin(), a.end());
    std::vector<char> seen(N.n_bus, 0);
    parent_line.assign(N.n_bus, -1);
    order.clear();
    auto walk = [&](int root) {
        std::vector<std::pair<int, size_t>> st{{root, 0}};
        seen[root] = 1;
        order.push_back(root);
        while (!st.empty()) {
            auto& [b, k] = st.back();
            if (k >= adj[b].size()) { st.pop_back(); continue; }
            const int e = adj[b][k++];
            const int o = N.line_from[e] == b ? N.line_to[e] : N.line_from[e];
            if (!seen[o]) {
                seen[o] = 1;
                parent_line[o] = e;
                order.push_back(o);
                st.push_back({o, 0});
            }
        }
    };
    if (N.n_bus > 0) walk(N.root);
    for (int b = 0; b < N.n_bus; ++b)
        if (!seen[b]) walk(b);
}

lopf_status build_partition(const Net& N, const Canon& P, int32_t world, const int32_t* bus_owner_in,
                            PartSpec& out, std::string& err) {
    if (world < 1) { err = "world must be >= 1"; return LOPF_E_ARG; }
    out = PartSpec();
    out.world = world;
    std::vector<int32_t> order, parent_line;
    dfs_buses(N, order, parent_line);
    // anchor bus of every subsystem
    std::vector<int32_t> anchor(P.S, 0);
    for (int64_t s = 0; s < P.S; ++s) {
        if (P.kind[s] == BUS) anchor[s] = P.comp[s];
        else if (P.kind[s] == LEAF) anchor[s] = P.leaf[s];
        else {
            const int e = P.comp[s], a = N.line_from[e], b = N.line_to[e];
            anchor[s] = parent_line[b] == e ? b : a;         // the end whose parent line is e
        }
    }
    out.bus_owner.assign(N.n_bus, 0);
    if (bus_owner_in) {
        for (int b = 0; b < N.n_bus; ++b) {
            if (bus_owner_in[b] < 0 || bus_owner_in[b] >= world) {
                err = "bus_owner[" + std::to_string(b) + "] out of range";
                return LOPF_E_ARG;
            }
            out.bus_owner[b] = bus_owner_in[b];
        }
    } else {                                                 // balanced contiguous preorder intervals
        std::vector<int64_t> w(N.n_bus, 0);
        int64_t total = 0;
        for (int64_t s = 0; s < P.S; ++s) { w[anchor[s]] += P.n_s[s]; total += P.n_s[s]; }
        int64_t acc = 0;
        int r = 0;
        for (int32_t b : order) {
            // move to the next rank once this one holds its share (never leave a rank empty of buses)
            while (r < world - 1 && acc >= (total * (r + 1) + world - 1) / world) ++r;
            out.bus_owner[b] = r;
            acc += w[b];
        }
    }
    out.sub_owner.resize(P.S);
    for (int64_t s = 0; s < P.S; ++s) out.sub_owner[s] = out.bus_owner[anchor[s]];
    // boundary copies
    std::vector<int32_t> copy_owner(P.nc);
    for (int64_t s = 0; s < P.S; ++s)
        for (int64_t k = P.sub_ptr[s]; k < P.sub_ptr[s + 1]; ++k) copy_owner[k] = out.sub_owner[s];
    out.bidx.assign(P.nc, -1);
    int32_t nb = 0;
    for (int64_t g = 0; g < P.n; ++g) {
        const int64_t q0 = P.seg_ptr[g], q1 = P.seg_ptr[g + 1];
        bool multi = false;
        for (int64_t q = q0 + 1; q < q1; ++q)
            if (copy_owner[P.seg_copy[q]] != copy_owner[P.seg_copy[q0]]) multi = true;
        if (multi)
            for (int64_t q = q0; q < q1; ++q) out.bidx[P.seg_copy[q]] = nb++;
    }
    out.n_bnd = nb;
    out.copy_owner = std::move(copy_owner);
    return LOPF_OK;
}

}  // namespace lopf

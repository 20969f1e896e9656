// C ABI of liblopf (include/lopf.h): argument checking, handle lifetime, device arena binding,
// launch orchestration and canonical-order getters.  No exception crosses this boundary.
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include "internal.h"

using namespace lopf;

struct lopf_handle {
    Net net;
    Canon cp;
    Layout lay;
    lopf_options opt{};
    void* arena = nullptr;
    size_t arena_bytes = 0;
    bool bound = false;
    bool registered = false;
    int grid = 0;
    DevProblem dp{};
    ResProblem rp{};
    BatchProblem bp{};
    BatchOps bo;
    std::vector<ScenResult> scen_res;              // host copy of the last batch results
    PartSpec part;                                 // partitioned mode (lay.part != 0)
    uint32_t epoch = 0;                            // resident launches so far (exchange tag epoch)
    std::vector<void*> ipc_open;                   // peer allocations opened by lopf_ipc_open (closed at destroy)
    std::vector<uint64_t> peer_tab;                // [world] device pointers of every rank's p2p entry buffer
    DevProblem p2p_arg{};                          // host copy of the p2p launch argument (kept for the async H2D)
    void* nccl_comm = nullptr;                     // library-owned NCCL communicator (lopf_part_nccl_init)
    bool resident() const { return lay.kernel == 2; }
    bool parted() const { return lay.part != 0; }
    bool batch() const { return lay.kernel == 3; }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

static thread_local std::string g_err;

static lopf_status fail(lopf_status st, const std::string& msg) {
    g_err = msg;
    return st;
}
static lopf_status cuda_fail(cudaError_t e, const char* where) {
    g_err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return LOPF_E_CUDA;
}
#define CUDA_TRY(call, where)                      \
    do {                                           \
        cudaError_t _e = (call);                   \
        if (_e != cudaSuccess) return cuda_fail(_e, where); \
    } while (0)

static constexpr int kMaxGrid = 4096;

// Pinned staging for device -> host reads into caller (pageable) memory: a DMA into pinned memory plus a
// host copy is several times faster than a staged pageable copy (x of the 8500 shape: ~0.05 vs 0.3 ms).
static thread_local void* g_pin = nullptr;
static thread_local size_t g_pin_bytes = 0;
static void* pinned(size_t bytes) {
    if (bytes > g_pin_bytes) {
        if (g_pin) cudaFreeHost(g_pin);
        g_pin = nullptr;
        g_pin_bytes = 0;
        if (cudaMallocHost(&g_pin, bytes) != cudaSuccess) { cudaGetLastError(); g_pin = nullptr; return nullptr; }
        g_pin_bytes = bytes;
    }
    return g_pin;
}

// (T) device arrays (reading F1) <-> host fp64: n elements of esz bytes at `dev`.  Synchronous.
static cudaError_t d2h_elems(double* out, const void* dev, size_t n, int esz, cudaStream_t s) {
    void* stage = pinned((size_t)esz * n);
    cudaError_t e;
    if (!stage) {                                              // no pinned memory: direct (staged) copy
        if (esz == 8) {
            e = cudaMemcpyAsync(out, dev, 8 * n, cudaMemcpyDeviceToHost, s);
            return e == cudaSuccess ? cudaStreamSynchronize(s) : e;
        }
        std::vector<float> tmp(n);
        e = cudaMemcpyAsync(tmp.data(), dev, 4 * n, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        for (size_t i = 0; e == cudaSuccess && i < n; ++i) out[i] = (double)tmp[i];
        return e;
    }
    e = cudaMemcpyAsync(stage, dev, (size_t)esz * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    if (esz == 8) std::memcpy(out, stage, 8 * n);
    else for (size_t i = 0; i < n; ++i) out[i] = (double)static_cast<const float*>(stage)[i];
    return cudaSuccess;
}
static cudaError_t h2d_elems(void* dev, const double* in, size_t n, int esz, cudaStream_t s) {
    if (esz == 8) {
        cudaError_t e = cudaMemcpyAsync(dev, in, 8 * n, cudaMemcpyHostToDevice, s);
        return e == cudaSuccess ? cudaStreamSynchronize(s) : e;    // `in` may be a temporary
    }
    std::vector<float> tmp(n);
    for (size_t i = 0; i < n; ++i) tmp[i] = (float)in[i];
    cudaError_t e = cudaMemcpyAsync(dev, tmp.data(), 4 * n, cudaMemcpyHostToDevice, s);
    return e == cudaSuccess ? cudaStreamSynchronize(s) : e;
}
static lopf_status check_precision(const lopf_options& o) {
    if (o.precision != 0 && o.precision != 32 && o.precision != 64)
        return fail(LOPF_E_ARG, "precision must be 0 / 64 (fp64) or 32 (fp32)");
    if (o.block_threads != 0)
        return fail(LOPF_E_ARG, "block_threads must be 0 (block sizes are fixed per kernel; see lopf_sizes.block)");
    if (o.reserved[1] != 0)
        return fail(LOPF_E_ARG, "options.reserved[1] must be 0 (the phase-skip diagnostics are a build flag, LOPF_DIAG_SKIP)");
    if (o.adapt_every < 0) return fail(LOPF_E_ARG, "adapt_every must be >= 0");
    if (o.coarse < 0) return fail(LOPF_E_ARG, "coarse must be >= 0");
    if (o.adapt_every > 0 && ((o.adapt_mu != 0 && !(o.adapt_mu > 1)) || (o.adapt_tau != 0 && !(o.adapt_tau > 1))))
        return fail(LOPF_E_ARG, "residual balancing needs adapt_mu > 1 and adapt_tau > 1");
    return LOPF_OK;
}

// The image uploaded by bind covers the packed problem; the fetch staging (lopf_fetch_async) goes after it.
static void add_fetch_stage(lopf_handle* h) {
    Layout& L = h->lay;
    if (L.image_bytes == 0) L.image_bytes = L.image.size();
    if (h->batch() || h->parted()) return;
    L.off_fetch = (L.bytes + 255) & ~(size_t)255;
    // also the slot-ordered x_s / lambda gather of the resident layout (lopf_get_state: one kernel, one copy)
    const size_t res_gather = h->resident() ? 16 * (size_t)L.total_slots : 0;
    L.bytes = L.off_fetch + std::max(64 + 8 * (size_t)h->cp.n, res_gather);
}

extern "C" {

int32_t lopf_abi_version(void) { return LOPF_ABI_VERSION; }

const char* lopf_last_error(void) { return g_err.c_str(); }

lopf_status lopf_options_default(lopf_options* o) {
    if (!o) return fail(LOPF_E_ARG, "options pointer is NULL");
    std::memset(o, 0, sizeof(*o));
    o->rho = 100.0;
    o->eps_rel = 1e-3;
    o->max_iter = 1000000; // reading C21
    o->trace_cap = 4096;
    return LOPF_OK;
}

lopf_status lopf_setup(const lopf_network* net, const lopf_options* opt, lopf_handle** out) {
    g_err.clear();
    if (!out) return fail(LOPF_E_ARG, "out handle pointer is NULL");
    *out = nullptr;
    lopf_options o;
    if (opt) o = *opt; else lopf_options_default(&o);
    if (!(o.rho > 0) || !std::isfinite(o.rho)) return fail(LOPF_E_ARG, "rho must be > 0 (SPEC.md:186)");
    if (!(o.eps_rel > 0) || !std::isfinite(o.eps_rel)) return fail(LOPF_E_ARG, "eps_rel must be > 0 (SPEC.md:186)");
    if (o.max_iter < 0) return fail(LOPF_E_ARG, "max_iter must be >= 0");
    if (o.trace_every < 0) return fail(LOPF_E_ARG, "trace_every must be >= 0");
    if (o.kernel < 0 || o.kernel > 2) return fail(LOPF_E_ARG, "kernel must be 0 (auto), 1 or 2");
    if (check_precision(o) != LOPF_OK) return LOPF_E_ARG;
    lopf_handle* h = new (std::nothrow) lopf_handle();
    if (!h) return fail(LOPF_E_ARG, "out of host memory");
    h->opt = o;
    std::string err;
    try {
        lopf_status st = copy_network(net, h->net, err);
        if (st == LOPF_OK) st = build_canon(h->net, h->opt, h->cp, err);
        if (st == LOPF_OK && h->opt.adapt_every > 0) {
            if (h->opt.adapt_mu == 0) h->opt.adapt_mu = 10.0;
            if (h->opt.adapt_tau == 0) h->opt.adapt_tau = 2.0;
            if (h->opt.kernel == 2) { st = LOPF_E_ARG; err = "residual balancing (adapt_every > 0) runs on the streaming kernel"; }
        }
        if (st == LOPF_OK) {
            if (h->opt.kernel == 2) {
                st = pack_resident(h->net, h->cp, h->opt, h->lay, err);
            } else if (h->opt.kernel == 1) {
                st = pack_streaming(h->net, h->cp, h->opt, kMaxGrid, h->lay, err);
            } else {                                      // auto: operators on chip when they fit (fp64)
                std::string e2;
                st = h->opt.adapt_every > 0 ? LOPF_E_ARG : pack_resident(h->net, h->cp, h->opt, h->lay, e2);
                if (st != LOPF_OK) st = pack_streaming(h->net, h->cp, h->opt, kMaxGrid, h->lay, err);
            }
        }
        if (st != LOPF_OK) { delete h; return fail(st, err); }
        add_fetch_stage(h);
    } catch (const std::bad_alloc&) {
        delete h;
        return fail(LOPF_E_ARG, "out of host memory during setup");
    } catch (const std::exception& ex) {
        delete h;
        return fail(LOPF_E_ARG, std::string("setup failed: ") + ex.what());
    }
    *out = h;
    return LOPF_OK;
}

lopf_status lopf_setup_batch(const lopf_network* net, const lopf_options* opt, int32_t n_scen, const double* load_scale,
                             lopf_handle** out) {
    g_err.clear();
    if (!out) return fail(LOPF_E_ARG, "out handle pointer is NULL");
    *out = nullptr;
    lopf_options o;
    if (opt) o = *opt; else lopf_options_default(&o);
    if (!(o.rho > 0) || !std::isfinite(o.rho)) return fail(LOPF_E_ARG, "rho must be > 0 (SPEC.md:186)");
    if (!(o.eps_rel > 0) || !std::isfinite(o.eps_rel)) return fail(LOPF_E_ARG, "eps_rel must be > 0 (SPEC.md:186)");
    if (o.max_iter < 0) return fail(LOPF_E_ARG, "max_iter must be >= 0");
    if (n_scen <= 0 || !load_scale) return fail(LOPF_E_ARG, "n_scen must be > 0 with a load_scale array");
    if (o.adapt_every != 0) return fail(LOPF_E_ARG, "residual balancing is not available on batch handles");
    if (o.coarse > 1) return fail(LOPF_E_ARG, "coarse partitions are not available on batch handles");
    if (n_scen > kBatchMaxScen)
        return fail(LOPF_E_ARG, "n_scen > " + std::to_string(kBatchMaxScen) + " per handle: shard the scenarios");
    if (check_precision(o) != LOPF_OK) return LOPF_E_ARG;
    lopf_handle* h = new (std::nothrow) lopf_handle();
    if (!h) return fail(LOPF_E_ARG, "out of host memory");
    h->opt = o;
    std::string err;
    try {
        lopf_status st = copy_network(net, h->net, err);
        if (st == LOPF_OK) st = build_canon(h->net, h->opt, h->cp, err);
        if (st == LOPF_OK) st = build_batch_ops(h->net, h->cp, n_scen, load_scale, h->bo, err);
        if (st == LOPF_OK) st = pack_batch(h->net, h->cp, h->bo, h->opt, h->lay, err);
        if (st != LOPF_OK) { delete h; return fail(st, err); }
        add_fetch_stage(h);
    } catch (const std::bad_alloc&) {
        delete h;
        return fail(LOPF_E_ARG, "out of host memory during setup");
    } catch (const std::exception& ex) {
        delete h;
        return fail(LOPF_E_ARG, std::string("setup failed: ") + ex.what());
    }
    *out = h;
    return LOPF_OK;
}

lopf_status lopf_setup_part(const lopf_network* net, const lopf_options* opt, int32_t rank, int32_t world,
                            const int32_t* bus_owner, lopf_handle** out) {
    g_err.clear();
    if (!out) return fail(LOPF_E_ARG, "out handle pointer is NULL");
    *out = nullptr;
    lopf_options o;
    if (opt) o = *opt; else lopf_options_default(&o);
    if (!(o.rho > 0) || !std::isfinite(o.rho)) return fail(LOPF_E_ARG, "rho must be > 0 (SPEC.md:186)");
    if (!(o.eps_rel > 0) || !std::isfinite(o.eps_rel)) return fail(LOPF_E_ARG, "eps_rel must be > 0 (SPEC.md:186)");
    if (o.max_iter < 0) return fail(LOPF_E_ARG, "max_iter must be >= 0");
    if (world < 1 || rank < 0 || rank >= world) return fail(LOPF_E_ARG, "need 0 <= rank < world");
    if (o.adapt_every != 0) return fail(LOPF_E_ARG, "residual balancing is not available on partitioned handles");
    if (o.coarse > 1) return fail(LOPF_E_ARG, "coarse partitions are not available on partitioned handles");
    if (check_precision(o) != LOPF_OK) return LOPF_E_ARG;
    lopf_handle* h = new (std::nothrow) lopf_handle();
    if (!h) return fail(LOPF_E_ARG, "out of host memory");
    h->opt = o;
    h->opt.trace_every = 0;
    std::string err;
    try {
        lopf_status st = copy_network(net, h->net, err);
        if (st == LOPF_OK) st = build_canon(h->net, h->opt, h->cp, err);
        if (st == LOPF_OK) st = build_partition(h->net, h->cp, world, bus_owner, h->part, err);
        if (st == LOPF_OK) st = pack_streaming(h->net, h->cp, h->opt, kMaxGrid, h->lay, err, &h->part, rank);
        if (st != LOPF_OK) { delete h; return fail(st, err); }
        add_fetch_stage(h);
    } catch (const std::bad_alloc&) {
        delete h;
        return fail(LOPF_E_ARG, "out of host memory during setup");
    } catch (const std::exception& ex) {
        delete h;
        return fail(LOPF_E_ARG, std::string("setup failed: ") + ex.what());
    }
    *out = h;
    return LOPF_OK;
}

lopf_status lopf_part_info(const lopf_handle* h, int64_t* xbuf_offset, int64_t* xbuf_doubles, int32_t* n_bnd,
                           int32_t* n_imp) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->parted()) return fail(LOPF_E_STATE, "not a partitioned handle (lopf_setup_part)");
    if (xbuf_offset) *xbuf_offset = (int64_t)h->lay.off_xbuf;
    if (xbuf_doubles) *xbuf_doubles = (int64_t)h->lay.n_bnd + 8LL * h->lay.world;
    if (n_bnd) *n_bnd = h->lay.n_bnd;
    if (n_imp) *n_imp = h->lay.n_imp;
    return LOPF_OK;
}

lopf_status lopf_part_owner(const lopf_handle* h, int32_t* bus_owner, int32_t* copy_owner, int32_t* bidx) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->parted()) return fail(LOPF_E_STATE, "not a partitioned handle (lopf_setup_part)");
    if (bus_owner) std::copy(h->part.bus_owner.begin(), h->part.bus_owner.end(), bus_owner);
    if (copy_owner) std::copy(h->part.copy_owner.begin(), h->part.copy_owner.end(), copy_owner);
    if (bidx) std::copy(h->part.bidx.begin(), h->part.bidx.end(), bidx);
    return LOPF_OK;
}

lopf_status lopf_part_sweep(lopf_handle* h, void* stream) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->parted()) return fail(LOPF_E_STATE, "not a partitioned handle (lopf_setup_part)");
    if (!h->bound) return fail(LOPF_E_STATE, "lopf_part_sweep before lopf_bind");
    DevProblem P = h->dp;
    P.max_iter = 1;
    P.test = 0;
    std::string err;
    lopf_status st = launch_solve(P, h->grid, stream, err);
    return st == LOPF_OK ? LOPF_OK : fail(st, err);
}

lopf_status lopf_part_import(lopf_handle* h, void* stream) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->parted()) return fail(LOPF_E_STATE, "not a partitioned handle (lopf_setup_part)");
    if (!h->bound) return fail(LOPF_E_STATE, "lopf_part_import before lopf_bind");
    DevProblem P = h->dp;
    P.test = 1;
    std::string err;
    lopf_status st = launch_part_import(P, stream, err);
    if (st != LOPF_OK) return fail(st, err);
    CUDA_TRY(cudaMemsetAsync(h->dp.xbuf, 0, sizeof(double) * ((size_t)h->lay.n_bnd + 8 * (size_t)h->lay.world),
                             (cudaStream_t)stream), "exchange clear");
    return LOPF_OK;
}

lopf_status lopf_sizes_get(const lopf_handle* h, lopf_sizes* sz) {
    if (!h || !sz) return fail(LOPF_E_ARG, "NULL argument");
    std::memset(sz, 0, sizeof(*sz));
    const Canon& P = h->cp;
    sz->S = P.S; sz->n = P.n; sz->m = P.m; sz->n_copies = P.nc;
    int64_t psym = 0;
    int mx = 0, mm = 0;
    for (int64_t s = 0; s < P.S; ++s) {
        psym += (int64_t)P.n_s[s] * (P.n_s[s] + 1) / 2;
        mx = std::max(mx, P.n_s[s]);
        mm = std::max(mm, P.m_raw[s]);
    }
    sz->p_sym = psym;
    sz->max_ns = mx; sz->max_ms = mm;
    sz->n_tasks = h->lay.n_tasks;
    sz->n_slots = h->lay.n_slots;
    sz->device_bytes = (int64_t)h->lay.bytes;
    sz->abar_doubles = h->lay.abar_doubles;
    // algorithmic bytes per sweep: packed symmetric Abar + bbar of load-bearing
    // subsystems + 6 per-copy streams (lambda, x_s rd+wr; u wr+rd) + 4 per-global (x wr+rd, lo, hi)
    // + c nonzeros, in fp64; plus the int32 copy->global map and CSR.
    int64_t nbbar = 0, psym_var = 0;
    for (int64_t s = 0; s < P.S; ++s) {
        bool any = false;
        for (int64_t r = P.b_ptr[s]; r < P.b_ptr[s + 1]; ++r) any |= P.b[r] != 0.0;
        if (any) {
            nbbar += P.n_s[s];
            psym_var += (int64_t)P.n_s[s] * (P.n_s[s] + 1) / 2;
        }
    }
    const int64_t E = h->lay.esz;           // 8 (fp64) or 4 (fp32 variant): the (T) arrays
    sz->alg_bytes = E * (psym + nbbar + 6 * P.nc + 4 * P.n + h->lay.n_obj) + 4 * (2 * P.nc + P.n + 1);
    if (h->batch()) {                       // per batch sweep: what all scenarios share once (the operators of the
        const int64_t ns = h->lay.n_scen;   // subsystems without a load, lo, hi, c), per scenario the rest: its
        sz->alg_bytes = E * ((psym - psym_var) + 2 * P.n + h->lay.n_obj +     // operators and b-bar, the
                             ns * (psym_var + nbbar + 6 * P.nc + 2 * P.n)) +   // 6 N_c iterate terms, x (w + r)
                        4 * (2 * P.nc + P.n + 1);
    }
    sz->kernel = h->lay.kernel;
    if (h->resident()) {                    // diagnostics: boundary tasks, largest SMEM footprint
        int mt = 0;
        for (const auto& c : h->lay.hdr) mt = std::max(mt, c.n_tasks);
        sz->reserved[0] = mt;                 // largest task count of a CTA
        sz->reserved[1] = h->lay.max_smem;
    }
    sz->grid = h->resident() ? h->lay.G : h->grid;
    sz->block = h->resident() ? kResBlock : h->batch() ? batch_block(h->lay.task_rows_max, h->lay.esz) : stream_block(h->lay.rmax, h->lay.esz);
    sz->n_scen = h->batch() ? h->lay.n_scen : 0;
    sz->upload_bytes = (int64_t)h->lay.image.size();
    sz->fetch_bytes = (h->batch() || h->parted()) ? 0 : (int64_t)(64 + 8 * h->cp.n);
    return LOPF_OK;
}

lopf_status lopf_bind(lopf_handle* h, void* arena, size_t bytes, void* stream) {
    if (!h || !arena) return fail(LOPF_E_ARG, "NULL argument");
    if (bytes < h->lay.bytes) return fail(LOPF_E_ARG, "arena smaller than lopf_sizes.device_bytes");
    if (((uintptr_t)arena) & 255) return fail(LOPF_E_ARG, "arena must be 256-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    if (!h->registered) {   // pin the host image once so every (re)bind is a DMA from pinned memory
        if (cudaHostRegister(h->lay.image.data(), h->lay.image.size(), cudaHostRegisterDefault) == cudaSuccess)
            h->registered = true;
        else
            cudaGetLastError();
    }
    if (!h->ev0) {
        CUDA_TRY(cudaEventCreate(&h->ev0), "cudaEventCreate");
        CUDA_TRY(cudaEventCreate(&h->ev1), "cudaEventCreate");
    }
    CUDA_TRY(cudaMemcpyAsync(arena, h->lay.image.data(), h->lay.image.size(), cudaMemcpyHostToDevice, s), "bind H2D");
    const Layout& L = h->lay;
    uint8_t* b = (uint8_t*)arena;
    if (h->batch()) {                              // lane = scenario layout (pack_batch.cpp, batch.cu)
        BatchProblem& B = h->bp;
        B = BatchProblem{};
        B.n_scen = L.n_scen;
        B.n_grp = L.n_grp;
        B.n_rows = L.n_rows;
        B.n_tasks = (int32_t)L.n_tasks;
        B.ve = L.ve;
        B.ns_max = L.ns_max;
        B.trmax = L.task_rows_max;
        B.esz = L.esz;
        B.n_obj = (int32_t)L.n_obj;
        B.n = h->cp.n;
        B.rows = (const BRow*)(b + L.off_brow);
        B.subs = (const BSub*)(b + L.off_bsub);
        B.tasks = (const BTask*)(b + L.off_btask);
        B.seg_rows = (const int32_t*)(b + L.off_bseg);
        B.gpar = b + L.off_gpar;
        B.spool = b + L.off_bspool;
        B.vpool = b + L.off_bvpool;
        B.x0 = b + L.off_x0;
        B.xl = b + L.off_xl;
        B.lam = b + L.off_lam;
        B.u0 = b + L.off_u0;
        B.u1 = b + L.off_u1;
        B.x = b + L.off_x;
        B.partial = (double*)(b + L.off_bpart);
        B.res = (ScenResult*)(b + L.off_bres);
        B.stopped = (int32_t*)(b + L.off_bstop);
        B.gact = (uint32_t*)(b + L.off_bgact);
        B.cnt = (unsigned long long*)(b + L.off_bcnt);
        B.wpre = (const long long*)(b + L.off_bwpre);
        B.torder = (const int32_t*)(b + L.off_btorder);
        B.tunit_ptr = (const int32_t*)(b + L.off_btunp);
        B.tunits = (const int32_t*)(b + L.off_btun);
        B.obj_idx = (const int32_t*)(b + L.off_objidx);
        B.obj_c = (const double*)(b + L.off_objc);
        B.ctrl = (DevCtrl*)(b + L.off_ctrl);
        B.stage = (double*)(b + L.off_bstage);
        B.rho = h->opt.rho;
        B.inv_rho = 1.0 / h->opt.rho;
        B.eps_rel = h->opt.eps_rel;
        h->dp = DevProblem{};
        h->dp.ctrl = B.ctrl;
        std::string err;
        int grid = 0;
        lopf_status st = query_batch_grid(L.task_rows_max, L.esz, &grid, err);
        if (st != LOPF_OK) return fail(st, err);
        h->grid = grid;
        st = launch_reset_batch(B, stream, err);
        if (st != LOPF_OK) return fail(st, err);
        h->arena = arena;
        h->arena_bytes = bytes;
        h->bound = true;
        return LOPF_OK;
    }
    if (h->resident()) {
        std::string err;
        int sms = 0, optin = 0;
        lopf_status st = resident_capacity(&sms, &optin, err);
        if (st != LOPF_OK) return fail(st, err);
        if (L.G > sms) return fail(LOPF_E_ARG, "resident layout needs " + std::to_string(L.G) + " CTAs but the device has " +
                                                   std::to_string(sms) + " SMs (set max_ctas or kernel = 1)");
        if (L.max_smem + 4096 > optin) return fail(LOPF_E_ARG, "resident layout exceeds the per-CTA shared memory");
        ResProblem& R = h->rp;
        R.hdr = (const CtaHdr*)(b + L.off_hdr);
        R.blobs = b + L.off_blobs;
        R.xchg = (double*)(b + L.off_xchg);
        R.flags = (unsigned long long*)(b + L.off_flags);
        R.partial = (double*)(b + L.off_partial);
        R.ctrl = (DevCtrl*)(b + L.off_ctrl);
        R.trace = (double*)(b + L.off_trace);
        R.x = b + L.off_x;
        R.obj_idx = (const int32_t*)(b + L.off_objidx);
        R.obj_c = (const double*)(b + L.off_objc);
        R.x0 = b + L.off_x0r;
        R.n_exp = L.n_exp;
        R.G = L.G;
        R.n_obj = (int32_t)L.n_obj;
        R.trace_cap = L.trace_cap;
        R.trace_every = h->opt.trace_every;
        R.total_slots = L.total_slots;
        R.max_smem = L.max_smem;
        R.rho = h->opt.rho;
        R.inv_rho = 1.0 / h->opt.rho;
        R.eps_rel = h->opt.eps_rel;
        R.prof = h->opt.reserved[0] ? (long long*)(b + L.off_prof) : nullptr;   // diagnostics switch
        R.esz = L.esz;
        h->dp = DevProblem{};
        h->dp.ctrl = R.ctrl;
        h->dp.x = R.x;
        h->dp.trace = R.trace;
        h->grid = L.G;
        h->arena = arena;
        h->arena_bytes = bytes;
        h->bound = true;
        return LOPF_OK;
    }
    DevProblem& P = h->dp;
    P.n_tasks = (int32_t)L.n_tasks;
    P.rmax = L.rmax;
    P.esz = L.esz;
    P.n_slots = (int32_t)L.n_slots;
    P.n = h->cp.n;
    P.tasks = (const int4*)(b + L.off_tasks);
    P.s_meta = (const SlotMeta*)(b + L.off_meta);
    P.s_bbar = (const double*)(b + L.off_bbar);
    P.xl = (double*)(b + L.off_xl);
    P.lam = (double*)(b + L.off_lam);
    P.u0 = (double*)(b + L.off_u0);
    P.u1 = (double*)(b + L.off_u1);
    P.x0 = (const double*)(b + L.off_x0);
    P.gbnd = (const double2*)(b + L.off_gpar);
    P.gcost = (const double*)(b + L.off_gcost);
    P.seg_ptr = (const int32_t*)(b + L.off_segptr);
    P.seg_slot = (const int32_t*)(b + L.off_segslot);
    P.x = (double*)(b + L.off_x);
    P.abar = (const double*)(b + L.off_abar);
    P.partial = (double*)(b + L.off_partial);
    P.ctrl = (DevCtrl*)(b + L.off_ctrl);
    P.trace = (double*)(b + L.off_trace);
    P.obj_idx = (const int32_t*)(b + L.off_objidx);
    P.obj_c = (const double*)(b + L.off_objc);
    P.n_obj = (int32_t)L.n_obj;
    P.trace_cap = L.trace_cap;
    P.trace_every = h->opt.trace_every;
    P.rho = h->opt.rho;
    P.inv_rho = 1.0 / h->opt.rho;
    P.eps_rel = h->opt.eps_rel;
    P.adapt_every = h->opt.adapt_every;
    P.adapt_mu = h->opt.adapt_mu;
    P.adapt_tau = h->opt.adapt_tau;
    P.part = L.part; P.rank = L.rank; P.world = L.world; P.n_bnd = L.n_bnd;
    P.n_imp = L.n_imp; P.ghost0 = L.ghost0;
    P.xbuf = L.part ? (double*)(b + L.off_xbuf) : nullptr;
    P.s_exp = L.part ? (const int32_t*)(b + L.off_sexp) : nullptr;
    P.imp = L.part ? (const int32_t*)(b + L.off_imp) : nullptr;
    P.p2p = 0;
    P.xstride = (int64_t)L.n_bnd + 8 * (int64_t)L.world;
    if (L.part) {                                  // peer table: this rank's own entry (world 1 runs as is)
        P.peer_xe = (double2* const*)(b + L.off_peer);
        P.xent = (double2*)(b + L.off_xent);
        if (h->peer_tab.size() != (size_t)L.world) h->peer_tab.assign((size_t)L.world, 0);   // a re-bind keeps peers
        h->peer_tab[L.rank] = (uint64_t)(uintptr_t)P.xent;
        CUDA_TRY(cudaMemcpyAsync(b + L.off_peer, h->peer_tab.data(), 8 * h->peer_tab.size(), cudaMemcpyHostToDevice,
                                 s), "peer table H2D");
    }
    std::string err;
    int grid = 0;
    lopf_status st = query_grid(L.rmax, L.esz, &grid, err);
    if (st != LOPF_OK) return fail(st, err);
    grid = std::min(grid, kMaxGrid);
    if (h->opt.grid_cap > 0) grid = std::min(grid, h->opt.grid_cap);   // test hook: cap the grid
    h->grid = grid;
    P.grid = grid;
    h->arena = arena;
    h->arena_bytes = bytes;
    h->bound = true;
    return LOPF_OK;
}

lopf_status lopf_reset(lopf_handle* h, void* stream) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->bound) return fail(LOPF_E_STATE, "lopf_reset before lopf_bind");
    std::string err;
    lopf_status st = h->resident() ? launch_reset_resident(h->rp, stream, err)
                     : h->batch() ? launch_reset_batch(h->bp, stream, err)
                                  : launch_reset(h->dp, stream, err);
    if (st == LOPF_OK && h->parted()) {            // both exchange parities and the p2p sweep flags
        CUDA_TRY(cudaMemsetAsync(h->dp.xbuf, 0, sizeof(double) * (size_t)h->dp.xstride, (cudaStream_t)stream),
                 "exchange clear");
        CUDA_TRY(cudaMemsetAsync(h->dp.xent, 0, 16 * 2 * (size_t)h->dp.xstride, (cudaStream_t)stream), "entry clear");
    }
    return st == LOPF_OK ? LOPF_OK : fail(st, err);
}

lopf_status lopf_part_p2p_info(const lopf_handle* h, int64_t* entry_offset, int64_t* entry_bytes) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->parted()) return fail(LOPF_E_STATE, "not a partitioned handle (lopf_setup_part)");
    if (entry_offset) *entry_offset = (int64_t)h->lay.off_xent;
    if (entry_bytes) *entry_bytes = 16 * 2 * ((int64_t)h->lay.n_bnd + 8 * (int64_t)h->lay.world);
    return LOPF_OK;
}

lopf_status lopf_part_connect(lopf_handle* h, const uint64_t* peer_entries, void* stream) {
    if (!h || !peer_entries) return fail(LOPF_E_ARG, "NULL argument");
    if (!h->parted() || !h->bound) return fail(LOPF_E_STATE, "lopf_part_connect needs a bound partitioned handle");
    const int W = h->lay.world;
    for (int q = 0; q < W; ++q) {
        if (!peer_entries[q]) return fail(LOPF_E_ARG, "peer pointer " + std::to_string(q) + " is NULL");
        h->peer_tab[q] = peer_entries[q];
    }
    if (h->peer_tab[h->lay.rank] != (uint64_t)(uintptr_t)h->dp.xent)
        return fail(LOPF_E_ARG, "peer_entries[rank] must be this handle's own entry buffer");
    CUDA_TRY(cudaMemcpyAsync((uint8_t*)h->arena + h->lay.off_peer, h->peer_tab.data(), 8 * h->peer_tab.size(),
                             cudaMemcpyHostToDevice, (cudaStream_t)stream), "peer table H2D");
    return LOPF_OK;
}

static lopf_status p2p_arg(lopf_handle* h, int64_t max_iter, int32_t test) {
    if (!h || !h->parted() || !h->bound) return fail(LOPF_E_STATE, "p2p solve needs bound partitioned handles");
    for (int q = 0; q < h->lay.world; ++q)
        if (!h->peer_tab[q])
            return fail(LOPF_E_STATE, "rank " + std::to_string(h->lay.rank) + " is not connected to rank " +
                                          std::to_string(q) + " (lopf_part_connect)");
    h->p2p_arg = h->dp;
    h->p2p_arg.p2p = 1;
    h->p2p_arg.max_iter = max_iter;
    h->p2p_arg.test = test ? 1 : 0;
    return LOPF_OK;
}

lopf_status lopf_part_solve_p2p(lopf_handle* h, int64_t max_iter, int32_t test, void* stream) {
    if (max_iter < 0) return fail(LOPF_E_ARG, "max_iter must be >= 0");
    lopf_status st = p2p_arg(h, max_iter, test);
    if (st != LOPF_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    DevProblem* dev = (DevProblem*)((uint8_t*)h->arena + h->lay.off_parr);
    CUDA_TRY(cudaMemcpyAsync(dev, &h->p2p_arg, sizeof(DevProblem), cudaMemcpyHostToDevice, s), "p2p argument H2D");
    CUDA_TRY(cudaMemsetAsync(h->dp.ctrl, 0, 2 * sizeof(unsigned long long), s), "control clear");
    CUDA_TRY(cudaMemsetAsync(&h->dp.ctrl->trace_rows, 0, sizeof(long long), s), "control clear");
    CUDA_TRY(cudaEventRecord(h->ev0, s), "cudaEventRecord");
    std::string err;
    const int g = std::min(h->grid, p2p_max_group(h->lay.rmax, h->lay.esz, 1));
    if (max_iter > 0) {
        st = launch_p2p(dev, &h->p2p_arg, 1, g, h->lay.rmax, h->lay.esz, stream, err);
        if (st != LOPF_OK) return fail(st, err);
    }
    CUDA_TRY(cudaEventRecord(h->ev1, s), "cudaEventRecord");
    return LOPF_OK;
}

lopf_status lopf_part_emulate(lopf_handle* const* hs, int32_t world, int64_t max_iter, int32_t test, void* stream) {
    if (!hs || world < 1) return fail(LOPF_E_ARG, "need world >= 1 handles");
    if (max_iter < 0) return fail(LOPF_E_ARG, "max_iter must be >= 0");
    std::vector<uint64_t> xe(world);
    int rmax = 1, esz = 0;
    for (int q = 0; q < world; ++q) {
        lopf_handle* h = hs[q];
        if (!h || !h->parted() || !h->bound || h->lay.world != world || h->lay.rank != q)
            return fail(LOPF_E_ARG, "handle " + std::to_string(q) + " is not rank " + std::to_string(q) + " of a bound " +
                                        std::to_string(world) + "-rank partition");
        xe[q] = (uint64_t)(uintptr_t)h->dp.xent;
        rmax = std::max(rmax, h->lay.rmax);
        if (esz && esz != h->lay.esz) return fail(LOPF_E_ARG, "ranks of one emulation need the same precision");
        esz = h->lay.esz;
    }
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<DevProblem> args(world);
    for (int q = 0; q < world; ++q) {
        lopf_status st = lopf_part_connect(hs[q], xe.data(), stream);
        if (st != LOPF_OK) return st;
        st = p2p_arg(hs[q], max_iter, test);
        if (st != LOPF_OK) return st;
        args[q] = hs[q]->p2p_arg;
        CUDA_TRY(cudaMemsetAsync(hs[q]->dp.ctrl, 0, 2 * sizeof(unsigned long long), s), "control clear");
    }
    DevProblem* dev = (DevProblem*)((uint8_t*)hs[0]->arena + hs[0]->lay.off_parr);   // world entries
    hs[0]->p2p_arg = args[0];
    CUDA_TRY(cudaMemcpyAsync(dev, args.data(), sizeof(DevProblem) * world, cudaMemcpyHostToDevice, s), "p2p arguments H2D");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");             // `args` is a temporary
    const int g = p2p_max_group(rmax, esz, world);
    if (g < 1) return fail(LOPF_E_CUDA, "p2p emulation: no co-resident grid");
    std::string err;
    if (max_iter > 0) {
        lopf_status st = launch_p2p(dev, nullptr, world, g, rmax, esz, stream, err);
        if (st != LOPF_OK) return fail(st, err);
    }
    return LOPF_OK;
}

// ---- library-owned NCCL communicator for the host-driven partitioned mode ------------------------------
// libnccl.so.2 is opened at first use (the one torch has loaded, if any); its absence is LOPF_E_NCCL.
struct NcclApi {
    int (*get_unique_id)(void*) = nullptr;
    int (*comm_init_rank)(void**, int, const void*, int) = nullptr;   // ncclUniqueId passed by value (128 B)
    int (*all_reduce)(const void*, void*, size_t, int, int, void*, void*) = nullptr;
    int (*comm_destroy)(void*) = nullptr;
    const char* (*error_string)(int) = nullptr;
    bool ok = false;
};
struct NcclId { char b[128]; };
typedef int (*nccl_init_by_value_t)(void**, int, NcclId, int);
static NcclApi& nccl() {
    static NcclApi a;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (lib) {
            a.get_unique_id = (int (*)(void*))dlsym(lib, "ncclGetUniqueId");
            a.comm_init_rank = (int (*)(void**, int, const void*, int))dlsym(lib, "ncclCommInitRank");
            a.all_reduce = (int (*)(const void*, void*, size_t, int, int, void*, void*))dlsym(lib, "ncclAllReduce");
            a.comm_destroy = (int (*)(void*))dlsym(lib, "ncclCommDestroy");
            a.error_string = (const char* (*)(int))dlsym(lib, "ncclGetErrorString");
            a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy && a.error_string;
        }
    }
    return a;
}
static lopf_status nccl_fail(int r, const char* where) {
    g_err = std::string("NCCL error in ") + where + ": " + (nccl().error_string ? nccl().error_string(r) : "?");
    return LOPF_E_NCCL;
}

lopf_status lopf_nccl_unique_id(void* out) {
    if (!out) return fail(LOPF_E_ARG, "NULL argument");
    if (!nccl().ok) return fail(LOPF_E_NCCL, "libnccl.so.2 not available");
    const int r = nccl().get_unique_id(out);
    return r ? nccl_fail(r, "ncclGetUniqueId") : LOPF_OK;
}

lopf_status lopf_part_nccl_init(lopf_handle* h, const void* unique_id) {
    if (!h || !unique_id) return fail(LOPF_E_ARG, "NULL argument");
    if (!h->parted()) return fail(LOPF_E_STATE, "not a partitioned handle (lopf_setup_part)");
    if (!nccl().ok) return fail(LOPF_E_NCCL, "libnccl.so.2 not available");
    if (h->nccl_comm) return LOPF_OK;
    NcclId id;
    std::memcpy(id.b, unique_id, 128);
    void* comm = nullptr;
    const int r = ((nccl_init_by_value_t)(void*)nccl().comm_init_rank)(&comm, h->lay.world, id, h->lay.rank);
    if (r) return nccl_fail(r, "ncclCommInitRank");
    h->nccl_comm = comm;
    return LOPF_OK;
}

lopf_status lopf_part_step(lopf_handle* h, void* stream) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->nccl_comm) return fail(LOPF_E_STATE, "lopf_part_step needs lopf_part_nccl_init");
    lopf_status st = lopf_part_sweep(h, stream);
    if (st != LOPF_OK) return st;
    const int r = nccl().all_reduce(h->dp.xbuf, h->dp.xbuf, (size_t)h->dp.xstride, /*ncclFloat64*/ 8, /*ncclSum*/ 0,
                                    h->nccl_comm, stream);
    if (r) return nccl_fail(r, "ncclAllReduce");
    return lopf_part_import(h, stream);
}

// ---- CUDA IPC of a device allocation (for lopf_part_connect across processes on one node) -------------
// The driver's cuMemGetAddressRange gives the allocation base of an arbitrary device pointer (a torch
// tensor lives inside a caching-allocator block); libcuda is opened at first use so the library still
// loads on machines without a driver.
typedef int (*cuMemGetAddressRange_t)(unsigned long long*, size_t*, unsigned long long);
static cuMemGetAddressRange_t get_range_fn() {
    static cuMemGetAddressRange_t fn = nullptr;
    if (!fn) {
        void* lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        if (lib) fn = (cuMemGetAddressRange_t)dlsym(lib, "cuMemGetAddressRange_v2");
    }
    return fn;
}

lopf_status lopf_ipc_export(const void* dev_ptr, void* out) {
    if (!dev_ptr || !out) return fail(LOPF_E_ARG, "NULL argument");
    cuMemGetAddressRange_t fn = get_range_fn();
    if (!fn) return fail(LOPF_E_CUDA, "libcuda.so.1 / cuMemGetAddressRange not available");
    unsigned long long base = 0;
    size_t size = 0;
    if (fn(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0) return fail(LOPF_E_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t hd;
    CUDA_TRY(cudaIpcGetMemHandle(&hd, (void*)(uintptr_t)base), "cudaIpcGetMemHandle");
    std::memcpy(out, &hd, sizeof(hd));
    const int64_t off = (int64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
    std::memcpy((char*)out + sizeof(hd), &off, 8);
    return LOPF_OK;
}

lopf_status lopf_ipc_open(lopf_handle* h, const void* in, void** dev_ptr) {
    if (!h || !in || !dev_ptr) return fail(LOPF_E_ARG, "NULL argument");
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, in, sizeof(hd));
    int64_t off = 0;
    std::memcpy(&off, (const char*)in + sizeof(hd), 8);
    void* base = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    h->ipc_open.push_back(base);
    *dev_ptr = (char*)base + off;
    return LOPF_OK;
}

lopf_status lopf_solve_async(lopf_handle* h, int64_t max_iter, int32_t test, void* stream) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->bound) return fail(LOPF_E_STATE, "solve before lopf_bind");
    if (h->parted()) return fail(LOPF_E_STATE, "partitioned handle: drive it with lopf_part_sweep / lopf_part_import");
    if (max_iter < 0) return fail(LOPF_E_ARG, "max_iter must be >= 0");
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(cudaEventRecord(h->ev0, s), "cudaEventRecord");
    std::string err;
    lopf_status st;
    if (h->resident()) {
        ResProblem R = h->rp;
        R.max_iter = max_iter;
        R.test = test ? 1 : 0;
        R.epoch = ++h->epoch;
        st = launch_resident(R, stream, err);
    } else if (h->batch()) {
        BatchProblem B = h->bp;
        B.max_iter = max_iter;
        B.test = test ? 1 : 0;
        st = launch_batch(B, h->grid, stream, err);
    } else {
        DevProblem P = h->dp;
        P.max_iter = max_iter;
        P.test = test ? 1 : 0;
        st = launch_solve(P, h->grid, stream, err);
    }
    if (st != LOPF_OK) return fail(st, err);
    CUDA_TRY(cudaEventRecord(h->ev1, s), "cudaEventRecord");
    return LOPF_OK;
}

static lopf_status fetch_batch(lopf_handle* h, cudaStream_t s) {
    h->scen_res.resize(h->lay.n_scen);
    CUDA_TRY(cudaMemcpyAsync(h->scen_res.data(), h->bp.res, sizeof(ScenResult) * h->lay.n_scen, cudaMemcpyDeviceToHost, s),
             "batch results D2H");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return LOPF_OK;
}

lopf_status lopf_result_get(lopf_handle* h, void* stream, lopf_result* res) {
    if (!h || !res) return fail(LOPF_E_ARG, "NULL argument");
    if (!h->bound) return fail(LOPF_E_STATE, "result before lopf_bind");
    if (h->batch()) {
        lopf_status st = fetch_batch(h, (cudaStream_t)stream);
        if (st != LOPF_OK) return st;
        std::memset(res, 0, sizeof(*res));
        bool all = true, num = false;
        int64_t worst = -1;
        for (int32_t i = 0; i < h->lay.n_scen; ++i) {
            const ScenResult& R = h->scen_res[i];
            all &= R.status == 1;
            num |= R.status == 3;
            if (worst < 0 || R.iters > h->scen_res[worst].iters) worst = i;
            res->objective += R.objective;
        }
        const ScenResult& W = h->scen_res[worst];
        res->iters = W.iters;
        res->pres = W.res[0]; res->dres = W.res[1]; res->eps_prim = W.res[2]; res->eps_dual = W.res[3];
        res->outcome = all ? LOPF_CONVERGED : LOPF_MAX_ITER;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, h->ev0, h->ev1) == cudaSuccess) res->solve_ms = ms;
        else cudaGetLastError();
        if (num) return fail(LOPF_E_NUMERIC, "non-finite residual sum in a batch scenario");
        return LOPF_OK;
    }
    DevCtrl c;
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(cudaMemcpyAsync(&c, h->dp.ctrl, sizeof(DevCtrl), cudaMemcpyDeviceToHost, s), "result D2H");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    std::memset(res, 0, sizeof(*res));
    res->outcome = c.outcome;
    res->iters = c.iters;
    res->pres = c.res[0]; res->dres = c.res[1]; res->eps_prim = c.res[2]; res->eps_dual = c.res[3];
    res->objective = c.objective;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, h->ev0, h->ev1) == cudaSuccess) res->solve_ms = ms;
    else cudaGetLastError();
    if (c.numeric) return fail(LOPF_E_NUMERIC, "non-finite residual sum detected on the device at sweep " +
                                                   std::to_string(c.iters));
    return LOPF_OK;
}

lopf_status lopf_get_rho(lopf_handle* h, void* stream, double* rho, int64_t* changes) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->bound) return fail(LOPF_E_STATE, "get_rho before lopf_bind");
    if (h->opt.adapt_every == 0 || h->resident() || h->batch()) {
        if (rho) *rho = h->opt.rho;
        if (changes) *changes = 0;
        return LOPF_OK;
    }
    DevCtrl c;
    CUDA_TRY(cudaMemcpyAsync(&c, h->dp.ctrl, sizeof(DevCtrl), cudaMemcpyDeviceToHost, (cudaStream_t)stream), "rho D2H");
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream), "cudaStreamSynchronize");
    if (rho) *rho = c.rho_cur;
    if (changes) *changes = c.rho_changes;
    return LOPF_OK;
}

lopf_status lopf_fetch_async(lopf_handle* h, void* stream, void* host_buf) {
    if (!h || !host_buf) return fail(LOPF_E_ARG, "NULL argument");
    if (!h->bound) return fail(LOPF_E_STATE, "fetch before lopf_bind");
    if (h->batch() || h->parted()) return fail(LOPF_E_STATE, "lopf_fetch_async serves single-problem handles");
    uint8_t* stage = (uint8_t*)h->arena + h->lay.off_fetch;
    std::string err;
    lopf_status st = launch_fetch(h->dp.ctrl, h->dp.x, h->cp.n, h->lay.esz, stage, stream, err);
    if (st != LOPF_OK) return fail(st, err);
    CUDA_TRY(cudaMemcpyAsync(host_buf, stage, 64 + 8 * (size_t)h->cp.n, cudaMemcpyDeviceToHost, (cudaStream_t)stream),
             "fetch D2H");
    return LOPF_OK;
}

lopf_status lopf_run(lopf_handle* h, int64_t k, int32_t test, void* stream, lopf_result* res) {
    lopf_status st = lopf_solve_async(h, k, test, stream);
    if (st != LOPF_OK) return st;
    if (k == 0) {
        if (res) std::memset(res, 0, sizeof(*res)), res->outcome = LOPF_MAX_ITER;
        return LOPF_OK;
    }
    return res ? lopf_result_get(h, stream, res) : LOPF_OK;
}

lopf_status lopf_solve(lopf_handle* h, void* stream, lopf_result* res) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    return lopf_run(h, h->opt.max_iter, 1, stream, res);
}

lopf_status lopf_get_decomposition(const lopf_handle* h, int32_t* kind, int32_t* comp, int32_t* leaf, int32_t* m_s,
                                   int32_t* n_s, int64_t* sub_ptr, int32_t* copy_global) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    const Canon& P = h->cp;
    if (kind) std::copy(P.kind.begin(), P.kind.end(), kind);
    if (comp) std::copy(P.comp.begin(), P.comp.end(), comp);
    if (leaf) std::copy(P.leaf.begin(), P.leaf.end(), leaf);
    if (m_s) std::copy(P.m_raw.begin(), P.m_raw.end(), m_s);
    if (n_s) std::copy(P.n_s.begin(), P.n_s.end(), n_s);
    if (sub_ptr) std::copy(P.sub_ptr.begin(), P.sub_ptr.end(), sub_ptr);
    if (copy_global) std::copy(P.copy_global.begin(), P.copy_global.end(), copy_global);
    return LOPF_OK;
}

lopf_status lopf_get_consensus(const lopf_handle* h, int64_t* row_ptr, int32_t* copy_idx) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (row_ptr) std::copy(h->cp.seg_ptr.begin(), h->cp.seg_ptr.end(), row_ptr);
    if (copy_idx) std::copy(h->cp.seg_copy.begin(), h->cp.seg_copy.end(), copy_idx);
    return LOPF_OK;
}

lopf_status lopf_get_globals(const lopf_handle* h, int32_t* role, int32_t* comp, int32_t* phase, double* c, double* lo,
                             double* hi) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    const Canon& P = h->cp;
    for (int64_t i = 0; i < P.n; ++i) {
        if (role) role[i] = P.var[i].role;
        if (comp) comp[i] = P.var[i].comp;
        if (phase) phase[i] = P.var[i].phase;
    }
    if (c) std::copy(P.c.begin(), P.c.end(), c);
    if (lo) std::copy(P.lo.begin(), P.lo.end(), lo);
    if (hi) std::copy(P.hi.begin(), P.hi.end(), hi);
    return LOPF_OK;
}

lopf_status lopf_get_operator(const lopf_handle* h, int64_t s, double* abar, double* bbar) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    const Canon& P = h->cp;
    if (s < 0 || s >= P.S) return fail(LOPF_E_ARG, "subsystem index out of range");
    if (abar) std::copy(P.abar.begin() + P.abar_ptr[s], P.abar.begin() + P.abar_ptr[s + 1], abar);
    if (bbar) std::copy(P.bbar.begin() + P.sub_ptr[s], P.bbar.begin() + P.sub_ptr[s + 1], bbar);
    return LOPF_OK;
}

lopf_status lopf_get_subsystem(const lopf_handle* h, int64_t s, double* A, double* b, int32_t* m_out) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    const Canon& P = h->cp;
    if (s < 0 || s >= P.S) return fail(LOPF_E_ARG, "subsystem index out of range");
    if (A) std::copy(P.A.begin() + P.a_ptr[s], P.A.begin() + P.a_ptr[s + 1], A);
    if (b) std::copy(P.b.begin() + P.b_ptr[s], P.b.begin() + P.b_ptr[s + 1], b);
    if (m_out) *m_out = P.m_s[s];
    return LOPF_OK;
}

// slot-ordered x_s / lambda of the current device iterate (streaming: flat slot arrays; resident:
// per-CTA blob regions concatenated in global slot order)
static lopf_status fetch_slots(lopf_handle* h, cudaStream_t s, std::vector<double>& xl, std::vector<double>& lm) {
    const Layout& L = h->lay;
    xl.assign(L.n_slots, 0.0);
    lm.assign(L.n_slots, 0.0);
    if (!h->resident()) {
        CUDA_TRY(d2h_elems(xl.data(), h->dp.xl, L.n_slots, L.esz, s), "state D2H");
        CUDA_TRY(d2h_elems(lm.data(), h->dp.lam, L.n_slots, L.esz, s), "state D2H");
    } else {                                       // one gather kernel over the CTA blobs, one copy
        uint8_t* stage = (uint8_t*)h->arena + L.off_fetch;
        std::string err;
        lopf_status st = launch_gather_resident(h->rp, stage, s, err);
        if (st != LOPF_OK) return fail(st, err);
        std::vector<double> both(2 * (size_t)L.n_slots);
        CUDA_TRY(d2h_elems(both.data(), stage, both.size(), 8, s), "state D2H");
        std::copy(both.begin(), both.begin() + L.n_slots, xl.begin());
        std::copy(both.begin() + L.n_slots, both.end(), lm.begin());
    }
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return LOPF_OK;
}

lopf_status lopf_get_state(lopf_handle* h, void* stream, double* x, double* x_loc, double* lam) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->bound) return fail(LOPF_E_STATE, "get_state before lopf_bind");
    if (h->batch()) return fail(LOPF_E_STATE, "batch handle: use lopf_get_state_scen");
    cudaStream_t s = (cudaStream_t)stream;
    const Layout& L = h->lay;
    if (x) CUDA_TRY(d2h_elems(x, h->dp.x, h->cp.n, L.esz, s), "state D2H");
    if (x_loc || lam) {
        std::vector<double> xl, lm;
        lopf_status st = fetch_slots(h, s, xl, lm);
        if (st != LOPF_OK) return st;
        for (int64_t k = 0; k < h->cp.nc; ++k) {
            const bool here = !h->parted() || h->part.copy_owner[k] == h->lay.rank;   // partitioned: own copies
            if (x_loc) x_loc[k] = here ? xl[L.slot_of_copy[k]] : NAN;
            if (lam) lam[k] = here ? lm[L.slot_of_copy[k]] : NAN;
        }
    } else {
        CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
    if (x && h->parted())                          // x_g is this rank's where its first copy is
        for (int64_t g = 0; g < h->cp.n; ++g)
            if (h->part.copy_owner[h->cp.seg_copy[h->cp.seg_ptr[g]]] != h->lay.rank) x[g] = NAN;
    return LOPF_OK;
}

lopf_status lopf_set_state(lopf_handle* h, void* stream, const double* x_loc, const double* lam) {
    if (!h || !x_loc || !lam) return fail(LOPF_E_ARG, "NULL argument");
    if (h->parted()) return fail(LOPF_E_STATE, "lopf_set_state is not supported on a partitioned handle");
    if (h->batch()) return fail(LOPF_E_STATE, "lopf_set_state is not supported on a batch handle (the u parity is "
                                              "shared by all scenarios)");
    if (!h->bound) return fail(LOPF_E_STATE, "set_state before lopf_bind");
    cudaStream_t s = (cudaStream_t)stream;
    const Layout& L = h->lay;
    std::vector<double> xl(L.n_slots, 0.0), lm(L.n_slots, 0.0), u(L.n_slots, 0.0), z(L.n_slots, 0.0);
    const double inv_rho = 1.0 / h->opt.rho;
    for (int64_t k = 0; k < h->cp.nc; ++k) {
        const int32_t sl = L.slot_of_copy[k];
        xl[sl] = x_loc[k];
        lm[sl] = lam[k];
        u[sl] = x_loc[k] - lam[k] * inv_rho;
    }
    if (!h->resident()) {
        CUDA_TRY(h2d_elems(h->dp.xl, xl.data(), L.n_slots, L.esz, s), "state H2D");
        CUDA_TRY(h2d_elems(h->dp.lam, lm.data(), L.n_slots, L.esz, s), "state H2D");
        CUDA_TRY(h2d_elems(h->dp.u0, u.data(), L.n_slots, L.esz, s), "state H2D");
    } else {
        for (int c = 0; c < L.G; ++c) {
            const CtaHdr& H = L.hdr[c];
            uint8_t* blob = h->rp.blobs + H.blob_off;
            CUDA_TRY(h2d_elems(blob + H.off_xl0, xl.data() + H.slot_base, H.n_slots, L.esz, s), "state H2D");
            CUDA_TRY(h2d_elems(blob + H.off_lam0, lm.data() + H.slot_base, H.n_slots, L.esz, s), "state H2D");
        }
    }
    CUDA_TRY(cudaMemsetAsync(&h->dp.ctrl->total, 0, sizeof(long long), s), "state memset");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return LOPF_OK;
}

lopf_status lopf_get_trace(lopf_handle* h, void* stream, double* buf, int64_t cap, int64_t* n_rows) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->bound) return fail(LOPF_E_STATE, "get_trace before lopf_bind");
    cudaStream_t s = (cudaStream_t)stream;
    DevCtrl c;
    CUDA_TRY(cudaMemcpyAsync(&c, h->dp.ctrl, sizeof(DevCtrl), cudaMemcpyDeviceToHost, s), "trace D2H");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    int64_t rows = std::min<int64_t>(c.trace_rows, cap);
    if (buf && rows > 0) {
        CUDA_TRY(cudaMemcpyAsync(buf, h->dp.trace, sizeof(double) * 5 * rows, cudaMemcpyDeviceToHost, s), "trace D2H");
        CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
    if (n_rows) *n_rows = rows;
    return LOPF_OK;
}

lopf_status lopf_get_batch_results(lopf_handle* h, void* stream, int64_t* iters, int32_t* outcome, double* res,
                                   double* objective) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->batch() || !h->bound) return fail(LOPF_E_STATE, "batch results need a bound batch handle");
    lopf_status st = fetch_batch(h, (cudaStream_t)stream);
    if (st != LOPF_OK) return st;
    for (int32_t i = 0; i < h->lay.n_scen; ++i) {
        const ScenResult& R = h->scen_res[i];
        if (iters) iters[i] = R.iters;
        if (outcome) outcome[i] = R.status == 1 ? LOPF_CONVERGED : R.status == 3 ? (int32_t)LOPF_E_NUMERIC : LOPF_MAX_ITER;
        if (res) for (int q = 0; q < 4; ++q) res[4 * i + q] = R.res[q];
        if (objective) objective[i] = R.objective;
    }
    return LOPF_OK;
}

lopf_status lopf_get_state_scen(lopf_handle* h, void* stream, int32_t scen, double* x, double* x_loc, double* lam) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->batch() || !h->bound) return fail(LOPF_E_STATE, "per-scenario state needs a bound batch handle");
    if (scen < 0 || scen >= h->lay.n_scen) return fail(LOPF_E_ARG, "scenario index out of range");
    cudaStream_t s = (cudaStream_t)stream;
    const Layout& L = h->lay;
    std::string err;
    lopf_status st = launch_gather_scen(h->bp, scen, stream, err);     // one gather kernel, one D2H
    if (st != LOPF_OK) return fail(st, err);
    const size_t nr = (size_t)L.n_rows, n = (size_t)h->cp.n;
    std::vector<double> stage(2 * nr + n);
    CUDA_TRY(d2h_elems(stage.data(), h->bp.stage, stage.size(), 8, s), "state D2H");
    for (int64_t k = 0; k < h->cp.nc; ++k) {
        if (x_loc) x_loc[k] = stage[L.slot_of_copy[k]];
        if (lam) lam[k] = stage[nr + L.slot_of_copy[k]];
    }
    if (x) std::copy(stage.begin() + 2 * nr, stage.end(), x);
    return LOPF_OK;
}

lopf_status lopf_get_operator_scen(const lopf_handle* h, int64_t s, int32_t scen, double* abar, double* bbar) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    const Canon& P = h->cp;
    if (s < 0 || s >= P.S) return fail(LOPF_E_ARG, "subsystem index out of range");
    if (!h->batch()) return lopf_get_operator(h, s, abar, bbar);
    if (scen < 0 || scen >= h->lay.n_scen) return fail(LOPF_E_ARG, "scenario index out of range");
    const int32_t v = h->bo.vidx[s];
    if (v < 0) return lopf_get_operator(h, s, abar, bbar);
    const size_t a0 = (size_t)scen * h->bo.VA + h->bo.va_off[v], b0 = (size_t)scen * h->bo.VB + h->bo.vb_off[v];
    if (abar) std::copy(h->bo.abar.begin() + a0, h->bo.abar.begin() + a0 + (size_t)P.n_s[s] * P.n_s[s], abar);
    if (bbar) std::copy(h->bo.bbar.begin() + b0, h->bo.bbar.begin() + b0 + P.n_s[s], bbar);
    return LOPF_OK;
}

lopf_status lopf_get_profile(lopf_handle* h, void* stream, int64_t* buf, int64_t cap, int64_t* n_rows) {
    if (!h) return fail(LOPF_E_ARG, "NULL handle");
    if (!h->bound || !h->resident() || !h->rp.prof) return fail(LOPF_E_STATE, "profiling needs the resident kernel with diagnostics enabled");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t rows = std::min<int64_t>(41 * (int64_t)h->lay.G, cap);   // G counter rows, then timeline events
    CUDA_TRY(cudaMemcpyAsync(buf, h->rp.prof, sizeof(int64_t) * 4 * rows, cudaMemcpyDeviceToHost, s), "profile D2H");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    if (n_rows) *n_rows = rows;
    return LOPF_OK;
}

void lopf_destroy(lopf_handle* h) {
    if (!h) return;
    for (void* p : h->ipc_open) cudaIpcCloseMemHandle(p);
    if (h->nccl_comm && nccl().ok) nccl().comm_destroy(h->nccl_comm);
    if (h->registered) cudaHostUnregister(h->lay.image.data());
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    cudaGetLastError();
    delete h;
}

}  // extern "C"

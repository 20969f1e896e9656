// Internal data structures of liblopf (NOT part of the ABI; see include/lopf.h).
//
// Host side (setup.cpp): an independent C++ implementation of the LP assembly
// (PAPER.md:109-227), the component decomposition and the operator
// precompute by Cholesky.  Device side (kernels.cu): the fused ADMM
// sweep.  pack.cpp turns the canonical problem into the device layouts described in
// DESIGN.md §4.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <vector_types.h>

#include "../../include/lopf.h"

namespace lopf {

enum Role : int8_t { PG = 0, QG, W, PB, QB, PD, QD, PF, QF, PT, QT };
enum Kind : int32_t { BUS = 0, LINE = 1, LEAF = 2, COARSE = 3 };

struct Var {
    int8_t role;
    int8_t phase;
    int32_t comp;
};

// Host copy of the network (validated).
struct Net {
    int32_t n_bus = 0, n_line = 0, n_gen = 0, n_load = 0, root = 0;
    std::vector<uint8_t> bus_ph, line_ph, gen_ph, load_ph, load_conn;
    std::vector<double> bus_wmin, bus_wmax, bus_gsh, bus_bsh;
    std::vector<int32_t> line_from, line_to, gen_bus, load_bus;
    std::vector<double> line_r, line_x, line_gsf, line_bsf, line_gst, line_bst, line_tau;
    std::vector<double> line_pmin, line_pmax, line_qmin, line_qmax;
    std::vector<double> gen_pmin, gen_pmax, gen_qmin, gen_qmax;
    std::vector<double> load_alpha, load_beta, load_a, load_b;
};

// Canonical problem: globals, subsystems, operators (everything in canonical order).
struct Canon {
    int64_t n = 0, m = 0, S = 0, nc = 0;
    std::vector<Var> var;
    std::vector<double> c, lo, hi;
    std::vector<int32_t> kind, comp, leaf, m_s, n_s;      // [S]; m_s after row reduction
    std::vector<int32_t> m_raw;                            // [S] rows before reduction
    std::vector<int64_t> sub_ptr;                          // [S+1] copy offsets
    std::vector<int32_t> copy_global;                      // [nc]
    std::vector<int64_t> seg_ptr;                          // [n+1]
    std::vector<int32_t> seg_copy;                         // [nc]
    std::vector<int64_t> a_ptr;                            // [S+1] offsets of dense A_s (reduced rows)
    std::vector<double> A, b;                              // dense A_s row-major; b_s (b_ptr = row offsets)
    std::vector<int64_t> b_ptr;                            // [S+1]
    std::vector<int64_t> abar_ptr;                         // [S+1] offsets of dense n_s x n_s Abar_s
    std::vector<double> abar, bbar;                        // bbar [nc]
    std::vector<double> x0;                                // [nc] initial x_s
};

// ---- device layout shared by pack.cpp and kernels.cu ---------------------------------------
// Slot info bit fields (streaming kernel).
constexpr int kInfoBaseMask = 0x3F;        // slot index (in its task) of the subsystem's first row
constexpr int kInfoCost = 1 << 6;          // the global has c != 0 (a p^g column): read c/rho
constexpr int kInfoExport = 1 << 7;        // partitioned mode: boundary copy, its u goes to the exchange buffer
constexpr int kInfoValid = 1 << 8;
constexpr int kInfoFirst = 1 << 9;         // first copy (canonical) of its global: writes x_g
constexpr int kInfoInline = 1 << 10;       // segment slots stored inline (nu <= 4)
constexpr int kInfoBbar = 1 << 11;         // the subsystem has a nonzero b-bar (load-bearing): read it
constexpr int kInfoNuShift = 12;           // nu (4 bits, capped at 15; used when inline)
constexpr int kInfoNsShift = 16;           // n_s (6 bits; packed tasks)
constexpr int kInfoPoffShift = 22;         // offset (doubles) of the subsystem's packed Abar in its task
// Task record {slot_off, abar_off, kmax | plen, R | flags}
constexpr int kTaskPacked = 1 << 4;        // packed task: .z = block doubles, kmax in bits 8..15 of .w
constexpr int kTaskDirect = 1 << 5;        // packed task whose block exceeds the stage: read from HBM
constexpr int kTaskKmaxShift = 8;
constexpr int kTaskVar = 1 << 6;           // batch: the task's operator block is per scenario (holds a load)
constexpr int kTaskUsedShift = 16;         // packed task: slots in use (rounded up to 4), bits 16..23 of .w
constexpr int kTaskHalves = 2;             // streaming packer: max 32-slot halves per packed task
#ifndef LOPF_PACK_BUDGET
#define LOPF_PACK_BUDGET 448
#endif
constexpr int kPackBudget = LOPF_PACK_BUDGET;  // operator-block entries (fp64 or fp32) per staged task (per-warp SMEM stage)

struct DevCtrl {                           // 256 B, device-resident control block
    unsigned long long arrive;             // barrier arrivals of this launch
    unsigned long long flag;               // (iteration << 2) | (stop << 1) | numeric
    long long total;                       // sweeps since reset (u ping-pong parity)
    long long iters;                       // sweeps executed by the last launch
    int outcome, numeric;
    double res[4];                         // pres, dres, eps_prim, eps_dual of the last sweep
    double objective;
    long long trace_rows;
    long long stopped;                     // partitioned mode: the termination test has fired
    double rho_cur;                        // residual balancing (F2): the penalty in force
    long long rho_changes;                 // ... and how often it changed since the reset
    unsigned long long arrive2;            // second barrier counter (u re-formed after a rho change)
    double pad[15];
};

// Per-slot metadata of the streaming / batch layouts, one 24-byte record (one bulk copy per task):
// the inline segment slots (nu <= 4, canonical copy order), the info bit field and the global index.
struct alignas(8) SlotMeta {
    int2 n01, n23;
    int32_t info, g;
};
static_assert(sizeof(SlotMeta) == 24, "SlotMeta is 24 bytes");

// Arrays marked (T) hold doubles when esz == 8 and floats when esz == 4 (the fp32 variant, reading F1:
// the paper's GPU precision); the kernels cast them to the element type they were
// instantiated for.  Residual sums, partials, trace, objective coefficients and the exchange are fp64.
struct DevProblem {                        // kernel argument (pointers into the arena)
    int32_t n_tasks, n_slots, grid, rmax;  // rmax: widest task (selects the kernel instantiation)
    int32_t esz;                           // element size of operators / iterate / globals: 8 (fp64) or 4 (fp32)
    int64_t n;
    const int4* tasks;                     // {slot_off, abar_off, kmax, R}
    const SlotMeta* s_meta;                // per-slot {inline segment slots, info, global}: one record
    const void* s_bbar;                    // (T)
    void* xl;                              // (T)
    void* lam;                             // (T)
    void* u0;                              // (T)
    void* u1;                              // (T)
    const void* x0;                        // (T) initial x_s per slot
    const void* gbnd;                      // (T) {lo, hi} per global
    const void* gcost;                     // (T) c/rho per global (read for kInfoCost slots only)
    const int32_t* seg_ptr;                // [n+1] into seg_slot
    const int32_t* seg_slot;               // [nc] slots in canonical copy order
    void* x;                               // (T) [n]
    const void* abar;                      // (T) packed operator pool
    double* partial;                       // [grid * 8]
    DevCtrl* ctrl;
    double* trace;                         // [trace_cap * 5]
    const int32_t* obj_idx;                // globals with c != 0
    const double* obj_c;
    int32_t n_obj, trace_cap, trace_every, test;
    double rho, inv_rho, eps_rel;
    long long max_iter;
    int32_t adapt_every, pad_a;            // residual balancing every k sweeps (0 = fixed rho; F2)
    double adapt_mu, adapt_tau;
    // partitioned mode (config 5): one sweep per launch, exchange through `xbuf`
    int32_t part, rank, world, n_bnd;      // n_bnd boundary-copy slots, then world x 8 residual slots
    double* xbuf;
    const int32_t* s_exp;                  // [n_slots] exchange slot of an exported copy (kInfoExport)
    const int32_t* imp;                    // [n_imp] exchange slot feeding each ghost slot
    int32_t n_imp, ghost0;                 // ghost slots ghost0 .. ghost0 + n_imp - 1 (after the task slots)
    // device-initiated exchange: every rank's tagged exchange entries {value, sweep + 1} [2][xstride]
    int32_t p2p, pad_p;
    int64_t xstride;                       // n_bnd + 8 world entries per parity
    double2* const* peer_xe;               // [world] each rank's entry buffer (this rank's at [rank])
    double2* xent;                         // this rank's entry buffer
};

// ---- resident kernel (operators + iterate in shared memory) -----------------------------------
// Every CTA owns a DFS-contiguous chunk of subsystems.  Its BLOB (global memory) is copied into
// SMEM at kernel start; the iterate (x_s, lambda, u) lives in SMEM for the whole launch and is
// written back at the end.  Offsets are bytes from the blob start.
#ifndef LOPF_RES_BLOCK
#define LOPF_RES_BLOCK 768
#endif
constexpr int kResBlock = LOPF_RES_BLOCK;     // worker warps + 1 reducer warp (768: 80 registers, no spills)
constexpr int kResSmemBudget = 222 * 1024;    // dynamic SMEM per CTA (227 KB usable on sm_100, minus static)
// sinfo: base (bits 0-5, first slot of the subsystem in its task) | valid (bit 6) | first (bit 7: this slot
// is the canonical first copy of a global whose x this CTA outputs) | consensus flags of the slot's global
// (bit 14) | gl (bits 15-31).  Every copy a CTA reads has an SMEM slot: its own copies [0, n_slots), the
// zero slot n_slots (x = lambda = 0), and a ghost slot per copy owned by another CTA (x = u imported from the
// exchange buffer by each task that reads it, lambda = 0).  A global with nu <= 4 has a record grec of the
// slots of its copies in canonical order, padded with the zero slot; one with nu > 4 ("slow") has gxb =
// {first entry, nu} of its slot list in gseg.
constexpr int kResValid = 1 << 6;
constexpr int kResFirst = 1 << 7;
constexpr int kResSlow = 1 << 14;             // nu > 4: the global's list in gseg
constexpr int kResGlShift = 15;

struct CtaHdr {                               // 128 B, one per CTA
    int32_t n_tasks, n_slots, n_glob, n_seg, n_ghost;
    int32_t blob_bytes, smem_bytes;
    // blob (global and SMEM): constant part then the state (x_s, lambda of sweep parity 0)
    int32_t off_abar, off_bbar, off_gpar, off_tasks, off_sinfo, off_sexp, off_grec, off_gxb, off_gseg,
        off_gimp, off_xl0, off_lam0;
    int32_t off_gown;                         // blob only, past blob_bytes (read from global memory at exit)
    // SMEM only (after the blob)
    int32_t off_xl1, off_lam1, off_xout, off_dst, dst_stride;
    int32_t slot_base;
    long long blob_off;
    int32_t pad[1];
};
static_assert(sizeof(CtaHdr) <= 128, "CtaHdr is loaded by the first 32 threads");

struct ResProblem {                           // resident kernel argument
    const CtaHdr* hdr;
    uint8_t* blobs;
    double* xchg;                             // [2][n_exp] {u, tag} 16-byte boundary entries (by sweep parity)
    double* partial;                          // [2][G][8] residual partials (ping-pong by sweep parity)
    unsigned long long* flags;                // [G] sweeps published by each CTA (+1), zeroed per launch
    DevCtrl* ctrl;
    double* trace;
    void* x;                                  // (T) [n] solution
    const int32_t* obj_idx;
    const double* obj_c;
    const void* x0;                           // (T) [total slots] initial x_s, blob slot order
    int32_t n_exp, G, n_obj, test;
    int32_t trace_cap, trace_every, total_slots, max_smem;
    double rho, inv_rho, eps_rel;
    long long max_iter;
    long long* prof;                          // diagnostics: [G][4] cycles (work, publish+wait, -, sweeps) or NULL
    uint32_t epoch;                           // launch number (> 0): high half of the exchange tags
    int32_t esz;                              // element size of the SMEM state / blob arrays: 8 fp64, 4 fp32 (F1)
};

// ---- batch kernel (config 4): lane = scenario ------------------------------------
// Scenarios form groups of 32 (group g, lane l = scenario 32 g + l).  Every per-scenario array is
// [group][entry][32]: one warp instruction touches one 256-byte line for 32 scenarios, and every
// structural datum (rows, subsystems, shared operators) is the same for the 32 lanes (uniform loads).
// Rows are the copies in depth-first subsystem order; a work item is (group, task), a task a DFS run
// of subsystems.

struct ScenResult {                            // 64 B per scenario (device)
    long long iters;                           // sweeps executed in the last launch
    long long total;                           // sweeps since reset (state parity)
    int status;                                // 0 running, 1 converged, 2 max_iter, 3 numeric
    int pad;
    double res[4];
    double objective;
};

constexpr int kBFirst = 1;                     // BRow.info: canonical first copy of its global (writes x_g)
constexpr int kBInline = 2;                    // segment rows inline (nu <= 4), else {offset, count} in seg_rows
constexpr int kBNuShift = 8;                   // nu in bits 8..15 (inline rows)
struct alignas(8) BRow {                       // 24 B per row (copy)
    int32_t g, info;
    int32_t n0, n1, n2, n3;                    // the segment's rows in canonical copy order (inline), or n0 = offset,
};                                             // n1 = count into seg_rows
static_assert(sizeof(BRow) == 24, "BRow is 24 bytes");
constexpr int kBVar = 1;                       // BSub.flags: per-scenario operator (the subsystem holds a load)
constexpr int kBBbar = 2;                      // ... with a nonzero b-bar after the triangle
// Per-scenario operator entries of an n_s-row subsystem in the quad-block upper layout (pack_batch.cpp):
// block q (rows 4q..4q+3) holds 4 entries for every column k in [4q, 4 ceil(n_s / 4)).
#ifdef __CUDACC__
#define LOPF_HD __host__ __device__
#else
#define LOPF_HD
#endif
#ifndef LOPF_BATCH_VQB64
#define LOPF_BATCH_VQB64 0                     // per-scenario operator layout, fp64: 1 quad-block upper, 0 packed
#endif                                         // upper triangle, row-major (A/B: 312 -> 307 us per batch sweep)
#ifndef LOPF_BATCH_VQB32
#define LOPF_BATCH_VQB32 1                     // the same for fp32 (A/B: quad-block 209 us, packed 257)
#endif
LOPF_HD constexpr bool batch_vqb(int esz) { return esz == 8 ? LOPF_BATCH_VQB64 : LOPF_BATCH_VQB32; }
LOPF_HD constexpr int batch_var_entries(int ns, bool vqb) {
    return vqb ? 8 * ((ns + 3) / 4) * ((ns + 3) / 4 + 1) : ns * (ns + 1) / 2;
}
struct BSub {                                  // 16 B per subsystem (DFS order)
    int32_t row0, ns, op, flags;               // op: shared dense Abar offset (T entries) or var-pool entry offset
};
struct BTask {                                 // 32 B per task: a DFS run of subsystems
    int32_t sub0, sub1, row0, row1;
    int32_t vop0, vop1;                        // its per-scenario operator entries [vop0, vop1) (contiguous)
    int32_t pad[2];
};

struct BatchProblem {
    int32_t n_scen, n_grp, n_rows, n_tasks, ve, ns_max, esz, n_obj;
    int64_t n;                                 // globals
    const BRow* rows;
    const BSub* subs;
    const BTask* tasks;
    const int32_t* seg_rows;                   // segments of nu > 4
    const void* gpar;                          // (T) [n][4] {c/rho, lo, hi, 1/nu}
    const void* spool;                         // (T) dense n_s x n_s Abar of the shared subsystems
    const void* vpool;                         // (T) [group][ve][32] packed upper triangle (+ b-bar) of load subsystems
    const void* x0;                            // (T) [n_rows] initial x_s
    void *xl, *lam, *u0, *u1;                  // (T) [group][n_rows][32]
    void* x;                                   // (T) [group][n][32]
    double* partial;                           // [group][n_tasks][5][32] residual sums per item
    ScenResult* res;                           // [n_scen]
    int32_t* stopped;                          // [n_scen] converged / non-finite: frozen
    uint32_t* gact;                            // [2][n_grp] group has an active scenario, by sweep parity
    unsigned long long* cnt;                   // barrier arrivals
    const long long* wpre;                     // [n_tasks + 1] prefix of the per-task cost weights (work split)
    const int32_t* torder;                     // [n_tasks] tasks by decreasing cost weight (dynamic hand-out order)
    const int32_t* tunit_ptr;                  // [n_tasks * kBatchTeamWarps + 1] each (task, team warp)'s units
    const int32_t* tunits;                     // unit = (subsystem - task.sub0) << 8 | row quad, per warp ascending
    const int32_t* obj_idx;
    const double* obj_c;
    DevCtrl* ctrl;
    double* stage;                             // gather staging for the per-scenario getters
    double rho, inv_rho, eps_rel;
    long long max_iter;
    int32_t test, trmax;                       // trmax: rows of the largest task
};
constexpr int kBatchMaxScen = 8192;            // scenarios per batch handle
constexpr int kBatchMaxGrp = kBatchMaxScen / 32;
#ifndef LOPF_BATCH_TASK_ROWS
#define LOPF_BATCH_TASK_ROWS 40
#endif
#ifndef LOPF_BATCH_TASK_ROWS32
#define LOPF_BATCH_TASK_ROWS32 48
#endif
constexpr int kBatchTaskRows = LOPF_BATCH_TASK_ROWS;     // rows per task (target; whole subsystems), fp64
constexpr int kBatchTaskRows32 = LOPF_BATCH_TASK_ROWS32; // the same for the fp32 variant (A/B: 40 / 48 best)
#ifndef LOPF_BATCH_TW
#define LOPF_BATCH_TW 4
#endif
constexpr int kBatchTeamWarps = LOPF_BATCH_TW;          // warps per team of the batch kernel
#ifndef LOPF_BATCH_LPT
#define LOPF_BATCH_LPT 1                               // units to team warps: 1 cost-balanced (LPT), 0 round robin
#endif

// Arena layout: byte offsets of every array (all 256-byte aligned).
struct Layout {
    int32_t kernel = 1;
    int64_t n_tasks = 0, n_slots = 0, abar_doubles = 0, n_obj = 0;
    int32_t rmax = 1;                     // streaming: widest task (R)
    int32_t staged = 0;                   // batch: 1 when no task reads its operator block from HBM (kTaskDirect)
    int32_t esz = 8;                      // streaming / batch: element size of the (T) arrays (8 fp64, 4 fp32)
    // partitioned mode
    int32_t part = 0, rank = 0, world = 1, n_bnd = 0, n_imp = 0, ghost0 = 0;
    size_t off_sexp = 0, off_imp = 0, off_xbuf = 0, off_xent = 0, off_peer = 0, off_parr = 0;
    size_t off_tasks = 0, off_meta = 0, off_bbar = 0, off_xl = 0, off_lam = 0,
           off_u0 = 0, off_u1 = 0, off_x0 = 0, off_gpar = 0, off_gcost = 0, off_segptr = 0, off_segslot = 0, off_x = 0, off_abar = 0,
           off_partial = 0, off_ctrl = 0, off_trace = 0, off_objidx = 0, off_objc = 0;
    size_t bytes = 0;
    int32_t max_grid = 0, trace_cap = 0;
    std::vector<int32_t> slot_of_copy;     // [nc] canonical copy -> slot (resident: global slot id)
    std::vector<uint8_t> image;            // host image of the whole arena (initial state included)
    // resident kernel
    int32_t G = 0, n_exp = 0, max_smem = 0, total_slots = 0;
    size_t off_hdr = 0, off_blobs = 0, off_xchg = 0, off_x0r = 0, off_prof = 0, off_flags = 0;
    std::vector<CtaHdr> hdr;               // host copy of the per-CTA headers
    std::vector<int32_t> slot_cta;         // [total slots] CTA of a global slot id
    // streaming task composition (kept for the batch packer): subsystems and block offsets per task
    std::vector<int4> trec;
    std::vector<int32_t> tsub_ptr, tsub_s, tsub_poff;
    // batch kernel (config 4, lane = scenario)
    int32_t n_scen = 0, n_grp = 0, ns_max = 0, n_rows = 0, n_bsub = 0, ve = 0;
    int32_t task_rows_max = 0;             // rows of the largest task (team kernel SMEM)
    size_t off_brow = 0, off_bsub = 0, off_btask = 0, off_bseg = 0, off_bspool = 0, off_bvpool = 0, off_bpart = 0,
           off_bres = 0, off_bstop = 0, off_bgact = 0, off_bcnt = 0, off_bwpre = 0, off_bstage = 0,
           off_btorder = 0, off_btunp = 0, off_btun = 0;
    size_t image_bytes = 0;                // bytes of `image` uploaded by bind (0: the whole arena); the rest is
                                           // device state initialised by the reset kernels
    size_t off_fetch = 0;                  // staging of lopf_fetch_async (result record + x as fp64), after the image
};

// Scenario batches (config 4): per-scenario operators of the subsystems that hold a load (their
// A_s depends on the load level through VDLM-1/2); every other subsystem shares the base operator.
struct BatchOps {
    int32_t n_scen = 0;
    std::vector<int64_t> vsub;                 // varying subsystems (canonical ids, ascending)
    std::vector<int32_t> vidx;                 // [S] index into vsub or -1
    std::vector<int64_t> va_off, vb_off;       // [V+1] offsets (doubles) of Abar (n_s^2) / bbar (n_s) per scenario
    int64_t VA = 0, VB = 0;                    // doubles per scenario
    std::vector<double> abar, bbar;            // [n_scen][VA], [n_scen][VB]
};

// setup.cpp
lopf_status build_canon(const Net& net, const lopf_options& opt, Canon& out, std::string& err);
lopf_status build_batch_ops(const Net& base, const Canon& cp, int32_t n_scen, const double* scale, BatchOps& out,
                            std::string& err);
lopf_status copy_network(const lopf_network* src, Net& dst, std::string& err);
// pack.cpp
std::vector<int64_t> dfs_order(const Net& N, const Canon& P);

// Feeder partition over `world` ranks (partition.cpp).
struct PartSpec {
    int32_t world = 1, n_bnd = 0;
    std::vector<int32_t> bus_owner;        // [n_bus]
    std::vector<int32_t> sub_owner;        // [S]
    std::vector<int32_t> copy_owner;       // [nc]
    std::vector<int32_t> bidx;             // [nc] exchange slot of a boundary copy, else -1
};
lopf_status build_partition(const Net& N, const Canon& P, int32_t world, const int32_t* bus_owner, PartSpec& out,
                            std::string& err);
lopf_status pack_streaming(const Net& N, const Canon& cp, const lopf_options& opt, int max_grid, Layout& lay, std::string& err,
                           const PartSpec* part = nullptr, int32_t rank = 0);
void init_state_image(const Canon& cp, Layout& lay);
// pack_resident.cpp: returns LOPF_E_ARG (with err) when the problem does not fit max_ctas CTAs
lopf_status pack_resident(const Net& net, const Canon& cp, const lopf_options& opt, Layout& lay, std::string& err);
// pack_batch.cpp
lopf_status pack_batch(const Net& N, const Canon& cp, const BatchOps& bo, const lopf_options& opt, Layout& lay,
                       std::string& err);
// kernels.cu
// Streaming / batch CTA (one per SM): warps x 2 SMEM stages of kPackBudget operator entries each.  Measured
// (tools/ab_stream.py): the best split keeps ~448 entries per stage and as many warps as SMEM then allows --
// 16 warps for fp64 (3.5 KB of operators per stage), 24 for fp32 (1.75 KB).
#ifndef LOPF_STREAM_WARPS_F64
#define LOPF_STREAM_WARPS_F64 16
#endif
#ifndef LOPF_STREAM_WARPS_F32
#define LOPF_STREAM_WARPS_F32 24
#endif
constexpr int kStreamWarpsF64 = LOPF_STREAM_WARPS_F64;
constexpr int kStreamWarpsF32 = LOPF_STREAM_WARPS_F32;
constexpr int kStreamWarpsWide = 12;         // ... when tasks of R > 2 exist (n_s > 64, the S = 1 path)
int stream_block(int rmax, int esz);
lopf_status launch_solve(const DevProblem& P, int grid, void* stream, std::string& err);
lopf_status launch_reset(const DevProblem& P, void* stream, std::string& err);
lopf_status launch_part_import(const DevProblem& P, void* stream, std::string& err);
lopf_status launch_p2p(const DevProblem* parr_dev, const DevProblem* one, int world_here, int gsize, int rmax, int esz,
                       void* stream, std::string& err);
int p2p_max_group(int rmax, int esz, int world_here);
lopf_status launch_fetch(const DevCtrl* ctrl, const void* x, int64_t n, int esz, void* stage, void* stream, std::string& err);
lopf_status query_grid(int rmax, int esz, int* grid, std::string& err);
lopf_status launch_resident(const ResProblem& P, void* stream, std::string& err);
lopf_status launch_reset_resident(const ResProblem& P, void* stream, std::string& err);
lopf_status launch_gather_resident(const ResProblem& P, void* stage, void* stream, std::string& err);
lopf_status resident_capacity(int* sms, int* smem_optin, std::string& err);
// batch.cu
int batch_block(int trmax, int esz);
int batch_smem(int trmax, int esz);
lopf_status query_batch_grid(int trmax, int esz, int* grid, std::string& err);
lopf_status launch_batch(const BatchProblem& B, int grid, void* stream, std::string& err);
lopf_status launch_reset_batch(const BatchProblem& B, void* stream, std::string& err);
lopf_status launch_gather_scen(const BatchProblem& B, int32_t scen, void* stream, std::string& err);

}  // namespace lopf

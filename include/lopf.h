/*
 * lopf.h — C ABI of the B200-native solver-free consensus ADMM for linearized,
 * multi-phase, unbalanced distribution OPF (arXiv 2310.09410, Ryu / Byeon / Kim).
 *
 * The library (paper_2310_09410_b200/liblopf.so) exposes the two calls the method
 * needs — a setup call and a solve call — plus getters for parity checking:
 *
 *   lopf_setup   CPU, once: validate the network (Table I), assemble
 *                the linearized OPF LP (eqs. (2)-(5)), decompose it
 *                component-wise with leaf merging into subsystems
 *                (A_s, b_s) and 0-1 maps B_s, and precompute
 *                Abar_s = A_s^T (A_s A_s^T)^-1 A_s - I and bbar_s = A_s^T (A_s A_s^T)^-1 b_s
 *                (closed_2; Algorithm 1 lines 2-3) and pack them for
 *                the device.
 *   lopf_bind    copy the packed problem host -> device into a caller-owned arena.
 *   lopf_solve   Algorithm 1 on the GPU until (termination)
 *                 or max_iter: global update closed_1 (PAPER.md:305-310,
 *                rho restored — DESIGN.md reading C1), local update closed_2, dual update
 *                ADMM-3, residuals; no host synchronisation per iteration.
 *   lopf_run     exactly k iterations (the termination test optional) — fixed-K parity.
 *
 * Conventions
 *   - All arrays in / out are plain host pointers unless stated "device".  Setup copies
 *     every input, so the caller may free its arrays as soon as lopf_setup returns.
 *   - Phases: bitmask a = 1, b = 2, c = 4.  Per-phase arrays have 3 slots [.. * 3]
 *     (slot 0 = phase a); slots of absent phases are ignored.  3x3 impedance blocks are
 *     row-major [.. * 9].
 *   - Output arrays are caller-allocated and sized from lopf_sizes_get(); everything
 *     is in CANONICAL order (reading C12); internal device layouts never leak.
 *   - Device memory: one caller-owned region (e.g. a torch uint8 CUDA tensor) of at least
 *     lopf_sizes.device_bytes bytes, 256-byte aligned; the library sub-allocates it and
 *     never frees it.  Streams are cudaStream_t passed as void* (0 = legacy default).
 *   - No exceptions cross the ABI.  Every call returns a lopf_status; on error
 *     lopf_last_error() (thread-local) describes it, naming the offending component or
 *     subsystem.  Reaching max_iter is an OUTCOME (LOPF_MAX_ITER), not an error.
 *   - A handle is not thread-safe; distinct handles are independent.
 */
#ifndef LOPF_H
#define LOPF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOPF_ABI_VERSION 3

typedef struct lopf_handle lopf_handle;

typedef enum {
    LOPF_OK = 0,
    LOPF_E_ARG = 1,            /* bad option / null pointer / size mismatch */
    LOPF_E_NETWORK = 2,        /* network validation failed */
    LOPF_E_ORPHAN = 3,         /* a global variable belongs to no subsystem (nu_i = 0) */
    LOPF_E_INFEASIBLE_SUB = 4, /* a subsystem's equality rows are inconsistent */
    LOPF_E_RANK = 5,           /* A_s A_s^T not positive definite even after row reduction */
    LOPF_E_CUDA = 6,           /* CUDA runtime error (message has the CUDA error string) */
    LOPF_E_NCCL = 7,           /* NCCL failure in the library-owned communicator (lopf_part_nccl_*) */
    LOPF_E_NUMERIC = 8,        /* non-finite residual detected on the device */
    LOPF_E_STATE = 9           /* call out of order (e.g. solve before bind) */
} lopf_status;

typedef enum { LOPF_CONVERGED = 0, LOPF_MAX_ITER = 2 } lopf_outcome;   /* SPEC.md:393 exit codes 0 / 2 */

/* Network, structure of arrays (Table I).  All pointers host, caller-owned. */
typedef struct {
    int32_t n_bus, n_line, n_gen, n_load, root_bus;
    const uint8_t *bus_phases;                                      /* [n_bus] */
    const double *bus_wmin, *bus_wmax, *bus_gsh, *bus_bsh;          /* [n_bus*3]: w bounds, g^sh, b^sh */
    const int32_t *line_from, *line_to;                             /* [n_line] bus indices (i = from) */
    const uint8_t *line_phases;                                     /* [n_line] */
    const double *line_r, *line_x;                                  /* [n_line*9] 3x3 row-major */
    const double *line_gs_from, *line_bs_from;                      /* [n_line*3] g^s_eij, b^s_eij */
    const double *line_gs_to, *line_bs_to;                          /* [n_line*3] g^s_eji, b^s_eji */
    const double *line_tau;                                         /* [n_line*3] tap ratio > 0 */
    const double *line_pmin, *line_pmax, *line_qmin, *line_qmax;    /* [n_line*3] flow bounds */
    const int32_t *gen_bus;                                         /* [n_gen] */
    const uint8_t *gen_phases;                                      /* [n_gen] */
    const double *gen_pmin, *gen_pmax, *gen_qmin, *gen_qmax;        /* [n_gen*3] */
    const int32_t *load_bus;                                        /* [n_load] */
    const uint8_t *load_phases, *load_conn;                         /* [n_load]; conn 0 wye, 1 delta (3-phase only) */
    const double *load_alpha, *load_beta, *load_a, *load_b;         /* [n_load*3] VDLM-1/2 data */
} lopf_network;

typedef struct {
    double rho;            /* penalty rho > 0 (paper default 100) */
    double eps_rel;        /* relative tolerance > 0 (paper default 1e-3) */
    int64_t max_iter;      /* >= 0 */
    int32_t trace_every;   /* 0: no trace; k > 0: record (t, pres, dres, eps_prim, eps_dual) every k sweeps */
    int32_t trace_cap;     /* rows of trace kept on the device (0 = default 4096) */
    int32_t single;        /* 1: one subsystem holding every row (S = 1) */
    int32_t kernel;        /* 0 auto, 1 streaming (operators in HBM/L2), 2 resident (operators in SMEM) */
    int32_t block_threads; /* must be 0: block sizes are fixed per kernel at build time (lopf_sizes.block) */
    int32_t max_ctas;      /* resident kernel: CTAs available (one per SM; 0 = 148, the B200 SM count) */
    int32_t grid_cap;      /* streaming kernel: cap on the persistent grid (0 = occupancy x SMs; test hook) */
    int32_t reserved[2];   /* [0] = 1: per-CTA phase cycle counters (lopf_get_profile); [1] must be 0 */
    int32_t precision;     /* 0 or 64: fp64 (the parity path); 32: fp32 operators, iterate and arithmetic — the
                              paper's GPU precision (reading F1).  Residual sums,
                              the termination test and the objective stay fp64.  All three kernels. */
    int32_t adapt_every;   /* 0: fixed rho (the paper's Algorithm 1).  k > 0: residual balancing (PAPER.md:394,
                              DESIGN.md reading F2) — after a sweep t that fails the test with t % k == 0,
                              rho <- adapt_tau rho if pres > adapt_mu dres, rho <- rho / adapt_tau if
                              dres > adapt_mu pres.  Abar_s, bbar_s are rho-free, so only the scalar
                              changes, on the device, with no host round trip.  Streaming kernel only (kernel 0 picks
                              it; kernel 2, batch and partitioned handles are LOPF_E_ARG). */
    int32_t coarse;        /* 0 / 1: component-wise subsystems.  B > 1: the coarse-partition regime
                              (closed form for any S >= 1): consecutive runs of B
                              component subsystems in depth-first order merged into one larger subsystem (kind 3,
                              DESIGN.md reading C25).  n_s up to 256 (larger is LOPF_E_ARG at pack time). */
    double adapt_mu;       /* > 1 (0 = default 10) */
    double adapt_tau;      /* > 1 (0 = default 2) */
} lopf_options;

typedef struct {
    int64_t S, n, m, n_copies, p_sym, n_tasks, n_slots, device_bytes;
    int64_t abar_doubles;  /* entries (fp64 or fp32, see precision) of the packed operator pool */
    int64_t alg_bytes;     /* algorithmic bytes per iteration (DESIGN.md §4.6 byte model; a batch handle: per
                              batch sweep, what the scenarios share counted once) */
    int32_t kernel;        /* kernel actually selected (1 streaming, 2 resident, 3 batch) */
    int32_t grid;          /* CTAs of the persistent launch (known after bind) */
    int32_t block;         /* threads per CTA */
    int32_t max_ns, max_ms;
    int32_t n_scen;        /* scenarios of a batch handle (lopf_setup_batch), else 0 */
    int32_t reserved[2];
    int64_t upload_bytes;  /* bytes lopf_bind copies host -> device (the packed problem; device-only state excluded) */
    int64_t fetch_bytes;   /* bytes of the host buffer lopf_fetch_async fills (single-problem handles) */
} lopf_sizes;

typedef struct {
    int32_t outcome;       /* lopf_outcome */
    int32_t reserved0;
    int64_t iters;         /* sweeps executed, K */
    double pres, dres, eps_prim, eps_dual;   /* of the last sweep */
    double objective;      /* c^T x of the last global x */
    double solve_ms;       /* device time of the iteration launch (CUDA events) */
} lopf_result;

/* Fill *o with the paper's defaults: rho 100, eps_rel 1e-3, max_iter 1e6. */
lopf_status lopf_options_default(lopf_options *o);

/* CPU setup (see top of file).  On success *out owns host copies of everything.
 * Errors: LOPF_E_ARG, LOPF_E_NETWORK, LOPF_E_ORPHAN, LOPF_E_INFEASIBLE_SUB, LOPF_E_RANK. */
lopf_status lopf_setup(const lopf_network *net, const lopf_options *opt, lopf_handle **out);

lopf_status lopf_sizes_get(const lopf_handle *h, lopf_sizes *sz);

/* Batch of n_scen load scenarios of one network (BASELINE.json configs[3]): scenario s scales every
 * load's (a, b) by load_scale[s * n_load + l] (> 0).  Each scenario is an independent run of
 * Algorithm 1 with its own (termination) test; only the operators of subsystems that hold a load
 * differ between scenarios (VDLM-1/2).  lopf_solve / lopf_run / lopf_reset then act
 * on every scenario; lopf_result reports iters = max over scenarios, outcome = CONVERGED iff every
 * scenario converged, objective = sum of the scenarios' objectives.  Canonical getters describe the
 * shared structure; per-scenario data comes from the *_scen getters below. */
lopf_status lopf_setup_batch(const lopf_network *net, const lopf_options *opt, int32_t n_scen,
                             const double *load_scale, lopf_handle **out);

/* Per-scenario outcome of the last batch launch: iters [n_scen], outcome [n_scen] (0 converged,
 * 2 max_iter, 8 numeric), res [n_scen*4] {pres, dres, eps_prim, eps_dual}, objective [n_scen]. */
lopf_status lopf_get_batch_results(lopf_handle *h, void *cuda_stream, int64_t *iters, int32_t *outcome,
                                   double *res, double *objective);

/* Scenario scen's iterate (canonical order): x [n], x_loc, lam [n_copies]; any pointer may be NULL. */
lopf_status lopf_get_state_scen(lopf_handle *h, void *cuda_stream, int32_t scen, double *x, double *x_loc,
                                double *lam);

/* Scenario scen's operator of subsystem s: abar [n_s*n_s], bbar [n_s]. */
lopf_status lopf_get_operator_scen(const lopf_handle *h, int64_t s, int32_t scen, double *abar, double *bbar);

/* ---- partitioned mode (config 5: one feeder over `world` GPUs) ----
 * Every rank calls lopf_setup_part with the SAME network and options.  The buses are split into
 * `world` contiguous depth-first intervals balanced by work (bus_owner == NULL) or as given by
 * bus_owner [n_bus] (values in [0, world)); subsystems follow their anchor bus (BUS: the bus,
 * LINE: the end away from the substation, LEAF: the leaf bus).  A rank keeps only its subsystems;
 * the copies its globals share with other ranks (boundary copies) travel through an exchange
 * buffer of n_bnd + 8*world doubles inside the arena: per sweep
 *     lopf_part_sweep(h, s)      one sweep (a4-a7) of this rank's subsystems; writes its boundary
 *                                copies' u and its five residual sums into its own exchange slots
 *     <sum-allreduce of the exchange buffer over the ranks>     (NCCL, caller-side)
 *     lopf_part_import(h, s)     the other ranks' u into this rank's ghost slots; the termination
 *                                test on the rank-ordered residual sums; clears
 *                                the exchange buffer for the next sweep.
 * Each slot is written by exactly one rank, so the sum is an exact gather, and the consensus of a
 * boundary global adds its copies in canonical order on every rank: iterates are bit-identical to
 * the single-GPU streaming kernel.  After termination both calls are no-ops.  lopf_result_get
 * reports K (iters), the residuals and this rank's share of the objective (sum over ranks = c^T x);
 * lopf_get_state returns this rank's copies and the globals whose first copy is here, NaN elsewhere.
 * lopf_solve / lopf_run / lopf_set_state return LOPF_E_STATE on a partitioned handle. */
lopf_status lopf_setup_part(const lopf_network *net, const lopf_options *opt, int32_t rank, int32_t world,
                            const int32_t *bus_owner, lopf_handle **out);
/* Exchange buffer location: byte offset in the arena, length in doubles; boundary slots; ghost slots. */
lopf_status lopf_part_info(const lopf_handle *h, int64_t *xbuf_offset, int64_t *xbuf_doubles, int32_t *n_bnd,
                           int32_t *n_imp);
/* The partition: bus_owner [n_bus], copy_owner [n_copies], exchange slot of every copy or -1 [n_copies]. */
lopf_status lopf_part_owner(const lopf_handle *h, int32_t *bus_owner, int32_t *copy_owner, int32_t *bidx);
lopf_status lopf_part_sweep(lopf_handle *h, void *cuda_stream);
lopf_status lopf_part_import(lopf_handle *h, void *cuda_stream);

/* Host-driven partitioned sweeps with a library-owned NCCL communicator (libnccl.so.2 opened at first use;
 * failures are LOPF_E_NCCL): rank 0 creates an id (128 bytes) and every rank passes the same bytes to
 * lopf_part_nccl_init; lopf_part_step = lopf_part_sweep + ncclAllReduce(sum, fp64) of the exchange buffer on
 * `stream` + lopf_part_import, all stream-ordered (capturable in a CUDA graph). */
lopf_status lopf_nccl_unique_id(void *out128);
lopf_status lopf_part_nccl_init(lopf_handle *h, const void *unique_id128);
lopf_status lopf_part_step(lopf_handle *h, void *cuda_stream);

/* ---- partitioned mode with a device-initiated exchange ----------------
 * One persistent launch per solve and rank, no host and no collective library in the loop: the kernel
 * stores every boundary copy's u as a tagged entry {u, sweep + 1} straight into each rank's entry buffer
 * (peer memory over NVLink / NVSwitch), each entry ONE 128-bit system-scope store; the last CTA of a rank
 * stores the rank's five residual sums the same way, then reads every rank's sums and its own ghost values,
 * each when its tag says "this sweep", copies the ghosts in and takes the (termination) decision on the
 * rank-ordered sums -- identical on every rank, iterates bit-identical to the single-GPU streaming kernel.
 * No flags and no fences cross GPUs; entry buffers are double-buffered by sweep parity (a rank cannot run
 * two sweeps ahead of a reader of its entries, because it waits for that reader's sums of the sweep in
 * between).  Each rank: lopf_part_p2p_info -> its entry buffer (offset in the arena, bytes); peers'
 * buffers are mapped with lopf_ipc_export / lopf_ipc_open (CUDA IPC, same node); lopf_part_connect(
 * peer_entries[world]: device pointers valid in this process, [rank] = its own); lopf_reset on every rank
 * and a host barrier; lopf_part_solve_p2p.  lopf_result_get reports K, residuals and this rank's objective
 * share.  Every rank's launch must be resident at the same time (one process per GPU). */
lopf_status lopf_part_p2p_info(const lopf_handle *h, int64_t *entry_offset, int64_t *entry_bytes);
lopf_status lopf_part_connect(lopf_handle *h, const uint64_t *peer_entries, void *cuda_stream);
lopf_status lopf_part_solve_p2p(lopf_handle *h, int64_t max_iter, int32_t test, void *cuda_stream);
/* All `world` ranks (hs[q] = rank q, bound on ONE GPU) as one cooperative launch (rank q = CTAs
 * [q g, (q+1) g)), connected through local memory: the same kernel and protocol as lopf_part_solve_p2p,
 * for testing the multi-rank path with fewer GPUs than ranks. */
lopf_status lopf_part_emulate(lopf_handle *const *hs, int32_t world, int64_t max_iter, int32_t test, void *cuda_stream);
/* CUDA IPC: out [72] = the cudaIpcMemHandle of the allocation holding dev_ptr + the offset of dev_ptr in
 * it; lopf_ipc_open maps such a record into this process (closed when h is destroyed). */
lopf_status lopf_ipc_export(const void *dev_ptr, void *out);
lopf_status lopf_ipc_open(lopf_handle *h, const void *in, void **dev_ptr);

/* Copy the packed problem into the caller's device arena (device pointer, >= device_bytes,
 * 256-byte aligned) on `stream`, and reset the iterate to the initial point of PAPER.md:495.
 * May be called again (e.g. to re-upload for an end-to-end timing). */
lopf_status lopf_bind(lopf_handle *h, void *device_arena, size_t bytes, void *cuda_stream);

/* Reset the device iterate to the initial point (lambda = 0; x_s = 1 / midpoint / 0). */
lopf_status lopf_reset(lopf_handle *h, void *cuda_stream);

/* Run until (termination) or max_iter, starting from the current device iterate.
 * Synchronises `stream` once at the end to fill *res. */
lopf_status lopf_solve(lopf_handle *h, void *cuda_stream, lopf_result *res);

/* Run exactly k sweeps (test = 0) or at most k sweeps stopping at (termination) (test = 1). */
lopf_status lopf_run(lopf_handle *h, int64_t k, int32_t test, void *cuda_stream, lopf_result *res);

/* Asynchronous variant for CUDA-graph capture / timing: enqueue the solve on `stream`
 * without synchronising; fetch the result later with lopf_result_get. */
lopf_status lopf_solve_async(lopf_handle *h, int64_t max_iter, int32_t test, void *cuda_stream);
lopf_status lopf_result_get(lopf_handle *h, void *cuda_stream, lopf_result *res);

/* Stream-ordered read-back of a solve (no host synchronisation): one small kernel gathers the result
 * record and the solution x into the arena, one cudaMemcpyAsync copies them to `host_buf` (fetch_bytes
 * from lopf_sizes; pinned memory makes the copy asynchronous).  Layout of host_buf: a lopf_result
 * (solve_ms = 0: take it from lopf_result_get or your own events), padded to 64 bytes, then x as n
 * doubles in canonical order.  The caller waits on its own event / stream before reading host_buf.
 * LOPF_E_STATE on batch and partitioned handles (use lopf_get_batch_results / lopf_result_get). */
lopf_status lopf_fetch_async(lopf_handle *h, void *cuda_stream, void *host_buf);

/* The penalty in force on the device (the fixed rho, or the residual-balancing one after the last solve)
 * and the number of changes since the last reset / bind. */
lopf_status lopf_get_rho(lopf_handle *h, void *cuda_stream, double *rho, int64_t *changes);

/* Canonical decomposition: kind (0 BUS, 1 LINE, 2 LEAF, 3 COARSE run), comp (bus or line index, run index),
 * leaf_bus (-1 unless LEAF), m_s, n_s [S]; sub_ptr [S+1] copy offsets; copy_global [n_copies]. */
lopf_status lopf_get_decomposition(const lopf_handle *h, int32_t *kind, int32_t *comp, int32_t *leaf_bus,
                                   int32_t *m_s, int32_t *n_s, int64_t *sub_ptr, int32_t *copy_global);

/* Consensus map global -> copies (I_si): row_ptr [n+1], copy_idx [n_copies]. */
lopf_status lopf_get_consensus(const lopf_handle *h, int64_t *row_ptr, int32_t *copy_idx);

/* Global variable catalog (canonical order) and LP data: role codes 0 pg 1 qg 2 w 3 pb 4 qb
 * 5 pd 6 qd 7 p_eij 8 q_eij 9 p_eji 10 q_eji; comp; phase slot; c, lo, hi (+-inf allowed). */
lopf_status lopf_get_globals(const lopf_handle *h, int32_t *role, int32_t *comp, int32_t *phase,
                             double *c, double *lo, double *hi);

/* Subsystem s's precomputed operator: abar [n_s*n_s] row-major, bbar [n_s]. */
lopf_status lopf_get_operator(const lopf_handle *h, int64_t s, double *abar, double *bbar);

/* Subsystem s's dense A_s [m_s*n_s] row-major and b_s [m_s] (after any row reduction m_s may shrink;
 * *m_out receives the row count). */
lopf_status lopf_get_subsystem(const lopf_handle *h, int64_t s, double *A, double *b, int32_t *m_out);

/* Device iterate -> host (canonical order): x [n] (last global update), x_loc, lam [n_copies].
 * Any pointer may be NULL.  Synchronous on `stream`. */
lopf_status lopf_get_state(lopf_handle *h, void *cuda_stream, double *x, double *x_loc, double *lam);

/* Host -> device iterate (canonical order); x_loc, lam [n_copies] (warm start / resume). */
lopf_status lopf_set_state(lopf_handle *h, void *cuda_stream, const double *x_loc, const double *lam);

/* Trace rows {t, pres, dres, eps_prim, eps_dual} of the last solve: buf [cap*5]. */
lopf_status lopf_get_trace(lopf_handle *h, void *cuda_stream, double *buf, int64_t cap, int64_t *n_rows);

/* Diagnostics (resident kernel, options.reserved[0] = 1): per-CTA cycle counters of the last launch,
 * rows {work, publish + neighbour wait, 0, sweeps}: buf [cap*4].  The counters perturb the timing.
 * Rows G .. 33G-1 (cap > G) hold the event timeline of a LOPF_RES_TIMELINE diagnostics build. */
lopf_status lopf_get_profile(lopf_handle *h, void *cuda_stream, int64_t *buf, int64_t cap, int64_t *n_rows);

void lopf_destroy(lopf_handle *h);

/* Thread-local description of the last error (empty string if none). */
const char *lopf_last_error(void);

/* Library / ABI version (LOPF_ABI_VERSION). */
int32_t lopf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LOPF_H */

/*
 * mgm.h -- C ABI of libmgm, a B200-native (sm_100a, fp64) implementation of the solve path
 * of the meshfree geometric multilevel (MGM) method, arXiv 2204.06154.
 *
 * Citations: P:n = line n of the paper text; O1..O17 = the readings written out
 * in DESIGN.md ("Readings of the paper").
 *
 * Problem: solve L_h u = f on a point cloud X_h of a closed surface, with
 *   L_h = I - mu D_h   (shifted surface Poisson, problem = 0), or
 *   L_h = D_h          (surface Poisson, problem = 1; solved as the bordered system
 *                       [L 1; 1^T 0][u; lambda] = [f; 0]),
 * D_h the RBF-FD or GFD Laplace-Beltrami matrix.  MGM (Alg. 2,
 * P:361-378; Alg. 3) is used standalone or as the right preconditioner of
 * GMRES.
 *
 * Conventions (all entry points):
 *  - No C++ types cross this boundary.  Every call returns mgm_status; nothing throws.
 *  - Host arrays ("host") are read during the call only and may be freed afterwards.
 *  - Device arrays ("device") are caller-owned, contiguous fp64 buffers on the ctx's GPU.
 *  - User vectors are in the caller's ORIGINAL point order; the library applies and undoes
 *    its internal ordering (Morton order, O1, in place of RCM, P:283/P:390/P:404).
 *  - Calls are ordered on the given CUDA stream (cudaStream_t passed as void*, NULL = the
 *    legacy default stream).  A ctx is not re-entrant: one call at a time per ctx.
 *  - On error, mgm_last_error() returns a message and the failing index (stencil centre,
 *    fine row, or pivot) where one exists.
 */
#ifndef MGM_H
#define MGM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mgm_ctx mgm_ctx; /* opaque; owns the device hierarchy, workspaces, graphs */

typedef enum {
    MGM_OK = 0,
    MGM_ERR_ARG = 1,        /* invalid argument (sizes, parameters, NULL pointers)          */
    MGM_ERR_UNISOLVENT = 2, /* RBF-FD/GFD stencil system singular; index = stencil centre   */
    MGM_ERR_SINGULAR = 3,   /* transfer system (index = fine row) or coarse LU (index = pivot) */
    MGM_ERR_BREAKDOWN = 4,  /* GMRES breakdown with a nonzero residual                       */
    MGM_ERR_CUDA = 5,       /* CUDA runtime error                                             */
    MGM_ERR_NCCL = 6,       /* NCCL missing or failed (multi-GPU)                             */
    MGM_ERR_OOM = 7,        /* device allocation failed                                       */
    MGM_ERR_INPUT = 8       /* duplicate points / non-finite input; index = offending point  */
} mgm_status;

/* Discretisation of the surface operator (Section 2 of the paper). */
typedef struct {
    int method;       /* 0 = PHS RBF-FD, 1 = GFD                     */
    int poly_degree;  /* ell: degree of the tangent-plane polynomials, 0..8          */
    int phs_k;        /* k: PHS kernel r^(2k+1), 1 <= k <= ell (k=0 has no Laplacian) */
    int stencil_n;    /* n: stencil size incl. the centre, nearest in R^3; <= 96      */
    double gfd_alpha; /* alpha of the GFD Gaussian weight exactly as written at P:185-187,
                         w_i = exp(-alpha |x_1 - x_i|^2 / (rho_1^2 + rho_i^2)), rho_k the radius
                         of point k's own projected stencil.  NOTE (O5): the paper's
                         Table 1 value alpha = 4 reproduces its Table 3 iteration counts only
                         when 16 (= 4 x 4) is passed here; the cfg2-GFD workload passes 16.    */
    int problem;      /* 0 = shifted (L = I - mu D), 1 = Poisson (L = D, mean-zero border)   */
    double mu;        /* mu > 0 of the shifted problem                                 */
} mgm_stencil_params;

/* Multilevel parameters (Section 4; Table 1). */
typedef struct {
    int num_levels;     /* p; 0 = the paper's rule p = floor(log(N/n_min)/log 4) + 1 */
    int n_min;          /* N_min for the rule above (Table 1: 250)                            */
    int coarsen_factor; /* N_{j+1} = floor(N_j / factor); the paper uses 4            */
    int interp_m;       /* m: nearest coarse points per interpolation stencil, <= 16   */
    int nu1, nu2;       /* pre-/post-smoothing sweeps                                  */
    int smoother;       /* 0 forward GS both, 1 backward both, 2 forward pre/backward post    */
    int restart;        /* GMRES restart length (<= 128)                                       */
} mgm_level_params;

typedef struct {
    int iterations;            /* GMRES: preconditioner applications in Arnoldi; standalone: V-cycles */
    int converged;             /* 1 if the stopping test was met                                        */
    double final_rel_residual; /* true ||b - A x||_2 / ||b||_2 at exit                                  */
    double* history;           /* caller-owned host buffer (or NULL): relative residual per iteration   */
    int history_cap;           /* capacity of history                                                   */
    double lambda;             /* Poisson mode: Lagrange multiplier of the border               */
    double setup_ms;           /* device+host time of mgm_setup                                         */
    double solve_ms;           /* device time of this solve (CUDA events on the stream)                 */
} mgm_report;

/* Device memory of a ctx: every device allocation the ctx makes (hierarchy, workspaces,
 * setup scratch) calls alloc(bytes, user) and later release(ptr, user) on the ctx's device;
 * alloc returns NULL on failure (-> MGM_ERR_OOM), pointers must be 256-byte aligned.
 * Passing NULL to mgm_setup (or alloc == NULL) uses cudaMalloc / cudaFree.  The callbacks
 * are called from the thread that calls into the library, inside mgm_* calls only.  The
 * Python binding passes PyTorch's caching allocator (paper_2204_06154_b200.torch_allocator). */
typedef struct {
    void* (*alloc)(size_t bytes, void* user);
    void (*release)(void* ptr, void* user);
    void* user;
} mgm_allocator;

/* Build the hierarchy (Alg. 2) on the current CUDA device.
 * points, normals: host, n_points x 3 row-major fp64 (normals unit length).  Copied.
 * allocator: host struct (copied) or NULL.
 * On success *out receives a new ctx (free with mgm_destroy).  Errors: MGM_ERR_ARG,
 * MGM_ERR_INPUT (index = point), MGM_ERR_UNISOLVENT (index = centre, original order),
 * MGM_ERR_SINGULAR, MGM_ERR_CUDA, MGM_ERR_OOM.  If out is non-NULL and the failure happened
 * after allocation, *out is set to a ctx that only carries the error (query with
 * mgm_last_error, then mgm_destroy). */
mgm_status mgm_setup(const double* points, const double* normals, int64_t n_points,
                     const mgm_stencil_params* stencil, const mgm_level_params* levels,
                     const mgm_allocator* allocator, void* cuda_stream, mgm_ctx** out);

/* One V(nu1,nu2)-cycle (Alg. 3): u <- MGM(f, u).
 * f_dev, u_dev: device, n_points fp64, original order; u_dev is the initial guess on entry
 * and the result on exit.  Poisson mode: lambda starts at 0 and is not returned. */
mgm_status mgm_vcycle(mgm_ctx* ctx, const double* f_dev, double* u_dev, void* cuda_stream);

/* Solve L u = rhs (Poisson: the bordered system) to ||rhs - L x|| / ||rhs|| <= tol.
 * krylov = 1: right-preconditioned GMRES(restart) with one V-cycle from a zero guess as the
 *             preconditioner; on one GPU (shifted problems) each restart cycle
 *             runs as ONE CUDA-graph launch whose WHILE node iterates the Arnoldi steps with
 *             the Givens rotations on the device (MGM_HOST_GMRES=1: host-driven loop, same
 *             arithmetic up to rounding); the preconditioned vectors z_k = M v_k are kept
 *             (restart x N fp64 of device memory) and x += Z y ends a restart cycle;
 *             krylov = 0: standalone MGM;
 * krylov = 2: right-preconditioned BiCGSTAB: report.iterations counts
 *             preconditioner applications (two per step) and report.history holds the
 *             relative residual after every half step; on a rho/omega breakdown it restarts
 *             once from the current iterate, then returns converged = 0.
 * rhs_dev, x_dev: device, n_points fp64, original order (multi-GPU: the rank's local block in
 * mgm_local_rows order).  x0_dev: the initial guess (device, same layout; may alias x_dev) or
 * NULL for x0 = 0 -- the paper's applications warm-start from the previous time step
 * (P:711).  GMRES then starts from r0 = rhs - L x0, BiCGSTAB likewise, standalone MGM from
 * u = x0; the stopping test stays ||rhs - L x|| / ||rhs|| <= tol.  x_dev receives the
 * solution.  rhs = 0 gives x = 0 with 0 iterations (whatever x0).  Non-convergence within
 * maxit is NOT an error (converged = 0).  report may be NULL. */
mgm_status mgm_solve(mgm_ctx* ctx, const double* rhs_dev, const double* x0_dev, double* x_dev, double tol,
                     int maxit, int krylov, mgm_report* report, void* cuda_stream);

/* Same as mgm_solve with HOST vectors (pinned or pageable): copies rhs (and x0) in and x out
 * on the stream inside the call (the end-to-end path). */
mgm_status mgm_solve_host(mgm_ctx* ctx, const double* rhs_host, const double* x0_host, double* x_host,
                          double tol, int maxit, int krylov, mgm_report* report, void* cuda_stream);

mgm_status mgm_destroy(mgm_ctx* ctx);

/* ---- multi-right-hand-side solves (the paper's applications solve
 * many systems with one operator) ---------------------------------
 * K right-hand sides share every pass over the operators: each colour kernel, SpMV and
 * transfer reads its operator once for all K (vectors interleaved [row][K] inside; widths
 * 2, 4, 8 -- K is padded with zero columns).  The per-(row, RHS) arithmetic is that of the
 * single-RHS kernels, so each column of a batched V-cycle equals a single V-cycle (up to
 * the coarsest solve, which uses the explicit inverse of L_p).  Shifted problems, one GPU,
 * coarsest level <= 4096 rows; otherwise MGM_ERR_ARG.
 * f_dev, u_dev, rhs_dev, x_dev: device, K column-major vectors of n_points fp64 in
 * original order (column k at ptr + k*n_points).
 * mgm_vcycle_batch: one V-cycle per column (u in: guess, out: result).
 * mgm_solve_batch: from x = 0 on every column, krylov = 0: standalone MGM until
 * every column's ||f - L x|| / ||f|| <= tol or maxit; reports[K] (may be NULL): iterations =
 * the first cycle at which that column met tol, final_rel_residual after the last cycle.
 * krylov = 1: K independent MGM-GMRES(restart) processes (right preconditioning, CGS2, as
 * mgm_solve) sharing each batched V-cycle and SpMV; a column that meets tol stops
 * iterating (its own count in reports[k].iterations, true final residual). */
mgm_status mgm_vcycle_batch(mgm_ctx* ctx, int K, const double* f_dev, double* u_dev, void* cuda_stream);
mgm_status mgm_solve_batch(mgm_ctx* ctx, int K, const double* rhs_dev, double* x_dev, double tol, int maxit,
                           int krylov, mgm_report* reports, void* cuda_stream);

/* ---- multi-GPU ----------------------------------
 * One process per GPU.  Every rank calls mgm_setup with the SAME cloud and parameters (the
 * setup is deterministic, so every rank builds the same hierarchy), then mgm_dist_attach.
 * The attach partitions the hierarchy: rank q owns the points whose level-0 Morton index lies
 * in [floor(qN/P), floor((q+1)N/P)) -- on every level a coarse point stays with the owner of
 * its level-0 point, so each level is split into Morton row blocks -- and keeps, on the
 * distributed levels 0..D-1, only its own rows of L_j, P_j, R_j plus GHOST copies of the rows
 * its operators read (the undistributed device arrays are freed).  D: the levels with at
 * least MGM_DIST_MIN_ROWS rows per rank (environment at attach, default 16384; MGM_DIST_LEVELS
 * forces D), never the V-cycle's bottom; levels >= D (and the dense bottom) run redundantly on
 * every rank after an all-gather of the restricted residual.  Halos of ghost values only:
 * after every colour of a Gauss-Seidel sweep (that colour's values), after interpolation +
 * correction and before a restriction or SpMV (all ghosts); NCCL grouped send/receive,
 * captured in the V-cycle's CUDA graph; Krylov inner products (and the Poisson border dots):
 * rank-local reduction + ncclAllReduce.  Every local operator row keeps the undistributed
 * row's entries and threads in the same order, so a V-cycle of the shifted problem is bitwise
 * the single-GPU one; Krylov iterates agree with it to rounding (the inner products are
 * summed in another order).  Shifted and Poisson problems.
 * From then on mgm_vcycle / mgm_solve are collective (every rank calls them) and take the
 * rank's LOCAL vectors: n_local entries in the order mgm_local_rows returns.  Not available
 * on an attached ctx: the batched solves, mgm_apply, mgm_export_level of a distributed level.
 *
 * Peer-store halos (MGM_P2P=1 in the environment at attach): instead of pack + NCCL send /
 * receive, one kernel per halo stores every boundary value straight into the peer's ghost slot
 * (peer memory mapped with cudaIpcOpenMemHandle, handles all-gathered over NCCL) and its last
 * CTA publishes a per-peer push count (st.release.sys into the peer's flag array); a one-CTA
 * kernel then waits (ld.acquire.sys) for the counts it expects from its peers.  Requires the
 * default allocator (no mgm_allocator) and at most 16 peers per level.  With fake ranks the
 * same stores run, ordered by the group instead of the flags.
 *
 * mgm_nccl_unique_id: rank 0 creates the 128-byte NCCL id (host buffer id128); the caller
 * broadcasts it to the other ranks (e.g. torch.distributed).  MGM_ERR_NCCL if
 * libnccl.so.2 cannot be loaded.
 * mgm_dist_attach: rank in [0, nranks); id128 = that id (host, 128 bytes, copied).  The
 * communicator is created on the ctx's device and destroyed by mgm_destroy.  Errors:
 * MGM_ERR_ARG (bad rank / already attached / a one-level hierarchy), MGM_ERR_NCCL. */
mgm_status mgm_nccl_unique_id(void* id128);
mgm_status mgm_dist_attach(mgm_ctx* ctx, int rank, int nranks, const void* id128);

/* The rows this rank owns: *n_local = their count, original_ids[n_local] (host, may be NULL)
 * = their original point indices, in the order of the rank's local vectors (the rank's
 * level-0 points in Morton order).  Unattached ctx: all n_points rows, identity order. */
mgm_status mgm_local_rows(const mgm_ctx* ctx, int64_t* n_local, int64_t* original_ids);

/* Distribution diagnostics: *dist_levels = D (0 unattached), *ghosts = ghost rows of this rank
 * over the distributed levels, *halo_values_per_vcycle = ghost values this rank receives in
 * one V-cycle (x 8 bytes = its halo volume). */
mgm_status mgm_dist_info(const mgm_ctx* ctx, int* dist_levels, int64_t* ghosts, int64_t* halo_values_per_vcycle);

/* Communication-only timing (collective): replays the halo exchanges and the all-gather of one
 * V-cycle in their V-cycle order without any compute, `reps` times, on the stream; then
 * `reps` sum-allreduces of 16 doubles (one Krylov multi-dot).  *halo_ms_per_vcycle and
 * *allreduce_us are this rank's device times (CUDA events); take the max over ranks.
 * MGM_ERR_ARG on an unattached ctx. */
mgm_status mgm_dist_comm_time(mgm_ctx* ctx, int reps, double* halo_ms_per_vcycle, double* allreduce_us,
                              void* cuda_stream);

/* Test hook: R "fake" ranks on ONE GPU in one process.  mgm_fake_group_create makes a group of
 * nranks; each rank's ctx (its own mgm_setup) attaches with mgm_dist_attach_fake and is then
 * driven by its own host thread, calling the same collective entry points as with NCCL.  The
 * transport copies between the ranks' device buffers (CUDA events + a host barrier) instead
 * of NCCL: the distributed code path is otherwise unchanged.  V-cycles run eagerly (no CUDA
 * graph).  Destroy the group after every ctx attached to it. */
mgm_status mgm_fake_group_create(int nranks, void** group);
mgm_status mgm_fake_group_destroy(void* group);
mgm_status mgm_dist_attach_fake(mgm_ctx* ctx, int rank, void* group);

/* Message of the last failure on this ctx (or of the last failed mgm_setup on this thread
 * when ctx is NULL); *failing_index (if non-NULL) receives the index or -1. */
const char* mgm_last_error(const mgm_ctx* ctx, int64_t* failing_index);

/* ---------------- introspection and test hooks (not on the timed path) ---------------- */

mgm_status mgm_num_levels(const mgm_ctx* ctx, int* p);

/* Level j (0 = finest): rows, stored nonzeros of L_j (symbolic pattern), nonzeros of the
 * interpolation P_j = I_{j+1}^j (0 on the coarsest level), number of GS colours (0 on the
 * coarsest), and the bytes the solve-phase layout of level j occupies on the device. */
mgm_status mgm_level_info(const mgm_ctx* ctx, int level, int64_t* n_rows, int64_t* nnz_L,
                          int64_t* nnz_P, int* n_colours, int64_t* stored_bytes);

/* Copy level j's discrete structures to HOST buffers (any may be NULL), in the library's
 * level ordering ("lib order": rows grouped by colour, Morton order within a colour):
 *   ids[n_rows]          original point index of each row
 *   L_ptr[n_rows+1], L_col[nnz_L] (lib-order column), L_val[nnz_L]: CSR of L_j, columns
 *                        ascending in Morton order with the diagonal first
 *   colour[n_rows]       GS colour of each row (all 0 on the coarsest level)
 *   P_ptr[n_rows+1], P_col[nnz_P] (next level's lib order), P_val[nnz_P]: CSR of P_j
 *   border[n_rows]       Poisson border vector c_j (c_1 = 1, c_{j+1} = P_j^T c_j) */
mgm_status mgm_export_level(const mgm_ctx* ctx, int level, int64_t* ids, int64_t* L_ptr,
                            int32_t* L_col, double* L_val, int32_t* colour, int64_t* P_ptr,
                            int32_t* P_col, double* P_val, double* border);

/* Fine-level stencil weights c_ij as computed on the GPU, host output
 * w[n_points * stencil_n] and stencil indices sten[n_points * stencil_n] (original point
 * indices, centre first, O2 order), both in ORIGINAL row order. */
mgm_status mgm_export_weights(const mgm_ctx* ctx, double* w, int64_t* sten);

/* Operators on level j, device vectors in lib order (n_j entries; Poisson: n_j + 1 with the
 * multiplier last):
 *   MGM_OP_SPMV      y = L_j x                         (Poisson: [L x + c x_N; c^T x])
 *   MGM_OP_SWEEP     y = x after ONE forward colour GS sweep with rhs f; y may == x
 *   MGM_OP_RESIDUAL  y = f - L_j x                     (Poisson: bordered)
 *   MGM_OP_RESTRICT  y (n_{j+1}) = R_j x               (Poisson: multiplier copied)
 *   MGM_OP_INTERP    y (n_j) = P_j x (x has n_{j+1})   (Poisson: multiplier copied)
 *   MGM_OP_COARSE    y = L_p^{-1} x on the coarsest level (level ignored)
 *   MGM_OP_SWEEP_ZG  y = ONE forward colour GS sweep from the zero guess with rhs f, by the
 *                    zero-guess kernel (reads the diagonal and earlier-colour entries only;
 *                    the level's u is filled with NaN first to show it is never read); x is
 *                    ignored; shifted problems only
 *   MGM_OP_PRECOND   y = M x, the V-cycle from the zero guess the Krylov solvers apply
 *                    (level ignored; level-0 lib order; u starts as NaN when zero-guess
 *                    sweeps are used)
 * f is used by SWEEP and RESIDUAL only. */
enum { MGM_OP_SPMV = 0, MGM_OP_SWEEP = 1, MGM_OP_RESIDUAL = 2, MGM_OP_RESTRICT = 3,
       MGM_OP_INTERP = 4, MGM_OP_COARSE = 5, MGM_OP_SWEEP_ZG = 6, MGM_OP_PRECOND = 7 };
mgm_status mgm_apply(mgm_ctx* ctx, int level, int op, const double* x_dev, const double* f_dev,
                     double* y_dev, void* cuda_stream);

/* Per-kernel-class device timing (CUDA events around every launch of that class on the
 * solve stream; adds events, use only for measurement).  cls: 0 = level-0 GS colour sweep
 * kernels (full sweeps), 1 = level-0 SpMV, 2 = whole V-cycle, 3 = level-0 GS colour kernels
 * of the first presmooth from a zero guess (Krylov preconditioner; reads diagonal +
 * earlier-colour entries only).  enable = 1 resets the accumulators. */
mgm_status mgm_timing_enable(mgm_ctx* ctx, int cls, int enable);
/* total_ms = sum of event-measured durations, launches = number of timed launches,
 * alg_bytes = algorithmic bytes those launches move (DESIGN.md byte model). */
mgm_status mgm_timing_read(mgm_ctx* ctx, int cls, double* total_ms, int64_t* launches,
                           double* alg_bytes);

/* Algorithmic bytes of one V-cycle and one GMRES Arnoldi step k (DESIGN.md byte model). */
mgm_status mgm_bytes_model(const mgm_ctx* ctx, double* vcycle_bytes, double* spmv_bytes);

/* Number of kernels launched by one V-cycle (graph nodes). */
mgm_status mgm_vcycle_kernel_count(const mgm_ctx* ctx, int64_t* count);

/* Diagnostics (not on the timed path).  With MGM_TRACE set in the environment at
 * mgm_setup, the V-cycle graph contains one-thread stamp kernels between Alg. 3 stages
 * that record %globaltimer (ns) once their predecessor has finished.  Copies the stamps
 * of the last V-cycle into stamps_ns[cap] (host), *n = count (0 when tracing is off), and
 * newline-separated stage labels into labels[label_cap] (may be NULL).  MGM_ERR_ARG if
 * cap < *n. */
mgm_status mgm_trace_read(const mgm_ctx* ctx, uint64_t* stamps_ns, int cap, int* n, char* labels, int label_cap);

/* Stored entries of level `level`'s operator that a forward Gauss-Seidel sweep from a zero
 * guess reads (the diagonal and the earlier-colour columns of every row; k_gs_colour ZG,
 * used for the first presmooth sweep on levels >= 1 and, inside the Krylov solvers, on
 * level 0), or nnz(L_j) when zero-guess sweeps are not used (Poisson, backward presmooth,
 * MGM_NO_ZG).  For byte models. */
mgm_status mgm_level_zg_nnz(const mgm_ctx* ctx, int level, int64_t* nnz_zg);

/* The dense bottom of the V-cycle: Alg. 3 lines 6-14 for the
 * levels >= J from e_J = 0 are linear in r_J; setup builds their matrix B_J
 * (n_J x n_J, Poisson n_J + 1) from the unit vectors with the library's own level kernels and
 * every V-cycle applies it as one dense HBM-bound kernel.  J = the first level >= 1 with at
 * most MGM_DENSE_MAX rows (environment at mgm_setup, default 4096; 0 = off).  *level = J or
 * -1 (off), *rows = its dimension, *bytes = the bytes of B_J read per apply. */
mgm_status mgm_dense_bottom_info(const mgm_ctx* ctx, int* level, int64_t* rows, int64_t* bytes);

/* Diagnostics: start time (%globaltimer, ns) of every phase of the one-kernel bottom of the
 * last V-cycle (MGM_TRACE set at setup), *n = number of phases (0 if tracing is off or the
 * bottom kernel is not used); meta[4*q..] = {op, local, rows, threads per row} (may be NULL). */
mgm_status mgm_bottom_trace_read(const mgm_ctx* ctx, uint64_t* stamps_ns, int cap, int* n, int32_t* meta);

/* Diagnostics: fine per-phase timeline of the bottom kernel (MGM_TRACE=2 at setup): for
 * thread 0 of the first and of the last CTA of the cluster, 8 SM-clock readings per phase
 * {phase start, operator row in registers, row sum ready, value broadcast, stores issued,
 * cluster arrive done, next rows' loads issued, cluster wait done} (slots 0,7,1,2,3,4,5,6 in
 * that order of the array: clk[cta][phase][slot]).  clk holds 2*8*cap int64; *n = phases. */
mgm_status mgm_bottom_ftrace_read(const mgm_ctx* ctx, int64_t* clk, int cap, int* n);

/* ---------------- host-only hooks of the setup's discrete steps (no GPU needed) --------
 * They run the same host code mgm_setup uses, so discrete-structure parity with the
 * oracle can be checked on a CPU-only machine. */

/* Morton order (O1, replaces RCM of P:283): perm[new] = old.  host arrays. */
mgm_status mgm_host_morton(const double* points, int64_t n, int64_t* perm);
/* k nearest `points` of each query (O2 order: squared distance, then index).
 * out[nq * k] int32 indices into points. */
mgm_status mgm_host_knn(const double* points, int64_t n, const double* queries, int64_t nq,
                        int k, int32_t* out);
/* The same kNN lists computed on the GPU (the path mgm_setup takes for k <= 64): host
 * arrays in and out, copied through device buffers on the current device.  MGM_ERR_ARG for
 * k < 1, k > n or k > 64; MGM_ERR_CUDA on a CUDA error. */
mgm_status mgm_device_knn(const double* points, int64_t n, const double* queries, int64_t nq,
                          int k, int32_t* out);
/* Weighted sample elimination of n points down to nt (O8). keep[nt] ascending. */
mgm_status mgm_host_wse(const double* points, int64_t n, int64_t nt, int64_t* keep);
/* The same elimination on the GPU (the path mgm_setup takes unless MGM_HOST_WSE=1): host
 * arrays in and out, copied through device buffers on the current device.  keep[nt]
 * ascending, equal to mgm_host_wse's.  MGM_ERR_ARG for nt < 1 or nt > n; MGM_ERR_INPUT for
 * duplicate points or no non-degenerate radius; MGM_ERR_CUDA on a CUDA error. */
mgm_status mgm_device_wse(const double* points, int64_t n, int64_t nt, int64_t* keep);
/* Greedy colouring (O11) of sym(pattern) minus the diagonal, vertices in index order.
 * CSR pattern ptr[n+1], col[ptr[n]]; colour[n] out; *n_colours out. */
mgm_status mgm_host_colouring(int64_t n, const int64_t* ptr, const int32_t* col, int32_t* colour,
                              int* n_colours);

/* Partition tables of one level for `rank` of `nranks` (the host code mgm_dist_attach runs;
 * DESIGN.md "Multi-GPU").  Rows are the level's lib order (colour-major: ascending rows =
 * ascending colours); owner[n] = owning rank of each row.  L_ptr/L_col: pattern of L_j;
 * P_ptr/P_col (n rows -> nc coarse, owner_c[nc]): P_j, whose transpose R_j reads this level
 * (NULL if none); Pf_ptr/Pf_col (nf fine rows -> n, owner_f[nf]): P_{j-1}, which reads this level
 * (NULL on level 0).  Outputs (host, caller-allocated; any may be NULL): rows[n] owned rows
 * (ascending, *n_rows); ghosts[n] ghost rows sorted by (owner, row) (*n_ghosts); peers[nranks]
 * (*n_peers); send_rows[n] per peer concatenated (rows the peer reads that this rank owns);
 * send_off / recv_off [nranks + 1] per-peer offsets into send_rows / ghosts;
 * send_coff / recv_coff [nranks * (ncol + 1)] per peer the absolute offset of each colour's
 * slice.  No GPU needed. */
mgm_status mgm_host_partition_level(int64_t n, const int64_t* L_ptr, const int32_t* L_col, const int32_t* colour,
                                    int ncol, const int32_t* owner, int64_t nc, const int64_t* P_ptr,
                                    const int32_t* P_col, const int32_t* owner_c, int64_t nf, const int64_t* Pf_ptr,
                                    const int32_t* Pf_col, const int32_t* owner_f, int nranks, int rank,
                                    int64_t* n_rows, int64_t* rows, int64_t* n_ghosts, int64_t* ghosts, int* n_peers,
                                    int32_t* peers, int64_t* send_rows, int64_t* send_off, int64_t* recv_off,
                                    int64_t* send_coff, int64_t* recv_coff);

#ifdef __cplusplus
}
#endif
#endif /* MGM_H */

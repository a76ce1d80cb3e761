/*
 * mq_b200.h — C ABI of libmq_b200.so, the B200 (sm_100a) drop-in for the hot
 * path of the reference `mqsolve` (arXiv 1611.06721): the repeated PCG solve
 * of the singular nonconducting curl-curl block K_n, the SPE/CSPE and POD
 * start vectors, the Brauer K_c(a_c) update and the explicit-Euler update.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/mqsolve):
 *   mq_ctx_create / mq_partition_export   model.py:438-470 (_Topology, partition)
 *   mq_pcg_solve_host / mq_pcg_solve_dev  krylov.py:174-250 (pcg_solve) on K_n
 *   mq_csr_*                              krylov.py:161-171 + 174-250 for a
 *                                         general CsrMatrix operator (sparse.py:50-176)
 *   mq_kn_apply                           schur.py:189-191 (_kn_scipy @ x)
 *   mq_strategy_* (start/observe)         startvec.py:315-472 (StartVectorStrategy,
 *                                         CspeStrategy, PodStrategy, previous)
 *   mq_solve_kn                           schur.py:239-264 (SchurOperator.solve_kn)
 *   mq_kc_apply                           model.py:507-509 (kc_apply closure)
 *   mq_euler_step / mq_recover_an         schur.py:379-419
 *   mq_run_explicit                       schur.py:474-607 (time loop, fixed dt)
 *
 * Conventions
 *   Return codes: MQ_OK, MQ_NOT_CONVERGED (SolveReport.converged = False ->
 *   StepFailureError upstream), MQ_INDEFINITE (IndefiniteOperatorError),
 *   MQ_INVALID (ValueError), MQ_CUDA_ERROR (RuntimeError), MQ_NONFINITE
 *   (StepFailureError, non-finite conducting state).  mq_last_error() returns
 *   the message of the most recent failure on the calling thread.
 *   Host vectors are in the reference's compact order (ascending global edge
 *   id, model.py:455-464).  Device vectors ("_dev") are in the padded
 *   device layout of length mq_dev_len(); entries off the partition are 0.
 *   One context is driven by one host thread (single-writer),
 *   on the context's own CUDA stream.  The caller owns host buffers; the
 *   context owns device buffers.
 */
#ifndef MQ_B200_H
#define MQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MQ_OK 0
#define MQ_NOT_CONVERGED 1
#define MQ_INDEFINITE 2
#define MQ_INVALID 3
#define MQ_CUDA_ERROR 4
#define MQ_NONFINITE 5

/* RHS families, startvec.py:45-50 */
#define MQ_FAM_SOURCE 0
#define MQ_FAM_COUPLING_CURRENT 1
#define MQ_FAM_COUPLING_PREVIOUS 2

/* strategies, startvec.py:457-472 */
#define MQ_STRAT_ZERO 0
#define MQ_STRAT_PREVIOUS 1
#define MQ_STRAT_CSPE 2
#define MQ_STRAT_POD 3

typedef struct mq_ctx mq_ctx;

/* GridSpec + conductor Material + air reluctivity (model.py:70-155, 438). */
typedef struct mq_grid_desc {
  int32_t nx, ny, nz;
  double h;
  const int8_t *material; /* nx*ny*nz, C order; 0 air, 1 conductor, 2 coil */
  double nu_air;          /* air reluctivity (model.py:439) */
  double kappa;           /* conductor conductivity */
  double brauer_k1, brauer_k2, brauer_k3; /* nu = k1 exp(k2 B^2) + k3 */
  double kn_diag;         /* assembled K_n diagonal; 0 -> derived */
  double kn_off;          /* assembled |K_n| off-diagonal; 0 -> derived */
} mq_grid_desc;

/* SolveReport (krylov.py:75-79) plus operator applications. */
typedef struct mq_solve_report {
  int32_t iterations;
  int32_t converged;
  double final_rel_residual;
  int64_t applies;
} mq_solve_report;

/* Start-vector / solver configuration (schur.py:177-207, krylov.py:57-72). */
typedef struct mq_solver_cfg {
  int32_t strategy;  /* MQ_STRAT_* */
  int32_t max_cols;  /* CSPE basis cap */
  int32_t n_pod;     /* POD ring size */
  int32_t max_iter;
  double eps_pod;
  double rel_tol;
  double abs_tol;
  double drop_tol;   /* CSPE drop tolerance (schur.py:207: = rel_tol) */
} mq_solver_cfg;

/* Per-family diagnostics (startvec.py:392-454, schur.py:217-263). */
typedef struct mq_diag {
  int64_t solves[3];
  int64_t iterations[3];
  int64_t pcg_applies;
  int64_t maintenance_applies;
  int32_t basis_cols[3];   /* CSPE: basis size per family */
  int32_t pod_k;           /* POD: last retained modes */
  double pod_info;         /* POD: last kept information */
  double min_pod_info;     /* POD: min over projections (1.0 if none) */
  int64_t columns_accepted[3];
  int64_t columns_dropped[3];
  int64_t evictions[3];
} mq_diag;

/* ---- context ------------------------------------------------------------ */
const char *mq_last_error(void);
int mq_device_count(int32_t *count);
int mq_device_sm_count(int32_t device, int32_t *sms);
/* page-locked host memory (result arrays of the Python mirror) */
int mq_host_alloc(int64_t bytes, void **out);
int mq_host_free(void *p);
/* MQ_INVALID when a padded device vector would hold 2^31 entries or more
 * (about 890^3 cells: 16 GB per vector; the fused PCG kernels index entries
 * with 32-bit integers) */
int mq_ctx_create(const mq_grid_desc *desc, int32_t device, mq_ctx **out);
void mq_ctx_destroy(mq_ctx *ctx);
int64_t mq_n_n(const mq_ctx *ctx);     /* nonconducting interior dofs */
int64_t mq_n_c(const mq_ctx *ctx);     /* conducting dofs */
int64_t mq_dev_len(const mq_ctx *ctx); /* padded device vector length */
int mq_kn_coefficients(const mq_ctx *ctx, double *diag, double *off, double *jacobi_inv);
/* bit-exact partition check: global edge ids, ascending (model.py:455-462) */
int mq_partition_export(const mq_ctx *ctx, int64_t *noncond_global, int64_t *cond_global);
/* global edge id -> compact nonconducting index (-1 if not a K_n dof) */
int mq_map_global_to_noncond(const mq_ctx *ctx, const int64_t *gid, int64_t n, int64_t *out);
int mq_ctx_sync(mq_ctx *ctx);
/* optional external stream (cudaStream_t as void*; NULL restores own) */
int mq_ctx_set_stream(mq_ctx *ctx, void *stream);
/* Run this context's PCG kernel on a slice of `sms` SMs (0 = whole GPU), so
 * that several contexts (ensemble members, configs[3]) step concurrently on
 * their own streams.  No reference counterpart (its members run one by one). */
int mq_ctx_set_sm_budget(mq_ctx *ctx, int32_t sms);
/* Which fused PCG kernel this context launches and its grid (diagnostics). */
int mq_pcg_kernel_info(const mq_ctx *ctx, char *name, int32_t cap, int32_t *grid);

/* ---- device vectors (padded layout) ------------------------------------- */
int mq_vec_alloc(mq_ctx *ctx, double **dev);            /* zero-filled */
int mq_vec_free(mq_ctx *ctx, double *dev);
int mq_vec_upload(mq_ctx *ctx, const double *host_compact, double *dev);
int mq_vec_download(mq_ctx *ctx, const double *dev, double *host_compact);

/* ---- K_n operator (schur.py:189-191) ------------------------------------ */
int mq_kn_apply_dev(mq_ctx *ctx, const double *x_dev, double *y_dev);
int mq_kn_apply_host(mq_ctx *ctx, const double *x, double *y);

/* ---- PCG on K_n with Jacobi (krylov.py:174-250) -------------------------
 * x0 may be NULL (start from zero, r = b, no initial application). */
int mq_pcg_solve_dev(mq_ctx *ctx, const double *b_dev, const double *x0_dev,
                     double *x_dev, double rel_tol, double abs_tol,
                     int32_t max_iter, int32_t use_jacobi, mq_solve_report *rep);
int mq_pcg_solve_host(mq_ctx *ctx, const double *b, const double *x0, double *x,
                      double rel_tol, double abs_tol, int32_t max_iter,
                      int32_t use_jacobi, mq_solve_report *rep);

/* ---- member-batched PCG on K_n (BASELINE configs[3]) --------
 * nb = 1, 2, 4 or 8 right-hand sides of the same K_n solved in one launch
 * (krylov.py:174-250 per member, per-member alpha / beta / stopping test; a
 * converged member is frozen).  b, x0 (may be NULL), x: host, member-major
 * (member m's compact vector at offset m * n_n); reports: nb records;
 * kernel_ms (optional): the launch's device time. */
int mq_pcg_solve_batched_host(mq_ctx *ctx, int32_t nb, const double *b, const double *x0, double *x,
                              double rel_tol, double abs_tol, int32_t max_iter, int32_t use_jacobi,
                              mq_solve_report *reports, double *kernel_ms);

/* ---- PCG on a general CSR operator (krylov.py:161-250) ------------------
 * int32 column indices, int64 row pointers; inv_diag NULL = no
 * preconditioner.  All pointers are HOST; the solve runs on `device`. */
int mq_csr_pcg_solve(int32_t device, int64_t n, const int64_t *row_ptr,
                     const int32_t *col_idx, const double *values,
                     const double *b, const double *x0, double *x,
                     const double *inv_diag, double rel_tol, double abs_tol,
                     int32_t max_iter, mq_solve_report *rep);
int mq_csr_spmv(int32_t device, int64_t nrows, int64_t ncols,
                const int64_t *row_ptr, const int32_t *col_idx,
                const double *values, const double *x, double *y);

/* ---- device-resident CSR operator (models given as matrices) -----------
 * The reference's manifest path (bench.py:228-313 load_model, model.py:640-689
 * export_model) gives a PartitionedSystem of CSR blocks with no grid behind
 * it.  mq_csr_op uploads one block once (K_n, K_cn, its transpose or K_c);
 * PCG solves (krylov.py:174-250, replaces pcg_solve(a=CsrMatrix) at
 * mq/schur.py:253 through the module-global rebinding) and SpMVs
 * (sparse.py:179-184, CsrMatrix.matvec) reuse it.  inv_diag: the Jacobi
 * inverse (krylov.py:90-94), NULL if never used.  Host vectors. */
typedef struct mq_csr_op mq_csr_op;
int mq_csr_op_create(int32_t device, int64_t nrows, int64_t ncols,
                     const int64_t *row_ptr, const int32_t *col_idx,
                     const double *values, const double *inv_diag, mq_csr_op **out);
int mq_csr_op_destroy(mq_csr_op *op);
int mq_csr_op_pcg(mq_csr_op *op, const double *b, const double *x0, double *x,
                  int32_t use_inv, double rel_tol, double abs_tol, int32_t max_iter,
                  mq_solve_report *rep);
int mq_csr_op_spmv(mq_csr_op *op, const double *x, double *y);

/* ---- solver: strategy + families + conducting block ---------------------
 * One solver per context.  pattern: compact source pattern (n_n). */
int mq_solver_init(mq_ctx *ctx, const mq_solver_cfg *cfg, const double *pattern);
int mq_solver_reset(mq_ctx *ctx);
/* SchurOperator.solve_kn: rhs/y device vectors; reports iterations */
int mq_solve_kn(mq_ctx *ctx, int32_t family, const double *rhs_dev, double *y_dev,
                mq_solve_report *rep);
/* StartVectorStrategy pieces on device vectors */
int mq_strategy_start(mq_ctx *ctx, int32_t family, const double *rhs_dev, double *x0_dev);
int mq_strategy_observe(mq_ctx *ctx, int32_t family, const double *y_dev);
int mq_diagnostics(mq_ctx *ctx, mq_diag *out);
/* CSPE cache contents of one family (compact host, column-major n_n x k) */
int mq_cspe_export(mq_ctx *ctx, int32_t family, int32_t *k, double *basis,
                   double *products, double *galerkin);

/* ---- conducting block -------------------------------------------------- */
/* K_c(state) x on host compact n_c vectors (model.py:507-509) */
int mq_kc_apply_host(mq_ctx *ctx, const double *state, const double *x, double *y);
/* y_n = K_cn^T a_c (host n_c -> host n_n) and y_c = K_cn x_n */
int mq_kcn_t_apply_host(mq_ctx *ctx, const double *a_c, double *y_n);
int mq_kcn_apply_host(mq_ctx *ctx, const double *x_n, double *y_c);
/* M_c diagonal (model.py:486-491) */
int mq_mc_diag(mq_ctx *ctx, double *mc_diag);

/* state a_c lives on device; set/get in compact host order */
int mq_state_set(mq_ctx *ctx, const double *a_c, double t);
int mq_state_get(mq_ctx *ctx, double *a_c, double *t);
/* explicit_euler_step: two solves (SOURCE at t+dt with waveform value
 * wave_new, COUPLING_PREVIOUS), then the Euler update (schur.py:379-405) */
int mq_euler_step(mq_ctx *ctx, double dt, double wave_new, int64_t step_index,
                  mq_solve_report *rep_src, mq_solve_report *rep_cpl);
/* recover_an at the current state (schur.py:408-419); a_n to host if non-NULL */
int mq_recover_an(mq_ctx *ctx, double wave_now, double *a_n_host,
                  mq_solve_report *rep_src, mq_solve_report *rep_cpl);
/* One-call host forms of explicit_euler_step((a_c, t), dt, op) and
 * recover_an(op, a_c, t) (schur.py:379-419): upload a_c (compact host order),
 * run, return a_c_next / a_n; a single stream synchronisation per call. */
int mq_euler_step_host(mq_ctx *ctx, const double *a_c, double t, double dt, double wave_new,
                       int64_t step_index, double *a_c_next,
                       mq_solve_report *rep_src, mq_solve_report *rep_cpl);
int mq_recover_an_host(mq_ctx *ctx, const double *a_c, double t, double wave_now, double *a_n_host,
                       mq_solve_report *rep_src, mq_solve_report *rep_cpl);

/* a_n = y_src - y_cpl of the most recent recovery / step solves (host n_n) */
int mq_last_an(mq_ctx *ctx, double *a_n_host);

/* Device-resident time loop: n_steps Euler steps with per-step dt[] and
 * waveform wave[] (wave[m] = waveform(t_m) for m = 0..n_steps, t_0 = start),
 * recover_an after every step when recover_every_step != 0 (output rows).
 * iters_out (optional, 4*n_steps int32): per step [src, cpl_prev, src_rec,
 * cpl_cur]; a_c_hist (optional, n_steps*n_c) states after each step.
 * Host sync only at the end.  use_graph != 0 replays one captured step. */
int mq_run_explicit(mq_ctx *ctx, int64_t n_steps, const double *dt,
                    const double *wave, int32_t recover_every_step,
                    int32_t use_graph, int32_t *iters_out, double *a_c_hist,
                    int64_t *failed_step);

/* mq_run_explicit that also records a_n = y_src - y_cpl of every step's
 * recovery (a_n_hist, n_steps*n_n, compact order; needs
 * recover_every_step != 0): the per-step A-field (a_c, a_n) of the run. */
int mq_run_explicit_states(mq_ctx *ctx, int64_t n_steps, const double *dt,
                           const double *wave, int32_t recover_every_step,
                           int32_t use_graph, int32_t *iters_out, double *a_c_hist,
                           double *a_n_hist, int64_t *failed_step);

/* The same loop in three calls: prepare (tables, counters), enqueue n steps
 * (asynchronous), finish (sync, error check, iteration log). */
int mq_run_prepare(mq_ctx *ctx, int64_t n_steps, const double *dt, const double *wave,
                   int32_t recover_every_step);
int mq_run_steps(mq_ctx *ctx, int64_t n, int32_t use_graph, double *a_c_hist_dev);
int mq_run_finish(mq_ctx *ctx, int32_t *iters_out, int64_t *failed_step);

/* B probe: mean |B| over probe cells (model.py:415-425 probe_b; default cell
 * set model.py:562-566, built by the host).  Cells are global cell ids and
 * must be conductor cells (their B depends on a_c only).  n = 0 clears.
 * Once set, every step of mq_run_steps also logs B_probe of its new state;
 * mq_run_probe_log copies the first n entries of the current run. */
int mq_probe_set(mq_ctx *ctx, const int64_t *cells, int64_t n);
int mq_probe_b(mq_ctx *ctx, const double *a_c_host /* NULL = current state */, double *out);
int mq_run_probe_log(mq_ctx *ctx, int64_t n, double *out);
/* Per-step strategy diagnostics of the current run, 8 doubles per step:
 * [0..2] CSPE basis size of families SOURCE, COUPLING_CURRENT,
 * COUPLING_PREVIOUS after that step's inserts; [3,4] POD (last_k, last_info)
 * after the Euler step's solves; [5,6] the same after the recovery's solves;
 * [7] unused.  The host folds them into the trace columns basis_cols, pod_k,
 * pod_info as the reference's _WindowStats / emit_row (schur.py:448-467,
 * 524-538). */
int mq_run_diag_log(mq_ctx *ctx, int64_t n, double *out);

/* Spectral estimate lambda_max(M_c^-1 K_S(a_ref)) by power iteration
 * (schur.py:327-376): v0 = normalised start vector (host n_c), a_ref NULL = 0.
 * dt = safety * 2 / lambda. */
int mq_estimate_cfl(mq_ctx *ctx, const double *a_ref, const double *v0, int32_t power_iters,
                    double power_tol, double safety, double rel_tol, int32_t max_iter,
                    double *lambda_out, double *dt_out, int32_t *used_out, int64_t *pcg_applies);

/* ---- i-slab distributed K_n PCG (BASELINE configs[4]) --------------------
 * A slab context owns node planes [i_lo, i_hi) of the global grid
 * (partition restricted bit-exactly); local planes -1 and n = i_hi - i_lo
 * are ghost planes refreshed by the host's halo exchange.  Each phase
 * returns this rank's partial sums (host); the host allreduces them over the
 * ranks and drives krylov.py:174-250's control flow (slab.py). */
int mq_ctx_create_slab(const mq_grid_desc *desc, int32_t i_lo, int32_t i_hi, int32_t device,
                       mq_ctx **out);
/* {C, Si, Sj, off, total, n_planes}: plane l of component c occupies
 * [c*C + (l+1)*Si, c*C + (l+2)*Si) */
int mq_layout(const mq_ctx *ctx, int64_t *out6);
int mq_slab_buffers(mq_ctx *ctx, double **r, double **pa, double **pb, double **ap);
int mq_slab_init(mq_ctx *ctx, const double *b_dev, double *x_dev, int32_t x0_mode,
                 int32_t use_jacobi, double *part3);
int mq_slab_k1(mq_ctx *ctx, double *x_dev, int32_t first, double beta, double alpha_prev,
               int32_t pold_is_a, int32_t use_jacobi, double *part1);
int mq_slab_k2(mq_ctx *ctx, double alpha, int32_t use_jacobi, double *part2);
int mq_slab_final(mq_ctx *ctx, double *x_dev, double alpha, int32_t p_is_a);

/* Fused slab PCG (configs[4]): one persistent kernel per rank runs the
 * stencil passes, the ghost-plane stores into the neighbour ranks and the
 * cross-rank all-reduce (mailbox + arrival counter in every rank's memory)
 * with no host round trip per iteration (krylov.py:174-250 per iteration).
 * _local: all nranks slab contexts of this process on one GPU, emulated as
 * the CTA groups of one cooperative launch.  b/x: per rank device vectors in
 * the slab layout (x is also the start vector when x0_given). */
int mq_slab_fused_solve_local(mq_ctx **ctxs, int32_t nranks, const double *const *b, double *const *x,
                              int32_t x0_given, double rel_tol, double abs_tol, int32_t max_iter,
                              int32_t use_jacobi, mq_solve_report *report);
/* One rank per process (one GPU each): exchange kIpcBufs (9) CUDA IPC
 * handles per rank (r, p_a, p_b, x, mailbox, counter, r2, ap, ap2; 64 bytes
 * each) with
 * mq_slab_ipc_export / an all-gather / mq_slab_ipc_import, then every rank
 * calls mq_slab_fused_solve_peer; the neighbours' ghost planes, mailboxes
 * and counters are written over NVLink by the kernel itself. */
int mq_slab_ipc_export(mq_ctx *ctx, const double *x_dev, void *handles_out);
int mq_slab_ipc_import(mq_ctx *ctx, int32_t rank, int32_t nranks, const void *all_handles,
                       const int32_t *nplanes, double *x_dev);
int mq_slab_fused_solve_peer(mq_ctx *ctx, const double *b_dev, int32_t x0_given, double rel_tol,
                             double abs_tol, int32_t max_iter, int32_t use_jacobi, mq_solve_report *report);

/* ---- sharded explicit step over i-slabs (BASELINE configs[4]) -----------
 * The SchurOperator step (schur.py:379-419) with the K_n-sized vectors of a
 * slab context (mq_ctx_create_slab) and the CSPE / previous / zero start
 * vectors (startvec.py:158-225, 345-431).  Every reduction leaves this rank's
 * partial sums (MQ_SS_NPART doubles) in `part`; the host sums them over the
 * ranks in rank order and hands the totals back as `tot`, so every rank takes
 * the same decisions on the same scalars.  The conducting state a_c (full
 * grid, compact order) is replicated on every rank; each rank integrates the
 * conducting edges whose node plane it owns (mq_ss_owned).  The host drives
 * the sequence (paper_1611_06721_b200/slabstep.py), the halo exchanges and
 * the PCG (mq_slab_fused_solve_local / _peer). */
#define MQ_SS_NPART 34
/* pattern_local: the source pattern on the slab's own dofs (slab compact order) */
int mq_ss_init(mq_ctx *ctx, const mq_solver_cfg *cfg, const double *pattern_local);
/* {n_c of the grid, owned conducting edges, conductor cells, K_cn^T rows of the slab} */
int mq_ss_info(mq_ctx *ctx, int64_t *out4);
int mq_ss_owned(mq_ctx *ctx, int64_t *idx);
/* 0 rhs_src, 1 rhs_cpl, 2 y_src, 3 y_cpl, 4 y_cur, 5 w2 (CGS vector), 6 y_cpl - y_src */
int mq_ss_vec(mq_ctx *ctx, int32_t which, double **out);
int mq_ss_state_set(mq_ctx *ctx, const double *a_c);
int mq_ss_state_get(mq_ctx *ctx, double *a_c);
/* which 0: rhs_src = pattern * wave (schur.py:81-82); 1: rhs_cpl = K_cn^T a_c (schur.py:394) */
int mq_ss_rhs(mq_ctx *ctx, int32_t which, double wave);
/* SubspaceCache.project (startvec.py:207-225) in two halves around the all-reduce */
int mq_ss_project(mq_ctx *ctx, int32_t family, int32_t rhs_which, double *part);
int mq_ss_start(mq_ctx *ctx, int32_t family, const double *tot, double *x_dev);
/* solution x (slab vector) -> the family's solution vector; rep counted in diagnostics */
int mq_ss_store(mq_ctx *ctx, int32_t family, const double *x_dev, const mq_solve_report *rep);
/* SubspaceCache.insert (startvec.py:158-199), phases 0..5 (solver_slab.cuh) */
int mq_ss_observe(mq_ctx *ctx, int32_t family, int32_t phase, const double *tot, double *part, int32_t *flag);
/* Euler update (schur.py:392-404): prep forms y_cpl - y_src (halo next), then
 * the owned conducting edges' new values (owned order); MQ_NONFINITE on a
 * non-finite state */
int mq_ss_euler_prep(mq_ctx *ctx);
int mq_ss_euler(mq_ctx *ctx, double dt, double *owned_out);
/* a_n = y_src - y_cur of the last recovery on the slab's dofs (schur.py:408-419) */
int mq_ss_an(mq_ctx *ctx, double *a_n_local);
int mq_ss_diag(mq_ctx *ctx, mq_diag *out);
/* CSPE cache of one family on this slab (as mq_cspe_export, slab compact order) */
int mq_ss_cspe_export(mq_ctx *ctx, int32_t family, int32_t *k, double *basis, double *products, double *galerkin);

/* Guard check: count the off-partition entries (boundary, conducting, guard
 * and padding positions; a slab's ghost planes excepted) that are not 0 in
 * every device vector the context owns (PCG scratch, user vectors, the
 * solver's caches and work vectors).  The stencils read those entries as
 * boundary values, so any stray write there shows; tests run it after runs
 * (memory-safety evidence on a pool where compute-sanitizer is closed). */
int mq_guard_check(mq_ctx *ctx, int64_t *bad_entries, int32_t *bad_vectors, int32_t *checked);

/* ---- timing (CUDA events on the context stream) ------------------------- */
/* Sum of the device times of the PCG launches of the last step (when PCG
 * timing is enabled with mq_pcg_stats(..., 1)). */
int mq_pcg_collect(mq_ctx *ctx, double *ms, int32_t *n_events);
int mq_timer_start(mq_ctx *ctx);
int mq_timer_stop(mq_ctx *ctx, double *ms);
/* cumulative device time and launch count of the PCG kernels */
int mq_pcg_stats(mq_ctx *ctx, double *pcg_ms, int64_t *pcg_iterations,
                 int64_t *launches, int32_t enable);
int mq_kernel_launches(mq_ctx *ctx, int64_t *count);
/* %globaltimer stamps of the last PCG launch (CTA 0), when the context was
 * created with MQ_PCG_TRACE set: [start, then per iteration K1 end, barrier
 * 1 end, K2 end, barrier 2 end] for the first 64 iterations. */
int mq_pcg_trace(mq_ctx *ctx, uint64_t *stamps, int32_t n);
int mq_l2_flush(mq_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* MQ_B200_H */

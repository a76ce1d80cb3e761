// The mq_ctx object and the launchers shared between translation units.
#pragma once

#include <cuda_runtime.h>

#include <set>
#include <vector>

#include "mq_internal.h"

namespace mq {

constexpr int MAXS = 32;      // max CSPE columns / POD snapshots per family
constexpr int kEvPool = 16;   // PCG launches timed per step

// Small per-family state kept on the device (startvec.py:118-225, 239-309).
// Vectors live in slots; order[] maps logical column -> slot so that FIFO
// eviction (startvec.py:180-184) and column drops (startvec.py:201-205)
// never move vector data.
struct FamDev {
  int k;                 // CSPE basis size / POD snapshots held
  int order[MAXS];       // logical -> slot
  int head;              // POD: next ring slot
  int kprime;            // CSPE: columns left after a pending eviction
  int new_slot;          // CSPE: slot receiving the accepted column
  int accept;            // CSPE: insert decision of the current observe
  int x0_mode;           // PCG start mode chosen by the last start vector
  int podk;              // POD: retained modes of the last projection
  int has_last;          // previous strategy
  int pending;           // CSPE: a deferred insert of the last recovery's solution waits
  int skip;              // CSPE: the current (gated) insert is a no-op
  double nv2, nw2;       // CSPE: squared norms of the raw / orthogonalised vector
  double nrm;            // CSPE: ||w|| used to normalise
  double pod_info;       // POD: kept information of the last projection
  double pod_sigma[MAXS];
  double G[MAXS * MAXS]; // CSPE Galerkin (logical order) / POD Gram (slot order)
  double d[MAXS + 2];    // scratch dot products
  double coef[MAXS];
  double W[MAXS * MAXS]; // POD: basis combination, W[l*MAXS+j] (l: logical snapshot)
  double Gk[MAXS * MAXS];// POD Galerkin scratch
  long long products, accepted, dropped, evictions, pod_applies;
  long long proj_count;
  double gs[MAXS + 2];   // POD: one-pass Galerkin sums before the scatter into Gk / d
};

// Device-wide run state of the stepper.
struct RunDev {
  unsigned int err;       // first error code (MQ_*), 0 = none
  int err_family;
  long long err_step;
  long long step;         // steps taken (device counter)
  long long solve_idx;    // solves logged
  long long pcg_applies;
  double min_pod_info;
  int any_pod;
  int pod_last_k;
  double pod_last_info;
};

struct SolverHost;
struct SlabPeer;
struct SlabStepHost;

}  // namespace mq

struct mq_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  int sms = 148;
  mq_grid_desc desc{};
  std::vector<int8_t> material;
  mq::Topology topo;
  double kn_diag = 0, kn_off = 0, jac_inv = 0;
  // device topology
  uint32_t *d_mask = nullptr;
  int32_t *d_nc_pad = nullptr;
  double *d_stage = nullptr;
  // PCG scratch
  double *d_r = nullptr, *d_p0 = nullptr, *d_p1 = nullptr, *d_ap = nullptr;
  double *d_ap2 = nullptr;  // Ap of odd iterations (pcg_resident1_kernel, pcg_tma1_kernel)
  double *d_r2 = nullptr;   // r of odd iterations (pcg_tma1_kernel)
  double *d_tmp0 = nullptr, *d_tmp1 = nullptr;
  double *d_partials = nullptr;
  mq::GridBar *d_bar = nullptr;
  double *d_mbox = nullptr;              // fused slab PCG: rank mailbox
  unsigned long long *d_mcount = nullptr; // [arrival counter, epoch]
  mq::PcgOut *d_out = nullptr;
  mq::PcgOut *h_out = nullptr;
  unsigned long long *d_trace = nullptr;
  int pcg_grid = 1;
  int pcg_variant = 0;        // 0: TMA brick kernel, 1: thread-per-row, 2: smem-resident
  mq::BrickGeo geo{};
  int brick_grid = 1;
  mq::BrickGeo res_geo{};
  int res_grid = 0;
  // conducting block (device)
  int64_t *d_kcn_ptr = nullptr;
  int32_t *d_kcn_col = nullptr;
  int8_t *d_kcn_sgn = nullptr;
  int32_t *d_kcnt_row = nullptr;
  int64_t *d_kcnt_ptr = nullptr;
  int32_t *d_kcnt_src = nullptr;
  int8_t *d_kcnt_sgn = nullptr;
  double *d_minv = nullptr;
  int32_t *d_f_edge = nullptr;
  int8_t *d_f_sgn = nullptr;
  double *d_f_base = nullptr;
  int32_t *d_f_cell = nullptr;
  int32_t *d_cell_face = nullptr;
  int32_t *d_e_face = nullptr;
  int8_t *d_e_sgn = nullptr;
  double *d_cell_nu = nullptr;
  double *d_ac = nullptr, *d_ac_next = nullptr, *d_ac_x = nullptr, *d_yc = nullptr;
  double two_h4 = 0;
  double t_now = 0;
  // solver
  mq::SolverHost *solver = nullptr;
  mq::SlabPeer *peer = nullptr;  // fused slab PCG across processes (IPC-mapped neighbours)
  mq::SlabStepHost *sstep = nullptr;  // sharded explicit step on a slab context (solver_slab.cuh)
  int slab_lo = 0, slab_hi = 0;       // node planes [lo, hi) of a slab context (0, 0: whole grid)
  // bookkeeping
  std::vector<void *> allocs;
  std::set<double *> vecs;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_pcg0 = nullptr, ev_pcg1 = nullptr;
  bool pcg_timing = false;
  double pcg_ms = 0;
  int64_t pcg_iters = 0, pcg_launches = 0;
  int64_t launches = 0;
  cudaEvent_t ev_pool[2 * 16] = {};
  int ev_n = 0;
  int sm_budget = 0;  // 0 = all SMs; else the PCG kernel runs on this many SMs
  void *flush_buf = nullptr;
  unsigned flush_val = 1;
};

namespace mq {

struct StencilPcgArgs;
struct CsrPcgArgs;

int ctx_alloc(mq_ctx *ctx, void **p, size_t bytes);
int ctx_pcg(mq_ctx *ctx, const double *b, double *x, int x0_mode, double rel_tol, double abs_tol, int max_iter,
            int use_jac, mq_solve_report *rep);
int conducting_init(mq_ctx *ctx);
void solver_free(mq_ctx *ctx);
void slab_peer_free(mq_ctx *ctx);
void slab_step_free(mq_ctx *ctx);
void solver_graph_reset(mq_ctx *ctx);

int coop_grid(const void *kernel, int want_blocks, int *out);
int launch_pcg_stencil(const StencilPcgArgs &args, int grid, cudaStream_t s);
int pcg_stencil_grid(int64_t words, int *out);
int launch_pcg_csr(const CsrPcgArgs &args, int grid, cudaStream_t s);
int pcg_csr_grid(int64_t n, int *out);
int brick_pcg_setup(const Lay &L, int nx, int ny, int nz, int sm_cap, int *grid, BrickGeo *geo);
bool tma_single_reduction(const BrickGeo &g);  // pcg_tma1_kernel (one grid barrier per iteration) is launched
int launch_pcg_brick(const StencilPcgArgs &args, const BrickGeo &geo, int grid, cudaStream_t s);
struct KnMulti;
int kn_multi_prepare(const Lay &L, const BrickGeo &geo, const uint32_t *mask, double dg, double of,
                     double *const *x, double *const *y, int nvec, const int *kptr, int sms, KnMulti **out);
int kn_multi_launch(const KnMulti *k, cudaStream_t s);
void kn_multi_free(KnMulti *k);
int launch_kn_apply_brick(const Lay &L, const BrickGeo &geo, const uint32_t *mask, double dg, double of,
                          const double *x, double *y, int sms, cudaStream_t s);
int launch_pcg_ctx(mq_ctx *ctx, const StencilPcgArgs &args);
int resident_pcg_setup(int nx, int ny, int nz, int *grid, BrickGeo *geo);
int launch_pcg_resident(const StencilPcgArgs &args, const BrickGeo &geo, int grid, cudaStream_t s);
bool resident_single_reduction(int li_max);
// MQ_PCG_STRESS=<ns>: test-only delay of some CTAs after every grid barrier of
// the resident kernels (results must not change: they depend on no timing)
int pcg_stress_ns();
int launch_kn_apply(const Lay &L, const uint32_t *mask, double dg, double of, const double *x, double *y, int sms,
                    cudaStream_t s);
int launch_scatter(int64_t n, const int32_t *idx, const double *src, double *dst, int sms, cudaStream_t s);
int launch_gather(int64_t n, const int32_t *idx, const double *src, double *dst, int sms, cudaStream_t s);
int launch_csr_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *va, const double *x, double *y,
                    int sms, cudaStream_t s);

}  // namespace mq

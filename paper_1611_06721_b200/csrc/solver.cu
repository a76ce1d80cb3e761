// Device-resident SchurOperator: start-vector strategies, solve_kn, the
// Brauer K_c update, the explicit-Euler update and the time loop.
//
// Reference (pkg/src/mqsolve):
//   SubspaceCache.insert/project ..... startvec.py:158-225 (CGS2, FIFO, bordered Galerkin)
//   _cholesky_lower / _solve_spd ..... startvec.py:59-79
//   pod_start_vector / SnapshotBuffer  startvec.py:239-309
//   strategies ....................... startvec.py:345-472
//   solve_kn ......................... schur.py:239-264
//   kc_apply (Brauer) ................ model.py:107-125, 492-509
//   explicit_euler_step / recover_an . schur.py:379-419
//   run_explicit ..................... schur.py:474-607
//
// All decisions (accept/drop/evict, pivot failures, POD truncation, solve
// failures) are taken on the device, so a whole time step is a fixed kernel
// sequence that can be captured once in a CUDA graph and replayed; the host
// reads iteration logs and error words only at the end of a run.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "mq_ctx.h"
#include "mq_device.cuh"

namespace mq {

// ---------------------------------------------------------------------------
// host-side solver object
// ---------------------------------------------------------------------------
struct StepParams {
  double dt;        // step size of the current step
  double wave_new;  // waveform(t + dt)
  double wave_now;  // waveform(t) used by recover_an
  long long step;   // 1-based step index for error messages
};

struct SolverHost {
  mq_solver_cfg cfg{};
  FamDev *d_fam = nullptr;  // 3 families
  RunDev *d_run = nullptr;
  StepParams *d_par = nullptr;
  // slot tables (device arrays of device pointers)
  double **d_U[3] = {nullptr, nullptr, nullptr};
  double **d_KU[3] = {nullptr, nullptr, nullptr};
  double **d_X[3] = {nullptr, nullptr, nullptr};
  double **d_B = nullptr, **d_KB = nullptr;
  std::vector<double *> h_U[3], h_KU[3], h_X[3], h_B, h_KB;
  double *last[3] = {nullptr, nullptr, nullptr};
  double *w1 = nullptr, *w2 = nullptr;
  double *rhs_src = nullptr, *rhs_cpl = nullptr, *y_src = nullptr, *y_cpl = nullptr;
  double *y_cur = nullptr;  // recovery's coupling solution (y_cpl may still be read by the side stream)
  // source pattern (sparse: padded index + value)
  int32_t *d_pat_idx = nullptr;
  double *d_pat_val = nullptr;
  int64_t n_pat = 0;
  // reduction scratch
  double *d_red = nullptr;
  unsigned int *d_cnt = nullptr;
  int red_grid = 1;
  // logs
  int32_t *d_log = nullptr;
  int64_t log_cap = 0;
  double *d_dt_tab = nullptr, *d_wave_tab = nullptr;
  int64_t tab_cap = 0;
  std::vector<void *> mem;
  int *d_iota = nullptr;  // identity order 0..MAXS-1
  cudaGraphExec_t graph_exec = nullptr;
  // one-call graphs of the host-facing mq_euler_step / mq_recover_an
  cudaGraphExec_t euler_graph = nullptr, recover_graph = nullptr;
  int64_t euler_launches = 0, recover_launches = 0;
  bool graph_ok = true;
  int64_t launches_per_step = 0;
  bool recover_every_step = true;
  int kb = 32;  // compile-time basis bound used for the tall-skinny kernels
  int per_step = 4;
  int64_t n_planned = 0, n_enqueued = 0;
  // overlap: the source family's cache update runs on a side stream on the
  // SMs the shared-memory-resident PCG kernel leaves idle, while the coupling
  // solve runs (own reduction scratch and CGS vectors)
  bool overlap = false;
  int side_grid = 0;
  cudaStream_t side = nullptr;
  // fork slots: 0/1 source update in the step / recovery, 2 coupling-previous
  // update, 3 deferred coupling-current insert, 4 deferred coupling-previous
  // insert (host-facing calls)
  static constexpr int kSlots = 5;
  cudaEvent_t ev_fork[kSlots] = {}, ev_join[kSlots] = {};
  bool pend[kSlots] = {};  // forks not yet joined (host-side, per enqueue sequence)
  // CSPE: a coupling family's insert is deferred into the next call's (or
  // step's) side stream; maybe_pending[fam] = one may wait on the device
  bool defer_cur = false;
  bool maybe_pending[3] = {false, false, false};
  double *d_red2 = nullptr, *w1b = nullptr, *w2b = nullptr;
  unsigned int *d_cnt2 = nullptr;
  // B probe (model.py:415-425): conductor-cell list indices, per-cell scratch,
  // per-step log of the current run
  int32_t *d_probe = nullptr, *d_probe_plan = nullptr;
  double *d_probe_vals = nullptr, *d_probe_log = nullptr, *d_probe_leaf = nullptr;
  unsigned int *d_probe_ctr = nullptr;  // k_probe's last-block ticket
  int probe_grid = 1;
  int64_t n_probe = 0, probe_cap = 0;
  // per-step strategy diagnostics of the current run (trace columns
  // basis_cols / pod_k / pod_info, schur.py:448-467,524-538): kDiagW doubles
  // per step, see k_dlog_k / k_dlog_pod
  double *d_dlog = nullptr;
  int64_t dlog_cap = 0;
  double *d_probe_out = nullptr;
  // POD: K B_j on the TMA brick march (grids run by pcg_tma_kernel), one
  // tensor map per basis slot per family (the k of the family's projection)
  KnMulti *kn_multi[3] = {nullptr, nullptr, nullptr};
  // POD: the eigen-decomposition of a family's snapshot Gram matrix depends
  // only on its ring, final once the family's push is done, so it runs on a
  // side stream right after the push (one CTA next to the TMA PCG kernel,
  // which leaves CTA slots free) and is joined before the family's next
  // projection or at the end of the call (MQ_EIG_AHEAD=0 disables)
  bool eig_ahead = false;
  cudaStream_t eig_side = nullptr;
  cudaEvent_t ev_ef[3] = {}, ev_ej[3] = {};
  bool eig_pend[3] = {false, false, false};
  // page-locked landing block of the host-facing calls: run status, the two
  // iteration counts and the probe value come back in one copy batch and one
  // stream synchronisation per call
  struct HostStage {
    RunDev run;
    int32_t it[2];
    double probe;
  } *h_st = nullptr;
  // B probe of the device state, computed by the host-facing recovery call
  // with its results (same kernel, same state, same cells as mq_probe_b) so
  // that the probe_b() that follows needs no device round trip; cleared by
  // every call that writes the state or the probe cells
  bool probe_cached = false;
  double probe_cache = 0.0;
};

static int s_alloc(mq_ctx *ctx, SolverHost *s, void **p, size_t bytes) {
  MQ_CUDA(cudaMalloc(p, bytes));
  MQ_CUDA(cudaMemsetAsync(*p, 0, bytes, ctx->stream));
  s->mem.push_back(*p);
  return MQ_OK;
}

void solver_graph_reset(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  if (!s) return;
  if (s->graph_exec) {
    cudaGraphExecDestroy(s->graph_exec);
    s->graph_exec = nullptr;
  }
  if (s->euler_graph) {
    cudaGraphExecDestroy(s->euler_graph);
    s->euler_graph = nullptr;
  }
  if (s->recover_graph) {
    cudaGraphExecDestroy(s->recover_graph);
    s->recover_graph = nullptr;
  }
}

void solver_free(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  if (!s) return;
  solver_graph_reset(ctx);
  for (int f = 0; f < 3; ++f) kn_multi_free(s->kn_multi[f]);
  if (s->eig_side) {
    cudaStreamSynchronize(s->eig_side);
    cudaStreamDestroy(s->eig_side);
  }
  for (int f = 0; f < 3; ++f) {
    if (s->ev_ef[f]) cudaEventDestroy(s->ev_ef[f]);
    if (s->ev_ej[f]) cudaEventDestroy(s->ev_ej[f]);
  }
  if (s->side) cudaStreamDestroy(s->side);
  for (int q = 0; q < SolverHost::kSlots; ++q) {
    if (s->ev_fork[q]) cudaEventDestroy(s->ev_fork[q]);
    if (s->ev_join[q]) cudaEventDestroy(s->ev_join[q]);
  }
  for (void *p : s->mem) cudaFree(p);
  cudaFree(s->d_probe);
  cudaFree(s->d_probe_vals);
  cudaFree(s->d_probe_log);
  cudaFree(s->d_dlog);
  cudaFree(s->d_probe_plan);
  cudaFree(s->d_probe_leaf);
  cudaFree(s->d_probe_ctr);
  if (s->h_st) cudaFreeHost(s->h_st);
  delete s;
  ctx->solver = nullptr;
}

// ---------------------------------------------------------------------------
// reduction helper: NQ runtime values per thread -> out[q] via last block
// ---------------------------------------------------------------------------
constexpr int RQ = MAXS + 2;  // max values reduced by one kernel

// Single-thread family bookkeeping run by thread 0 of the last block of the
// reduction that produced its inputs (one kernel boundary less per step of
// the CSPE/POD chains): the CSPE projection solve, the insert gates and
// decision, the Galerkin commit, the POD push commit.
enum PostKind : int { POST_NONE = 0, POST_PROJECT, POST_GATE, POST_GATE_C2, POST_DECIDE, POST_COMMIT, POST_POD_PUSH,
                      POST_GAL_SCATTER };
struct Post {
  int kind = POST_NONE;
  FamDev *f = nullptr;
  int max_cols = 0;
  int n_pod = 0;
  double drop_tol = 0.0;
};
__device__ void run_post(const Post &p);

__device__ __forceinline__ void last_block_reduce(double *acc, int nq, double *partials, unsigned int *counter,
                                                  double *out, const Post &post = Post()) {
  __shared__ double sm[RQ * kWarps];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  for (int q = 0; q < nq; ++q) {
    double v = warp_sum(acc[q]);
    if (lane == 0) sm[q * kWarps + warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < nq) {
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s = add(s, sm[threadIdx.x * kWarps + w]);
    partials[(int64_t)threadIdx.x * G + blockIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(counter, 1u) == (unsigned)G - 1);
  __syncthreads();
  if (is_last) {
    // every thread of the last block takes a strided share of each row of
    // partials; fixed-order warp and block sums (deterministic).  A serial
    // sum of G partials per value by one thread costs G dependent L2 loads.
    __threadfence();
    for (int q = 0; q < nq; ++q) {
      double s = 0.0;
      for (int b = threadIdx.x; b < G; b += blockDim.x) s = add(s, __ldcg(partials + (int64_t)q * G + b));
      s = warp_sum(s);
      if (lane == 0) sm[q * kWarps + warp] = s;
    }
    __syncthreads();
    if (threadIdx.x < nq) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s = add(s, sm[threadIdx.x * kWarps + w]);
      out[threadIdx.x] = s;
    }
    if (threadIdx.x == 0) *counter = 0u;
    if (post.kind != POST_NONE) {
      __syncthreads();
      if (threadIdx.x == 0) run_post(post);
    }
  }
}

#define FOR_ACTIVE(L, mask)                                                                  \
  for (int64_t w_ = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); w_ < (L).words;         \
       w_ += (int64_t)gridDim.x * kWarps)                                                    \
    if (((mask)[w_] >> (threadIdx.x & 31)) & 1u)

// Flat passes over pairs of padded entries: every device vector is 0 off the
// partition, so dots and linear combinations need no mask (the outputs stay
// 0 there).  KB bounds the number of basis vectors (compile-time register
// budget), UN pairs per thread are in flight per stream.
#ifndef MQ_TS_UNROLL
#define MQ_TS_UNROLL 2
#endif
template <int KB>
struct Unroll {
  static constexpr int value = KB <= 8 ? MQ_TS_UNROLL : 1;
};

// d[j] = A_{order[j]} . v  (j < k), d[k] = v . v when selfdot
template <int KB>
__global__ void __launch_bounds__(kBlock) k_mdot(int64_t npair, double *const *tab, const int *order,
                                                 const int *kptr, const double *__restrict__ v, int selfdot,
                                                 double *out, double *partials, unsigned int *counter,
                                                 Post post, const int *skip) {
  if (skip && *skip) return;  // gated deferred insert with nothing pending
  __shared__ const double2 *ptr[KB];
  const int k = *kptr;
  if (threadIdx.x < k) ptr[threadIdx.x] = reinterpret_cast<const double2 *>(tab[order[threadIdx.x]]);
  __syncthreads();
  double acc[KB + 2];
#pragma unroll
  for (int q = 0; q < KB + 2; ++q) acc[q] = 0.0;
  const double2 *v2 = reinterpret_cast<const double2 *>(v);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < npair; p0 += Unroll<KB>::value * stride) {
    double2 vv[Unroll<KB>::value], uu[Unroll<KB>::value][KB];
#pragma unroll
    for (int u = 0; u < Unroll<KB>::value; ++u) {
      const int64_t p = p0 + u * stride;
      if (p < npair) {
        vv[u] = __ldcg(v2 + p);
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j < k) uu[u][j] = __ldcg(ptr[j] + p);
      }
    }
#pragma unroll
    for (int u = 0; u < Unroll<KB>::value; ++u) {
      if (p0 + u * stride >= npair) break;
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < k) {
          acc[j] = add(acc[j], mul(uu[u][j].x, vv[u].x));
          acc[j] = add(acc[j], mul(uu[u][j].y, vv[u].y));
        }
      if (selfdot) {
        acc[KB] = add(acc[KB], mul(vv[u].x, vv[u].x));
        acc[KB] = add(acc[KB], mul(vv[u].y, vv[u].y));
      }
    }
  }
  if (selfdot) acc[k] = acc[KB];
  last_block_reduce(acc, k + (selfdot ? 1 : 0), partials, counter, out, post);
}

// out = in - sum_j c_j A_{order[j]};  d[j] = A_{order[j]} . out (j < ndot), d[ndot] = out.out
template <int KB>
__global__ void __launch_bounds__(kBlock) k_axpy_dots(int64_t npair, double *const *tab, const int *order,
                                                      const int *kptr, const double *c, const double *in,
                                                      double *outv, int ndot_is_k, double *dout,
                                                      double *partials, unsigned int *counter, const int *gate,
                                                      Post post) {
  if (gate && !*gate) return;
  __shared__ const double2 *ptr[KB];
  __shared__ double cs[KB];
  const int k = *kptr;
  if (threadIdx.x < k) {
    ptr[threadIdx.x] = reinterpret_cast<const double2 *>(tab[order[threadIdx.x]]);
    cs[threadIdx.x] = c[threadIdx.x];
  }
  __syncthreads();
  const int nd = ndot_is_k ? k : 0;
  double acc[KB + 2];
#pragma unroll
  for (int q = 0; q < KB + 2; ++q) acc[q] = 0.0;
  const double2 *in2 = reinterpret_cast<const double2 *>(in);
  double2 *out2 = reinterpret_cast<double2 *>(outv);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < npair; p0 += Unroll<KB>::value * stride) {
    double2 iv[Unroll<KB>::value], uu[Unroll<KB>::value][KB];
#pragma unroll
    for (int u = 0; u < Unroll<KB>::value; ++u) {
      const int64_t p = p0 + u * stride;
      if (p < npair) {
        iv[u] = __ldcg(in2 + p);
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j < k) uu[u][j] = __ldcg(ptr[j] + p);
      }
    }
#pragma unroll
    for (int u = 0; u < Unroll<KB>::value; ++u) {
      const int64_t p = p0 + u * stride;
      if (p >= npair) break;
      double tx = 0.0, ty = 0.0;
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < k) {
          tx = (j == 0) ? mul(cs[0], uu[u][0].x) : add(tx, mul(cs[j], uu[u][j].x));
          ty = (j == 0) ? mul(cs[0], uu[u][0].y) : add(ty, mul(cs[j], uu[u][j].y));
        }
      const double ox = sub(iv[u].x, tx), oy = sub(iv[u].y, ty);
      out2[p] = make_double2(ox, oy);
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < nd) {
          acc[j] = add(acc[j], mul(uu[u][j].x, ox));
          acc[j] = add(acc[j], mul(uu[u][j].y, oy));
        }
      acc[KB] = add(acc[KB], mul(ox, ox));
      acc[KB] = add(acc[KB], mul(oy, oy));
    }
  }
  acc[nd] = acc[KB];
  last_block_reduce(acc, nd + 1, partials, counter, dout, post);
}

// out = sum_j c_j A_{order[j]} (0 when k == 0)
template <int KB>
__device__ __forceinline__ void comb_body(int64_t npair, double *const *tab, const int *order, int k,
                                          const double *c, double *outv) {
  __shared__ const double2 *ptr[KB];
  __shared__ double cs[KB];
  if (threadIdx.x < k) {
    ptr[threadIdx.x] = reinterpret_cast<const double2 *>(tab[order[threadIdx.x]]);
    cs[threadIdx.x] = c[threadIdx.x];
  }
  __syncthreads();
  double2 *out2 = reinterpret_cast<double2 *>(outv);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < npair; p0 += Unroll<KB>::value * stride) {
    double2 uu[Unroll<KB>::value][KB];
#pragma unroll
    for (int u = 0; u < Unroll<KB>::value; ++u) {
      const int64_t p = p0 + u * stride;
      if (p < npair) {
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j < k) uu[u][j] = __ldcg(ptr[j] + p);
      }
    }
#pragma unroll
    for (int u = 0; u < Unroll<KB>::value; ++u) {
      const int64_t p = p0 + u * stride;
      if (p >= npair) break;
      double tx = 0.0, ty = 0.0;
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < k) {
          tx = (j == 0) ? mul(cs[0], uu[u][0].x) : add(tx, mul(cs[j], uu[u][j].x));
          ty = (j == 0) ? mul(cs[0], uu[u][0].y) : add(ty, mul(cs[j], uu[u][j].y));
        }
      out2[p] = make_double2(tx, ty);
    }
  }
}

template <int KB>
__global__ void __launch_bounds__(kBlock) k_comb(int64_t npair, double *const *tab, const int *order,
                                                 const int *kptr, const double *c, double *outv) {
  comb_body<KB>(npair, tab, order, *kptr, c, outv);
}

// the same for lo < k <= KB only (k read on the device: a small-k and a
// large-k instance are both launched, exactly one of them runs)
template <int KB>
__global__ void __launch_bounds__(kBlock) k_comb_range(int64_t npair, double *const *tab, const int *order,
                                                       const int *kptr, const double *c, double *outv, int lo) {
  const int k = *kptr;
  if (k <= lo || k > KB) return;
  comb_body<KB>(npair, tab, order, k, c, outv);
}

// CSPE: u = w/nrm into U[slot], ku = K u into KU[slot], cross_j = U_{order[j]}.ku (j<kprime), diag = u.ku
template <int KB>
__global__ void __launch_bounds__(kBlock) k_cspe_product(Lay L, const uint32_t *__restrict__ mask, double dg,
                                                         double of, FamDev *f, double *const *Utab,
                                                         double *const *KUtab, const double *__restrict__ w,
                                                         double *partials, unsigned int *counter, Post post) {
  if (!f->accept) return;
  __shared__ const double *ptr[MAXS];
  const int kp = f->kprime;
  if (threadIdx.x < kp) ptr[threadIdx.x] = Utab[f->order[threadIdx.x]];
  __syncthreads();
  double *U = Utab[f->new_slot];
  double *KU = KUtab[f->new_slot];
  const double nrm = f->nrm;
  double acc[KB + 2];
#pragma unroll
  for (int q = 0; q < KB + 2; ++q) acc[q] = 0.0;
  FOR_ACTIVE(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    const int c = e < L.C ? 0 : (e < 2 * L.C ? 1 : 2);
    auto u = [&](int64_t q) { return w[q] / nrm; };
    const double ue = u(e);
    const double ku = stencil_row(c, e, L, dg, of, u);
    U[e] = ue;
    KU[e] = ku;
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < kp) acc[j] = add(acc[j], mul(__ldcg(ptr[j] + e), ku));
    acc[KB] = add(acc[KB], mul(ue, ku));
  }
  acc[kp] = acc[KB];
  last_block_reduce(acc, kp + 1, partials, counter, f->d + 0, post);
}

// POD basis for podk <= KMAX as one flat 16-byte pass (snapshots are 0
// off the partition, so B is too): B_j = (sum_l X_{order[l]} W[l][j]) /
// sigma_j in the order of k_pod_basis (l ascending from l = 0)
constexpr int kBasisFlatMax = 8;

template <int K>
__device__ __forceinline__ void basis_body(int64_t npair, int m, const double2 *const *xp, double2 *const *bp,
                                           const double *Wt, const double *sg) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npair; p += stride) {
    double tx[K], ty[K];
    {
      const double2 x0 = __ldcg(xp[0] + p);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        tx[j] = mul(x0.x, Wt[j]);
        ty[j] = mul(x0.y, Wt[j]);
      }
    }
#pragma unroll 6
    for (int l = 1; l < m; ++l) {
      const double2 xv = __ldcg(xp[l] + p);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        tx[j] = add(tx[j], mul(xv.x, Wt[l * kBasisFlatMax + j]));
        ty[j] = add(ty[j], mul(xv.y, Wt[l * kBasisFlatMax + j]));
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) bp[j][p] = make_double2(tx[j] / sg[j], ty[j] / sg[j]);
  }
}

// POD basis for podk <= 8 as one flat 16-byte pass (snapshots are 0 off the
// partition, so B is too): B_j = (sum_l X_{order[l]} W[l][j]) / sigma_j in
// the order of k_pod_basis (l ascending from l = 0); the body is instantiated
// for the exact k (the FP64 work per loaded value is k multiply-adds)
__global__ void __launch_bounds__(kBlock) k_pod_basis_flat(int64_t npair, FamDev *f, double *const *Xtab,
                                                           double *const *Btab) {
  __shared__ const double2 *xp[MAXS];
  __shared__ double2 *bp[kBasisFlatMax];
  __shared__ double Wt[MAXS * kBasisFlatMax];
  __shared__ double sg[kBasisFlatMax];
  const int m = f->k, kk = f->podk;
  if (kk == 0 || kk > kBasisFlatMax) return;
  if (threadIdx.x < m) xp[threadIdx.x] = reinterpret_cast<const double2 *>(Xtab[f->order[threadIdx.x]]);
  if (threadIdx.x < kk) {
    bp[threadIdx.x] = reinterpret_cast<double2 *>(Btab[threadIdx.x]);
    sg[threadIdx.x] = f->pod_sigma[threadIdx.x];
  }
  for (int q = threadIdx.x; q < MAXS * kBasisFlatMax; q += blockDim.x) {
    const int l = q / kBasisFlatMax, j = q % kBasisFlatMax;
    Wt[q] = f->W[l * MAXS + j];
  }
  __syncthreads();
  switch (kk) {
    case 1: basis_body<1>(npair, m, xp, bp, Wt, sg); break;
    case 2: basis_body<2>(npair, m, xp, bp, Wt, sg); break;
    case 3: basis_body<3>(npair, m, xp, bp, Wt, sg); break;
    case 4: basis_body<4>(npair, m, xp, bp, Wt, sg); break;
    case 5: basis_body<5>(npair, m, xp, bp, Wt, sg); break;
    case 6: basis_body<6>(npair, m, xp, bp, Wt, sg); break;
    case 7: basis_body<7>(npair, m, xp, bp, Wt, sg); break;
    default: basis_body<8>(npair, m, xp, bp, Wt, sg); break;
  }
}

// POD Galerkin for podk <= 5 in one flat pass over B, K B and the rhs (all 0
// off the partition): gs[j*k + i] = B_i . KB_j, gs[k*k + i] = B_i . rhs,
// scattered into Gk / d by the last block (POST_GAL_SCATTER)
template <int K>
__device__ __forceinline__ void gal_body(int64_t npair, double *const *Btab, double *const *KBtab,
                                         const double *rhs, double *acc) {
  const double2 *B[K], *KB[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    B[i] = reinterpret_cast<const double2 *>(Btab[i]);
    KB[i] = reinterpret_cast<const double2 *>(KBtab[i]);
  }
  const double2 *R = reinterpret_cast<const double2 *>(rhs);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npair; p += stride) {
    double2 b[K], kb[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      b[i] = __ldcg(B[i] + p);
      kb[i] = __ldcg(KB[i] + p);
    }
    const double2 r = __ldcg(R + p);
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int i = 0; i < K; ++i) {
        acc[j * K + i] = add(acc[j * K + i], mul(b[i].x, kb[j].x));
        acc[j * K + i] = add(acc[j * K + i], mul(b[i].y, kb[j].y));
      }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      acc[K * K + i] = add(acc[K * K + i], mul(b[i].x, r.x));
      acc[K * K + i] = add(acc[K * K + i], mul(b[i].y, r.y));
    }
  }
}

constexpr int kGalFusedMax = 5;  // k*k + k <= RQ

__global__ void __launch_bounds__(kBlock) k_pod_galerkin_fused(int64_t npair, FamDev *f, double *const *Btab,
                                                               double *const *KBtab, const double *__restrict__ rhs,
                                                               double *partials, unsigned int *counter) {
  const int kk = f->podk;
  if (kk == 0 || kk > kGalFusedMax) return;
  double acc[kGalFusedMax * kGalFusedMax + kGalFusedMax];
#pragma unroll
  for (int q = 0; q < kGalFusedMax * kGalFusedMax + kGalFusedMax; ++q) acc[q] = 0.0;
  switch (kk) {
    case 1: gal_body<1>(npair, Btab, KBtab, rhs, acc); break;
    case 2: gal_body<2>(npair, Btab, KBtab, rhs, acc); break;
    case 3: gal_body<3>(npair, Btab, KBtab, rhs, acc); break;
    case 4: gal_body<4>(npair, Btab, KBtab, rhs, acc); break;
    default: gal_body<5>(npair, Btab, KBtab, rhs, acc); break;
  }
  Post post;
  post.kind = POST_GAL_SCATTER;
  post.f = f;
  last_block_reduce(acc, kk * kk + kk, partials, counter, f->gs, post);
}

// POD push as one flat 16-byte pass: the snapshot copy and its Gram row
template <int KB>
__global__ void __launch_bounds__(kBlock) k_pod_push_flat(int64_t npair, FamDev *f, double *const *Xtab, int n_pod,
                                                          const double *__restrict__ y, double *partials,
                                                          unsigned int *counter, Post post) {
  __shared__ const double2 *ptr[MAXS];
  const int m = f->k;
  const int slot = (m < n_pod) ? m : f->order[0];
  const int first = (m < n_pod) ? 0 : 1;
  const int nother = m - first;
  if (threadIdx.x < nother) ptr[threadIdx.x] = reinterpret_cast<const double2 *>(Xtab[f->order[first + threadIdx.x]]);
  __syncthreads();
  double2 *X = reinterpret_cast<double2 *>(Xtab[slot]);
  const double2 *Y = reinterpret_cast<const double2 *>(y);
  double acc[KB + 2];
#pragma unroll
  for (int q = 0; q < KB + 2; ++q) acc[q] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npair; p += stride) {
    const double2 yv = __ldcg(Y + p);
    double2 u[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < nother) u[j] = __ldcg(ptr[j] + p);
    X[p] = yv;
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < nother) {
        acc[j] = add(acc[j], mul(u[j].x, yv.x));
        acc[j] = add(acc[j], mul(u[j].y, yv.y));
      }
    acc[KB] = add(acc[KB], mul(yv.x, yv.x));
    acc[KB] = add(acc[KB], mul(yv.y, yv.y));
  }
  acc[nother] = acc[KB];
  last_block_reduce(acc, nother + 1, partials, counter, f->d, post);
}

// POD: B_j = (sum_l X_{order[l]} W[l][j]) / sigma_j  for j < podk
__global__ void __launch_bounds__(kBlock) k_pod_basis(Lay L, const uint32_t *__restrict__ mask, FamDev *f,
                                                      double *const *Xtab, double *const *Btab) {
  __shared__ const double *xp[MAXS];
  __shared__ double *bp[MAXS];
  __shared__ double Wt[MAXS * MAXS];
  __shared__ double sg[MAXS];
  const int m = f->k, kk = f->podk;
  if (kk <= kBasisFlatMax) return;  // k_pod_basis_flat did it (or nothing to do)
  if (threadIdx.x < m) xp[threadIdx.x] = Xtab[f->order[threadIdx.x]];
  if (threadIdx.x < kk) { bp[threadIdx.x] = Btab[threadIdx.x]; sg[threadIdx.x] = f->pod_sigma[threadIdx.x]; }
  for (int q = threadIdx.x; q < MAXS * MAXS; q += blockDim.x) Wt[q] = f->W[q];
  __syncthreads();
  FOR_ACTIVE(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    double x[MAXS];
    for (int l = 0; l < m; ++l) x[l] = xp[l][e];
    for (int j = 0; j < kk; ++j) {
      double t = mul(x[0], Wt[0 * MAXS + j]);
      for (int l = 1; l < m; ++l) t = add(t, mul(x[l], Wt[l * MAXS + j]));
      bp[j][e] = t / sg[j];
    }
  }
}

// POD: KB_j = K B_j for j < podk (blockIdx.y = j)
__global__ void __launch_bounds__(kBlock) k_spmv_multi(Lay L, const uint32_t *__restrict__ mask, double dg, double of,
                                                       const FamDev *f, double *const *Btab, double *const *KBtab) {
  const int j = blockIdx.y;
  if (j >= f->podk) return;
  const double *B = Btab[j];
  double *KB = KBtab[j];
  FOR_ACTIVE(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    const int c = e < L.C ? 0 : (e < 2 * L.C ? 1 : 2);
    KB[e] = stencil_row(c, e, L, dg, of, [&](int64_t q) { return B[q]; });
  }
}

// POD Galerkin: blockIdx.y = j < podk -> Gk[i][j] = B_i . KB_j; j == podk -> d[i] = B_i . rhs
template <int KB>
__global__ void __launch_bounds__(kBlock) k_pod_galerkin(Lay L, const uint32_t *__restrict__ mask, FamDev *f,
                                                         double *const *Btab, double *const *KBtab,
                                                         const double *__restrict__ rhs, double *partials,
                                                         unsigned int *counters) {
  const int j = blockIdx.y;
  const int kk = f->podk;
  if (j > kk || kk <= kGalFusedMax) return;  // k_pod_galerkin_fused did it
  __shared__ const double *bp[MAXS];
  if (threadIdx.x < kk) bp[threadIdx.x] = Btab[threadIdx.x];
  __syncthreads();
  const double *v = (j < kk) ? KBtab[j] : rhs;
  double acc[KB + 2];
#pragma unroll
  for (int q = 0; q < KB + 2; ++q) acc[q] = 0.0;
  FOR_ACTIVE(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    const double vv = __ldcg(v + e);
#pragma unroll
    for (int i = 0; i < KB; ++i)
      if (i < kk) acc[i] = add(acc[i], mul(__ldcg(bp[i] + e), vv));
  }
  double *out = (j < kk) ? (f->Gk + (int64_t)j * MAXS) : f->d;  // Gk stored column j contiguous
  last_block_reduce(acc, kk, partials + (int64_t)j * RQ * gridDim.x, counters + j, out);
}

// POD push: copy y into the ring slot and update the Gram row/column
template <int KB>
__global__ void __launch_bounds__(kBlock) k_pod_push(Lay L, const uint32_t *__restrict__ mask, FamDev *f,
                                                     double *const *Xtab, int n_pod, const double *__restrict__ y,
                                                     double *partials, unsigned int *counter, Post post) {
  __shared__ const double *ptr[MAXS];
  const int m = f->k;
  const int slot = (m < n_pod) ? m : f->order[0];
  // other snapshots staying in the ring (logical order), excluding the evicted one
  const int first = (m < n_pod) ? 0 : 1;
  const int nother = m - first;
  if (threadIdx.x < nother) ptr[threadIdx.x] = Xtab[f->order[first + threadIdx.x]];
  __syncthreads();
  double *X = Xtab[slot];
  double acc[KB + 2];
#pragma unroll
  for (int q = 0; q < KB + 2; ++q) acc[q] = 0.0;
  FOR_ACTIVE(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    const double yv = __ldcg(y + e);
    X[e] = yv;
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < nother) acc[j] = add(acc[j], mul(__ldcg(ptr[j] + e), yv));
    acc[KB] = add(acc[KB], mul(yv, yv));
  }
  acc[nother] = acc[KB];
  last_block_reduce(acc, nother + 1, partials, counter, f->d, post);
}

// ---------------------------------------------------------------------------
// small dense kernels (one CTA)
// ---------------------------------------------------------------------------
// Cholesky with the reference's pivot rule (startvec.py:59-74); returns the
// failing column or -1.  a: n x n row-major with leading dimension MAXS.
__device__ int chol_small(const double *a, double *low, int n) {
  for (int q = 0; q < n * MAXS; ++q) low[q] = 0.0;
  for (int j = 0; j < n; ++j) {
    double dot = 0.0;
    for (int l = 0; l < j; ++l) dot = (l == 0) ? mul(low[j * MAXS], low[j * MAXS]) : add(dot, mul(low[j * MAXS + l], low[j * MAXS + l]));
    const double gjj = a[j * MAXS + j];
    const double s = sub(gjj, dot);
    if (!isfinite(s) || s <= 1e-12 * fabs(gjj) || s <= 0.0) return j;
    const double ljj = sqrt(s);
    low[j * MAXS + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double t = 0.0;
      for (int l = 0; l < j; ++l) t = (l == 0) ? mul(low[i * MAXS], low[j * MAXS]) : add(t, mul(low[i * MAXS + l], low[j * MAXS + l]));
      low[i * MAXS + j] = sub(a[i * MAXS + j], t) / ljj;
    }
  }
  return -1;
}

// L L^T c = rhs (startvec.py:77-79)
__device__ void chol_solve_small(const double *low, const double *rhs, double *c, int n) {
  double y[MAXS];
  for (int i = 0; i < n; ++i) {
    double t = rhs[i];
    for (int l = 0; l < i; ++l) t = sub(t, mul(low[i * MAXS + l], y[l]));
    y[i] = t / low[i * MAXS + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double t = y[i];
    for (int l = i + 1; l < n; ++l) t = sub(t, mul(low[l * MAXS + i], c[l]));
    c[i] = t / low[i * MAXS + i];
  }
}

__device__ void drop_logical(FamDev *f, int j, double *beta) {
  const int k = f->k;
  for (int a = j; a + 1 < k; ++a) {
    f->order[a] = f->order[a + 1];
    if (beta) beta[a] = beta[a + 1];
  }
  for (int r = 0, rr = 0; r < k; ++r) {
    if (r == j) continue;
    for (int c = 0, cc = 0; c < k; ++c) {
      if (c == j) continue;
      f->G[rr * MAXS + cc] = f->G[r * MAXS + c];
      ++cc;
    }
    ++rr;
  }
  f->k = k - 1;
}

// CSPE project (startvec.py:207-225): f->d holds beta = U^T rhs
__device__ void cspe_project_small(FamDev *f) {
  __shared__ double low[MAXS * MAXS];
  double beta[MAXS];
  for (int j = 0; j < f->k; ++j) beta[j] = f->d[j];
  while (f->k > 0) {
    const int bad = chol_small(f->G, low, f->k);
    if (bad >= 0) {
      drop_logical(f, bad, beta);
      f->dropped += 1;
      continue;
    }
    chol_solve_small(low, beta, f->coef, f->k);
    break;
  }
  f->x0_mode = f->k > 0 ? 1 : 0;
}

// CSPE observe, after ||v||: reject zero / non-finite (startvec.py:166-170)
__device__ void cspe_gate(FamDev *f) {
  const double nv = sqrt(f->d[f->k]);
  f->nv2 = nv;
  if (nv == 0.0 || !isfinite(nv)) {
    f->accept = 0;
    f->dropped += 1;
  } else {
    f->accept = 1;
    for (int j = 0; j < f->k; ++j) f->coef[j] = f->d[j];
  }
}

// CGS pass 2 uses the coefficients of pass 1's dot products
__device__ void cspe_gate_c2(FamDev *f) {
  if (!f->accept) return;
  for (int j = 0; j < f->k; ++j) f->coef[j] = f->d[j];
}

// after the second CGS pass: drop test, FIFO eviction, slot choice (startvec.py:175-186)
__device__ void cspe_decide(FamDev *f, const double *nw2, int max_cols, double drop_tol) {
  if (!f->accept) return;
  const double nw = sqrt(*nw2);
  if (nw < drop_tol * f->nv2) {
    f->accept = 0;
    f->dropped += 1;
    return;
  }
  f->nrm = nw;
  if (f->k == max_cols) {
    const int slot = f->order[0];
    drop_logical(f, 0, nullptr);
    f->evictions += 1;
    f->new_slot = slot;
  } else {
    // first slot not referenced by the logical order
    for (int s = 0; s < MAXS; ++s) {
      bool used = false;
      for (int j = 0; j < f->k; ++j) used |= (f->order[j] == s);
      if (!used) { f->new_slot = s; break; }
    }
  }
  f->kprime = f->k;
}

// bordered Galerkin update (startvec.py:187-199); f->d = [cross..., diag]
__device__ void cspe_commit(FamDev *f) {
  if (!f->accept) return;
  const int k = f->kprime;
  for (int j = 0; j < k; ++j) {
    f->G[k * MAXS + j] = f->d[j];
    f->G[j * MAXS + k] = f->d[j];
  }
  f->G[k * MAXS + k] = f->d[k];
  f->order[k] = f->new_slot;
  f->k = k + 1;
  f->products += 1;
  f->accepted += 1;
}

// POD push bookkeeping: Gram row/column from f->d (logical order of the
// remaining snapshots, then the new one)
__device__ void pod_push_commit(FamDev *f, int n_pod) {
  const int m = f->k;
  int slot;
  if (m < n_pod) {
    slot = m;
    f->order[m] = slot;
    f->k = m + 1;
  } else {
    slot = f->order[0];
    for (int a = 0; a + 1 < m; ++a) f->order[a] = f->order[a + 1];
    f->order[m - 1] = slot;
  }
  const int nother = f->k - 1;
  for (int j = 0; j < nother; ++j) {
    const int sj = f->order[j];
    f->G[slot * MAXS + sj] = f->d[j];
    f->G[sj * MAXS + slot] = f->d[j];
  }
  f->G[slot * MAXS + slot] = f->d[nother];
}

// one-pass Galerkin sums -> Gk (column j contiguous) and d
__device__ void gal_scatter(FamDev *f) {
  const int k = f->podk;
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) f->Gk[j * MAXS + i] = f->gs[j * k + i];
  for (int i = 0; i < k; ++i) f->d[i] = f->gs[k * k + i];
}

__device__ void run_post(const Post &p) {
  switch (p.kind) {
    case POST_GAL_SCATTER: gal_scatter(p.f); break;
    case POST_PROJECT: cspe_project_small(p.f); break;
    case POST_GATE: cspe_gate(p.f); break;
    case POST_GATE_C2: cspe_gate_c2(p.f); break;
    case POST_DECIDE: cspe_decide(p.f, p.f->d, p.max_cols, p.drop_tol); break;
    case POST_COMMIT: cspe_commit(p.f); break;
    case POST_POD_PUSH: pod_push_commit(p.f, p.n_pod); break;
    default: break;
  }
}

// POD: eigen-decomposition of the logical Gram matrix by parallel cyclic
// Jacobi (replaces LAPACK syevd, startvec.py:285-294), truncation, basis
// combination W = V_k (divided by sigma in k_pod_basis).
#ifndef MQ_EIG_ABS
#define MQ_EIG_ABS 1e-16
#endif
__global__ void __launch_bounds__(256) k_pod_eig(FamDev *f, double eps_pod) {
  // rows padded to an odd number of doubles: the column updates walk a
  // column with consecutive threads, which a 32-double row stride would put
  // in one shared-memory bank
  constexpr int LDA = MAXS + 1;
  __shared__ double A[MAXS * LDA];
  __shared__ double V[MAXS * LDA];
  __shared__ double cs[MAXS / 2], sn[MAXS / 2];
  __shared__ int pp[MAXS / 2], qq[MAXS / 2];
  __shared__ int perm[MAXS];
  __shared__ double lam[MAXS], sig[MAXS];
  __shared__ int s_k;
  __shared__ int s_done;
  const int m = f->k;
  if (m == 0) {
    if (threadIdx.x == 0) { f->podk = 0; f->x0_mode = 0; }
    return;
  }
  const int mm = m + (m & 1);  // even size for the round-robin tournament
  for (int q = threadIdx.x; q < mm * mm; q += blockDim.x) {
    const int r = q / mm, c = q % mm;
    double v = 0.0;
    if (r < m && c < m) v = f->G[f->order[r] * MAXS + f->order[c]];
    A[r * LDA + c] = v;
    V[r * LDA + c] = (r == c) ? 1.0 : 0.0;
  }
  __shared__ double s_tr;
  __shared__ int s_rot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int r = 0; r < m; ++r) tr += fabs(A[r * LDA + r]);
    s_tr = tr;
  }
  __syncthreads();
  const int npair = mm / 2;
  // cyclic sweeps until a sweep rotates nothing: a pair is skipped when its
  // coupling is negligible relative to its diagonal entries (1e-15) or to
  // the trace (1e-18) -- the Gram matrices of nearly dependent snapshots
  // carry noise-level eigenvalues whose couplings never fall below a
  // relative threshold
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < mm - 1; ++round) {
      if (threadIdx.x < npair) {
        // round-robin pairing: player mm-1 fixed, others rotate
        const int t = threadIdx.x;
        int a = (t == 0) ? mm - 1 : (round + t) % (mm - 1);
        int b = (round + mm - 1 - t) % (mm - 1);
        if (t == 0) b = round % (mm - 1);
        const int p = a < b ? a : b, q = a < b ? b : a;
        pp[t] = p;
        qq[t] = q;
        const double apq = A[p * LDA + q];
        double c = 1.0, s = 0.0;
        const double app = A[p * LDA + p], aqq = A[q * LDA + q];
        if (apq != 0.0 && fabs(apq) > 1e-15 * sqrt(fabs(app * aqq)) && fabs(apq) > MQ_EIG_ABS * s_tr) {
          atomicAdd(&s_rot, 1);
          const double th = (A[q * LDA + q] - A[p * LDA + p]) / (2.0 * apq);
          const double tt = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
          c = 1.0 / sqrt(tt * tt + 1.0);
          s = tt * c;
        }
        cs[t] = c;
        sn[t] = s;
      }
      __syncthreads();
      // rows: row_p' = c row_p - s row_q ; row_q' = s row_p + c row_q
      for (int it = threadIdx.x; it < npair * mm; it += blockDim.x) {
        const int t = it / mm, col = it % mm;
        const int p = pp[t], q = qq[t];
        const double c = cs[t], s = sn[t];
        const double ap = A[p * LDA + col], aq = A[q * LDA + col];
        A[p * LDA + col] = c * ap - s * aq;
        A[q * LDA + col] = s * ap + c * aq;
      }
      __syncthreads();
      // columns of A and V
      for (int it = threadIdx.x; it < npair * mm; it += blockDim.x) {
        const int t = it / mm, row = it % mm;
        const int p = pp[t], q = qq[t];
        const double c = cs[t], s = sn[t];
        const double ap = A[row * LDA + p], aq = A[row * LDA + q];
        A[row * LDA + p] = c * ap - s * aq;
        A[row * LDA + q] = s * ap + c * aq;
        const double vp = V[row * LDA + p], vq = V[row * LDA + q];
        V[row * LDA + p] = c * vp - s * vq;
        V[row * LDA + q] = s * vp + c * vq;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) s_done = s_rot == 0;
    __syncthreads();
    if (s_done) break;
  }
  if (threadIdx.x == 0) {
    // sort descending (startvec.py:287-289), sigma = sqrt(clip(lambda, 0));
    // shared-memory work only: the family state is written after the barrier
    for (int i = 0; i < m; ++i) { perm[i] = i; lam[i] = A[i * LDA + i]; }
    for (int i = 0; i < m; ++i)
      for (int j = i + 1; j < m; ++j)
        if (lam[perm[j]] > lam[perm[i]]) { int t = perm[i]; perm[i] = perm[j]; perm[j] = t; }
    double total = 0.0;
    for (int i = 0; i < m; ++i) {
      const double l = lam[perm[i]];
      sig[i] = sqrt(l > 0.0 ? l : 0.0);
      total += sig[i];
    }
    int k = 0;
    if (sig[0] != 0.0)
      for (int i = 0; i < m; ++i) k += (sig[i] / sig[0] > eps_pod) ? 1 : 0;
    s_k = k;
    f->nrm = total;
    f->podk = k;
    f->x0_mode = 0;
  }
  __syncthreads();
  const int k = s_k;
  for (int i = threadIdx.x; i < m; i += blockDim.x) f->pod_sigma[i] = sig[i];
  for (int q = threadIdx.x; q < m * k; q += blockDim.x) {
    const int l = q / k, j = q % k;
    f->W[l * MAXS + j] = V[l * LDA + perm[j]];
  }
}

// POD Galerkin solve with the k-decrement retry (startvec.py:298-309)
__global__ void k_pod_solve(FamDev *f, RunDev *run) {
  if (threadIdx.x != 0) return;
  __shared__ double low[MAXS * MAXS];
  __shared__ double g[MAXS * MAXS];
  int k = f->podk;
  const int applications = k;
  if (f->k == 0) return;  // empty buffer: zero start vector, no bookkeeping
  if (f->pod_sigma[0] == 0.0) {
    f->podk = 0;
    f->pod_info = 0.0;
    run->pod_last_k = 0;
    run->pod_last_info = 0.0;
    f->x0_mode = 0;
    return;
  }
  // Gk column j contiguous: Gk[j*MAXS + i] = B_i . KB_j = g[i][j]
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      const double gij = f->Gk[j * MAXS + i], gji = f->Gk[i * MAXS + j];
      g[i * MAXS + j] = mul(0.5, add(gij, gji));
    }
  while (k > 0) {
    if (chol_small(g, low, k) >= 0) { --k; continue; }
    chol_solve_small(low, f->d, f->coef, k);
    break;
  }
  f->pod_applies += applications;
  f->podk = k;
  double kept = 0.0;
  for (int i = 0; i < k; ++i) kept += f->pod_sigma[i];
  const double info = k > 0 ? kept / f->nrm : 0.0;
  f->pod_info = info;
  run->pod_last_k = k;
  run->pod_last_info = info;
  if (k > 0) {
    run->any_pod = 1;
    if (info < run->min_pod_info) run->min_pod_info = info;
  }
  f->x0_mode = k > 0 ? 1 : 0;
}

__global__ void k_prev_start(FamDev *f) {
  if (threadIdx.x == 0) f->x0_mode = f->has_last ? 1 : 0;
}

__global__ void k_set_mode(FamDev *f, int mode) {
  if (threadIdx.x == 0) f->x0_mode = mode;
}

__global__ void k_prev_mark(FamDev *f) {
  if (threadIdx.x == 0) f->has_last = 1;
}

// copy active entries (x0 from a stored vector) when the mode says so
__global__ void __launch_bounds__(kBlock) k_copy_if(Lay L, const uint32_t *__restrict__ mask, const FamDev *f,
                                                    const double *__restrict__ src, double *__restrict__ dst) {
  if (f->x0_mode != 1) return;
  FOR_ACTIVE(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    dst[e] = src[e];
  }
}

__global__ void __launch_bounds__(kBlock) k_copy(Lay L, const uint32_t *__restrict__ mask,
                                                 const double *__restrict__ src, double *__restrict__ dst) {
  FOR_ACTIVE(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    dst[e] = src[e];
  }
}

// record one solve (schur.py:255-263)
__global__ void k_post_solve(const PcgOut *o, RunDev *run, FamDev *fams, int fam, int32_t *log, long long log_cap,
                             const StepParams *par) {
  if (threadIdx.x != 0) return;
  const PcgOut r = *o;
  if (r.status == 99) return;  // skipped after an earlier failure
  if (r.status != MQ_OK && run->err == 0) {
    run->err = r.status == MQ_NOT_CONVERGED ? MQ_NOT_CONVERGED : r.status;
    run->err_family = fam;
    run->err_step = par ? par->step : -1;
  }
  const long long i = run->solve_idx;
  if (log && i < log_cap) log[i] = r.iterations;
  run->solve_idx = i + 1;
  run->pcg_applies += r.applies;
}

// ---- per-step diagnostics log ---------------------------------------------
// Row m (0-based step of the run) of the log, kDiagW doubles:
//   [0..2] CSPE basis size of each family after that step's inserts
//   [3,4]  POD (last_k, last_info) sampled after the Euler step's solves
//   [5,6]  POD (last_k, last_info) sampled after the recovery's solves
// The host reduces them as the reference's _WindowStats and emit_row do.
constexpr int kDiagW = 8;

// row = par->step - shift (a deferred insert runs one step late)
__global__ void k_dlog_k(const FamDev *f, int fam, const StepParams *par, double *log, long long cap, int shift) {
  if (threadIdx.x != 0 || !log) return;
  const long long m = par->step - shift;
  if (m >= 0 && m < cap) log[m * kDiagW + fam] = (double)f->k;
}

__global__ void k_dlog_pod(const RunDev *run, const StepParams *par, double *log, long long cap, int col) {
  if (threadIdx.x != 0 || !log) return;
  const long long m = par->step - 1;
  if (m >= 0 && m < cap) {
    log[m * kDiagW + col] = (double)run->pod_last_k;
    log[m * kDiagW + col + 1] = run->pod_last_info;
  }
}

// ---- conducting block ---------------------------------------------------
struct CondArgs {
  int64_t n_c, n_cells, n_rows_t;
  const int64_t *kcn_ptr; const int32_t *kcn_col; const int8_t *kcn_sgn;
  const int32_t *kcnt_row; const int64_t *kcnt_ptr; const int32_t *kcnt_src; const int8_t *kcnt_sgn;
  const int32_t *f_edge; const int8_t *f_sgn; const double *f_base; const int32_t *f_cell;
  const int32_t *cell_face; const int32_t *e_face; const int8_t *e_sgn;
  const double *minv;
  double of, h, two_h4, k1, k2, k3;
  int linear;
};

__device__ __forceinline__ double face_flux(const CondArgs &a, int64_t f, const double *x) {
  // c_cond row: cond edges in ascending compact order, csr sum from 0
  double s = 0.0;
  if (f < 0) return s;  // boundary face of a conductor cell: all edges PEC
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int32_t e = a.f_edge[4 * f + q];
    if (e >= 0) s = add(s, mul((double)a.f_sgn[4 * f + q], x[e]));
  }
  return s;
}

// squared flux density of conductor cell c (model.py:399-407): all edges of
// its faces are conducting, so the state alone determines it
__device__ __forceinline__ double cell_b2(const CondArgs &a, int64_t c, const double *state) {
  double f[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) f[q] = face_flux(a, a.cell_face[6 * c + q], state);
  return add(add(add(mul(f[0], f[0]), mul(f[1], f[1])), add(mul(f[2], f[2]), mul(f[3], f[3]))),
             add(mul(f[4], f[4]), mul(f[5], f[5]))) / a.two_h4;
}

// nu per conductor cell from the state (model.py:496-500, 107-125)
__global__ void k_cell_nu(CondArgs a, const double *__restrict__ state, double *__restrict__ nu) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < a.n_cells; c += (int64_t)gridDim.x * blockDim.x) {
    const double b2 = cell_b2(a, c, state);
    nu[c] = a.linear ? a.k3 : add(mul(a.k1, exp(mul(a.k2, b2))), a.k3);
  }
}

// numpy's pairwise summation of a float64 array (the add.reduce inner loop
// behind ndarray.mean): blocks of <= 128 summed with 8 accumulators, larger
// arrays split at an 8-aligned half.  The split tree depends only on n, so
// the host builds it once (probe_plan): leaves are summed in parallel, then
// one thread combines them in the tree's postfix order.
// (values written by other blocks: L2 loads)
__device__ double np_leaf_sum_cg(const double *v, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = add(r, __ldcg(v + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = __ldcg(v + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = add(r[j], __ldcg(v + i + j));
  double res = add(add(add(r[0], r[1]), add(r[2], r[3])), add(add(r[4], r[5]), add(r[6], r[7])));
  for (; i < n; ++i) res = add(res, __ldcg(v + i));
  return res;
}

// B_probe = mean(sqrt(b2[cells])) (model.py:415-425).  Every block computes
// |B| of a strided share of the cells; the last block to finish (ticket)
// sums the leaves in parallel and runs the tree.  plan = [n_leaves, n_prog,
// (start, len) per leaf, postfix program (leaf index or -1 = add)].  The value
// goes to log[par->step - 1] inside a run, else to *out.
__global__ void k_probe(CondArgs a, const int32_t *__restrict__ cells, int64_t n, const int32_t *__restrict__ plan,
                        const double *__restrict__ state, double *__restrict__ vals, double *__restrict__ leaf,
                        unsigned int *ctr, const StepParams *par, double *log, double *out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    vals[q] = sqrt(cell_b2(a, cells[q], state));
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(ctr, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int nl = plan[0], np = plan[1];
  for (int t = threadIdx.x; t < nl; t += blockDim.x) leaf[t] = np_leaf_sum_cg(vals + plan[2 + 2 * t], plan[3 + 2 * t]);
  __syncthreads();
  if (threadIdx.x != 0) return;
  *ctr = 0u;
  double st[64];
  int sp = 0;
  for (int i = 0; i < np; ++i) {
    const int op = plan[2 + 2 * nl + i];
    if (op >= 0) {
      st[sp++] = leaf[op];
    } else {
      const double rb = st[--sp];
      const double ra = st[--sp];
      st[sp++] = add(ra, rb);
    }
  }
  const double v = add(0.0, st[0]) / (double)n;
  if (log) log[par->step - 1] = v;
  else *out = v;
}

// y = K_c(state) x with nu precomputed (model.py:502-509)
__device__ __forceinline__ double kc_row(const CondArgs &a, int64_t e, const double *nu, const double *x) {
  double y = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int32_t f = a.e_face[4 * e + q];
    if (f < 0) continue;
    double fc = 0.0;  // face_by_cond @ nu (<= 2 terms)
    const int32_t c0 = a.f_cell[2 * f], c1 = a.f_cell[2 * f + 1];
    if (c0 >= 0) fc = add(fc, mul(0.5, nu[c0]));
    if (c1 >= 0) fc = add(fc, mul(0.5, nu[c1]));
    const double w = add(a.f_base[f], fc);
    const double v = mul(w / a.h, face_flux(a, f, x));
    y = add(y, mul((double)a.e_sgn[4 * e + q], v));
  }
  return y;
}

__global__ void k_kc_apply(CondArgs a, const double *__restrict__ nu, const double *__restrict__ x,
                           double *__restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.n_c; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = kc_row(a, e, nu, x);
}

// w_n = K_cn^T a_c into the (otherwise zero) padded vector (csc_matvec order)
__global__ void k_kcnt(CondArgs a, const double *__restrict__ ac, double *__restrict__ w) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.n_rows_t; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = a.kcnt_ptr[r]; q < a.kcnt_ptr[r + 1]; ++q) s = add(s, mul(a.kcnt_sgn[q] * a.of, ac[a.kcnt_src[q]]));
    w[a.kcnt_row[r]] = s;
  }
}

// y_c = K_cn x_n (csr order)
__global__ void k_kcn(CondArgs a, const double *__restrict__ xn, double *__restrict__ yc) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.n_c; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = a.kcn_ptr[e]; q < a.kcn_ptr[e + 1]; ++q) s = add(s, mul(a.kcn_sgn[q] * a.of, xn[a.kcn_col[q]]));
    yc[e] = s;
  }
}

// Euler update (schur.py:392-404):
//   rate = K_cn (y_cpl - y_src) - K_c(a_c) a_c ;  a_next = a_c + dt (minv rate)
__global__ void k_euler(CondArgs a, const double *__restrict__ nu, const double *__restrict__ ac,
                        const double *__restrict__ ycpl, const double *__restrict__ ysrc, double *__restrict__ anext,
                        const StepParams *par, RunDev *run) {
  if (run->err) return;
  const double dt = par->dt;
  bool bad = false;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.n_c; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = a.kcn_ptr[e]; q < a.kcn_ptr[e + 1]; ++q) {
      const int32_t col = a.kcn_col[q];
      s = add(s, mul(a.kcn_sgn[q] * a.of, sub(ycpl[col], ysrc[col])));
    }
    const double rate = sub(s, kc_row(a, e, nu, ac));
    const double v = add(ac[e], mul(dt, mul(a.minv[e], rate)));
    anext[e] = v;
    bad |= !isfinite(v);
  }
  if (bad) {
    if (atomicCAS(&run->err, 0u, (unsigned)MQ_NONFINITE) == 0u) {
      run->err_step = par->step;
      run->err_family = -1;
    }
  }
}

__global__ void k_copy_n(int64_t n, const double *__restrict__ src, double *__restrict__ dst, const RunDev *run) {
  if (run && run->err) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

// source rhs = pattern * waveform (schur.py:81-82): only the pattern support
__global__ void k_src_rhs(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ val,
                          const StepParams *par, int use_now, double *__restrict__ rhs) {
  const double s = use_now ? par->wave_now : par->wave_new;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    rhs[idx[q]] = mul(val[q], s);
}

__global__ void __launch_bounds__(kBlock) k_sub(Lay L, const uint32_t *__restrict__ mask, const double *__restrict__ a,
                                                const double *__restrict__ b, double *__restrict__ out) {
  FOR_ACTIVE(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    out[e] = sub(a[e], b[e]);
  }
}

__global__ void k_load_params(StepParams *par, const double *dt_tab, const double *wave_tab, RunDev *run) {
  if (threadIdx.x != 0) return;
  const long long m = run->step;
  par->dt = dt_tab[m];
  par->wave_new = wave_tab[m + 1];
  par->wave_now = wave_tab[m + 1];
  par->step = m + 1;
}

__global__ void k_step_done(RunDev *run, const StepParams *par, const double *ac, double *hist, int64_t n_c) {
  const long long m = par->step - 1;  // k_load_params set step = m + 1
  if (hist && !run->err)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_c; e += (int64_t)gridDim.x * blockDim.x)
      hist[m * n_c + e] = ac[e];
  if (blockIdx.x == 0 && threadIdx.x == 0) run->step = m + 1;
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static CondArgs cond_args(mq_ctx *ctx) {
  CondArgs a;
  const Topology &t = ctx->topo;
  a.n_c = (int64_t)t.c_pad.size();
  a.n_cells = t.n_cells_c;
  a.n_rows_t = (int64_t)t.kcnt_row.size();
  a.kcn_ptr = ctx->d_kcn_ptr; a.kcn_col = ctx->d_kcn_col; a.kcn_sgn = ctx->d_kcn_sgn;
  a.kcnt_row = ctx->d_kcnt_row; a.kcnt_ptr = ctx->d_kcnt_ptr; a.kcnt_src = ctx->d_kcnt_src; a.kcnt_sgn = ctx->d_kcnt_sgn;
  a.f_edge = ctx->d_f_edge; a.f_sgn = ctx->d_f_sgn; a.f_base = ctx->d_f_base; a.f_cell = ctx->d_f_cell;
  a.cell_face = ctx->d_cell_face; a.e_face = ctx->d_e_face; a.e_sgn = ctx->d_e_sgn;
  a.minv = ctx->d_minv;
  a.of = ctx->kn_off;
  a.h = ctx->desc.h;
  a.two_h4 = ctx->two_h4;
  a.k1 = ctx->desc.brauer_k1; a.k2 = ctx->desc.brauer_k2; a.k3 = ctx->desc.brauer_k3;
  a.linear = ctx->desc.brauer_k1 == 0.0;
  return a;
}

template <class T>
static int up(mq_ctx *ctx, T **dst, const std::vector<T> &src) {
  if (src.empty()) { *dst = nullptr; return MQ_OK; }
  int rc = ctx_alloc(ctx, (void **)dst, src.size() * sizeof(T));
  if (rc) return rc;
  MQ_CUDA(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return MQ_OK;
}

int conducting_init(mq_ctx *ctx) {
  const Topology &t = ctx->topo;
  int rc = 0;
  rc = rc ? rc : up(ctx, &ctx->d_kcn_ptr, t.kcn_ptr);
  rc = rc ? rc : up(ctx, &ctx->d_kcn_col, t.kcn_col);
  rc = rc ? rc : up(ctx, &ctx->d_kcn_sgn, t.kcn_sgn);
  rc = rc ? rc : up(ctx, &ctx->d_kcnt_row, t.kcnt_row);
  rc = rc ? rc : up(ctx, &ctx->d_kcnt_ptr, t.kcnt_ptr);
  rc = rc ? rc : up(ctx, &ctx->d_kcnt_src, t.kcnt_src);
  rc = rc ? rc : up(ctx, &ctx->d_kcnt_sgn, t.kcnt_sgn);
  std::vector<double> minv(t.mc_diag.size());
  for (size_t q = 0; q < minv.size(); ++q) minv[q] = 1.0 / t.mc_diag[q];  // schur.py:212
  rc = rc ? rc : up(ctx, &ctx->d_minv, minv);
  rc = rc ? rc : up(ctx, &ctx->d_f_edge, t.f_edge);
  rc = rc ? rc : up(ctx, &ctx->d_f_sgn, t.f_sgn);
  rc = rc ? rc : up(ctx, &ctx->d_f_base, t.f_base);
  rc = rc ? rc : up(ctx, &ctx->d_f_cell, t.f_cell);
  rc = rc ? rc : up(ctx, &ctx->d_cell_face, t.cell_face);
  rc = rc ? rc : up(ctx, &ctx->d_e_face, t.e_face);
  rc = rc ? rc : up(ctx, &ctx->d_e_sgn, t.e_sgn);
  const size_t nc = std::max<size_t>(1, t.c_pad.size());
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_cell_nu, sizeof(double) * std::max<int64_t>(1, t.n_cells_c));
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_ac, sizeof(double) * nc);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_ac_next, sizeof(double) * nc);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_ac_x, sizeof(double) * nc);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_yc, sizeof(double) * nc);
  ctx->two_h4 = 2.0 * std::pow(ctx->desc.h, 4.0);
  return rc;
}

static int grid_for(mq_ctx *ctx, int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > (int64_t)ctx->sms * 4) b = ctx->sms * 4;
  return (int)b;
}

static int stream_grid(mq_ctx *ctx) {
  int64_t b = (ctx->topo.L.words + kWarps - 1) / kWarps;
  if (b > (int64_t)ctx->sms * 4) b = ctx->sms * 4;
  return (int)std::max<int64_t>(1, b);
}

// dispatch a kernel template on the basis-size bound of the solver
#define KB_LAUNCH(kb, kern, grid, block, stream, ...)                       \
  do {                                                                    \
    if ((kb) <= 8) kern<8><<<(grid), (block), 0, (stream)>>>(__VA_ARGS__);  \
    else if ((kb) <= 16) kern<16><<<(grid), (block), 0, (stream)>>>(__VA_ARGS__); \
    else kern<32><<<(grid), (block), 0, (stream)>>>(__VA_ARGS__);          \
  } while (0)

#define LAUNCH_CHECK()                 \
  do {                                 \
    MQ_CUDA(cudaGetLastError());       \
    ctx->launches += 1;                \
  } while (0)

// ---- start vector -----------------------------------------------------
static int start_vector(mq_ctx *ctx, int fam, const double *rhs, double *x0) {
  SolverHost *s = ctx->solver;
  FamDev *f = s->d_fam + fam;
  const Lay &L = ctx->topo.L;
  cudaStream_t st = ctx->stream;
  const int G = s->red_grid;
  switch (s->cfg.strategy) {
    case MQ_STRAT_ZERO:
      k_set_mode<<<1, 32, 0, st>>>(f, 0);
      LAUNCH_CHECK();
      break;
    case MQ_STRAT_PREVIOUS:
      k_prev_start<<<1, 32, 0, st>>>(f);
      LAUNCH_CHECK();
      k_copy_if<<<stream_grid(ctx), kBlock, 0, st>>>(L, ctx->d_mask, f, s->last[fam], x0);
      LAUNCH_CHECK();
      break;
    case MQ_STRAT_CSPE: {
      // beta = U^T rhs; the last block then solves the projected system
      Post post;
      post.kind = POST_PROJECT;
      post.f = f;
      KB_LAUNCH(s->kb, k_mdot, G, kBlock, st, L.total / 2, s->d_U[fam], f->order, &f->k, rhs, 0, f->d, s->d_red,
                s->d_cnt, post, nullptr);
      LAUNCH_CHECK();
      KB_LAUNCH(s->kb, k_comb, G, kBlock, st, L.total / 2, s->d_U[fam], f->order, &f->k, f->coef, x0);
      LAUNCH_CHECK();
      break;
    }
    case MQ_STRAT_POD: {
      if (s->eig_ahead) {
        // the eigen-decomposition of this ring ran after the family's last
        // push (observe); an empty ring has podk = 0 from the reset
        if (s->eig_pend[fam]) {
          MQ_CUDA(cudaStreamWaitEvent(st, s->ev_ej[fam], 0));
          s->eig_pend[fam] = false;
        }
      } else {
        k_pod_eig<<<1, 256, 0, st>>>(f, s->cfg.eps_pod);
        LAUNCH_CHECK();
      }
      k_pod_basis_flat<<<G, kBlock, 0, st>>>(L.total / 2, f, s->d_X[fam], s->d_B);
      LAUNCH_CHECK();
      k_pod_basis<<<stream_grid(ctx), kBlock, 0, st>>>(L, ctx->d_mask, f, s->d_X[fam], s->d_B);
      LAUNCH_CHECK();
      if (s->kn_multi[fam]) {
        int rc2 = kn_multi_launch(s->kn_multi[fam], st);
        if (rc2) return rc2;
        ctx->launches += 1;
      } else {
        dim3 g2(stream_grid(ctx), s->cfg.n_pod);
        k_spmv_multi<<<g2, kBlock, 0, st>>>(L, ctx->d_mask, ctx->kn_diag, ctx->kn_off, f, s->d_B, s->d_KB);
        LAUNCH_CHECK();
      }
      dim3 g3(G, s->cfg.n_pod + 1);
      k_pod_galerkin_fused<<<G, kBlock, 0, st>>>(L.total / 2, f, s->d_B, s->d_KB, rhs, s->d_red, s->d_cnt + 1);
      LAUNCH_CHECK();
      KB_LAUNCH(s->kb, k_pod_galerkin, g3, kBlock, st, L, ctx->d_mask, f, s->d_B, s->d_KB, rhs, s->d_red,
                s->d_cnt + 1);
      LAUNCH_CHECK();
      k_pod_solve<<<1, 32, 0, st>>>(f, s->d_run);
      LAUNCH_CHECK();
      // small-k and large-k instances, exactly one runs (podk is on the device)
      k_comb_range<4><<<G, kBlock, 0, st>>>(L.total / 2, s->d_B, s->d_iota, &f->podk, f->coef, x0, -1);
      LAUNCH_CHECK();
      KB_LAUNCH(s->kb, k_comb_range, G, kBlock, st, L.total / 2, s->d_B, s->d_iota, &f->podk, f->coef, x0, 4);
      LAUNCH_CHECK();
      break;
    }
  }
  return MQ_OK;
}

// ---- observe ------------------------------------------------------------
// deferred CSPE insert (the recovery's coupling family, see enqueue_step)
__global__ void k_obs_gate(FamDev *f) {
  if (threadIdx.x != 0) return;
  if (f->pending) {
    f->pending = 0;
    f->skip = 0;
  } else {
    f->skip = 1;
    f->accept = 0;  // the chain's later kernels test accept
  }
}

__global__ void k_set_pending(FamDev *f) {
  if (threadIdx.x == 0) f->pending = 1;
}

// where a family's cache update runs: stream, reduction scratch, CGS vectors
struct ObsRes {
  cudaStream_t st;
  double *red;
  unsigned int *cnt;
  double *w1, *w2;
  int grid;
};

static ObsRes main_res(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  return ObsRes{ctx->stream, s->d_red, s->d_cnt, s->w1, s->w2, s->red_grid};
}

// gated: the insert runs only if the family has a deferred one pending
// (k_obs_gate); CSPE only
static int observe(mq_ctx *ctx, int fam, const double *y, const ObsRes &o, bool gated = false, int dlog_shift = 1) {
  SolverHost *s = ctx->solver;
  FamDev *f = s->d_fam + fam;
  const Lay &L = ctx->topo.L;
  cudaStream_t st = o.st;
  const int G = o.grid;
  switch (s->cfg.strategy) {
    case MQ_STRAT_ZERO:
      break;
    case MQ_STRAT_PREVIOUS:
      k_copy<<<G, kBlock, 0, st>>>(L, ctx->d_mask, y, s->last[fam]);
      LAUNCH_CHECK();
      k_prev_mark<<<1, 32, 0, st>>>(f);
      LAUNCH_CHECK();
      break;
    case MQ_STRAT_CSPE: {
      if (gated) {
        k_obs_gate<<<1, 32, 0, st>>>(f);
        LAUNCH_CHECK();
      }
      Post post;
      post.f = f;
      post.max_cols = s->cfg.max_cols;
      post.drop_tol = s->cfg.drop_tol;
      // ||v|| and U^T v in one pass, then the zero / non-finite gate
      post.kind = POST_GATE;
      KB_LAUNCH(s->kb, k_mdot, G, kBlock, st, L.total / 2, s->d_U[fam], f->order, &f->k, y, 1, f->d, o.red,
                o.cnt, post, gated ? &f->skip : nullptr);
      LAUNCH_CHECK();
      // CGS pass 1: w1 = v - U c1, c2 = U^T w1
      post.kind = POST_GATE_C2;
      KB_LAUNCH(s->kb, k_axpy_dots, G, kBlock, st, L.total / 2, s->d_U[fam], f->order, &f->k, f->coef, y, o.w1, 1, f->d,
                                        o.red, o.cnt, &f->accept, post);
      LAUNCH_CHECK();
      // CGS pass 2: w2 = w1 - U c2, ||w2||^2, then drop test / eviction / slot
      post.kind = POST_DECIDE;
      KB_LAUNCH(s->kb, k_axpy_dots, G, kBlock, st, L.total / 2, s->d_U[fam], f->order, &f->k, f->coef, o.w1, o.w2, 0,
                                        f->d, o.red, o.cnt, &f->accept, post);
      LAUNCH_CHECK();
      // u, K u, cross products, diagonal, then the bordered Galerkin commit
      post.kind = POST_COMMIT;
      KB_LAUNCH(s->kb, k_cspe_product, G, kBlock, st, L, ctx->d_mask, ctx->kn_diag, ctx->kn_off, f, s->d_U[fam], s->d_KU[fam],
                                           o.w2, o.red, o.cnt, post);
      LAUNCH_CHECK();
      k_dlog_k<<<1, 32, 0, st>>>(f, fam, s->d_par, s->d_dlog, s->dlog_cap, dlog_shift);
      LAUNCH_CHECK();
      break;
    }
    case MQ_STRAT_POD: {
      Post post;
      post.kind = POST_POD_PUSH;
      post.f = f;
      post.n_pod = s->cfg.n_pod;
      KB_LAUNCH(s->kb, k_pod_push_flat, G, kBlock, st, L.total / 2, f, s->d_X[fam], s->cfg.n_pod, y, o.red, o.cnt,
                post);
      LAUNCH_CHECK();
      if (s->eig_ahead) {
        MQ_CUDA(cudaEventRecord(s->ev_ef[fam], st));
        MQ_CUDA(cudaStreamWaitEvent(s->eig_side, s->ev_ef[fam], 0));
        k_pod_eig<<<1, 256, 0, s->eig_side>>>(f, s->cfg.eps_pod);
        LAUNCH_CHECK();
        MQ_CUDA(cudaEventRecord(s->ev_ej[fam], s->eig_side));
        s->eig_pend[fam] = true;
      }
      break;
    }
  }
  return MQ_OK;
}

// ---- one solve_kn (schur.py:239-264), device only ------------------------
static int solve_enqueue(mq_ctx *ctx, int fam, const double *rhs, double *y, bool observe_now = true) {
  SolverHost *s = ctx->solver;
  FamDev *f = s->d_fam + fam;
  int rc = start_vector(ctx, fam, rhs, y);
  if (rc) return rc;
  StencilPcgArgs a{};
  a.L = ctx->topo.L;
  a.mask = ctx->d_mask;
  a.dg = ctx->kn_diag;
  a.of = ctx->kn_off;
  a.inv = ctx->jac_inv;
  a.use_jac = 1;
  a.x0_mode = 0;
  a.b = rhs;
  a.x = y;
  a.r = ctx->d_r;
  a.pa = ctx->d_p0;
  a.pb = ctx->d_p1;
  a.ap = ctx->d_ap;
  a.ap2 = ctx->d_ap2;
  a.r2 = ctx->d_r2;
  a.stress_ns = pcg_stress_ns();
  a.rel_tol = s->cfg.rel_tol;
  a.abs_tol = s->cfg.abs_tol;
  a.max_iter = s->cfg.max_iter;
  a.partials = ctx->d_partials;
  a.bar = ctx->d_bar;
  a.out = ctx->d_out;
  a.x0_mode_dev = &f->x0_mode;
  a.err_word = &s->d_run->err;
  const bool timed = ctx->pcg_timing && ctx->ev_n < kEvPool;
  if (timed) MQ_CUDA(cudaEventRecordWithFlags(ctx->ev_pool[2 * ctx->ev_n], ctx->stream, cudaEventRecordExternal));
  rc = launch_pcg_ctx(ctx, a);
  if (rc) return rc;
  if (timed) {
    MQ_CUDA(cudaEventRecordWithFlags(ctx->ev_pool[2 * ctx->ev_n + 1], ctx->stream, cudaEventRecordExternal));
    ctx->ev_n += 1;
  }
  ctx->launches += 1;
  k_post_solve<<<1, 32, 0, ctx->stream>>>(ctx->d_out, s->d_run, s->d_fam, fam, s->d_log, s->log_cap, s->d_par);
  LAUNCH_CHECK();
  return observe_now ? observe(ctx, fam, y, main_res(ctx)) : MQ_OK;
}

// the source family's cache update on the side stream (fork), joined back
// into the main stream by join_side()
static int fork_observe(mq_ctx *ctx, int slot, int fam, const double *y, bool gated = false, int dlog_shift = 1) {
  SolverHost *s = ctx->solver;
  MQ_CUDA(cudaEventRecord(s->ev_fork[slot], ctx->stream));
  MQ_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork[slot], 0));
  int rc = observe(ctx, fam, y, ObsRes{s->side, s->d_red2, s->d_cnt2, s->w1b, s->w2b, s->side_grid}, gated,
                   dlog_shift);
  if (rc) return rc;
  MQ_CUDA(cudaEventRecord(s->ev_join[slot], s->side));
  s->pend[slot] = true;
  return MQ_OK;
}

// main stream waits for the side stream up to fork `slot` (side work is in
// issue order, so this also covers earlier forks)
static int join_side(mq_ctx *ctx, int slot) {
  SolverHost *s = ctx->solver;
  if (!s->pend[slot]) return MQ_OK;
  MQ_CUDA(cudaStreamWaitEvent(ctx->stream, s->ev_join[slot], 0));
  s->pend[slot] = false;
  return MQ_OK;
}

static int join_eigs(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  for (int f = 0; f < 3; ++f)
    if (s->eig_pend[f]) {
      MQ_CUDA(cudaStreamWaitEvent(ctx->stream, s->ev_ej[f], 0));
      s->eig_pend[f] = false;
    }
  return MQ_OK;
}

static int join_all(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  for (int q = 0; q < SolverHost::kSlots; ++q) {
    int rc = join_side(ctx, q);
    if (rc) return rc;
  }
  return join_eigs(ctx);
}

static int euler_enqueue(mq_ctx *ctx, bool join_tail, bool defer_cpl = false);

// join_tail: leave no side work pending (standalone calls); the stepper
// passes false and lets the recovery absorb the coupling family's update
// defer_cpl: leave the coupling family's insert pending on the device for
// the next call's side stream (host-facing calls, CSPE)
static int euler_enqueue(mq_ctx *ctx, bool join_tail, bool defer_cpl) {
  SolverHost *s = ctx->solver;
  const Topology &t = ctx->topo;
  CondArgs a = cond_args(ctx);
  cudaStream_t st = ctx->stream;
  const int64_t n_c = (int64_t)t.c_pad.size();
  // SOURCE at t + dt
  k_src_rhs<<<grid_for(ctx, s->n_pat), 256, 0, st>>>(s->n_pat, s->d_pat_idx, s->d_pat_val, s->d_par, 0, s->rhs_src);
  LAUNCH_CHECK();
  int rc = solve_enqueue(ctx, MQ_FAM_SOURCE, s->rhs_src, s->y_src, !s->overlap);
  if (rc) return rc;
  if (s->overlap) {
    rc = fork_observe(ctx, 0, MQ_FAM_SOURCE, s->y_src);
    if (rc) return rc;
  }
  // COUPLING_FROM_PREVIOUS_STATE with w = K_cn^T a_c
  k_kcnt<<<grid_for(ctx, a.n_rows_t), 256, 0, st>>>(a, ctx->d_ac, s->rhs_cpl);
  LAUNCH_CHECK();
  // the coupling family's update overlaps the Euler update and the recovery
  // when one follows in the same sequence; alone it would only trail the
  // call on the small side grid
  const bool fork_cpl = s->overlap && !join_tail && !defer_cpl;
  rc = solve_enqueue(ctx, MQ_FAM_COUPLING_PREVIOUS, s->rhs_cpl, s->y_cpl, !fork_cpl && !defer_cpl);
  if (rc) return rc;
  if (fork_cpl) {
    rc = fork_observe(ctx, 2, MQ_FAM_COUPLING_PREVIOUS, s->y_cpl);
    if (rc) return rc;
  }
  if (defer_cpl) {
    k_set_pending<<<1, 32, 0, st>>>(s->d_fam + MQ_FAM_COUPLING_PREVIOUS);
    LAUNCH_CHECK();
  }
  k_dlog_pod<<<1, 32, 0, st>>>(s->d_run, s->d_par, s->d_dlog, s->dlog_cap, 3);
  LAUNCH_CHECK();
  // Brauer + Euler update
  k_cell_nu<<<grid_for(ctx, a.n_cells), 256, 0, st>>>(a, ctx->d_ac, ctx->d_cell_nu);
  LAUNCH_CHECK();
  k_euler<<<grid_for(ctx, n_c), 256, 0, st>>>(a, ctx->d_cell_nu, ctx->d_ac, s->y_cpl, s->y_src, ctx->d_ac_next,
                                              s->d_par, s->d_run);
  LAUNCH_CHECK();
  k_copy_n<<<grid_for(ctx, n_c), 256, 0, st>>>(n_c, ctx->d_ac_next, ctx->d_ac, s->d_run);
  LAUNCH_CHECK();
  return join_tail ? join_all(ctx) : MQ_OK;
}

// defer: leave the coupling family's insert pending for the next step's
// side stream (stepper only)
static int recover_enqueue(mq_ctx *ctx, bool defer) {
  SolverHost *s = ctx->solver;
  CondArgs a = cond_args(ctx);
  cudaStream_t st = ctx->stream;
  // the source family's cache must be final before its projection
  int rc = join_side(ctx, 0);
  if (rc) return rc;
  k_src_rhs<<<grid_for(ctx, s->n_pat), 256, 0, st>>>(s->n_pat, s->d_pat_idx, s->d_pat_val, s->d_par, 1, s->rhs_src);
  LAUNCH_CHECK();
  rc = solve_enqueue(ctx, MQ_FAM_SOURCE, s->rhs_src, s->y_src, !s->overlap);
  if (rc) return rc;
  if (s->overlap) {
    rc = fork_observe(ctx, 1, MQ_FAM_SOURCE, s->y_src);
    if (rc) return rc;
  }
  k_kcnt<<<grid_for(ctx, a.n_rows_t), 256, 0, st>>>(a, ctx->d_ac, s->rhs_cpl);
  LAUNCH_CHECK();
  // a deferred insert of the previous recovery must finish before this
  // family projects and before y_cur is overwritten
  rc = join_side(ctx, 3);
  if (rc) return rc;
  rc = solve_enqueue(ctx, MQ_FAM_COUPLING_CURRENT, s->rhs_cpl, s->y_cur, !defer);
  if (rc) return rc;
  k_dlog_pod<<<1, 32, 0, st>>>(s->d_run, s->d_par, s->d_dlog, s->dlog_cap, 5);
  LAUNCH_CHECK();
  if (defer) {
    k_set_pending<<<1, 32, 0, st>>>(s->d_fam + MQ_FAM_COUPLING_CURRENT);
    LAUNCH_CHECK();
  }
  return join_all(ctx);
}

// The cached graphs of the host-facing calls.  With deferral (CSPE + overlap)
// each call starts with the other call's pending coupling insert on the side
// stream (gated: a no-op when nothing is pending on the device), under its own
// solves, and leaves its own coupling insert pending; otherwise every cache
// update completes inside the call.
static bool host_defer(const SolverHost *s) { return s->defer_cur && s->overlap; }

static int euler_enqueue_host(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  if (!host_defer(s)) return euler_enqueue(ctx, true);
  int rc = fork_observe(ctx, 3, MQ_FAM_COUPLING_CURRENT, s->y_cur, true);
  if (rc) return rc;
  return euler_enqueue(ctx, true, true);
}

static int recover_enqueue_host(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  if (!host_defer(s)) return recover_enqueue(ctx, false);
  int rc = fork_observe(ctx, 4, MQ_FAM_COUPLING_PREVIOUS, s->y_cpl, true);
  if (rc) return rc;
  return recover_enqueue(ctx, true);
}

// a deferred insert left by the stepper, run now (before any host-visible
// use of the families); a gated no-op if none is pending on the device
static const double *deferred_vec(SolverHost *s, int fam) {
  return fam == MQ_FAM_COUPLING_CURRENT ? s->y_cur : s->y_cpl;
}

static int flush_deferred(mq_ctx *ctx, unsigned keep = 0u) {
  SolverHost *s = ctx->solver;
  if (!s) return MQ_OK;
  for (int fam = MQ_FAM_COUPLING_CURRENT; fam <= MQ_FAM_COUPLING_PREVIOUS; ++fam) {
    if (!s->maybe_pending[fam] || (keep >> fam & 1u)) continue;
    s->maybe_pending[fam] = false;
    const int rc = observe(ctx, fam, deferred_vec(s, fam), main_res(ctx), true);
    if (rc) return rc;
  }
  return MQ_OK;
}

static int stage_status(mq_ctx *ctx, int64_t log_first) {
  SolverHost *s = ctx->solver;
  MQ_CUDA(cudaMemcpyAsync(&s->h_st->run, s->d_run, sizeof(RunDev), cudaMemcpyDeviceToHost, ctx->stream));
  if (log_first >= 0)
    MQ_CUDA(cudaMemcpyAsync(s->h_st->it, s->d_log + log_first, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost,
                            ctx->stream));
  return MQ_OK;
}

static int staged_run_status(mq_ctx *ctx, int64_t *failed_step) {
  const RunDev &r = ctx->solver->h_st->run;
  if (failed_step) *failed_step = r.err ? r.err_step : -1;
  if (r.err == 0) return MQ_OK;
  static const char *fam_name[3] = {"source", "coupling_current", "coupling_previous"};
  std::string where = r.err_step >= 0 ? " at step " + std::to_string(r.err_step) : std::string();
  if (r.err == MQ_NOT_CONVERGED)
    set_error(std::string("inner solve (") + (r.err_family >= 0 ? fam_name[r.err_family] : "?") +
              ") stalled" + where);
  else if (r.err == MQ_INDEFINITE)
    set_error(std::string("nonpositive curvature in inner solve (") +
              (r.err_family >= 0 ? fam_name[r.err_family] : "?") + ")" + where);
  else if (r.err == MQ_NONFINITE)
    set_error("non-finite conducting state" + where);
  else
    set_error("device failure (grid barrier watchdog)" + where);
  return (int)r.err;
}

static int check_run(mq_ctx *ctx, int64_t *failed_step) {
  int rc = stage_status(ctx, -1);
  if (rc) return rc;
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return staged_run_status(ctx, failed_step);
}

__global__ void k_reset_run(RunDev *run) {
  if (threadIdx.x != 0) return;
  run->err = 0;
  run->err_family = 0;
  run->err_step = 0;
  run->step = 0;
  run->solve_idx = 0;
}

// per-call fields only; strategy-wide counters persist (startvec.py:404-454)
static int reset_run(mq_ctx *ctx) {
  k_reset_run<<<1, 32, 0, ctx->stream>>>(ctx->solver->d_run);
  MQ_CUDA(cudaGetLastError());
  return MQ_OK;
}

static int init_run(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  RunDev r{};
  r.min_pod_info = 1.0;
  r.pod_last_info = 1.0;
  MQ_CUDA(cudaMemcpyAsync(s->d_run, &r, sizeof(RunDev), cudaMemcpyHostToDevice, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_solver_init(mq_ctx *ctx, const mq_solver_cfg *cfg, const double *pattern) {
  if (!ctx || !cfg) { set_error("NULL argument"); return MQ_INVALID; }
  if (cfg->strategy < 0 || cfg->strategy > 3) { set_error("unknown start-vector strategy"); return MQ_INVALID; }
  if (cfg->strategy == MQ_STRAT_CSPE && (cfg->max_cols < 1 || cfg->max_cols > MAXS)) {
    set_error("max_cols must lie in [1, 32]");
    return MQ_INVALID;
  }
  if (cfg->strategy == MQ_STRAT_POD && (cfg->n_pod < 1 || cfg->n_pod > MAXS)) {
    set_error("n_pod must lie in [1, 32]");
    return MQ_INVALID;
  }
  if (cfg->strategy == MQ_STRAT_POD && !(cfg->eps_pod > 0.0 && cfg->eps_pod < 1.0)) {
    set_error("eps_pod must lie in (0, 1)");
    return MQ_INVALID;
  }
  if (!(cfg->rel_tol > 0.0) || cfg->abs_tol < 0.0 || cfg->max_iter < 1) {
    set_error("invalid PCG configuration");
    return MQ_INVALID;
  }
  solver_free(ctx);
  SolverHost *s = new SolverHost();
  ctx->solver = s;
  s->cfg = *cfg;
  {
    const int bound = cfg->strategy == MQ_STRAT_CSPE ? cfg->max_cols : (cfg->strategy == MQ_STRAT_POD ? cfg->n_pod : 1);
    s->kb = bound <= 8 ? 8 : (bound <= 16 ? 16 : 32);
  }
  const Lay &L = ctx->topo.L;
  const size_t vb = sizeof(double) * L.total;
  int rc = 0;
  rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_fam, sizeof(FamDev) * 3);
  rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_run, sizeof(RunDev));
  rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_par, sizeof(StepParams));
  rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_probe_out, sizeof(double));
  if (!rc) {
    cudaError_t e = cudaMallocHost((void **)&s->h_st, sizeof(SolverHost::HostStage));
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMallocHost");
  }
  auto vec = [&](double **p) { return rc ? rc : (rc = s_alloc(ctx, s, (void **)p, vb)); };
  auto table = [&](double ***tab, std::vector<double *> &h, int n) {
    if (rc) return rc;
    h.assign(MAXS, nullptr);
    for (int q = 0; q < n && !rc; ++q) vec(&h[q]);
    if (rc) return rc;
    rc = s_alloc(ctx, s, (void **)tab, sizeof(double *) * MAXS);
    if (rc) return rc;
    cudaError_t e = cudaMemcpyAsync(*tab, h.data(), sizeof(double *) * MAXS, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "slot table");
    return rc;
  };
  for (int fam = 0; fam < 3; ++fam) {
    if (cfg->strategy == MQ_STRAT_CSPE) {
      table(&s->d_U[fam], s->h_U[fam], cfg->max_cols);
      table(&s->d_KU[fam], s->h_KU[fam], cfg->max_cols);
    } else if (cfg->strategy == MQ_STRAT_POD) {
      table(&s->d_X[fam], s->h_X[fam], cfg->n_pod);
    } else if (cfg->strategy == MQ_STRAT_PREVIOUS) {
      vec(&s->last[fam]);
    }
  }
  if (cfg->strategy == MQ_STRAT_POD) {
    table(&s->d_B, s->h_B, cfg->n_pod);
    table(&s->d_KB, s->h_KB, cfg->n_pod);
    // K B_j through the TMA march where the TMA PCG kernel runs (128^3 and
    // up); MQ_POD_SPMV=flat keeps the thread-per-row k_spmv_multi
    const char *ea = getenv("MQ_EIG_AHEAD");
    if (!rc && ctx->pcg_variant == 0 && ctx->brick_grid < ctx->sms * 2 && !(ea && ea[0] == '0')) {
      cudaError_t e = cudaStreamCreateWithFlags(&s->eig_side, cudaStreamNonBlocking);
      for (int f = 0; f < 3 && e == cudaSuccess; ++f) {
        e = cudaEventCreateWithFlags(&s->ev_ef[f], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_ej[f], cudaEventDisableTiming);
      }
      if (e != cudaSuccess) rc = cuda_fail(e, "eig side stream");
      else s->eig_ahead = true;
    }
    const char *sp = getenv("MQ_POD_SPMV");
    if (!rc && ctx->pcg_variant == 0 && !(sp && std::string(sp) == "flat"))
      for (int fam = 0; fam < 3 && !rc; ++fam)
        rc = kn_multi_prepare(L, ctx->geo, ctx->d_mask, ctx->kn_diag, ctx->kn_off, s->h_B.data(), s->h_KB.data(),
                              cfg->n_pod, &s->d_fam[fam].podk, ctx->sms, &s->kn_multi[fam]);
  }
  vec(&s->w1);
  vec(&s->w2);
  vec(&s->rhs_src);
  vec(&s->rhs_cpl);
  vec(&s->y_src);
  vec(&s->y_cpl);
  vec(&s->y_cur);
#ifndef MQ_RED_MULT
#define MQ_RED_MULT 2
#endif
  s->red_grid = std::max(1, std::min<int>(ctx->sms * MQ_RED_MULT, (int)((L.words + kWarps - 1) / kWarps)));
  rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_red, sizeof(double) * RQ * (size_t)s->red_grid * (MAXS + 2));
  rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_cnt, sizeof(unsigned int) * (MAXS + 4));
  // side stream for the overlapped source-family update: only with the
  // resident PCG kernel, which leaves SMs idle (MQ_OVERLAP=0 disables)
  {
    const char *ov = getenv("MQ_OVERLAP");
    const int idle = ctx->sms - ctx->res_grid;
    if (!rc && ctx->pcg_variant == 2 && idle >= 4 && !(ov && ov[0] == '0')) {
      s->side_grid = idle;
      vec(&s->w1b);
      vec(&s->w2b);
      rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_red2, sizeof(double) * RQ * (size_t)s->red_grid * (MAXS + 2));
      rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_cnt2, sizeof(unsigned int) * (MAXS + 4));
      if (!rc) {
        cudaError_t e = cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking);
        for (int q = 0; q < SolverHost::kSlots && e == cudaSuccess; ++q) {
          e = cudaEventCreateWithFlags(&s->ev_fork[q], cudaEventDisableTiming);
          if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_join[q], cudaEventDisableTiming);
        }
        if (e != cudaSuccess) rc = cuda_fail(e, "overlap stream");
        else {
          s->overlap = true;
          s->defer_cur = cfg->strategy == MQ_STRAT_CSPE;
        }
      }
    }
  }
  // sparse source pattern on its support
  if (!rc && pattern) {
    std::vector<int32_t> idx;
    std::vector<double> val;
    const auto &pad = ctx->topo.nc_pad;
    for (size_t q = 0; q < pad.size(); ++q)
      if (pattern[q] != 0.0) { idx.push_back(pad[q]); val.push_back(pattern[q]); }
    s->n_pat = (int64_t)idx.size();
    if (s->n_pat) {
      rc = s_alloc(ctx, s, (void **)&s->d_pat_idx, sizeof(int32_t) * idx.size());
      rc = rc ? rc : s_alloc(ctx, s, (void **)&s->d_pat_val, sizeof(double) * val.size());
      if (!rc) {
        cudaMemcpyAsync(s->d_pat_idx, idx.data(), sizeof(int32_t) * idx.size(), cudaMemcpyHostToDevice, ctx->stream);
        cudaMemcpyAsync(s->d_pat_val, val.data(), sizeof(double) * val.size(), cudaMemcpyHostToDevice, ctx->stream);
      }
    }
  }
  if (!rc) {
    int iota[MAXS];
    for (int q = 0; q < MAXS; ++q) iota[q] = q;
    rc = s_alloc(ctx, s, (void **)&s->d_iota, sizeof(iota));
    if (!rc) cudaMemcpyAsync(s->d_iota, iota, sizeof(iota), cudaMemcpyHostToDevice, ctx->stream);
  }
  if (!rc) rc = init_run(ctx);
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "solver init");
  }
  if (rc) solver_free(ctx);
  return rc;
}

int mq_solver_reset(mq_ctx *ctx) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  int rj = join_eigs(ctx);  // a running eigen-decomposition writes the family state
  if (rj) return rj;
  MQ_CUDA(cudaMemsetAsync(s->d_fam, 0, sizeof(FamDev) * 3, ctx->stream));
  for (bool &m : s->maybe_pending) m = false;  // the memset cleared any deferred insert
  s->probe_cached = false;
  return init_run(ctx);
}

int mq_solve_kn(mq_ctx *ctx, int32_t family, const double *rhs, double *y, mq_solve_report *rep) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  {
    const int frc = flush_deferred(ctx);
    if (frc) return frc;
  }
  if (family < 0 || family > 2) { set_error("unknown family"); return MQ_INVALID; }
  int rc = reset_run(ctx);
  if (rc) return rc;
  MQ_CUDA(cudaMemsetAsync(s->d_par, 0, sizeof(StepParams), ctx->stream));
  rc = solve_enqueue(ctx, family, rhs, y);
  if (rc) return rc;
  MQ_CUDA(cudaMemcpyAsync(ctx->h_out, ctx->d_out, sizeof(PcgOut), cudaMemcpyDeviceToHost, ctx->stream));
  rc = check_run(ctx, nullptr);
  const PcgOut &o = *ctx->h_out;
  if (rep) {
    rep->iterations = o.iterations;
    rep->converged = o.converged;
    rep->final_rel_residual = o.rel;
    rep->applies = o.applies;
  }
  return rc;
}

int mq_strategy_start(mq_ctx *ctx, int32_t family, const double *rhs, double *x0) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  {
    const int frc = flush_deferred(ctx);
    if (frc) return frc;
  }
  int rc = start_vector(ctx, family, rhs, x0);
  if (rc) return rc;
  // materialise zero start vectors
  FamDev f;
  MQ_CUDA(cudaMemcpyAsync(&f, s->d_fam + family, sizeof(FamDev), cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  if (f.x0_mode == 0) MQ_CUDA(cudaMemsetAsync(x0, 0, sizeof(double) * ctx->topo.L.total, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

int mq_strategy_observe(mq_ctx *ctx, int32_t family, const double *y) {
  if (!ctx->solver) { set_error("solver not initialised"); return MQ_INVALID; }
  {
    const int frc = flush_deferred(ctx);
    if (frc) return frc;
  }
  int rc = observe(ctx, family, y, main_res(ctx));
  if (!rc) rc = join_eigs(ctx);
  if (rc) return rc;
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

int mq_diagnostics(mq_ctx *ctx, mq_diag *out) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  {
    const int frc = flush_deferred(ctx);
    if (frc) return frc;
    const int jrc = join_eigs(ctx);
    if (jrc) return jrc;
  }
  FamDev f[3];
  RunDev r;
  MQ_CUDA(cudaMemcpyAsync(f, s->d_fam, sizeof(FamDev) * 3, cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaMemcpyAsync(&r, s->d_run, sizeof(RunDev), cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memset(out, 0, sizeof(*out));
  out->pcg_applies = r.pcg_applies;
  for (int q = 0; q < 3; ++q) {
    out->basis_cols[q] = s->cfg.strategy == MQ_STRAT_CSPE ? f[q].k : 0;
    out->columns_accepted[q] = f[q].accepted;
    out->columns_dropped[q] = f[q].dropped;
    out->evictions[q] = f[q].evictions;
    out->maintenance_applies += s->cfg.strategy == MQ_STRAT_CSPE ? f[q].products : f[q].pod_applies;
  }
  out->pod_k = r.pod_last_k;
  out->pod_info = r.pod_last_info;
  out->min_pod_info = r.any_pod ? r.min_pod_info : 1.0;
  return MQ_OK;
}

int mq_cspe_export(mq_ctx *ctx, int32_t family, int32_t *k, double *basis, double *products, double *galerkin) {
  SolverHost *s = ctx->solver;
  if (!s || s->cfg.strategy != MQ_STRAT_CSPE) { set_error("CSPE solver not initialised"); return MQ_INVALID; }
  FamDev f;
  MQ_CUDA(cudaMemcpyAsync(&f, s->d_fam + family, sizeof(FamDev), cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  *k = f.k;
  const int64_t n = (int64_t)ctx->topo.nc_pad.size();
  for (int j = 0; j < f.k; ++j) {
    if (basis) {
      int rc = mq_vec_download(ctx, s->h_U[family][f.order[j]], basis + j * n);
      if (rc) return rc;
    }
    if (products) {
      int rc = mq_vec_download(ctx, s->h_KU[family][f.order[j]], products + j * n);
      if (rc) return rc;
    }
  }
  if (galerkin)
    for (int r = 0; r < f.k; ++r)
      for (int c = 0; c < f.k; ++c) galerkin[r * f.k + c] = f.G[r * MAXS + c];
  return MQ_OK;
}

int mq_kc_apply_host(mq_ctx *ctx, const double *state, const double *x, double *y) {
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  CondArgs a = cond_args(ctx);
  cudaStream_t st = ctx->stream;
  MQ_CUDA(cudaMemcpyAsync(ctx->d_ac_next, state, sizeof(double) * n_c, cudaMemcpyHostToDevice, st));
  MQ_CUDA(cudaMemcpyAsync(ctx->d_ac_x, x, sizeof(double) * n_c, cudaMemcpyHostToDevice, st));
  k_cell_nu<<<grid_for(ctx, a.n_cells), 256, 0, st>>>(a, ctx->d_ac_next, ctx->d_cell_nu);
  LAUNCH_CHECK();
  k_kc_apply<<<grid_for(ctx, n_c), 256, 0, st>>>(a, ctx->d_cell_nu, ctx->d_ac_x, ctx->d_yc);
  LAUNCH_CHECK();
  MQ_CUDA(cudaMemcpyAsync(y, ctx->d_yc, sizeof(double) * n_c, cudaMemcpyDeviceToHost, st));
  MQ_CUDA(cudaStreamSynchronize(st));
  return MQ_OK;
}

int mq_kcn_t_apply_host(mq_ctx *ctx, const double *a_c, double *y_n) {
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  CondArgs a = cond_args(ctx);
  cudaStream_t st = ctx->stream;
  MQ_CUDA(cudaMemcpyAsync(ctx->d_ac_x, a_c, sizeof(double) * n_c, cudaMemcpyHostToDevice, st));
  MQ_CUDA(cudaMemsetAsync(ctx->d_tmp0, 0, sizeof(double) * ctx->topo.L.total, st));
  k_kcnt<<<grid_for(ctx, a.n_rows_t), 256, 0, st>>>(a, ctx->d_ac_x, ctx->d_tmp0);
  LAUNCH_CHECK();
  return mq_vec_download(ctx, ctx->d_tmp0, y_n);
}

int mq_kcn_apply_host(mq_ctx *ctx, const double *x_n, double *y_c) {
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  CondArgs a = cond_args(ctx);
  cudaStream_t st = ctx->stream;
  int rc = mq_vec_upload(ctx, x_n, ctx->d_tmp0);
  if (rc) return rc;
  k_kcn<<<grid_for(ctx, n_c), 256, 0, st>>>(a, ctx->d_tmp0, ctx->d_yc);
  LAUNCH_CHECK();
  MQ_CUDA(cudaMemcpyAsync(y_c, ctx->d_yc, sizeof(double) * n_c, cudaMemcpyDeviceToHost, st));
  MQ_CUDA(cudaStreamSynchronize(st));
  return MQ_OK;
}

int mq_mc_diag(mq_ctx *ctx, double *mc_diag) {
  std::memcpy(mc_diag, ctx->topo.mc_diag.data(), sizeof(double) * ctx->topo.mc_diag.size());
  return MQ_OK;
}

int mq_state_set(mq_ctx *ctx, const double *a_c, double t) {
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  if (ctx->solver) ctx->solver->probe_cached = false;
  if (a_c) MQ_CUDA(cudaMemcpyAsync(ctx->d_ac, a_c, sizeof(double) * n_c, cudaMemcpyHostToDevice, ctx->stream));
  else MQ_CUDA(cudaMemsetAsync(ctx->d_ac, 0, sizeof(double) * n_c, ctx->stream));
  ctx->t_now = t;
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

int mq_state_get(mq_ctx *ctx, double *a_c, double *t) {
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  if (a_c) MQ_CUDA(cudaMemcpyAsync(a_c, ctx->d_ac, sizeof(double) * n_c, cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  if (t) *t = ctx->t_now;
  return MQ_OK;
}

static void staged_report(mq_ctx *ctx, mq_solve_report *a, mq_solve_report *b) {
  const int32_t *it = ctx->solver->h_st->it;
  if (a) { a->iterations = it[0]; a->converged = 1; a->final_rel_residual = 0; a->applies = it[0] + 1; }
  if (b) { b->iterations = it[1]; b->converged = 1; b->final_rel_residual = 0; b->applies = it[1] + 1; }
}

static int ensure_log(mq_ctx *ctx, int64_t n) {
  SolverHost *s = ctx->solver;
  if (s->log_cap >= n) return MQ_OK;
  if (s->d_log) cudaFree(s->d_log);
  s->d_log = nullptr;
  MQ_CUDA(cudaMalloc(&s->d_log, sizeof(int32_t) * n));
  s->log_cap = n;
  solver_graph_reset(ctx);
  return MQ_OK;
}

// Enqueue fn once into a graph and replay it afterwards (the kernels read
// their per-call scalars from device memory, so the graph is call-invariant);
// eager launches while PCG timing events are recorded.
static int run_cached(mq_ctx *ctx, cudaGraphExec_t *g, int64_t *nlaunch, int (*fn)(mq_ctx *)) {
  SolverHost *s = ctx->solver;
  if (ctx->pcg_timing || !s->graph_ok) return fn(ctx);
  if (!*g) {
    cudaGraph_t gr = nullptr;
    const int64_t l0 = ctx->launches;
    cudaError_t e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      int r2 = fn(ctx);
      e = cudaStreamEndCapture(ctx->stream, &gr);
      if (r2 == MQ_OK && e == cudaSuccess) e = cudaGraphInstantiate(g, gr, 0);
      if (gr) cudaGraphDestroy(gr);
    }
    *nlaunch = ctx->launches - l0;
    ctx->launches = l0;
    if (e != cudaSuccess || !*g) {
      cudaGetLastError();
      *g = nullptr;
      return fn(ctx);
    }
  }
  MQ_CUDA(cudaGraphLaunch(*g, ctx->stream));
  ctx->launches += *nlaunch;
  return MQ_OK;
}

// Host-facing step and recovery.  Everything a call needs is enqueued on the
// context stream and the call synchronises once: state upload, parameters, the
// cached one-call graph, then the run status, the two iteration counts and the
// host result (a_c or a_n) come back in one batch of copies.
static int euler_call(mq_ctx *ctx, const double *a_c_in, double t, double dt, double wave_new, int64_t step_index,
                      double *a_c_out, mq_solve_report *rep_src, mq_solve_report *rep_cpl) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  if (dt < 0) { set_error("dt must be nonnegative"); return MQ_INVALID; }
  s->probe_cached = false;
  {
    const int frc = flush_deferred(ctx, host_defer(s) ? 1u << MQ_FAM_COUPLING_CURRENT : 0u);
    if (frc) return frc;
  }
  int rc = ensure_log(ctx, 4);
  if (rc) return rc;
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  if (a_c_in) {
    MQ_CUDA(cudaMemcpyAsync(ctx->d_ac, a_c_in, sizeof(double) * n_c, cudaMemcpyHostToDevice, ctx->stream));
    ctx->t_now = t;
  }
  rc = reset_run(ctx);
  if (rc) return rc;
  StepParams p{dt, wave_new, wave_new, (long long)step_index};
  MQ_CUDA(cudaMemcpyAsync(s->d_par, &p, sizeof(p), cudaMemcpyHostToDevice, ctx->stream));
  rc = run_cached(ctx, &s->euler_graph, &s->euler_launches, euler_enqueue_host);
  if (rc) return rc;
  if (host_defer(s)) {
    s->maybe_pending[MQ_FAM_COUPLING_CURRENT] = false;
    s->maybe_pending[MQ_FAM_COUPLING_PREVIOUS] = true;
  }
  rc = stage_status(ctx, 0);
  if (rc) return rc;
  if (a_c_out) MQ_CUDA(cudaMemcpyAsync(a_c_out, ctx->d_ac, sizeof(double) * n_c, cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t failed = -1;
  rc = staged_run_status(ctx, &failed);
  staged_report(ctx, rep_src, rep_cpl);
  if (!rc) ctx->t_now += dt;
  return rc;
}

static int recover_call(mq_ctx *ctx, const double *a_c_in, double t, double wave_now, double *a_n_host,
                        mq_solve_report *rep_src, mq_solve_report *rep_cpl) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  s->probe_cached = false;
  {
    const int frc = flush_deferred(ctx, host_defer(s) ? 1u << MQ_FAM_COUPLING_PREVIOUS : 0u);
    if (frc) return frc;
  }
  int rc = ensure_log(ctx, 4);
  if (rc) return rc;
  if (a_c_in) {
    const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
    MQ_CUDA(cudaMemcpyAsync(ctx->d_ac, a_c_in, sizeof(double) * n_c, cudaMemcpyHostToDevice, ctx->stream));
    ctx->t_now = t;
  }
  rc = reset_run(ctx);
  if (rc) return rc;
  StepParams p{0.0, wave_now, wave_now, -1};
  MQ_CUDA(cudaMemcpyAsync(s->d_par, &p, sizeof(p), cudaMemcpyHostToDevice, ctx->stream));
  rc = run_cached(ctx, &s->recover_graph, &s->recover_launches, recover_enqueue_host);
  if (rc) return rc;
  if (host_defer(s)) {
    s->maybe_pending[MQ_FAM_COUPLING_PREVIOUS] = false;
    s->maybe_pending[MQ_FAM_COUPLING_CURRENT] = true;
  }
  rc = stage_status(ctx, 0);
  if (rc) return rc;
  if (a_n_host) {
    // a_n = y_src - y_cur, gathered to the compact order; a failed run is
    // reported below and the copied values are then meaningless
    k_sub<<<stream_grid(ctx), kBlock, 0, ctx->stream>>>(ctx->topo.L, ctx->d_mask, s->y_src, s->y_cur, ctx->d_tmp1);
    LAUNCH_CHECK();
    const int64_t n = (int64_t)ctx->topo.nc_pad.size();
    rc = launch_gather(n, ctx->d_nc_pad, ctx->d_tmp1, ctx->d_stage, ctx->sms, ctx->stream);
    if (rc) return rc;
    ctx->launches += 1;
    MQ_CUDA(cudaMemcpyAsync(a_n_host, ctx->d_stage, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  const bool probe = s->n_probe > 0;
  if (probe) {
    k_probe<<<s->probe_grid, 256, 0, ctx->stream>>>(cond_args(ctx), s->d_probe, s->n_probe, s->d_probe_plan,
                                                    ctx->d_ac, s->d_probe_vals, s->d_probe_leaf, s->d_probe_ctr,
                                                    nullptr, nullptr, s->d_probe_out);
    LAUNCH_CHECK();
    MQ_CUDA(cudaMemcpyAsync(&s->h_st->probe, s->d_probe_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  }
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  rc = staged_run_status(ctx, nullptr);
  staged_report(ctx, rep_src, rep_cpl);
  if (probe && rc == MQ_OK) {
    s->probe_cache = s->h_st->probe;
    s->probe_cached = true;
  }
  return rc;
}

int mq_euler_step(mq_ctx *ctx, double dt, double wave_new, int64_t step_index, mq_solve_report *rep_src,
                  mq_solve_report *rep_cpl) {
  return euler_call(ctx, nullptr, 0.0, dt, wave_new, step_index, nullptr, rep_src, rep_cpl);
}

int mq_euler_step_host(mq_ctx *ctx, const double *a_c, double t, double dt, double wave_new, int64_t step_index,
                       double *a_c_next, mq_solve_report *rep_src, mq_solve_report *rep_cpl) {
  if (!a_c || !a_c_next) { set_error("NULL state array"); return MQ_INVALID; }
  return euler_call(ctx, a_c, t, dt, wave_new, step_index, a_c_next, rep_src, rep_cpl);
}

int mq_recover_an(mq_ctx *ctx, double wave_now, double *a_n_host, mq_solve_report *rep_src,
                  mq_solve_report *rep_cpl) {
  return recover_call(ctx, nullptr, 0.0, wave_now, a_n_host, rep_src, rep_cpl);
}

int mq_recover_an_host(mq_ctx *ctx, const double *a_c, double t, double wave_now, double *a_n_host,
                       mq_solve_report *rep_src, mq_solve_report *rep_cpl) {
  if (!a_c) { set_error("NULL state array"); return MQ_INVALID; }
  return recover_call(ctx, a_c, t, wave_now, a_n_host, rep_src, rep_cpl);
}

int mq_last_an(mq_ctx *ctx, double *a_n_host) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  k_sub<<<stream_grid(ctx), kBlock, 0, ctx->stream>>>(ctx->topo.L, ctx->d_mask, s->y_src, s->y_cur, ctx->d_tmp1);
  LAUNCH_CHECK();
  return mq_vec_download(ctx, ctx->d_tmp1, a_n_host);
}

// a_n = y_src - y_cur of the step's recovery in compact order (schur.py:416-419)
__global__ void k_an_record(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ y_src,
                            const double *__restrict__ y_cur, const StepParams *par, const RunDev *run,
                            double *__restrict__ out) {
  if (run->err) return;
  const long long m = par->step - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = idx[i];
    out[m * n + i] = sub(y_src[e], y_cur[e]);
  }
}

static int enqueue_step(mq_ctx *ctx, double *hist, double *hist_n = nullptr) {
  SolverHost *s = ctx->solver;
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  ctx->ev_n = 0;
  k_load_params<<<1, 32, 0, ctx->stream>>>(s->d_par, s->d_dt_tab, s->d_wave_tab, s->d_run);
  MQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  const bool defer = s->defer_cur && s->recover_every_step;
  if (defer) {
    // the previous recovery's coupling-family insert, under this step's
    // source and coupling solves (a no-op if none is pending)
    int r0 = fork_observe(ctx, 3, MQ_FAM_COUPLING_CURRENT, s->y_cur, true, 2);
    if (r0) return r0;
  }
  int rc = euler_enqueue(ctx, !s->recover_every_step);
  if (rc) return rc;
  if (s->recover_every_step) {
    rc = recover_enqueue(ctx, defer);
    if (rc) return rc;
    if (defer) s->maybe_pending[MQ_FAM_COUPLING_CURRENT] = true;
    if (hist_n) {
      const int64_t n_n = (int64_t)ctx->topo.nc_pad.size();
      k_an_record<<<grid_for(ctx, n_n), 256, 0, ctx->stream>>>(n_n, ctx->d_nc_pad, s->y_src, s->y_cur, s->d_par,
                                                               s->d_run, hist_n);
      MQ_CUDA(cudaGetLastError());
      ctx->launches += 1;
    }
  }
  if (s->n_probe > 0) {
    k_probe<<<s->probe_grid, 256, 0, ctx->stream>>>(cond_args(ctx), s->d_probe, s->n_probe, s->d_probe_plan,
                                                    ctx->d_ac, s->d_probe_vals, s->d_probe_leaf, s->d_probe_ctr,
                                                    s->d_par, s->d_probe_log, nullptr);
    MQ_CUDA(cudaGetLastError());
    ctx->launches += 1;
  }
  k_step_done<<<grid_for(ctx, n_c), 256, 0, ctx->stream>>>(s->d_run, s->d_par, ctx->d_ac, hist, n_c);
  MQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  return MQ_OK;
}

static void probe_plan(int64_t off, int64_t n, std::vector<int32_t> &leaves, std::vector<int32_t> &prog) {
  if (n <= 128) {
    prog.push_back((int32_t)(leaves.size() / 2));
    leaves.push_back((int32_t)off);
    leaves.push_back((int32_t)n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  probe_plan(off, n2, leaves, prog);
  probe_plan(off + n2, n - n2, leaves, prog);
  prog.push_back(-1);
}

int mq_probe_set(mq_ctx *ctx, const int64_t *cells, int64_t n) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  s->probe_cached = false;
  if (n < 0 || (n > 0 && !cells)) { set_error("invalid probe cell list"); return MQ_INVALID; }
  const std::vector<int64_t> &ids = ctx->topo.cell_ids;
  std::vector<int32_t> loc((size_t)n);
  for (int64_t q = 0; q < n; ++q) {
    auto it = std::lower_bound(ids.begin(), ids.end(), cells[q]);
    if (it == ids.end() || *it != cells[q]) {
      set_error("probe cell is not a conductor cell (the device probe reads the conducting state only)");
      return MQ_INVALID;
    }
    loc[q] = (int32_t)(it - ids.begin());
  }
  cudaFree(s->d_probe);
  cudaFree(s->d_probe_vals);
  cudaFree(s->d_probe_plan);
  cudaFree(s->d_probe_leaf);
  cudaFree(s->d_probe_ctr);
  s->d_probe = nullptr;
  s->d_probe_ctr = nullptr;
  s->d_probe_vals = s->d_probe_leaf = nullptr;
  s->d_probe_plan = nullptr;
  s->n_probe = 0;
  if (n > 0) {
    if (n > (int64_t)1 << 30) { set_error("probe cell set too large"); return MQ_INVALID; }
    std::vector<int32_t> leaves, prog;
    probe_plan(0, n, leaves, prog);
    std::vector<int32_t> plan = {(int32_t)(leaves.size() / 2), (int32_t)prog.size()};
    plan.insert(plan.end(), leaves.begin(), leaves.end());
    plan.insert(plan.end(), prog.begin(), prog.end());
    MQ_CUDA(cudaMalloc(&s->d_probe, sizeof(int32_t) * n));
    MQ_CUDA(cudaMalloc(&s->d_probe_vals, sizeof(double) * n));
    MQ_CUDA(cudaMalloc(&s->d_probe_leaf, sizeof(double) * (leaves.size() / 2)));
    MQ_CUDA(cudaMalloc(&s->d_probe_plan, sizeof(int32_t) * plan.size()));
    MQ_CUDA(cudaMalloc(&s->d_probe_ctr, sizeof(unsigned int)));
    MQ_CUDA(cudaMemset(s->d_probe_ctr, 0, sizeof(unsigned int)));
    s->probe_grid = (int)std::min<int64_t>((n + 255) / 256, ctx->sms);
    MQ_CUDA(cudaMemcpy(s->d_probe, loc.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    MQ_CUDA(cudaMemcpy(s->d_probe_plan, plan.data(), sizeof(int32_t) * plan.size(), cudaMemcpyHostToDevice));
  }
  s->n_probe = n;
  if (s->graph_exec) { cudaGraphExecDestroy(s->graph_exec); s->graph_exec = nullptr; }
  return MQ_OK;
}

int mq_probe_b(mq_ctx *ctx, const double *a_c_host, double *out) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  if (s->n_probe <= 0) { set_error("probe cell set is empty"); return MQ_INVALID; }
  if (!a_c_host && s->probe_cached) {
    *out = s->probe_cache;
    return MQ_OK;
  }
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  const double *state = ctx->d_ac;
  if (a_c_host) {
    MQ_CUDA(cudaMemcpyAsync(ctx->d_ac_x, a_c_host, sizeof(double) * n_c, cudaMemcpyHostToDevice, ctx->stream));
    state = ctx->d_ac_x;
  }
  k_probe<<<s->probe_grid, 256, 0, ctx->stream>>>(cond_args(ctx), s->d_probe, s->n_probe, s->d_probe_plan, state,
                                                  s->d_probe_vals, s->d_probe_leaf, s->d_probe_ctr, nullptr, nullptr,
                                                  s->d_probe_out);
  LAUNCH_CHECK();
  MQ_CUDA(cudaMemcpyAsync(&s->h_st->probe, s->d_probe_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  *out = s->h_st->probe;
  return MQ_OK;
}

int mq_run_probe_log(mq_ctx *ctx, int64_t n, double *out) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  if (s->n_probe <= 0) { set_error("probe cell set is empty"); return MQ_INVALID; }
  if (n < 0 || n > s->n_enqueued) { set_error("more probe rows than steps run"); return MQ_INVALID; }
  if (n > 0) MQ_CUDA(cudaMemcpy(out, s->d_probe_log, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return MQ_OK;
}

int mq_run_diag_log(mq_ctx *ctx, int64_t n, double *out) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  if (n < 0 || n > s->n_enqueued || n > s->dlog_cap) { set_error("more diagnostics rows than steps run"); return MQ_INVALID; }
  if (n > 0) MQ_CUDA(cudaMemcpy(out, s->d_dlog, sizeof(double) * kDiagW * n, cudaMemcpyDeviceToHost));
  return MQ_OK;
}

int mq_run_prepare(mq_ctx *ctx, int64_t n_steps, const double *dt, const double *wave,
                   int32_t recover_every_step) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  s->probe_cached = false;
  if (n_steps < 0) { set_error("n_steps must be nonnegative"); return MQ_INVALID; }
  {
    // a host call's deferred insert: the coupling-current one is absorbed by
    // the first step's side stream when the steps recover, the other runs now
    const bool absorb = s->defer_cur && recover_every_step;
    const int frc = flush_deferred(ctx, absorb ? 1u << MQ_FAM_COUPLING_CURRENT : 0u);
    if (frc) return frc;
  }
  const int per = recover_every_step ? 4 : 2;
  int rc = ensure_log(ctx, std::max<int64_t>(4, per * n_steps));
  if (rc) return rc;
  if (s->tab_cap < n_steps + 1) {
    if (s->d_dt_tab) cudaFree(s->d_dt_tab);
    if (s->d_wave_tab) cudaFree(s->d_wave_tab);
    MQ_CUDA(cudaMalloc(&s->d_dt_tab, sizeof(double) * (n_steps + 1)));
    MQ_CUDA(cudaMalloc(&s->d_wave_tab, sizeof(double) * (n_steps + 1)));
    s->tab_cap = n_steps + 1;
    if (s->graph_exec) { cudaGraphExecDestroy(s->graph_exec); s->graph_exec = nullptr; }
  }
  if ((recover_every_step != 0) != s->recover_every_step && s->graph_exec) {
    cudaGraphExecDestroy(s->graph_exec);
    s->graph_exec = nullptr;
  }
  if (s->dlog_cap < n_steps) {
    cudaFree(s->d_dlog);
    s->d_dlog = nullptr;
    MQ_CUDA(cudaMalloc(&s->d_dlog, sizeof(double) * kDiagW * n_steps));
    MQ_CUDA(cudaMemset(s->d_dlog, 0, sizeof(double) * kDiagW * n_steps));
    s->dlog_cap = n_steps;
    solver_graph_reset(ctx);  // every cached graph holds the log pointer
  }
  if (s->n_probe > 0 && s->probe_cap < n_steps) {
    cudaFree(s->d_probe_log);
    s->d_probe_log = nullptr;
    MQ_CUDA(cudaMalloc(&s->d_probe_log, sizeof(double) * n_steps));
    s->probe_cap = n_steps;
    if (s->graph_exec) { cudaGraphExecDestroy(s->graph_exec); s->graph_exec = nullptr; }
  }
  s->recover_every_step = recover_every_step != 0;
  s->per_step = per;
  s->n_planned = n_steps;
  s->n_enqueued = 0;
  if (n_steps > 0)
    MQ_CUDA(cudaMemcpyAsync(s->d_dt_tab, dt, sizeof(double) * n_steps, cudaMemcpyHostToDevice, ctx->stream));
  MQ_CUDA(cudaMemcpyAsync(s->d_wave_tab, wave, sizeof(double) * (n_steps + 1), cudaMemcpyHostToDevice, ctx->stream));
  rc = reset_run(ctx);
  if (rc) return rc;
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

static int run_steps(mq_ctx *ctx, int64_t n, int32_t use_graph, double *a_c_hist_dev, double *a_n_hist_dev);

int mq_run_steps(mq_ctx *ctx, int64_t n, int32_t use_graph, double *a_c_hist_dev) {
  return run_steps(ctx, n, use_graph, a_c_hist_dev, nullptr);
}

static int run_steps(mq_ctx *ctx, int64_t n, int32_t use_graph, double *a_c_hist_dev, double *a_n_hist_dev) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  if (s->n_enqueued + n > s->n_planned) { set_error("more steps than prepared"); return MQ_INVALID; }
  bool graphed = false;
  if (use_graph && !a_c_hist_dev && s->graph_ok) {
    if (!s->graph_exec) {
      cudaGraph_t g = nullptr;
      const int64_t l0 = ctx->launches;
      cudaError_t e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        int r2 = enqueue_step(ctx, nullptr);
        e = cudaStreamEndCapture(ctx->stream, &g);
        if (r2 == MQ_OK && e == cudaSuccess) e = cudaGraphInstantiate(&s->graph_exec, g, 0);
        if (g) cudaGraphDestroy(g);
      }
      s->launches_per_step = ctx->launches - l0;
      ctx->launches = l0;
      if (e != cudaSuccess || !s->graph_exec) {
        cudaGetLastError();
        s->graph_ok = false;
        s->graph_exec = nullptr;
      }
    }
    if (s->graph_exec) {
      graphed = true;
      for (int64_t m = 0; m < n; ++m) {
        MQ_CUDA(cudaGraphLaunch(s->graph_exec, ctx->stream));
        ctx->launches += s->launches_per_step;
      }
    }
  }
  if (!graphed) {
    for (int64_t m = 0; m < n; ++m) {
      int rc = enqueue_step(ctx, a_c_hist_dev, a_n_hist_dev);
      if (rc) return rc;
    }
  }
  s->n_enqueued += n;
  return MQ_OK;
}

int mq_run_finish(mq_ctx *ctx, int32_t *iters_out, int64_t *failed_step) {
  SolverHost *s = ctx->solver;
  if (!s) { set_error("solver not initialised"); return MQ_INVALID; }
  {
    const int frc = flush_deferred(ctx);
    if (frc) return frc;
  }
  int rc = check_run(ctx, failed_step);
  const int64_t n = s->n_enqueued;
  if (iters_out && n > 0)
    MQ_CUDA(cudaMemcpy(iters_out, s->d_log, sizeof(int32_t) * s->per_step * n, cudaMemcpyDeviceToHost));
  return rc;
}

int mq_run_explicit_states(mq_ctx *ctx, int64_t n_steps, const double *dt, const double *wave,
                           int32_t recover_every_step, int32_t use_graph, int32_t *iters_out, double *a_c_hist,
                           double *a_n_hist, int64_t *failed_step) {
  if (a_n_hist && !recover_every_step) { set_error("a_n history needs a recovery every step"); return MQ_INVALID; }
  int rc = mq_run_prepare(ctx, n_steps, dt, wave, recover_every_step);
  if (rc) return rc;
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  const int64_t n_n = (int64_t)ctx->topo.nc_pad.size();
  double *hist = nullptr, *hist_n = nullptr;
  if (a_c_hist && n_steps > 0) MQ_CUDA(cudaMalloc(&hist, sizeof(double) * n_c * n_steps));
  if (a_n_hist && n_steps > 0) {
    const cudaError_t e = cudaMalloc(&hist_n, sizeof(double) * n_n * n_steps);
    if (e != cudaSuccess) {
      cudaFree(hist);
      MQ_CUDA(e);
    }
  }
  rc = run_steps(ctx, n_steps, use_graph, hist, hist_n);
  int rc2 = mq_run_finish(ctx, iters_out, failed_step);
  if (rc == MQ_OK) rc = rc2;
  if (hist) {
    cudaMemcpy(a_c_hist, hist, sizeof(double) * n_c * n_steps, cudaMemcpyDeviceToHost);
    cudaFree(hist);
  }
  if (hist_n) {
    cudaMemcpy(a_n_hist, hist_n, sizeof(double) * n_n * n_steps, cudaMemcpyDeviceToHost);
    cudaFree(hist_n);
  }
  if (rc == MQ_OK) {
    double t = ctx->t_now;
    for (int64_t m = 0; m < n_steps; ++m) t += dt[m];
    ctx->t_now = t;
  }
  return rc;
}

int mq_run_explicit(mq_ctx *ctx, int64_t n_steps, const double *dt, const double *wave, int32_t recover_every_step,
                    int32_t use_graph, int32_t *iters_out, double *a_c_hist, int64_t *failed_step) {
  return mq_run_explicit_states(ctx, n_steps, dt, wave, recover_every_step, use_graph, iters_out, a_c_hist, nullptr,
                                failed_step);
}

// Power iteration for lambda_max(M_c^-1 K_S) (schur.py:327-376 with the
// detached inner solves of schur.py:297-313).  Inner PCG solves run on the
// device (warm-started from the previous inner solution, no family history);
// the n_c-sized Rayleigh-quotient algebra runs on the host in the reference's
// operation order.  v0: the normalised start vector (host, n_c).
int mq_estimate_cfl(mq_ctx *ctx, const double *a_ref, const double *v0, int32_t power_iters, double power_tol,
                    double safety, double rel_tol, int32_t max_iter, double *lambda_out, double *dt_out,
                    int32_t *used_out, int64_t *pcg_applies) {
  if (!(safety > 0.0 && safety <= 1.0)) { set_error("safety must lie in (0, 1]"); return MQ_INVALID; }
  if (power_iters < 1) { set_error("power_iters must be at least 1"); return MQ_INVALID; }
  if (ctx->solver) ctx->solver->probe_cached = false;
  const int64_t n_c = (int64_t)ctx->topo.c_pad.size();
  const Lay &L = ctx->topo.L;
  CondArgs a = cond_args(ctx);
  cudaStream_t st = ctx->stream;
  std::vector<double> v(v0, v0 + n_c), w(n_c), kc(n_c), ky(n_c), u(n_c);
  const std::vector<double> &mc = ctx->topo.mc_diag;
  std::vector<double> minv(n_c);
  for (int64_t e = 0; e < n_c; ++e) minv[e] = 1.0 / mc[e];
  double *d_w = nullptr, *d_y = nullptr;
  MQ_CUDA(cudaMalloc(&d_w, sizeof(double) * L.total));
  MQ_CUDA(cudaMalloc(&d_y, sizeof(double) * L.total));
  MQ_CUDA(cudaMemsetAsync(d_w, 0, sizeof(double) * L.total, st));
  MQ_CUDA(cudaMemsetAsync(d_y, 0, sizeof(double) * L.total, st));
  // nu of the linearisation state (a_ref = 0 when NULL)
  if (a_ref) MQ_CUDA(cudaMemcpyAsync(ctx->d_ac_next, a_ref, sizeof(double) * n_c, cudaMemcpyHostToDevice, st));
  else MQ_CUDA(cudaMemsetAsync(ctx->d_ac_next, 0, sizeof(double) * n_c, st));
  k_cell_nu<<<grid_for(ctx, a.n_cells), 256, 0, st>>>(a, ctx->d_ac_next, ctx->d_cell_nu);
  int rc = MQ_OK;
  double lam = 0.0, lam_prev = 0.0;
  bool have_prev = false;
  int used = power_iters;
  int64_t applies = 0;
  for (int it = 1; it <= power_iters && rc == MQ_OK; ++it) {
    cudaError_t e = cudaMemcpyAsync(ctx->d_ac_x, v.data(), sizeof(double) * n_c, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { rc = cuda_fail(e, "cfl upload"); break; }
    k_kcnt<<<grid_for(ctx, a.n_rows_t), 256, 0, st>>>(a, ctx->d_ac_x, d_w);
    mq_solve_report rep{};
    rc = ctx_pcg(ctx, d_w, d_y, it == 1 ? 2 : 1, rel_tol, 0.0, max_iter, 1, &rep);
    if (rc == MQ_NOT_CONVERGED) { set_error("spectral probe solve stalled"); break; }
    if (rc) break;
    applies += rep.applies;
    k_kc_apply<<<grid_for(ctx, n_c), 256, 0, st>>>(a, ctx->d_cell_nu, ctx->d_ac_x, ctx->d_yc);
    e = cudaMemcpyAsync(kc.data(), ctx->d_yc, sizeof(double) * n_c, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) {
      k_kcn<<<grid_for(ctx, n_c), 256, 0, st>>>(a, d_y, ctx->d_yc);
      e = cudaMemcpyAsync(ky.data(), ctx->d_yc, sizeof(double) * n_c, cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { rc = cuda_fail(e, "cfl products"); break; }
    double den = 0.0, num = 0.0, nu2 = 0.0;
    for (int64_t q = 0; q < n_c; ++q) {
      w[q] = kc[q] - ky[q];
      den += v[q] * (mc[q] * v[q]);
      num += v[q] * w[q];
    }
    lam = num / den;
    for (int64_t q = 0; q < n_c; ++q) {
      u[q] = minv[q] * w[q];
      nu2 += u[q] * u[q];
    }
    const double nu = std::sqrt(nu2);
    if (nu == 0.0) { set_error("power iteration collapsed to the nullspace"); rc = MQ_NOT_CONVERGED; break; }
    for (int64_t q = 0; q < n_c; ++q) v[q] = u[q] / nu;
    if (have_prev && std::fabs(lam - lam_prev) <= power_tol * std::fabs(lam)) { used = it; break; }
    lam_prev = lam;
    have_prev = true;
  }
  cudaFree(d_w);
  cudaFree(d_y);
  if (rc) return rc;
  if (!(lam > 0.0) || !std::isfinite(lam)) {
    set_error("spectral estimate is not positive");
    return MQ_NOT_CONVERGED;
  }
  *lambda_out = lam;
  *dt_out = safety * 2.0 / lam;
  if (used_out) *used_out = used;
  if (pcg_applies) *pcg_applies = applies;
  return MQ_OK;
}

int mq_pcg_collect(mq_ctx *ctx, double *ms, int32_t *n_events) {
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  double sum = 0.0;
  for (int i = 0; i < ctx->ev_n; ++i) {
    float f = 0.f;
    MQ_CUDA(cudaEventElapsedTime(&f, ctx->ev_pool[2 * i], ctx->ev_pool[2 * i + 1]));
    sum += f;
  }
  *ms = sum;
  if (n_events) *n_events = ctx->ev_n;
  return MQ_OK;
}

}  // extern "C"

#include "solver_slab.cuh"

// ---- guard check (memory-safety evidence without compute-sanitizer) ------
// Every device vector of a context holds exact zeros off the partition
// (boundary, conducting, guard and padding entries): the stencils read them as
// boundary values, so a stray write there changes results.  This counts the
// off-partition entries that are not 0 in every vector the context owns.
// Slab contexts: the ghost planes (neighbour values) are skipped.
namespace mq {
__global__ void k_guard(Lay L, const uint32_t *__restrict__ mask, const double *__restrict__ v, int64_t skip_lo,
                        int64_t skip_hi, unsigned long long *bad) {
  unsigned long long n = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L.total; e += (int64_t)gridDim.x * blockDim.x) {
    if ((mask[e >> 5] >> (e & 31)) & 1u) continue;
    const int64_t rel = e % L.C;  // position inside the component box
    if (rel < skip_lo || rel >= skip_hi) continue;
    if (v[e] != 0.0) ++n;
  }
  if (n) atomicAdd(bad, n);
}
}  // namespace mq

extern "C" int mq_guard_check(mq_ctx *ctx, int64_t *bad_entries, int32_t *bad_vectors, int32_t *checked) {
  if (!ctx || !bad_entries || !bad_vectors) { set_error("NULL argument"); return MQ_INVALID; }
  MQ_CUDA(cudaSetDevice(ctx->device));
  std::vector<const double *> vs = {ctx->d_r, ctx->d_p0, ctx->d_p1, ctx->d_ap, ctx->d_ap2, ctx->d_r2};
  for (double *p : ctx->vecs) vs.push_back(p);
  if (SolverHost *s = ctx->solver) {
    for (int f = 0; f < 3; ++f) {
      for (double *p : s->h_U[f]) vs.push_back(p);
      for (double *p : s->h_KU[f]) vs.push_back(p);
      for (double *p : s->h_X[f]) vs.push_back(p);
      vs.push_back(s->last[f]);
    }
    for (double *p : s->h_B) vs.push_back(p);
    for (double *p : s->h_KB) vs.push_back(p);
    for (double *p : {s->w1, s->w2, s->w1b, s->w2b, s->rhs_src, s->rhs_cpl, s->y_src, s->y_cpl, s->y_cur})
      vs.push_back(p);
  }
  if (SlabStepHost *s = ctx->sstep) {
    for (int f = 0; f < 3; ++f) {
      for (double *p : s->h_U[f]) vs.push_back(p);
      for (double *p : s->h_KU[f]) vs.push_back(p);
      vs.push_back(s->last[f]);
    }
    for (double *p : {s->rhs_src, s->rhs_cpl, s->y_src, s->y_cpl, s->y_cur, s->w1, s->w2, s->dvec}) vs.push_back(p);
  }
  const Lay &L = ctx->topo.L;
  // slab: owned planes are padded planes 1..n of each component box
  const bool slab = ctx->slab_hi > ctx->slab_lo;
  const int64_t lo = slab ? L.Si : 0, hi = slab ? (int64_t)(ctx->topo.nx + 1) * L.Si : L.C;
  unsigned long long *d_bad = nullptr;
  MQ_CUDA(cudaMalloc(&d_bad, sizeof(unsigned long long)));
  int64_t total = 0;
  int nbad = 0, n = 0;
  for (const double *v : vs) {
    if (!v) continue;
    ++n;
    cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), ctx->stream);
    k_guard<<<ctx->sms * 4, 256, 0, ctx->stream>>>(L, ctx->d_mask, v, lo, hi, d_bad);
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, d_bad, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) { cudaFree(d_bad); return cuda_fail(e, "guard check"); }
    total += (int64_t)h;
    nbad += h ? 1 : 0;
  }
  cudaFree(d_bad);
  *bad_entries = total;
  *bad_vectors = nbad;
  if (checked) *checked = n;
  return MQ_OK;
}


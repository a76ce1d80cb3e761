// Fused distributed K_n PCG over i-slabs (BASELINE configs[4]): one
// persistent kernel per rank does the stencil passes, the halo exchange and
// the cross-rank all-reduce, with no host round trip per iteration.
//
// Same algorithm and per-row arithmetic as pcg_stencil_kernel (krylov.py:
// 174-250), on a slab context (csrc/slab.cu layout: owned planes 0..n-1 and
// two ghost planes -1 and n).  Per iteration:
//   K1: p_new = M^-1 r + beta p_old (own rows; neighbours and ghosts on the
//       fly), Ap, deferred x update, partial p.Ap; every row of plane 0 /
//       n-1 also stores its p_new into the ghost plane of the neighbour rank
//       (peer memory over NVLink, or the same device when emulated)
//   -> rank all-reduce(p.Ap)
//   K2: r -= alpha Ap, partials r.r, r.z; plane 0 / n-1 rows store r into
//       the neighbours' ghost planes
//   -> rank all-reduce(r.r, r.z)
// The all-reduce doubles as the cross-rank barrier that orders the ghost
// stores before the next pass reads them: a rank's stores precede its
// release (red.release.sys on every rank's arrival counter), the readers
// acquire their counter before reading.  p ghosts are double-buffered like
// p itself (p_new of iteration i lands in the buffer the neighbour reads as
// p_old in iteration i+1 while it may still read the other one).
//
// All-reduce: a rank's group of CTAs first reduces its partials (group
// barrier, CTA order), CTA 0 then stores the rank total into slot
// [inst % RING][rank] of every rank's mailbox and bumps every rank's
// monotonic arrival counter; every CTA waits for its counter to reach
// nranks * (inst + 1) and sums the nranks slots in rank order, so all ranks
// hold bitwise-identical scalars and take identical branches.  Instances
// continue across solves (epoch kept on the device), so counters are never
// reset while a peer may be writing.
//
// With fewer GPUs than ranks the ranks are emulated as groups of CTAs of
// one cooperative launch on one GPU (groups wait on one another, so they
// must be co-resident: one launch, never several).
#include <algorithm>
#include <string>
#include <vector>

#include "mq_ctx.h"
#include "mq_device.cuh"
#include "slab_rank.cuh"

namespace mq {

__device__ __forceinline__ int comp_of_f(int64_t e, int64_t C) { return e < C ? 0 : (e < 2 * C ? 1 : 2); }

// store value v of own row e into the neighbours' ghost planes when e lies in
// plane 0 / n - 1 (component offsets of the receiving slab)
__device__ __forceinline__ void push_ghost(const SlabRank &me, int64_t e, double v, double *lo, double *hi) {
  const Lay &L = me.L;
  const int c = comp_of_f(e, L.C);
  const int64_t rel = e - c * L.C;
  const int64_t plane = rel / L.Si;  // padded plane index: own plane i is i + 1
  const int64_t jk = rel - plane * L.Si;
  if (plane == 1 && lo) lo[c * me.lo_C + me.lo_top + jk] = v;
  if (plane == me.n && hi) hi[c * me.hi_C + jk] = v;
}

__global__ void __launch_bounds__(kBlock) slab_pcg_fused_kernel(const SlabFusedArgs *__restrict__ Ap) {
  __shared__ double red[3 * kWarps];
  __shared__ double tot[4];
  const SlabFusedArgs &A = *Ap;
  const int Gr = gridDim.x / A.ngroups;
  const int g = blockIdx.x / Gr, lb = blockIdx.x % Gr;
  const SlabRank &me = A.rk[g];
  const int rank = A.rank0 + g;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wstride = (int64_t)Gr * kWarps;
  const int64_t w0 = (int64_t)lb * kWarps + warp;
  const Lay L = me.L;
  const uint32_t *__restrict__ mask = me.mask;
  const double dg = A.dg, of = A.of, inv = A.inv;
  const bool jac = A.use_jac != 0;
  double *x = me.x, *r = me.r, *ap = me.ap;
  const double *b = me.b;
  const unsigned long long base = *me.epoch;
  unsigned long long inst = base;
  int status = MQ_OK, iters = 0, converged = 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  double *pold = me.pa, *pnew = me.pb;
  double *lo_pold = me.lo_pa, *lo_pnew = me.lo_pb, *hi_pold = me.hi_pa, *hi_pnew = me.hi_pb;
  int applies = A.x0_mode == 1 ? 1 : 0;
  double v3[3] = {0.0, 0.0, 0.0};
  // ---- x0 ghosts, then the initial residual (krylov.py:209-218) ----
  if (A.x0_mode == 1) {
    for (int64_t w = w0; w < L.words; w += wstride) {
      if (!((mask[w] >> lane) & 1u)) continue;
      const int64_t e = w * 32 + lane;
      push_ghost(me, e, x[e], me.lo_x, me.hi_x);
    }
    double v0[1] = {0.0};
    if (!rank_allreduce<1>(me, A.nranks, rank, lb, Gr, inst++, v0, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
  }
  for (int64_t w = w0; w < L.words; w += wstride) {
    if (!((mask[w] >> lane) & 1u)) continue;
    const int64_t e = w * 32 + lane;
    const double bv = b[e];
    double rv = bv;
    if (A.x0_mode == 1) rv = sub(bv, stencil_row(comp_of_f(e, L.C), e, L, dg, of, [&](int64_t q) { return x[q]; }));
    else x[e] = 0.0;
    r[e] = rv;
    push_ghost(me, e, rv, me.lo_r, me.hi_r);
    const double z = jac ? mul(inv, rv) : rv;
    v3[0] = add(v3[0], mul(bv, bv));
    v3[1] = add(v3[1], mul(rv, rv));
    v3[2] = add(v3[2], mul(rv, z));
  }
  if (!rank_allreduce<3>(me, A.nranks, rank, lb, Gr, inst++, v3, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
  {
    bnorm = sqrt(v3[0]);
    const double target = fmax(A.rel_tol * bnorm, A.abs_tol);
    double rnorm = sqrt(v3[1]);
    rz = jac ? v3[2] : v3[1];
    auto relf = [&](double res) { return bnorm > 0.0 ? res / bnorm : (res == 0.0 ? 0.0 : INFINITY); };
    if (rnorm <= target) { converged = 1; rel = relf(rnorm); goto done; }
    double beta = 0.0, alpha_prev = 0.0;
    bool first = true;
    for (int it = 1; it <= A.max_iter; ++it) {
      // ---- K1 ----
      double v1[1] = {0.0};
      for (int64_t w = w0; w < L.words; w += wstride) {
        if (!((mask[w] >> lane) & 1u)) continue;
        const int64_t e = w * 32 + lane;
        auto pn = [&](int64_t q) {
          const double rq = r[q];
          const double z = jac ? mul(inv, rq) : rq;
          return first ? z : add(z, mul(beta, pold[q]));
        };
        const double pe = pn(e);
        const double av = stencil_row(comp_of_f(e, L.C), e, L, dg, of, pn);
        if (!first) x[e] = add(x[e], mul(alpha_prev, pold[e]));
        pnew[e] = pe;
        push_ghost(me, e, pe, lo_pnew, hi_pnew);
        ap[e] = av;
        v1[0] = add(v1[0], mul(pe, av));
      }
      ++applies;
      if (!rank_allreduce<1>(me, A.nranks, rank, lb, Gr, inst++, v1, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
      const double pap = v1[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; goto done; }
      alpha = rz / pap;
      // ---- K2 ----
      double v2[2] = {0.0, 0.0};
      for (int64_t w = w0; w < L.words; w += wstride) {
        if (!((mask[w] >> lane) & 1u)) continue;
        const int64_t e = w * 32 + lane;
        const double rv = sub(r[e], mul(alpha, ap[e]));
        r[e] = rv;
        push_ghost(me, e, rv, me.lo_r, me.hi_r);
        const double z = jac ? mul(inv, rv) : rv;
        v2[0] = add(v2[0], mul(rv, rv));
        v2[1] = add(v2[1], mul(rv, z));
      }
      if (!rank_allreduce<2>(me, A.nranks, rank, lb, Gr, inst++, v2, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
      rnorm = sqrt(v2[0]);
      iters = it;
      rel = relf(rnorm);
      const double rz_new = jac ? v2[1] : v2[0];
      if (rnorm <= target) { converged = 1; break; }
      if (!isfinite(rz_new)) { status = MQ_INDEFINITE; break; }
      beta = rz_new / rz;
      rz = rz_new;
      alpha_prev = alpha;
      first = false;
      double *t = pold; pold = pnew; pnew = t;
      t = lo_pold; lo_pold = lo_pnew; lo_pnew = t;
      t = hi_pold; hi_pold = hi_pnew; hi_pnew = t;
    }
    if (status == MQ_OK) {
      double *pdir = converged ? pnew : pold;
      for (int64_t w = w0; w < L.words; w += wstride) {
        if (!((mask[w] >> lane) & 1u)) continue;
        const int64_t e = w * 32 + lane;
        x[e] = add(x[e], mul(alpha, pdir[e]));
      }
      if (!converged) status = MQ_NOT_CONVERGED;
    }
  }
done:
  // every group leaves with the same instance count (identical control flow)
  if (lb == 0 && threadIdx.x == 0) {
    *me.epoch = inst;
    PcgOut o;
    o.iterations = iters;
    o.converged = converged;
    o.status = status;
    o.applies = applies;
    o.rel = rel;
    o.bnorm = bnorm;
    o.alpha = alpha;
    o.rz = rz;
    *me.out = o;
  }
}

int launch_pcg_tma_slab(const StencilPcgArgs *args, const SlabRank *ranks, const int *nplanes, int ngroups,
                        int nranks, int rank0, int ny, int nz, cudaStream_t s);

// MQ_SLAB_KERNEL=simple selects the thread-per-row kernel above; default: the
// TMA brick kernel (pcg_brick.cu: pcg_tma_slab_kernel)
static bool slab_use_tma() {
  const char *v = getenv("MQ_SLAB_KERNEL");
  return !(v && std::string(v) == "simple");
}

static int fused_ready(mq_ctx *ctx) {
  if (ctx->d_mbox) return MQ_OK;
  int rc = ctx_alloc(ctx, (void **)&ctx->d_mbox, sizeof(double) * kRing * kMaxRanks * kMbW);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_mcount, sizeof(unsigned long long) * 2);
  if (rc) return rc;
  MQ_CUDA(cudaMemsetAsync(ctx->d_mcount, 0, sizeof(unsigned long long) * 2, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

static int finish_report(mq_ctx *c0, mq_solve_report *rep) {
  const PcgOut &o = *c0->h_out;
  if (rep) {
    rep->iterations = o.iterations;
    rep->converged = o.converged;
    rep->final_rel_residual = o.rel;
    rep->applies = o.applies;
  }
  if (o.status == MQ_INDEFINITE) { set_error("nonpositive curvature or non-finite preconditioned residual"); return MQ_INDEFINITE; }
  if (o.status == MQ_CUDA_ERROR) { set_error("rank all-reduce or group barrier watchdog expired"); return MQ_CUDA_ERROR; }
  return o.status;
}

static void fill_rank(SlabRank &s, mq_ctx *ctx, const double *b, double *x) {
  s.L = ctx->topo.L;
  s.mask = ctx->d_mask;
  s.b = b;
  s.x = x;
  s.r = ctx->d_r;
  s.pa = ctx->d_p0;
  s.pb = ctx->d_p1;
  s.ap = ctx->d_ap;
  s.n = ctx->topo.nx;
  s.partials = ctx->d_partials;
  s.bar = ctx->d_bar;
  s.out = ctx->d_out;
  s.epoch = ctx->d_mcount + 1;
}

// the one-barrier TMA slab kernel's double buffers (r of odd, Ap of both
// iteration parities), allocated with the slab context
static bool has_one_barrier_buffers(const mq_ctx *ctx) { return ctx->d_r2 && ctx->d_ap && ctx->d_ap2; }

// ---- one rank per process: IPC-mapped neighbour buffers ------------------
constexpr int kIpcBufs = 9;  // r, pa, pb, x, mailbox, counter, r2, ap, ap2

struct SlabPeer {
  SlabRank rk{};
  int rank = 0, nranks = 1;
  double *x = nullptr;
  std::vector<void *> opened;  // IPC mappings to close
};

void slab_peer_free(mq_ctx *ctx) {
  if (!ctx->peer) return;
  for (void *p : ctx->peer->opened) cudaIpcCloseMemHandle(p);
  delete ctx->peer;
  ctx->peer = nullptr;
}

}  // namespace mq

using namespace mq;

extern "C" {

// All ranks' slabs in this process on one GPU, run as the groups of one
// cooperative launch (the single-GPU emulation of the multi-GPU kernel).
int mq_slab_fused_solve_local(mq_ctx **ctxs, int32_t nranks, const double *const *b, double *const *x,
                              int32_t x0_given, double rel_tol, double abs_tol, int32_t max_iter, int32_t use_jacobi,
                              mq_solve_report *rep) {
  if (!ctxs || nranks < 1 || nranks > kMaxRanks) { set_error("1..8 slab contexts required"); return MQ_INVALID; }
  if (!(rel_tol >= 0.0) || !(abs_tol >= 0.0) || max_iter < 0) { set_error("invalid PCG configuration"); return MQ_INVALID; }
  mq_ctx *c0 = ctxs[0];
  for (int q = 0; q < nranks; ++q) {
    if (ctxs[q]->device != c0->device) { set_error("local fused slabs must share one device"); return MQ_INVALID; }
    int rc = fused_ready(ctxs[q]);
    if (rc) return rc;
  }
  SlabFusedArgs A{};
  A.ngroups = nranks;
  A.nranks = nranks;
  A.rank0 = 0;
  A.dg = c0->kn_diag;
  A.of = c0->kn_off;
  A.inv = c0->jac_inv;
  A.use_jac = use_jacobi ? 1 : 0;
  A.x0_mode = x0_given ? 1 : 2;
  A.max_iter = max_iter;
  A.rel_tol = rel_tol;
  A.abs_tol = abs_tol;
  for (int q = 0; q < nranks; ++q) {
    SlabRank &s = A.rk[q];
    fill_rank(s, ctxs[q], b[q], x[q]);
    for (int p = 0; p < nranks; ++p) {
      s.mbox[p] = ctxs[p]->d_mbox;
      s.mcount[p] = ctxs[p]->d_mcount;
    }
    if (q > 0) {
      mq_ctx *lo = ctxs[q - 1];
      s.lo_x = x[q - 1];
      s.lo_r = lo->d_r;
      s.lo_pa = lo->d_p0;
      s.lo_pb = lo->d_p1;
      s.lo_r2 = lo->d_r2;
      s.lo_a = lo->d_ap;
      s.lo_a2 = lo->d_ap2;
      s.lo_C = lo->topo.L.C;
      s.lo_top = (int64_t)(lo->topo.nx + 1) * lo->topo.L.Si;
    }
    if (q + 1 < nranks) {
      mq_ctx *hi = ctxs[q + 1];
      s.hi_x = x[q + 1];
      s.hi_r = hi->d_r;
      s.hi_pa = hi->d_p0;
      s.hi_pb = hi->d_p1;
      s.hi_r2 = hi->d_r2;
      s.hi_a = hi->d_ap;
      s.hi_a2 = hi->d_ap2;
      s.hi_C = hi->topo.L.C;
    }
  }
  // every rank's epoch must agree (they only ever run together)
  cudaStream_t st = c0->stream;
  // the launch runs on rank 0's stream: the other ranks' streams may still
  // hold work writing this solve's inputs (b, x0 -- the sharded step queues
  // K_cn^T a_c and the start vector there), so they are drained first
  for (int q = 1; q < nranks; ++q) MQ_CUDA(cudaStreamSynchronize(ctxs[q]->stream));
  if (slab_use_tma()) {
    StencilPcgArgs sa[kMaxRanks];
    int np[kMaxRanks];
    for (int q = 0; q < nranks; ++q) {
      StencilPcgArgs &t = sa[q];
      t = StencilPcgArgs{};
      mq_ctx *c = ctxs[q];
      t.L = c->topo.L;
      t.mask = c->d_mask;
      t.dg = A.dg;
      t.of = A.of;
      t.inv = A.inv;
      t.use_jac = A.use_jac;
      t.x0_mode = A.x0_mode;
      t.b = b[q];
      t.x = x[q];
      t.r = c->d_r;
      t.pa = c->d_p0;
      t.pb = c->d_p1;
      t.ap = c->d_ap;
      t.ap2 = c->d_ap2;
      t.r2 = c->d_r2;
      t.rel_tol = rel_tol;
      t.stress_ns = pcg_stress_ns();
      t.abs_tol = abs_tol;
      t.max_iter = max_iter;
      t.partials = c->d_partials;
      t.bar = c->d_bar;
      t.out = c->d_out;
      np[q] = c->topo.nx;
    }
    int rc = launch_pcg_tma_slab(sa, A.rk, np, nranks, nranks, 0, c0->topo.ny, c0->topo.nz, st);
    if (rc) return rc;
    c0->launches += 1;
    cudaError_t e = cudaMemcpyAsync(c0->h_out, ctxs[0]->d_out, sizeof(PcgOut), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "fused slab PCG");
    return finish_report(c0, rep);
  }
  for (int q = 0; q < nranks; ++q) MQ_CUDA(cudaMemsetAsync(&ctxs[q]->d_bar->count, 0, sizeof(unsigned long long), st));
  SlabFusedArgs *dA = nullptr;
  MQ_CUDA(cudaMalloc(&dA, sizeof(SlabFusedArgs)));
  cudaError_t e = cudaMemcpyAsync(dA, &A, sizeof(A), cudaMemcpyHostToDevice, st);
  int per = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, slab_pcg_fused_kernel, kBlock, 0);
  int rc = MQ_OK;
  if (e == cudaSuccess && per < 1) { set_error("fused slab kernel cannot be resident"); rc = MQ_CUDA_ERROR; }
  if (e == cudaSuccess && rc == MQ_OK) {
    const int cap = c0->sms * std::min(per, 2);
    const int Gr = std::max(1, cap / nranks);
    void *params[] = {&dA};
    e = cudaLaunchCooperativeKernel((const void *)slab_pcg_fused_kernel, dim3(Gr * nranks), dim3(kBlock), params, 0,
                                    st);
    c0->launches += 1;
  }
  if (e == cudaSuccess && rc == MQ_OK) e = cudaMemcpyAsync(c0->h_out, ctxs[0]->d_out, sizeof(PcgOut), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(dA);
  if (e != cudaSuccess) return cuda_fail(e, "fused slab PCG");
  if (rc) return rc;
  return finish_report(c0, rep);
}


// Handles of this rank's r, p_a, p_b, x (x_dev), mailbox and counter,
// kIpcBufs x sizeof(cudaIpcMemHandle_t) bytes, to be exchanged between the
// ranks (torch.distributed all_gather on the host).
int mq_slab_ipc_export(mq_ctx *ctx, const double *x_dev, void *handles_out) {
  int rc = fused_ready(ctx);
  if (rc) return rc;
  if (!has_one_barrier_buffers(ctx)) { set_error("slab context without the one-barrier buffers"); return MQ_INVALID; }
  const void *bufs[kIpcBufs] = {ctx->d_r, ctx->d_p0, ctx->d_p1, x_dev, ctx->d_mbox, ctx->d_mcount,
                                ctx->d_r2, ctx->d_ap, ctx->d_ap2};
  cudaIpcMemHandle_t *h = reinterpret_cast<cudaIpcMemHandle_t *>(handles_out);
  for (int q = 0; q < kIpcBufs; ++q) MQ_CUDA(cudaIpcGetMemHandle(&h[q], const_cast<void *>(bufs[q])));
  return MQ_OK;
}

// all_handles: nranks x kIpcBufs handles in rank order; nplanes: owned
// planes per rank.  Maps the neighbours' r/p/x and every rank's mailbox and
// counter into this process (NVLink peer access), and remembers x_dev as the
// solution buffer of mq_slab_fused_solve_peer.
int mq_slab_ipc_import(mq_ctx *ctx, int32_t rank, int32_t nranks, const void *all_handles, const int32_t *nplanes,
                       double *x_dev) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) { set_error("invalid rank layout"); return MQ_INVALID; }
  int rc = fused_ready(ctx);
  if (rc) return rc;
  slab_peer_free(ctx);
  SlabPeer *P = new SlabPeer;
  P->rank = rank;
  P->nranks = nranks;
  P->x = x_dev;
  const cudaIpcMemHandle_t *h = reinterpret_cast<const cudaIpcMemHandle_t *>(all_handles);
  auto open = [&](int q, int k, void **out) -> int {
    if (q == rank) {
      void *own[kIpcBufs] = {ctx->d_r, ctx->d_p0, ctx->d_p1, x_dev, ctx->d_mbox, ctx->d_mcount,
                             ctx->d_r2, ctx->d_ap, ctx->d_ap2};
      *out = own[k];
      return MQ_OK;
    }
    cudaError_t e = cudaIpcOpenMemHandle(out, h[q * kIpcBufs + k], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    P->opened.push_back(*out);
    return MQ_OK;
  };
  SlabRank &s = P->rk;
  const Lay &L = ctx->topo.L;
  auto comp_stride = [&](int n) { return ((int64_t)(n + 2) * L.Si + 31) / 32 * 32; };
  for (int q = 0; q < nranks && rc == MQ_OK; ++q) {
    void *mb = nullptr, *mc = nullptr;
    rc = open(q, 4, &mb);
    rc = rc ? rc : open(q, 5, &mc);
    s.mbox[q] = (double *)mb;
    s.mcount[q] = (unsigned long long *)mc;
  }
  // neighbour buffers: r, pa, pb, x and the one-barrier r2, ap, ap2
  const int nb[7] = {0, 1, 2, 3, 6, 7, 8};
  if (rc == MQ_OK && rank > 0) {
    void *v[7];
    for (int k = 0; k < 7 && rc == MQ_OK; ++k) rc = open(rank - 1, nb[k], &v[k]);
    s.lo_r = (double *)v[0];
    s.lo_pa = (double *)v[1];
    s.lo_pb = (double *)v[2];
    s.lo_x = (double *)v[3];
    s.lo_r2 = (double *)v[4];
    s.lo_a = (double *)v[5];
    s.lo_a2 = (double *)v[6];
    s.lo_C = comp_stride(nplanes[rank - 1]);
    s.lo_top = (int64_t)(nplanes[rank - 1] + 1) * L.Si;
  }
  if (rc == MQ_OK && rank + 1 < nranks) {
    void *v[7];
    for (int k = 0; k < 7 && rc == MQ_OK; ++k) rc = open(rank + 1, nb[k], &v[k]);
    s.hi_r = (double *)v[0];
    s.hi_pa = (double *)v[1];
    s.hi_pb = (double *)v[2];
    s.hi_x = (double *)v[3];
    s.hi_r2 = (double *)v[4];
    s.hi_a = (double *)v[5];
    s.hi_a2 = (double *)v[6];
    s.hi_C = comp_stride(nplanes[rank + 1]);
  }
  ctx->peer = P;
  if (rc) { slab_peer_free(ctx); return rc; }
  return MQ_OK;
}

// This rank's part of the distributed solve (one CTA group on this GPU); all
// ranks call it with the same arguments.  b: this slab's right-hand side.
int mq_slab_fused_solve_peer(mq_ctx *ctx, const double *b, int32_t x0_given, double rel_tol, double abs_tol,
                             int32_t max_iter, int32_t use_jacobi, mq_solve_report *rep) {
  SlabPeer *P = ctx->peer;
  if (!P) { set_error("mq_slab_ipc_import first"); return MQ_INVALID; }
  if (!(rel_tol >= 0.0) || !(abs_tol >= 0.0) || max_iter < 0) { set_error("invalid PCG configuration"); return MQ_INVALID; }
  SlabRank rk = P->rk;
  fill_rank(rk, ctx, b, P->x);
  StencilPcgArgs t{};
  t.L = ctx->topo.L;
  t.mask = ctx->d_mask;
  t.dg = ctx->kn_diag;
  t.of = ctx->kn_off;
  t.inv = ctx->jac_inv;
  t.use_jac = use_jacobi ? 1 : 0;
  t.x0_mode = x0_given ? 1 : 2;
  t.b = b;
  t.x = P->x;
  t.r = ctx->d_r;
  t.pa = ctx->d_p0;
  t.pb = ctx->d_p1;
  t.ap = ctx->d_ap;
  t.ap2 = ctx->d_ap2;
  t.r2 = ctx->d_r2;
  t.rel_tol = rel_tol;
  t.stress_ns = pcg_stress_ns();
  t.abs_tol = abs_tol;
  t.max_iter = max_iter;
  t.partials = ctx->d_partials;
  t.bar = ctx->d_bar;
  t.out = ctx->d_out;
  const int np = ctx->topo.nx;
  int rc = launch_pcg_tma_slab(&t, &rk, &np, 1, P->nranks, P->rank, ctx->topo.ny, ctx->topo.nz, ctx->stream);
  if (rc) return rc;
  ctx->launches += 1;
  MQ_CUDA(cudaMemcpyAsync(ctx->h_out, ctx->d_out, sizeof(PcgOut), cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return finish_report(ctx, rep);
}

}  // extern "C"

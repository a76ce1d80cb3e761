// Member-batched PCG (BASELINE configs[3]): one persistent
// launch advances B independent right-hand sides of the same K_n (the
// ensemble members share K_n; only J and kappa differ), with the vectors
// interleaved [padded entry][member] so that every stencil neighbour load
// brings the B members' values in one contiguous 8·B-byte run and the mask
// and index work is done once per entry.  krylov.py:174-250 per member:
// per-member alpha / beta / stopping test, a member that has converged is
// frozen (its final x update is the deferred one of the next K1 pass), the
// launch ends when every member is done or the budget is spent.
//
// Same per-row arithmetic as pcg_stencil_kernel (pcg.cu): thread per (entry,
// member) slot, p_new formed on the fly at the 12 neighbours, two passes and
// two grid reductions per iteration.  Kept as the measured alternative to
// running the members one after another with the shared-memory-resident
// kernel: the batch's vectors cannot stay in shared memory.
#include <algorithm>
#include <vector>

#include "mq_ctx.h"
#include "mq_device.cuh"

namespace mq {

constexpr int kMaxBatch = 8;

struct BatchedArgs {
  Lay L;
  const uint32_t *mask;
  double dg, of, inv;
  int use_jac, x0_given, max_iter;
  double rel_tol, abs_tol;
  const double *b;  // [L.total][B]
  double *x, *r, *pa, *pb, *ap;
  double *partials;  // 3*B*G
  GridBar *bar;
  PcgOut *out;       // B records
};

__device__ __forceinline__ int comp_of_b(int64_t e, int64_t C) { return e < C ? 0 : (e < 2 * C ? 1 : 2); }

// block sums of NQ values per member; thread (q*B + m) of the block writes
// partials[(q*B + m)*G + block]
template <int B, int NQ>
__device__ __forceinline__ void member_block_partials(double (&v)[NQ], double *red, double *partials) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int o = 16; o >= B; o >>= 1) v[q] = add(v[q], __shfl_xor_sync(0xffffffffu, v[q], o));
  if (lane < B)
#pragma unroll
    for (int q = 0; q < NQ; ++q) red[(q * kWarps + warp) * B + lane] = v[q];
  __syncthreads();
  if (threadIdx.x < NQ * B) {
    const int q = threadIdx.x / B, m = threadIdx.x % B;
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s = add(s, red[(q * kWarps + w) * B + m]);
    partials[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
  }
  __syncthreads();
}

template <int B>
__device__ __forceinline__ double pick(const double (&arr)[B], int m) {
  double v = arr[0];
#pragma unroll
  for (int q = 1; q < B; ++q)
    if (q == m) v = arr[q];
  return v;
}

template <int B>
__device__ __forceinline__ int pick_int(const int (&arr)[B], int m) {
  int v = arr[0];
#pragma unroll
  for (int q = 1; q < B; ++q)
    if (q == m) v = arr[q];
  return v;
}

template <int B>
__global__ void __launch_bounds__(kBlock, 3) pcg_batched_kernel(BatchedArgs a) {
  __shared__ double red[3 * kWarps * kMaxBatch];
  __shared__ double tot[3 * kMaxBatch];
  const int G = gridDim.x;
  const int mb = threadIdx.x % B;  // this thread's member (the slot stride is a multiple of B)
  const Lay L = a.L;
  const uint32_t *__restrict__ mask = a.mask;
  const double dg = a.dg, of = a.of, inv = a.inv;
  const bool jac = a.use_jac != 0;
  double *x = a.x, *r = a.r, *ap = a.ap;
  const int64_t nslot = L.total * B;
  const int64_t s0 = (int64_t)blockIdx.x * kBlock + threadIdx.x, sstride = (int64_t)G * kBlock;
  // per-member state, identical in every thread of every CTA
  double bnorm[B], target[B], rz[B], alpha[B], beta[B], alpha_prev[B], rel[B];
  int state[B], iters[B], status[B];  // state 0 active, 1 done (final x update pending), 2 finished
  // ---- initial residual ----
  {
    double v[3] = {0.0, 0.0, 0.0};
    for (int64_t s = s0; s < nslot; s += sstride) {
      const int64_t e = s / B;
      if (!active(mask, e)) continue;
      const double bv = a.b[s];
      double rv = bv;
      if (a.x0_given) {
        const double axv = stencil_row(comp_of_b(e, L.C), e, L, dg, of, [&](int64_t q) { return x[q * B + mb]; });
        rv = sub(bv, axv);
      } else {
        x[s] = 0.0;
      }
      r[s] = rv;
      const double z = jac ? mul(inv, rv) : rv;
      v[0] = add(v[0], mul(bv, bv));
      v[1] = add(v[1], mul(rv, rv));
      v[2] = add(v[2], mul(rv, z));
    }
    member_block_partials<B, 3>(v, red, a.partials);
  }
  bool ok = grid_sync(a.bar);
  {
    double s3[3 * B];
    grid_partials_sum<3 * B>(a.partials, G, s3, tot);
#pragma unroll
    for (int m = 0; m < B; ++m) {
      bnorm[m] = sqrt(s3[0 * B + m]);
      target[m] = fmax(a.rel_tol * bnorm[m], a.abs_tol);
      const double rn = sqrt(s3[1 * B + m]);
      rz[m] = jac ? s3[2 * B + m] : s3[1 * B + m];
      rel[m] = bnorm[m] > 0.0 ? rn / bnorm[m] : (rn == 0.0 ? 0.0 : INFINITY);
      state[m] = rn <= target[m] ? 2 : 0;  // converged at the start: nothing to add to x
      iters[m] = 0;
      status[m] = MQ_OK;
      alpha[m] = beta[m] = alpha_prev[m] = 0.0;
    }
  }
  double *pold = a.pa, *pnew = a.pb;
  int it = 0;
  for (; ok && it < a.max_iter; ++it) {
    bool any = false;
#pragma unroll
    for (int m = 0; m < B; ++m) any |= state[m] == 0;
    if (!any) break;
    const int my_state = pick_int<B>(state, mb);
    const double my_beta = pick<B>(beta, mb), my_ap = pick<B>(alpha_prev, mb);
    const bool first = it == 0;
    // ---- K1 ----
    double v1[1] = {0.0};
    for (int64_t s = s0; s < nslot; s += sstride) {
      const int64_t e = s / B;
      if (my_state == 2 || !active(mask, e)) continue;
      if (my_state == 1) {  // converged last iteration: the final x += alpha p
        x[s] = add(x[s], mul(my_ap, pold[s]));
        continue;
      }
      auto pn = [&](int64_t q) {
        const double rq = r[q * B + mb];
        const double z = jac ? mul(inv, rq) : rq;
        return first ? z : add(z, mul(my_beta, pold[q * B + mb]));
      };
      const double pe = pn(e);
      const double av = stencil_row(comp_of_b(e, L.C), e, L, dg, of, pn);
      if (!first) x[s] = add(x[s], mul(my_ap, pold[s]));
      pnew[s] = pe;
      ap[s] = av;
      v1[0] = add(v1[0], mul(pe, av));
    }
    member_block_partials<B, 1>(v1, red, a.partials + 3 * B * (int64_t)G);
#pragma unroll
    for (int m = 0; m < B; ++m)
      if (state[m] == 1) state[m] = 2;
    ok = grid_sync(a.bar);
    if (!ok) break;
    double s1[B];
    grid_partials_sum<B>(a.partials + 3 * B * (int64_t)G, G, s1, tot);
#pragma unroll
    for (int m = 0; m < B; ++m) {
      if (state[m] != 0) continue;
      const double pap = s1[m];
      if (!isfinite(pap) || pap <= 0.0) {
        status[m] = MQ_INDEFINITE;
        iters[m] = it + 1;
        state[m] = 2;
        continue;
      }
      alpha[m] = rz[m] / pap;
    }
    const int st2 = pick_int<B>(state, mb);
    const double my_alpha = pick<B>(alpha, mb);
    // ---- K2 ----
    double v2[2] = {0.0, 0.0};
    for (int64_t s = s0; s < nslot; s += sstride) {
      const int64_t e = s / B;
      if (st2 != 0 || !active(mask, e)) continue;
      const double rv = sub(r[s], mul(my_alpha, ap[s]));
      r[s] = rv;
      const double z = jac ? mul(inv, rv) : rv;
      v2[0] = add(v2[0], mul(rv, rv));
      v2[1] = add(v2[1], mul(rv, z));
    }
    member_block_partials<B, 2>(v2, red, a.partials + 4 * B * (int64_t)G);
    ok = grid_sync(a.bar);
    if (!ok) break;
    double s2[2 * B];
    grid_partials_sum<2 * B>(a.partials + 4 * B * (int64_t)G, G, s2, tot);
#pragma unroll
    for (int m = 0; m < B; ++m) {
      if (state[m] != 0) continue;
      const double rn = sqrt(s2[m]);
      iters[m] = it + 1;
      rel[m] = bnorm[m] > 0.0 ? rn / bnorm[m] : (rn == 0.0 ? 0.0 : INFINITY);
      const double rz_new = jac ? s2[B + m] : s2[m];
      alpha_prev[m] = alpha[m];
      if (rn <= target[m]) { state[m] = 1; continue; }   // final update in the next K1
      if (!isfinite(rz_new)) { status[m] = MQ_INDEFINITE; state[m] = 2; continue; }
      beta[m] = rz_new / rz[m];
      rz[m] = rz_new;
    }
    double *t = pold; pold = pnew; pnew = t;
  }
  // members still pending a final update (converged in the last iteration
  // or out of budget): x += alpha p with their last direction (now pold)
  if (ok) {
    bool any = false;
#pragma unroll
    for (int m = 0; m < B; ++m) {
      if (state[m] == 0) { status[m] = MQ_NOT_CONVERGED; state[m] = 1; }
      any |= state[m] == 1;
    }
    if (any) {
      const int my_state = pick_int<B>(state, mb);
      const double my_ap = pick<B>(alpha_prev, mb);
      for (int64_t s = s0; s < nslot; s += sstride)
        if (my_state == 1 && active(mask, s / B)) x[s] = add(x[s], mul(my_ap, pold[s]));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
#pragma unroll
    for (int m = 0; m < B; ++m) {
      PcgOut o{};
      o.iterations = iters[m];
      o.converged = (ok && status[m] == MQ_OK) ? 1 : 0;
      o.status = ok ? status[m] : MQ_CUDA_ERROR;
      o.applies = iters[m] + (a.x0_given ? 1 : 0);
      o.rel = rel[m];
      o.bnorm = bnorm[m];
      a.out[m] = o;
    }
  }
}

template <int B>
static int launch_batched(const BatchedArgs &args, cudaStream_t s, int *grid_out) {
  int grid = 0;
  int rc = coop_grid((const void *)pcg_batched_kernel<B>, 0, &grid);
  if (rc) return rc;
  MQ_CUDA(cudaMemsetAsync(&args.bar->count, 0, sizeof(unsigned long long), s));
  BatchedArgs a = args;
  void *params[] = {&a};
  MQ_CUDA(cudaLaunchCooperativeKernel((const void *)pcg_batched_kernel<B>, dim3(grid), dim3(kBlock), params, 0, s));
  *grid_out = grid;
  return MQ_OK;
}

__global__ void k_interleave(int64_t n, int nb, const int32_t *__restrict__ pad, const double *__restrict__ src,
                             double *__restrict__ dst) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * nb; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = q / n, i = q % n;
    dst[(int64_t)pad[i] * nb + m] = src[q];
  }
}

__global__ void k_deinterleave(int64_t n, int nb, const int32_t *__restrict__ pad, const double *__restrict__ src,
                               double *__restrict__ dst) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * nb; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = q / n, i = q % n;
    dst[q] = src[(int64_t)pad[i] * nb + m];
  }
}

}  // namespace mq

using namespace mq;

extern "C" int mq_pcg_solve_batched_host(mq_ctx *ctx, int32_t nb, const double *b, const double *x0, double *x,
                                         double rel_tol, double abs_tol, int32_t max_iter, int32_t use_jacobi,
                                         mq_solve_report *reports, double *kernel_ms) {
  if (!ctx || !b || !x || !reports) { set_error("NULL argument"); return MQ_INVALID; }
  if (nb != 1 && nb != 2 && nb != 4 && nb != 8) { set_error("batch size must be 1, 2, 4 or 8"); return MQ_INVALID; }
  if (ctx->slab_hi > ctx->slab_lo) { set_error("batched PCG runs on a whole-grid context"); return MQ_INVALID; }
  if (!(rel_tol >= 0.0) || !(abs_tol >= 0.0) || max_iter < 0) { set_error("invalid PCG configuration"); return MQ_INVALID; }
  MQ_CUDA(cudaSetDevice(ctx->device));
  const Lay &L = ctx->topo.L;
  const int64_t n = (int64_t)ctx->topo.nc_pad.size();
  const size_t vb = sizeof(double) * (size_t)L.total * nb;
  std::vector<void *> mem;
  auto alloc = [&](size_t bytes) -> double * {
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    mem.push_back(p);
    cudaMemsetAsync(p, 0, bytes, ctx->stream);
    return static_cast<double *>(p);
  };
  double *db = alloc(vb), *dx = alloc(vb), *dr = alloc(vb), *dpa = alloc(vb), *dpb = alloc(vb), *dap = alloc(vb);
  double *dstage = alloc(sizeof(double) * n * nb);
  double *dpart = alloc(sizeof(double) * 5 * kMaxBatch * 3 * 148 * 8);
  PcgOut *dout = reinterpret_cast<PcgOut *>(alloc(sizeof(PcgOut) * kMaxBatch));
  GridBar *dbar = reinterpret_cast<GridBar *>(alloc(sizeof(GridBar)));
  int rc = MQ_OK;
  if (!db || !dx || !dr || !dpa || !dpb || !dap || !dstage || !dpart || !dout || !dbar) {
    for (void *p : mem) cudaFree(p);
    set_error("out of device memory (batched PCG)");
    return MQ_CUDA_ERROR;
  }
  cudaStream_t s = ctx->stream;
  const int g = std::min<int64_t>((n * nb + 255) / 256, ctx->sms * 8);
  cudaMemcpyAsync(dstage, b, sizeof(double) * n * nb, cudaMemcpyHostToDevice, s);
  k_interleave<<<g, 256, 0, s>>>(n, nb, ctx->d_nc_pad, dstage, db);
  if (x0) {
    cudaMemcpyAsync(dstage, x0, sizeof(double) * n * nb, cudaMemcpyHostToDevice, s);
    k_interleave<<<g, 256, 0, s>>>(n, nb, ctx->d_nc_pad, dstage, dx);
  }
  BatchedArgs a{};
  a.L = L;
  a.mask = ctx->d_mask;
  a.dg = ctx->kn_diag;
  a.of = ctx->kn_off;
  a.inv = ctx->jac_inv;
  a.use_jac = use_jacobi ? 1 : 0;
  a.x0_given = x0 ? 1 : 0;
  a.max_iter = max_iter;
  a.rel_tol = rel_tol;
  a.abs_tol = abs_tol;
  a.b = db;
  a.x = dx;
  a.r = dr;
  a.pa = dpa;
  a.pb = dpb;
  a.ap = dap;
  a.partials = dpart;
  a.bar = dbar;
  a.out = dout;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  int grid = 0;
  switch (nb) {
    case 1: rc = launch_batched<1>(a, s, &grid); break;
    case 2: rc = launch_batched<2>(a, s, &grid); break;
    case 4: rc = launch_batched<4>(a, s, &grid); break;
    default: rc = launch_batched<8>(a, s, &grid); break;
  }
  cudaEventRecord(e1, s);
  if (!rc) {
    k_deinterleave<<<g, 256, 0, s>>>(n, nb, ctx->d_nc_pad, dx, dstage);
    cudaMemcpyAsync(x, dstage, sizeof(double) * n * nb, cudaMemcpyDeviceToHost, s);
    PcgOut h[kMaxBatch];
    cudaMemcpyAsync(h, dout, sizeof(PcgOut) * nb, cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "batched PCG");
    if (!rc) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (kernel_ms) *kernel_ms = ms;
      for (int m = 0; m < nb; ++m) {
        reports[m].iterations = h[m].iterations;
        reports[m].converged = h[m].converged;
        reports[m].final_rel_residual = h[m].rel;
        reports[m].applies = h[m].applies;
        if (h[m].status == MQ_INDEFINITE && !rc) { set_error("nonpositive curvature in a batched member"); rc = MQ_INDEFINITE; }
        if (h[m].status == MQ_CUDA_ERROR && !rc) { set_error("grid barrier watchdog expired"); rc = MQ_CUDA_ERROR; }
      }
      if (!rc)
        for (int m = 0; m < nb; ++m)
          if (!h[m].converged) rc = MQ_NOT_CONVERGED;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (void *p : mem) cudaFree(p);
  return rc;
}

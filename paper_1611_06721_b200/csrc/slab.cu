// Phase kernels of the i-slab distributed K_n PCG (BASELINE configs[4]).
//
// The algorithm is krylov.py:174-250 with the same arithmetic as the
// single-device kernels; the slab owns node planes [ilo, ihi) and reads the
// neighbours' boundary planes from its two ghost planes, which the host
// refreshes (halo exchange) before every stencil pass.  Each phase leaves this
// rank's deterministic partial sums in a small device array; the host sums
// them over the ranks (allreduce) and takes the scalar decisions exactly like
// the reference, so every rank follows the same control flow.
//   init:  r = b - A x0 (or b), partials [b.b, r.r, r.z]
//   k1:    p_new = M^-1 r + beta p_old (also at neighbours/ghosts),
//          Ap = K_n p_new, x += alpha_prev p_old, partial p.Ap
//   k2:    r -= alpha Ap, partials [r.r, r.z]
//   final: x += alpha p
#include <algorithm>

#include "mq_ctx.h"
#include "mq_device.cuh"

namespace mq {

// block partials + last-block fixed-order reduce into out[0..NV)
template <int NV>
__device__ __forceinline__ void slab_reduce(double (&v)[NV], double *partials, unsigned int *counter, double *out) {
  __shared__ double sm[NV * kWarps];
  __shared__ bool last;
  block_sum<NV>(v, sm);
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) partials[q * G + blockIdx.x] = v[q];
    __threadfence();
    last = atomicAdd(counter, 1u) == (unsigned)G - 1;
  }
  __syncthreads();
  if (last) {
    // strided share per thread, fixed-order warp and block sums
    __threadfence();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int b = threadIdx.x; b < G; b += blockDim.x) s = add(s, __ldcg(partials + q * G + b));
      s = warp_sum(s);
      if (lane == 0) sm[q * kWarps + warp] = s;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s = add(s, sm[threadIdx.x * kWarps + w]);
      out[threadIdx.x] = s;
    }
    if (threadIdx.x == 0) *counter = 0u;
  }
}

#define SLAB_ROWS(L, mask)                                                                     \
  for (int64_t w_ = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); w_ < (L).words;          \
       w_ += (int64_t)gridDim.x * kWarps)                                                     \
    if (((mask)[w_] >> (threadIdx.x & 31)) & 1u)

__device__ __forceinline__ int comp_of_s(int64_t e, int64_t C) { return e < C ? 0 : (e < 2 * C ? 1 : 2); }

__global__ void __launch_bounds__(kBlock) k_slab_init(Lay L, const uint32_t *__restrict__ mask, double dg, double of,
                                                      double inv, int jac, int x0_mode, const double *__restrict__ b,
                                                      double *x, double *r, double *partials, unsigned int *counter,
                                                      double *out) {
  double v[3] = {0.0, 0.0, 0.0};
  SLAB_ROWS(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    const double bv = b[e];
    double rv = bv;
    if (x0_mode == 1) rv = sub(bv, stencil_row(comp_of_s(e, L.C), e, L, dg, of, [&](int64_t q) { return x[q]; }));
    r[e] = rv;
    const double z = jac ? mul(inv, rv) : rv;
    v[0] = add(v[0], mul(bv, bv));
    v[1] = add(v[1], mul(rv, rv));
    v[2] = add(v[2], mul(rv, z));
  }
  slab_reduce<3>(v, partials, counter, out);
}

__global__ void __launch_bounds__(kBlock) k_slab_zero_x(Lay L, const uint32_t *__restrict__ mask, double *x) {
  SLAB_ROWS(L, mask) { x[w_ * 32 + (threadIdx.x & 31)] = 0.0; }
}

__global__ void __launch_bounds__(kBlock) k_slab_k1(Lay L, const uint32_t *__restrict__ mask, double dg, double of,
                                                    double inv, int jac, int first, double beta, double alpha_prev,
                                                    const double *__restrict__ r, const double *__restrict__ pold,
                                                    double *__restrict__ pnew, double *__restrict__ ap, double *x,
                                                    double *partials, unsigned int *counter, double *out) {
  double v[1] = {0.0};
  SLAB_ROWS(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    auto pn = [&](int64_t q) {
      const double rq = r[q];
      const double z = jac ? mul(inv, rq) : rq;
      return first ? z : add(z, mul(beta, pold[q]));
    };
    const double pe = pn(e);
    const double av = stencil_row(comp_of_s(e, L.C), e, L, dg, of, pn);
    if (!first) x[e] = add(x[e], mul(alpha_prev, pold[e]));
    pnew[e] = pe;
    ap[e] = av;
    v[0] = add(v[0], mul(pe, av));
  }
  slab_reduce<1>(v, partials, counter, out);
}

__global__ void __launch_bounds__(kBlock) k_slab_k2(Lay L, const uint32_t *__restrict__ mask, double inv, int jac,
                                                    double alpha, double *r, const double *__restrict__ ap,
                                                    double *partials, unsigned int *counter, double *out) {
  double v[2] = {0.0, 0.0};
  SLAB_ROWS(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    const double rv = sub(r[e], mul(alpha, ap[e]));
    r[e] = rv;
    const double z = jac ? mul(inv, rv) : rv;
    v[0] = add(v[0], mul(rv, rv));
    v[1] = add(v[1], mul(rv, z));
  }
  slab_reduce<2>(v, partials, counter, out);
}

__global__ void __launch_bounds__(kBlock) k_slab_final(Lay L, const uint32_t *__restrict__ mask, double alpha,
                                                       const double *__restrict__ p, double *x) {
  SLAB_ROWS(L, mask) {
    const int64_t e = w_ * 32 + (threadIdx.x & 31);
    x[e] = add(x[e], mul(alpha, p[e]));
  }
}

template <class T>
static int slab_upload(mq_ctx *ctx, T **dst, const std::vector<T> &src) {
  if (src.empty()) { *dst = nullptr; return MQ_OK; }
  int rc = ctx_alloc(ctx, (void **)dst, src.size() * sizeof(T));
  if (rc) return rc;
  MQ_CUDA(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return MQ_OK;
}

static int slab_grid(mq_ctx *ctx) {
  int64_t g = (ctx->topo.L.words + kWarps - 1) / kWarps;
  if (g > (int64_t)ctx->sms * 4) g = ctx->sms * 4;
  return (int)std::max<int64_t>(1, g);
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_ctx_create_slab(const mq_grid_desc *desc, int32_t i_lo, int32_t i_hi, int32_t device, mq_ctx **out) {
  if (!desc || !out) { set_error("NULL argument"); return MQ_INVALID; }
  *out = nullptr;
  mq_ctx *ctx = new mq_ctx();
  ctx->desc = *desc;
  ctx->material.assign(desc->material, desc->material + (size_t)desc->nx * desc->ny * desc->nz);
  ctx->desc.material = ctx->material.data();
  std::string err;
  int rc = build_slab_topology(ctx->desc, i_lo, i_hi, ctx->topo, err);
  if (rc) { set_error(err); delete ctx; return rc; }
  ctx->device = device;
  ctx->slab_lo = i_lo;
  ctx->slab_hi = i_hi;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaSetDevice"); }
  e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaStreamCreate"); }
  ctx->stream = ctx->own_stream;
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  const double w = 0.5 * desc->nu_air + 0.5 * desc->nu_air;
  const double c = w / desc->h;
  ctx->kn_off = desc->kn_off > 0.0 ? desc->kn_off : c;
  ctx->kn_diag = desc->kn_diag > 0.0 ? desc->kn_diag : (((c + c) + c) + c);
  ctx->jac_inv = 1.0 / ctx->kn_diag;
  const Topology &t = ctx->topo;
  rc = 0;
  rc = rc ? rc : slab_upload(ctx, &ctx->d_mask, t.mask);
  rc = rc ? rc : slab_upload(ctx, &ctx->d_nc_pad, t.nc_pad);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_stage, sizeof(double) * std::max<int64_t>(1, (int64_t)t.nc_pad.size()));
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_r, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_p0, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_p1, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_ap, sizeof(double) * t.L.total);
  // double buffers of the one-barrier fused slab kernel (pcg_tma1_slab_kernel)
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_ap2, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_r2, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_tmp0, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_tmp1, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_partials, sizeof(double) * 8 * 1024);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_bar, sizeof(GridBar));
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_out, sizeof(PcgOut));
  if (!rc) {
    e = cudaMallocHost((void **)&ctx->h_out, sizeof(PcgOut));
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMallocHost");
  }
  if (!rc) {
    e = cudaEventCreate(&ctx->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaEventCreate");
  }
  ctx->pcg_variant = 1;  // stencil kernels with explicit neighbour loads
  if (!rc) {
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "slab setup");
  }
  if (rc) { mq_ctx_destroy(ctx); return rc; }
  *out = ctx;
  return MQ_OK;
}

int mq_layout(const mq_ctx *ctx, int64_t *out6) {
  const Lay &L = ctx->topo.L;
  out6[0] = L.C;
  out6[1] = L.Si;
  out6[2] = L.Sj;
  out6[3] = L.off;
  out6[4] = L.total;
  out6[5] = ctx->topo.nx;
  return MQ_OK;
}

int mq_slab_buffers(mq_ctx *ctx, double **r, double **pa, double **pb, double **ap) {
  if (r) *r = ctx->d_r;
  if (pa) *pa = ctx->d_p0;
  if (pb) *pb = ctx->d_p1;
  if (ap) *ap = ctx->d_ap;
  return MQ_OK;
}

// partial sums of the last phase (host, nq values); synchronises the stream
static int read_partials(mq_ctx *ctx, double *host, int nq) {
  MQ_CUDA(cudaMemcpyAsync(host, ctx->d_partials + 7 * 1024, sizeof(double) * nq, cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

int mq_slab_init(mq_ctx *ctx, const double *b, double *x, int32_t x0_mode, int32_t use_jacobi, double *part3) {
  const Lay &L = ctx->topo.L;
  const int G = slab_grid(ctx);
  unsigned int *counter = reinterpret_cast<unsigned int *>(ctx->d_bar);
  if (x0_mode != 1) {
    k_slab_zero_x<<<G, kBlock, 0, ctx->stream>>>(L, ctx->d_mask, x);
    MQ_CUDA(cudaGetLastError());
  }
  k_slab_init<<<G, kBlock, 0, ctx->stream>>>(L, ctx->d_mask, ctx->kn_diag, ctx->kn_off, ctx->jac_inv, use_jacobi,
                                              x0_mode, b, x, ctx->d_r, ctx->d_partials, counter,
                                              ctx->d_partials + 7 * 1024);
  MQ_CUDA(cudaGetLastError());
  ctx->launches += 1 + (x0_mode != 1);
  return read_partials(ctx, part3, 3);
}

int mq_slab_k1(mq_ctx *ctx, double *x, int32_t first, double beta, double alpha_prev, int32_t pold_is_a,
               int32_t use_jacobi, double *part1) {
  const Lay &L = ctx->topo.L;
  const int G = slab_grid(ctx);
  unsigned int *counter = reinterpret_cast<unsigned int *>(ctx->d_bar);
  const double *pold = pold_is_a ? ctx->d_p0 : ctx->d_p1;
  double *pnew = pold_is_a ? ctx->d_p1 : ctx->d_p0;
  k_slab_k1<<<G, kBlock, 0, ctx->stream>>>(L, ctx->d_mask, ctx->kn_diag, ctx->kn_off, ctx->jac_inv, use_jacobi, first,
                                            beta, alpha_prev, ctx->d_r, pold, pnew, ctx->d_ap, x, ctx->d_partials,
                                            counter, ctx->d_partials + 7 * 1024);
  MQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  return read_partials(ctx, part1, 1);
}

int mq_slab_k2(mq_ctx *ctx, double alpha, int32_t use_jacobi, double *part2) {
  const Lay &L = ctx->topo.L;
  const int G = slab_grid(ctx);
  unsigned int *counter = reinterpret_cast<unsigned int *>(ctx->d_bar);
  k_slab_k2<<<G, kBlock, 0, ctx->stream>>>(L, ctx->d_mask, ctx->jac_inv, use_jacobi, alpha, ctx->d_r, ctx->d_ap,
                                            ctx->d_partials, counter, ctx->d_partials + 7 * 1024);
  MQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  return read_partials(ctx, part2, 2);
}

int mq_slab_final(mq_ctx *ctx, double *x, double alpha, int32_t p_is_a) {
  const Lay &L = ctx->topo.L;
  k_slab_final<<<slab_grid(ctx), kBlock, 0, ctx->stream>>>(L, ctx->d_mask, alpha, p_is_a ? ctx->d_p0 : ctx->d_p1, x);
  MQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

}  // extern "C"

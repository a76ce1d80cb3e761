// PCG kernels (krylov.py:174-250) for the K_n stencil and for a general CSR
// operator, plus K_n SpMV and layout gather/scatter.
//
// One persistent cooperative kernel runs a whole solve: the loop control
// (stopping rule, breakdown checks, iteration budget) lives on the device and
// the host sees only the final SolveReport.  Every CTA reduces its part of a
// dot product into partials[], and after a grid barrier every CTA sums the
// partials in the same fixed order, so all CTAs hold bitwise-identical
// scalars and take the same branch.
//
// Stencil path: two passes per iteration over the padded layout.
//   K1: p_new = M^-1 r + beta p_old (also at the 12 neighbours, on the fly),
//       Ap = K_n p_new, x += alpha_prev p_old (deferred), partial p.Ap
//   K2: r -= alpha Ap, partials r.r and r.M^-1 r
// K1 streams r, p_old, x in and x, p_new, Ap out; K2 streams r, Ap in and r
// out: 9 vector streams = 72 B per dof and iteration.
#include <cooperative_groups.h>

#include "mq_device.cuh"

namespace mq {



__device__ __forceinline__ int comp_of(int64_t e, int64_t C) { return e < C ? 0 : (e < 2 * C ? 1 : 2); }

__global__ void __launch_bounds__(kBlock, 3) pcg_stencil_kernel(StencilPcgArgs a) {
  __shared__ double red[3 * kWarps];
  __shared__ double tot[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  const int64_t wstride = (int64_t)G * kWarps;
  const int64_t w0 = (int64_t)blockIdx.x * kWarps + warp;
  const Lay L = a.L;
  const uint32_t *__restrict__ mask = a.mask;
  const double dg = a.dg, of = a.of, inv = a.inv;
  const bool jac = a.use_jac != 0;
  double *x = a.x, *r = a.r, *ap = a.ap;
  const double *b = a.b;
  const int x0_mode = a.x0_mode_dev ? *a.x0_mode_dev : a.x0_mode;
  if (a.err_word && *((volatile const unsigned int *)a.err_word)) {
    // an earlier solve of this step failed: skip (uniform across CTAs)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      PcgOut o{};
      o.status = 99;
      *a.out = o;
    }
    return;
  }

  // ---- initial residual (krylov.py:209-218) ----
  double v3[3] = {0.0, 0.0, 0.0};
  for (int64_t w = w0; w < L.words; w += wstride) {
    const uint32_t m = mask[w];
    if (m == 0u) continue;
    if (!((m >> lane) & 1u)) continue;
    const int64_t e = w * 32 + lane;
    const double bv = b[e];
    double rv = bv;
    if (x0_mode == 1) {
      const int c = comp_of(e, L.C);
      const double axv = stencil_row(c, e, L, dg, of, [&](int64_t q) { return x[q]; });
      rv = sub(bv, axv);
    } else {
      x[e] = 0.0;
    }
    r[e] = rv;
    const double z = jac ? mul(inv, rv) : rv;
    v3[0] = add(v3[0], mul(bv, bv));
    v3[1] = add(v3[1], mul(rv, rv));
    v3[2] = add(v3[2], mul(rv, z));
  }
  block_sum<3>(v3, red);
  if (threadIdx.x == 0) {
    a.partials[0 * G + blockIdx.x] = v3[0];
    a.partials[1 * G + blockIdx.x] = v3[1];
    a.partials[2 * G + blockIdx.x] = v3[2];
  }
  int status = MQ_OK;
  int iters = 0;
  int converged = 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  double *pold = a.pa, *pnew = a.pb;
  int applies = (x0_mode == 2) ? 0 : 1;
  if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
  {
    double s3[3];
    grid_partials_sum<3>(a.partials, G, s3, tot);
    bnorm = sqrt(s3[0]);
    const double target = fmax(a.rel_tol * bnorm, a.abs_tol);
    double rnorm = sqrt(s3[1]);
    rz = jac ? s3[2] : s3[1];
    auto relf = [&](double res) { return bnorm > 0.0 ? res / bnorm : (res == 0.0 ? 0.0 : INFINITY); };
    if (rnorm <= target) { converged = 1; rel = relf(rnorm); goto done; }
    double beta = 0.0, alpha_prev = 0.0;
    bool first = true;
    for (int it = 1; it <= a.max_iter; ++it) {
      // ---- K1: p_new, Ap = K p_new, deferred x update, p.Ap ----
      double v1[1] = {0.0};
      for (int64_t w = w0; w < L.words; w += wstride) {
        const uint32_t m = mask[w];
        if (m == 0u) continue;
        if (!((m >> lane) & 1u)) continue;
        const int64_t e = w * 32 + lane;
        const int c = comp_of(e, L.C);
        auto pn = [&](int64_t q) {
          const double rq = r[q];
          const double z = jac ? mul(inv, rq) : rq;
          return first ? z : add(z, mul(beta, pold[q]));
        };
        const double pe = pn(e);
        const double av = stencil_row(c, e, L, dg, of, pn);
        if (!first) x[e] = add(x[e], mul(alpha_prev, pold[e]));
        pnew[e] = pe;
        ap[e] = av;
        v1[0] = add(v1[0], mul(pe, av));
      }
      block_sum<1>(v1, red);
      if (threadIdx.x == 0) a.partials[3 * G + blockIdx.x] = v1[0];
      ++applies;
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      double s1[1];
      grid_partials_sum<1>(a.partials + 3 * G, G, s1, tot);
      const double pap = s1[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; goto done; }
      alpha = rz / pap;
      // ---- K2: r -= alpha Ap, r.r, r.z ----
      double v2[2] = {0.0, 0.0};
      for (int64_t w = w0; w < L.words; w += wstride) {
        const uint32_t m = mask[w];
        if (m == 0u) continue;
        if (!((m >> lane) & 1u)) continue;
        const int64_t e = w * 32 + lane;
        const double rv = sub(r[e], mul(alpha, ap[e]));
        r[e] = rv;
        const double z = jac ? mul(inv, rv) : rv;
        v2[0] = add(v2[0], mul(rv, rv));
        v2[1] = add(v2[1], mul(rv, z));
      }
      block_sum<2>(v2, red);
      if (threadIdx.x == 0) {
        a.partials[4 * G + blockIdx.x] = v2[0];
        a.partials[5 * G + blockIdx.x] = v2[1];
      }
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      double s2[2];
      grid_partials_sum<2>(a.partials + 4 * G, G, s2, tot);
      rnorm = sqrt(s2[0]);
      iters = it;
      rel = relf(rnorm);
      const double rz_new = jac ? s2[1] : s2[0];
      if (rnorm <= target) { converged = 1; break; }
      if (!isfinite(rz_new)) { status = MQ_INDEFINITE; break; }
      beta = rz_new / rz;
      rz = rz_new;
      alpha_prev = alpha;
      first = false;
      double *t = pold; pold = pnew; pnew = t;
    }
    if (status == MQ_OK) {
      // ---- final x update with the last direction (krylov.py:238); after
      // an exhausted budget the last direction was already swapped into pold
      double *pdir = converged ? pnew : pold;
      for (int64_t w = w0; w < L.words; w += wstride) {
        const uint32_t m = mask[w];
        if (m == 0u) continue;
        if (!((m >> lane) & 1u)) continue;
        const int64_t e = w * 32 + lane;
        x[e] = add(x[e], mul(alpha, pdir[e]));
      }
      if (!converged) status = MQ_NOT_CONVERGED;
    }
  }
done:
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    PcgOut o;
    o.iterations = iters;
    o.converged = converged;
    o.status = status;
    o.applies = applies;
    o.rel = rel;
    o.bnorm = bnorm;
    o.alpha = alpha;
    o.rz = rz;
    *a.out = o;
  }
}

// y = K_n x on active rows (inactive rows untouched = 0).
__global__ void __launch_bounds__(kBlock) kn_apply_kernel(Lay L, const uint32_t *__restrict__ mask, double dg,
                                                          double of, const double *__restrict__ x,
                                                          double *__restrict__ y) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t w = (int64_t)blockIdx.x * kWarps + warp; w < L.words; w += (int64_t)gridDim.x * kWarps) {
    const uint32_t m = mask[w];
    if (!((m >> lane) & 1u)) continue;
    const int64_t e = w * 32 + lane;
    y[e] = stencil_row(comp_of(e, L.C), e, L, dg, of, [&](int64_t q) { return __ldg(x + q); });
  }
}

__global__ void scatter_kernel(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ src,
                               double *__restrict__ dst) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    dst[idx[q]] = src[q];
}

__global__ void gather_kernel(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ src,
                              double *__restrict__ dst) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    dst[q] = src[idx[q]];
}

// ---------------------------------------------------------------------------
// General CSR operator (compact vectors), three passes per iteration.
// ---------------------------------------------------------------------------


__device__ __forceinline__ double csr_row(const CsrPcgArgs &a, int64_t i, const double *v) {
  double s = 0.0;  // scipy csr_matvec: sum starts at Yx[i] = 0
  for (int64_t q = a.rp[i]; q < a.rp[i + 1]; ++q) s = add(s, mul(a.va[q], v[a.ci[q]]));
  return s;
}

__global__ void __launch_bounds__(kBlock) pcg_csr_kernel(CsrPcgArgs a) {
  __shared__ double red[3 * kWarps];
  __shared__ double tot[4];
  const int G = gridDim.x;
  const int64_t stride = (int64_t)G * kBlock;
  const int64_t i0 = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const bool pre = a.inv != nullptr;
  double v3[3] = {0.0, 0.0, 0.0};
  for (int64_t i = i0; i < a.n; i += stride) {
    const double bv = a.b[i];
    const double rv = a.has_x0 ? sub(bv, csr_row(a, i, a.x)) : bv;
    a.r[i] = rv;
    const double z = pre ? mul(a.inv[i], rv) : rv;
    v3[0] = add(v3[0], mul(bv, bv));
    v3[1] = add(v3[1], mul(rv, rv));
    v3[2] = add(v3[2], mul(rv, z));
  }
  block_sum<3>(v3, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) a.partials[q * G + blockIdx.x] = v3[q];
  int status = MQ_OK, iters = 0, converged = 0, applies = a.has_x0 ? 1 : 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
  {
    double s3[3];
    grid_partials_sum<3>(a.partials, G, s3, tot);
    bnorm = sqrt(s3[0]);
    const double target = fmax(a.rel_tol * bnorm, a.abs_tol);
    double rnorm = sqrt(s3[1]);
    rz = pre ? s3[2] : s3[1];
    auto relf = [&](double res) { return bnorm > 0.0 ? res / bnorm : (res == 0.0 ? 0.0 : INFINITY); };
    if (rnorm <= target) { converged = 1; rel = relf(rnorm); goto done; }
    double beta = 0.0;
    for (int it = 1; it <= a.max_iter; ++it) {
      for (int64_t i = i0; i < a.n; i += stride) {
        const double rv = a.r[i];
        const double z = pre ? mul(a.inv[i], rv) : rv;
        a.p[i] = (it == 1) ? z : add(z, mul(beta, a.p[i]));
      }
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      double v1[1] = {0.0};
      for (int64_t i = i0; i < a.n; i += stride) {
        const double av = csr_row(a, i, a.p);
        a.ap[i] = av;
        v1[0] = add(v1[0], mul(a.p[i], av));
      }
      block_sum<1>(v1, red);
      if (threadIdx.x == 0) a.partials[3 * G + blockIdx.x] = v1[0];
      ++applies;
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      double s1[1];
      grid_partials_sum<1>(a.partials + 3 * G, G, s1, tot);
      const double pap = s1[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; goto done; }
      alpha = rz / pap;
      double v2[2] = {0.0, 0.0};
      for (int64_t i = i0; i < a.n; i += stride) {
        a.x[i] = add(a.x[i], mul(alpha, a.p[i]));
        const double rv = sub(a.r[i], mul(alpha, a.ap[i]));
        a.r[i] = rv;
        const double z = pre ? mul(a.inv[i], rv) : rv;
        v2[0] = add(v2[0], mul(rv, rv));
        v2[1] = add(v2[1], mul(rv, z));
      }
      block_sum<2>(v2, red);
      if (threadIdx.x == 0) {
        a.partials[4 * G + blockIdx.x] = v2[0];
        a.partials[5 * G + blockIdx.x] = v2[1];
      }
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      double s2[2];
      grid_partials_sum<2>(a.partials + 4 * G, G, s2, tot);
      rnorm = sqrt(s2[0]);
      iters = it;
      rel = relf(rnorm);
      const double rz_new = pre ? s2[1] : s2[0];
      if (rnorm <= target) { converged = 1; break; }
      if (!isfinite(rz_new)) { status = MQ_INDEFINITE; break; }
      beta = rz_new / rz;
      rz = rz_new;
    }
    if (status == MQ_OK && !converged) status = MQ_NOT_CONVERGED;
  }
done:
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    PcgOut o;
    o.iterations = iters;
    o.converged = converged;
    o.status = status;
    o.applies = applies;
    o.rel = rel;
    o.bnorm = bnorm;
    o.alpha = alpha;
    o.rz = rz;
    *a.out = o;
  }
}

__global__ void csr_spmv_kernel(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                const double *__restrict__ va, const double *__restrict__ x,
                                double *__restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) s = add(s, mul(va[q], x[ci[q]]));
    y[i] = s;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
int coop_grid(const void *kernel, int want_blocks, int *out) {
  int dev = 0, sms = 0, per = 0;
  MQ_CUDA(cudaGetDevice(&dev));
  MQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  MQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kBlock, 0));
  if (per < 1) { set_error("PCG kernel cannot be resident"); return MQ_CUDA_ERROR; }
  int g = sms * per;
  if (want_blocks > 0 && want_blocks < g) g = want_blocks;
  if (g < 1) g = 1;
  *out = g;
  return MQ_OK;
}

int launch_pcg_stencil(const StencilPcgArgs &args, int grid, cudaStream_t s) {
  MQ_CUDA(cudaMemsetAsync(&args.bar->count, 0, sizeof(unsigned long long), s));
  StencilPcgArgs a = args;
  void *params[] = {&a};
  MQ_CUDA(cudaLaunchCooperativeKernel((const void *)pcg_stencil_kernel, dim3(grid), dim3(kBlock), params, 0, s));
  return MQ_OK;
}

int pcg_stencil_grid(int64_t words, int *out) {
  // one warp per mask word at least; never more CTAs than co-resident
  const int64_t want = (words + kWarps - 1) / kWarps;
  return coop_grid((const void *)pcg_stencil_kernel, (int)(want > (1 << 30) ? (1 << 30) : want), out);
}

int launch_pcg_csr(const CsrPcgArgs &args, int grid, cudaStream_t s) {
  MQ_CUDA(cudaMemsetAsync(&args.bar->count, 0, sizeof(unsigned long long), s));
  CsrPcgArgs a = args;
  void *params[] = {&a};
  MQ_CUDA(cudaLaunchCooperativeKernel((const void *)pcg_csr_kernel, dim3(grid), dim3(kBlock), params, 0, s));
  return MQ_OK;
}

int pcg_csr_grid(int64_t n, int *out) {
  const int64_t want = (n + kBlock - 1) / kBlock;
  return coop_grid((const void *)pcg_csr_kernel, (int)(want > (1 << 30) ? (1 << 30) : want), out);
}

int launch_kn_apply(const Lay &L, const uint32_t *mask, double dg, double of, const double *x, double *y,
                    int sms, cudaStream_t s) {
  int64_t blocks = (L.words + kWarps - 1) / kWarps;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  kn_apply_kernel<<<(int)blocks, kBlock, 0, s>>>(L, mask, dg, of, x, y);
  MQ_CUDA(cudaGetLastError());
  return MQ_OK;
}

int launch_scatter(int64_t n, const int32_t *idx, const double *src, double *dst, int sms, cudaStream_t s) {
  if (n <= 0) return MQ_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  scatter_kernel<<<(int)blocks, 256, 0, s>>>(n, idx, src, dst);
  MQ_CUDA(cudaGetLastError());
  return MQ_OK;
}

int launch_gather(int64_t n, const int32_t *idx, const double *src, double *dst, int sms, cudaStream_t s) {
  if (n <= 0) return MQ_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  gather_kernel<<<(int)blocks, 256, 0, s>>>(n, idx, src, dst);
  MQ_CUDA(cudaGetLastError());
  return MQ_OK;
}

int launch_csr_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *va, const double *x, double *y,
                    int sms, cudaStream_t s) {
  if (n <= 0) return MQ_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  csr_spmv_kernel<<<(int)blocks, 256, 0, s>>>(n, rp, ci, va, x, y);
  MQ_CUDA(cudaGetLastError());
  return MQ_OK;
}

}  // namespace mq

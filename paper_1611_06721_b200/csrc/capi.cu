// C ABI of libmq_b200: context, device vectors, K_n operator and PCG.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "mq_ctx.h"

namespace mq {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char *what) {
  g_err = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what;
  return MQ_CUDA_ERROR;
}

int ctx_alloc(mq_ctx *ctx, void **p, size_t bytes) {
  MQ_CUDA(cudaMalloc(p, bytes));
  MQ_CUDA(cudaMemsetAsync(*p, 0, bytes, ctx->stream));
  ctx->allocs.push_back(*p);
  return MQ_OK;
}

template <class T>
int upload(mq_ctx *ctx, T **dst, const std::vector<T> &src) {
  if (src.empty()) { *dst = nullptr; return MQ_OK; }
  int rc = ctx_alloc(ctx, (void **)dst, src.size() * sizeof(T));
  if (rc) return rc;
  MQ_CUDA(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return MQ_OK;
}

// Runs a stencil PCG solve on device vectors of the context.
int ctx_pcg(mq_ctx *ctx, const double *b, double *x, int x0_mode, double rel_tol, double abs_tol, int max_iter,
            int use_jac, mq_solve_report *rep) {
  if (!(rel_tol > 0.0) || abs_tol < 0.0 || max_iter < 1) {
    set_error("invalid PCG configuration (rel_tol > 0, abs_tol >= 0, max_iter >= 1)");
    return MQ_INVALID;
  }
  StencilPcgArgs a{};
  a.L = ctx->topo.L;
  a.mask = ctx->d_mask;
  a.dg = ctx->kn_diag;
  a.of = ctx->kn_off;
  a.inv = ctx->jac_inv;
  a.use_jac = use_jac;
  a.x0_mode = x0_mode;
  a.b = b;
  a.x = x;
  a.r = ctx->d_r;
  a.pa = ctx->d_p0;
  a.pb = ctx->d_p1;
  a.ap = ctx->d_ap;
  a.ap2 = ctx->d_ap2;
  a.r2 = ctx->d_r2;
  a.stress_ns = pcg_stress_ns();
  a.rel_tol = rel_tol;
  a.abs_tol = abs_tol;
  a.max_iter = max_iter;
  a.partials = ctx->d_partials;
  a.bar = ctx->d_bar;
  a.out = ctx->d_out;
  a.trace = ctx->d_trace;
  if (ctx->pcg_timing) MQ_CUDA(cudaEventRecord(ctx->ev_pcg0, ctx->stream));
  int rc = launch_pcg_ctx(ctx, a);
  if (rc) return rc;
  ctx->launches += 1;
  if (ctx->pcg_timing) MQ_CUDA(cudaEventRecord(ctx->ev_pcg1, ctx->stream));
  MQ_CUDA(cudaMemcpyAsync(ctx->h_out, ctx->d_out, sizeof(PcgOut), cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->pcg_timing) {
    float ms = 0.f;
    MQ_CUDA(cudaEventElapsedTime(&ms, ctx->ev_pcg0, ctx->ev_pcg1));
    ctx->pcg_ms += ms;
    ctx->pcg_iters += ctx->h_out->iterations;
  }
  const PcgOut &o = *ctx->h_out;
  if (rep) {
    rep->iterations = o.iterations;
    rep->converged = o.converged;
    rep->final_rel_residual = o.rel;
    rep->applies = o.applies;
  }
  if (o.status == MQ_INDEFINITE) {
    set_error("nonpositive curvature or non-finite preconditioned residual at iteration " +
              std::to_string(o.iterations));
    return MQ_INDEFINITE;
  }
  if (o.status == MQ_CUDA_ERROR) {
    set_error("grid barrier watchdog expired in the PCG kernel");
    return MQ_CUDA_ERROR;
  }
  return o.status;
}

int launch_pcg_ctx(mq_ctx *ctx, const StencilPcgArgs &args) {
  if (ctx->pcg_variant == 1) return launch_pcg_stencil(args, ctx->pcg_grid, ctx->stream);
  if (ctx->pcg_variant == 2) return launch_pcg_resident(args, ctx->res_geo, ctx->res_grid, ctx->stream);
  return launch_pcg_brick(args, ctx->geo, ctx->brick_grid, ctx->stream);
}

}  // namespace mq

using namespace mq;

extern "C" {

const char *mq_last_error(void) { return g_err.c_str(); }

int mq_device_count(int32_t *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) { *count = 0; return cuda_fail(e, "cudaGetDeviceCount"); }
  *count = n;
  return MQ_OK;
}

// Page-locked host memory for result arrays: device-to-host copies into it
// run at DMA speed instead of through the driver's pageable staging.
int mq_host_alloc(int64_t bytes, void **out) {
  if (bytes <= 0 || !out) { set_error("invalid host allocation"); return MQ_INVALID; }
  MQ_CUDA(cudaMallocHost(out, (size_t)bytes));
  return MQ_OK;
}

int mq_host_free(void *p) {
  if (p) MQ_CUDA(cudaFreeHost(p));
  return MQ_OK;
}

int mq_device_sm_count(int32_t device, int32_t *sms) {
  int n = 0;
  cudaError_t e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) { *sms = 0; return cuda_fail(e, "cudaDeviceGetAttribute"); }
  *sms = n;
  return MQ_OK;
}

int mq_ctx_create(const mq_grid_desc *desc, int32_t device, mq_ctx **out) {
  if (!desc || !out) { set_error("NULL argument"); return MQ_INVALID; }
  *out = nullptr;
  if (!(desc->nu_air > 0.0)) { set_error("air reluctivity must be positive"); return MQ_INVALID; }
  if (!(desc->kappa > 0.0)) { set_error("conductor material needs positive conductivity"); return MQ_INVALID; }
  if (desc->brauer_k1 < 0.0 || desc->brauer_k2 < 0.0 || !(desc->brauer_k3 > 0.0)) {
    set_error("invalid Brauer coefficients");
    return MQ_INVALID;
  }
  mq_ctx *ctx = new mq_ctx();
  ctx->desc = *desc;
  ctx->material.assign(desc->material, desc->material + (size_t)desc->nx * desc->ny * desc->nz);
  ctx->desc.material = ctx->material.data();
  std::string err;
  int rc = build_topology(ctx->desc, ctx->topo, err);
  if (rc) { set_error(err); delete ctx; return rc; }
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaSetDevice"); }
  e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaStreamCreate"); }
  ctx->stream = ctx->own_stream;
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  // K_n coefficients: off = w/h with w = 0.5 nu + 0.5 nu = nu exactly
  // (model.py:474-481); diag = four face terms summed in CSR order.
  const double h = desc->h;
  const double w = 0.5 * desc->nu_air + 0.5 * desc->nu_air;
  const double c = w / h;
  ctx->kn_off = desc->kn_off > 0.0 ? desc->kn_off : c;
  ctx->kn_diag = desc->kn_diag > 0.0 ? desc->kn_diag : (((c + c) + c) + c);
  // JacobiPreconditioner._inv = 1.0 / diag (krylov.py:94)
  ctx->jac_inv = 1.0 / ctx->kn_diag;
  const Topology &t = ctx->topo;
  rc = 0;
  rc = rc ? rc : upload(ctx, &ctx->d_mask, t.mask);
  rc = rc ? rc : upload(ctx, &ctx->d_nc_pad, t.nc_pad);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_stage, sizeof(double) * std::max<int64_t>(1, (int64_t)t.nc_pad.size()));
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_r, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_p0, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_p1, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_ap, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_tmp0, sizeof(double) * t.L.total);
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_tmp1, sizeof(double) * t.L.total);
  if (!rc) rc = pcg_stencil_grid(t.L.words, &ctx->pcg_grid);
  if (!rc) rc = brick_pcg_setup(t.L, t.nx, t.ny, t.nz, 0, &ctx->brick_grid, &ctx->geo);
  if (!rc) rc = resident_pcg_setup(t.nx, t.ny, t.nz, &ctx->res_grid, &ctx->res_geo);
  // Ap of odd iterations: the single-reduction resident kernel publishes Ap
  // double-buffered (a CTA's next Ap must not overwrite the values a slower
  // neighbour still has to load after the barrier)
  // (and so does the one-barrier TMA kernel, which also double-buffers r)
  if (!rc) rc = ctx_alloc(ctx, (void **)&ctx->d_ap2, sizeof(double) * t.L.total);
  if (!rc) rc = ctx_alloc(ctx, (void **)&ctx->d_r2, sizeof(double) * t.L.total);
  {
    // default: shared-memory-resident kernel when the bricks fit on chip,
    // else the TMA brick kernel; MQ_PCG_KERNEL=simple|brick|resident overrides
    const char *v = getenv("MQ_PCG_KERNEL");
    const std::string want = v ? v : "";
    ctx->pcg_variant = ctx->res_grid > 0 ? 2 : 0;
    if (want == "simple") ctx->pcg_variant = 1;
    else if (want == "brick") ctx->pcg_variant = 0;
    else if (want == "resident" && ctx->res_grid > 0) ctx->pcg_variant = 2;
  }
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_partials, sizeof(double) * 8 * (size_t)std::max(ctx->pcg_grid, 1024));
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_bar, sizeof(GridBar));
  rc = rc ? rc : ctx_alloc(ctx, (void **)&ctx->d_out, sizeof(PcgOut));
  if (!rc && getenv("MQ_PCG_TRACE")) rc = ctx_alloc(ctx, (void **)&ctx->d_trace, sizeof(unsigned long long) * 2048);
  if (!rc) {
    e = cudaMallocHost((void **)&ctx->h_out, sizeof(PcgOut));
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMallocHost");
  }
  if (!rc) {
    e = cudaEventCreate(&ctx->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev_pcg0);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev_pcg1);
    for (int q = 0; q < 2 * kEvPool && e == cudaSuccess; ++q) e = cudaEventCreate(&ctx->ev_pool[q]);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaEventCreate");
  }
  if (!rc) rc = conducting_init(ctx);
  if (!rc) {
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "context setup");
  }
  if (rc) { mq_ctx_destroy(ctx); return rc; }
  *out = ctx;
  return MQ_OK;
}

void mq_ctx_destroy(mq_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  solver_free(ctx);
  slab_step_free(ctx);
  slab_peer_free(ctx);
  for (void *p : ctx->allocs) cudaFree(p);
  for (double *p : ctx->vecs) cudaFree(p);
  if (ctx->h_out) cudaFreeHost(ctx->h_out);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->ev_pcg0) cudaEventDestroy(ctx->ev_pcg0);
  if (ctx->ev_pcg1) cudaEventDestroy(ctx->ev_pcg1);
  for (int q = 0; q < 2 * kEvPool; ++q)
    if (ctx->ev_pool[q]) cudaEventDestroy(ctx->ev_pool[q]);
  if (ctx->flush_buf) cudaFree(ctx->flush_buf);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int64_t mq_n_n(const mq_ctx *ctx) { return ctx ? (int64_t)ctx->topo.nc_pad.size() : -1; }
int64_t mq_n_c(const mq_ctx *ctx) { return ctx ? (int64_t)ctx->topo.c_pad.size() : -1; }
int64_t mq_dev_len(const mq_ctx *ctx) { return ctx ? ctx->topo.L.total : -1; }

int mq_kn_coefficients(const mq_ctx *ctx, double *diag, double *off, double *jacobi_inv) {
  if (!ctx) { set_error("NULL context"); return MQ_INVALID; }
  if (diag) *diag = ctx->kn_diag;
  if (off) *off = ctx->kn_off;
  if (jacobi_inv) *jacobi_inv = ctx->jac_inv;
  return MQ_OK;
}

int mq_partition_export(const mq_ctx *ctx, int64_t *noncond_global, int64_t *cond_global) {
  if (!ctx) { set_error("NULL context"); return MQ_INVALID; }
  if (noncond_global) std::memcpy(noncond_global, ctx->topo.nc_global.data(), ctx->topo.nc_global.size() * 8);
  if (cond_global) std::memcpy(cond_global, ctx->topo.c_global.data(), ctx->topo.c_global.size() * 8);
  return MQ_OK;
}

int mq_map_global_to_noncond(const mq_ctx *ctx, const int64_t *gid, int64_t n, int64_t *out) {
  if (!ctx) { set_error("NULL context"); return MQ_INVALID; }
  const auto &g = ctx->topo.nc_global;
  for (int64_t q = 0; q < n; ++q) {
    auto it = std::lower_bound(g.begin(), g.end(), gid[q]);
    out[q] = (it != g.end() && *it == gid[q]) ? (int64_t)(it - g.begin()) : -1;
  }
  return MQ_OK;
}

int mq_ctx_sync(mq_ctx *ctx) {
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

int mq_pcg_kernel_info(const mq_ctx *ctx, char *name, int32_t cap, int32_t *grid) {
  std::string n;
  int g = 0;
  if (ctx->pcg_variant == 1) { n = "pcg_stencil_kernel"; g = ctx->pcg_grid; }
  else if (ctx->pcg_variant == 2) {
    const int li = (ctx->res_geo.nx + ctx->res_geo.chunks - 1) / ctx->res_geo.chunks;
    n = std::string(resident_single_reduction(li) ? "pcg_resident1_kernel<" : "pcg_resident_kernel<") +
        std::to_string(li) + ">";
    g = ctx->res_grid;
  } else { n = tma_single_reduction(ctx->geo) ? "pcg_tma1_kernel" : "pcg_tma_kernel"; g = ctx->brick_grid; }
  if (name && cap > 0) {
    std::strncpy(name, n.c_str(), (size_t)cap - 1);
    name[cap - 1] = 0;
  }
  if (grid) *grid = g;
  return MQ_OK;
}

int mq_ctx_set_sm_budget(mq_ctx *ctx, int32_t sms) {
  int dev_sms = 0;
  MQ_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  if (sms < 0) { set_error("SM budget must be nonnegative"); return MQ_INVALID; }
  if (sms == 0 || sms >= dev_sms) {
    int rc = brick_pcg_setup(ctx->topo.L, ctx->topo.nx, ctx->topo.ny, ctx->topo.nz, 0, &ctx->brick_grid, &ctx->geo);
    if (rc) return rc;
    ctx->pcg_variant = ctx->res_grid > 0 ? 2 : 0;
    ctx->sm_budget = 0;
  } else {
    // a slice of the GPU: the TMA brick kernel sized for `sms` SMs (the
    // resident kernel needs one CTA per brick on the whole chip)
    int rc = brick_pcg_setup(ctx->topo.L, ctx->topo.nx, ctx->topo.ny, ctx->topo.nz, sms, &ctx->brick_grid, &ctx->geo);
    if (rc) return rc;
    ctx->pcg_variant = 0;
    ctx->sm_budget = sms;
  }
  solver_graph_reset(ctx);
  return MQ_OK;
}

int mq_ctx_set_stream(mq_ctx *ctx, void *stream) {
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return MQ_OK;
}

int mq_vec_alloc(mq_ctx *ctx, double **dev) {
  double *p = nullptr;
  MQ_CUDA(cudaMalloc((void **)&p, sizeof(double) * ctx->topo.L.total));
  MQ_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * ctx->topo.L.total, ctx->stream));
  ctx->vecs.insert(p);
  *dev = p;
  return MQ_OK;
}

int mq_vec_free(mq_ctx *ctx, double *dev) {
  auto it = ctx->vecs.find(dev);
  if (it == ctx->vecs.end()) { set_error("vector not owned by this context"); return MQ_INVALID; }
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->vecs.erase(it);
  MQ_CUDA(cudaFree(dev));
  return MQ_OK;
}

int mq_vec_upload(mq_ctx *ctx, const double *host, double *dev) {
  const int64_t n = (int64_t)ctx->topo.nc_pad.size();
  MQ_CUDA(cudaMemcpyAsync(ctx->d_stage, host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  int rc = launch_scatter(n, ctx->d_nc_pad, ctx->d_stage, dev, ctx->sms, ctx->stream);
  if (rc) return rc;
  ctx->launches += 1;
  return MQ_OK;
}

int mq_vec_download(mq_ctx *ctx, const double *dev, double *host) {
  const int64_t n = (int64_t)ctx->topo.nc_pad.size();
  int rc = launch_gather(n, ctx->d_nc_pad, dev, ctx->d_stage, ctx->sms, ctx->stream);
  if (rc) return rc;
  ctx->launches += 1;
  MQ_CUDA(cudaMemcpyAsync(host, ctx->d_stage, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

int mq_kn_apply_dev(mq_ctx *ctx, const double *x, double *y) {
  int rc = ctx->pcg_variant == 1
               ? launch_kn_apply(ctx->topo.L, ctx->d_mask, ctx->kn_diag, ctx->kn_off, x, y, ctx->sms, ctx->stream)
               : launch_kn_apply_brick(ctx->topo.L, ctx->geo, ctx->d_mask, ctx->kn_diag, ctx->kn_off, x, y,
                                       ctx->sms, ctx->stream);
  if (!rc) ctx->launches += 1;
  return rc;
}

int mq_kn_apply_host(mq_ctx *ctx, const double *x, double *y) {
  int rc = mq_vec_upload(ctx, x, ctx->d_tmp0);
  if (rc) return rc;
  rc = mq_kn_apply_dev(ctx, ctx->d_tmp0, ctx->d_tmp1);
  if (rc) return rc;
  return mq_vec_download(ctx, ctx->d_tmp1, y);
}

int mq_pcg_solve_dev(mq_ctx *ctx, const double *b, const double *x0, double *x, double rel_tol, double abs_tol,
                     int32_t max_iter, int32_t use_jacobi, mq_solve_report *rep) {
  int mode = 2;
  if (x0) {
    mode = 1;
    if (x0 != x) MQ_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * ctx->topo.L.total, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return ctx_pcg(ctx, b, x, mode, rel_tol, abs_tol, max_iter, use_jacobi, rep);
}

int mq_pcg_solve_host(mq_ctx *ctx, const double *b, const double *x0, double *x, double rel_tol, double abs_tol,
                      int32_t max_iter, int32_t use_jacobi, mq_solve_report *rep) {
  int rc = mq_vec_upload(ctx, b, ctx->d_tmp0);
  if (rc) return rc;
  if (x0) {
    rc = mq_vec_upload(ctx, x0, ctx->d_tmp1);
    if (rc) return rc;
  }
  rc = ctx_pcg(ctx, ctx->d_tmp0, ctx->d_tmp1, x0 ? 1 : 2, rel_tol, abs_tol, max_iter, use_jacobi, rep);
  if (rc != MQ_OK && rc != MQ_NOT_CONVERGED) return rc;
  int rc2 = mq_vec_download(ctx, ctx->d_tmp1, x);
  return rc2 ? rc2 : rc;
}

// ---- general CSR operator ---------------------------------------------
int mq_csr_pcg_solve(int32_t device, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                     const double *values, const double *b, const double *x0, double *x, const double *inv_diag,
                     double rel_tol, double abs_tol, int32_t max_iter, mq_solve_report *rep) {
  if (n < 0 || !row_ptr || !b || !x) { set_error("invalid CSR arguments"); return MQ_INVALID; }
  if (!(rel_tol > 0.0) || abs_tol < 0.0 || max_iter < 1) { set_error("invalid PCG configuration"); return MQ_INVALID; }
  MQ_CUDA(cudaSetDevice(device));
  const int64_t nnz = row_ptr[n];
  const size_t vb = sizeof(double) * (size_t)std::max<int64_t>(n, 1);
  int grid = 1;
  int rc = pcg_csr_grid(std::max<int64_t>(n, 1), &grid);
  if (rc) return rc;
  std::vector<void *> mem;
  auto alloc = [&](void **p, size_t bytes) -> int {
    MQ_CUDA(cudaMalloc(p, bytes));
    MQ_CUDA(cudaMemset(*p, 0, bytes));
    mem.push_back(*p);
    return MQ_OK;
  };
  int64_t *d_rp = nullptr; int32_t *d_ci = nullptr;
  double *d_va = nullptr, *d_b = nullptr, *d_x = nullptr, *d_r = nullptr, *d_p = nullptr, *d_ap = nullptr;
  double *d_inv = nullptr, *d_part = nullptr;
  GridBar *d_bar = nullptr; PcgOut *d_out = nullptr;
  rc = alloc((void **)&d_rp, sizeof(int64_t) * (n + 1));
  rc = rc ? rc : alloc((void **)&d_ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  rc = rc ? rc : alloc((void **)&d_va, sizeof(double) * std::max<int64_t>(nnz, 1));
  rc = rc ? rc : alloc((void **)&d_b, vb);
  rc = rc ? rc : alloc((void **)&d_x, vb);
  rc = rc ? rc : alloc((void **)&d_r, vb);
  rc = rc ? rc : alloc((void **)&d_p, vb);
  rc = rc ? rc : alloc((void **)&d_ap, vb);
  if (!rc && inv_diag) rc = alloc((void **)&d_inv, vb);
  rc = rc ? rc : alloc((void **)&d_part, sizeof(double) * 8 * (size_t)grid);
  rc = rc ? rc : alloc((void **)&d_bar, sizeof(GridBar));
  rc = rc ? rc : alloc((void **)&d_out, sizeof(PcgOut));
  PcgOut o{};
  if (!rc) {
    cudaMemcpy(d_rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice);
    if (nnz > 0) {
      cudaMemcpy(d_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice);
      cudaMemcpy(d_va, values, sizeof(double) * nnz, cudaMemcpyHostToDevice);
    }
    if (n > 0) {
      cudaMemcpy(d_b, b, sizeof(double) * n, cudaMemcpyHostToDevice);
      if (x0) cudaMemcpy(d_x, x0, sizeof(double) * n, cudaMemcpyHostToDevice);
      if (inv_diag) cudaMemcpy(d_inv, inv_diag, sizeof(double) * n, cudaMemcpyHostToDevice);
    }
    CsrPcgArgs a{};
    a.n = n; a.rp = d_rp; a.ci = d_ci; a.va = d_va; a.inv = d_inv; a.has_x0 = x0 != nullptr;
    a.b = d_b; a.x = d_x; a.r = d_r; a.p = d_p; a.ap = d_ap;
    a.rel_tol = rel_tol; a.abs_tol = abs_tol; a.max_iter = max_iter;
    a.partials = d_part; a.bar = d_bar; a.out = d_out;
    rc = launch_pcg_csr(a, grid, 0);
    if (!rc) {
      cudaError_t e = cudaMemcpy(&o, d_out, sizeof(PcgOut), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) rc = cuda_fail(e, "CSR PCG");
      else if (n > 0) cudaMemcpy(x, d_x, sizeof(double) * n, cudaMemcpyDeviceToHost);
    }
  }
  for (void *p : mem) cudaFree(p);
  if (rc) return rc;
  if (rep) {
    rep->iterations = o.iterations;
    rep->converged = o.converged;
    rep->final_rel_residual = o.rel;
    rep->applies = o.applies;
  }
  if (o.status == MQ_INDEFINITE) {
    set_error("nonpositive curvature or non-finite preconditioned residual at iteration " + std::to_string(o.iterations));
    return MQ_INDEFINITE;
  }
  if (o.status == MQ_CUDA_ERROR) { set_error("grid barrier watchdog expired in the CSR PCG kernel"); return MQ_CUDA_ERROR; }
  return o.status;
}

int mq_csr_spmv(int32_t device, int64_t nrows, int64_t ncols, const int64_t *row_ptr, const int32_t *col_idx,
                const double *values, const double *x, double *y) {
  MQ_CUDA(cudaSetDevice(device));
  const int64_t nnz = row_ptr[nrows];
  int64_t *d_rp = nullptr; int32_t *d_ci = nullptr; double *d_va = nullptr, *d_x = nullptr, *d_y = nullptr;
  MQ_CUDA(cudaMalloc(&d_rp, sizeof(int64_t) * (nrows + 1)));
  MQ_CUDA(cudaMalloc(&d_ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  MQ_CUDA(cudaMalloc(&d_va, sizeof(double) * std::max<int64_t>(nnz, 1)));
  MQ_CUDA(cudaMalloc(&d_x, sizeof(double) * std::max<int64_t>(ncols, 1)));
  MQ_CUDA(cudaMalloc(&d_y, sizeof(double) * std::max<int64_t>(nrows, 1)));
  cudaMemcpy(d_rp, row_ptr, sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice);
  if (nnz) {
    cudaMemcpy(d_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice);
    cudaMemcpy(d_va, values, sizeof(double) * nnz, cudaMemcpyHostToDevice);
  }
  if (ncols) cudaMemcpy(d_x, x, sizeof(double) * ncols, cudaMemcpyHostToDevice);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int rc = launch_csr_spmv(nrows, d_rp, d_ci, d_va, d_x, d_y, sms, 0);
  if (!rc && nrows) {
    cudaError_t e = cudaMemcpy(y, d_y, sizeof(double) * nrows, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "csr spmv");
  }
  cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_va); cudaFree(d_x); cudaFree(d_y);
  return rc;
}

// ---- timing ------------------------------------------------------------
int mq_timer_start(mq_ctx *ctx) {
  MQ_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
  return MQ_OK;
}

int mq_timer_stop(mq_ctx *ctx, double *ms) {
  MQ_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
  MQ_CUDA(cudaEventSynchronize(ctx->ev1));
  float f = 0.f;
  MQ_CUDA(cudaEventElapsedTime(&f, ctx->ev0, ctx->ev1));
  *ms = f;
  return MQ_OK;
}

int mq_pcg_stats(mq_ctx *ctx, double *pcg_ms, int64_t *pcg_iterations, int64_t *launches, int32_t enable) {
  if (pcg_ms) *pcg_ms = ctx->pcg_ms;
  if (pcg_iterations) *pcg_iterations = ctx->pcg_iters;
  if (launches) *launches = ctx->pcg_launches;
  if (enable >= 0) {
    ctx->pcg_timing = enable != 0;
    ctx->pcg_ms = 0.0;
    ctx->pcg_iters = 0;
    ctx->pcg_launches = 0;
  }
  return MQ_OK;
}

int mq_pcg_trace(mq_ctx *ctx, uint64_t *stamps, int32_t n) {
  if (!ctx->d_trace) { set_error("PCG tracing disabled (set MQ_PCG_TRACE)"); return MQ_INVALID; }
  MQ_CUDA(cudaMemcpy(stamps, ctx->d_trace, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return MQ_OK;
}

int mq_kernel_launches(mq_ctx *ctx, int64_t *count) {
  *count = ctx->launches;
  return MQ_OK;
}

int mq_l2_flush(mq_ctx *ctx) {
  const size_t bytes = (size_t)256 << 20;  // > 126 MB L2
  if (!ctx->flush_buf) MQ_CUDA(cudaMalloc(&ctx->flush_buf, bytes));
  MQ_CUDA(cudaMemsetAsync(ctx->flush_buf, ctx->flush_val++ & 0xff, bytes, ctx->stream));
  return MQ_OK;
}

}  // extern "C"

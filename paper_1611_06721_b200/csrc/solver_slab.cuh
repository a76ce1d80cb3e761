// Sharded explicit-Euler step over i-slabs (BASELINE configs[4]): the
// SchurOperator step of schur.py:379-419 with every K_n-sized vector split
// into the slabs of slab.cu / slab_fused.cu, one slab per rank.
//
// Included at the end of solver.cu: the start-vector kernels (k_mdot,
// k_axpy_dots, k_comb, k_cspe_product), the 1-thread CSPE decisions
// (run_post: cspe_project_small / gate / decide / commit) and the conducting
// kernels (k_cell_nu, kc_row) are the single-device ones, run on the slab's
// layout.  What changes is where the reductions end:
//
//   single device:  tall-skinny pass -> last-block reduce -> decision (one kernel)
//   slab:           tall-skinny pass -> last-block reduce = this rank's partial
//                   -> host all-reduce over the ranks (fixed rank order, the same
//                   bits on every rank) -> k_ss_post: decision on the totals
//
// so every rank takes the same accept / drop / evict decisions on the same
// scalars (startvec.py:158-225), and the rank-partial sums are the only
// difference from the single-device step.  Ghost planes: a vector that feeds
// a stencil (the orthogonalised CGS vector before K u, y_cpl - y_src before
// K_cn) gets one halo exchange from the host; all other vectors hold zeros in
// their ghost planes, so the flat dot products over the slab layout see only
// owned rows.
//
// Conducting block: a_c is small (n_c <= 0.7 M at 256^3) and replicated on
// every rank.  Brauer nu is recomputed per rank for all conductor cells
// (model.py:496-500); K_cn^T a_c is formed for the slab's own rows
// (csc_matvec order, sparse.py:186-193); each rank integrates the conducting
// edges whose node plane it owns (their K_cn rows reach one plane either side,
// i.e. the slab's ghost planes) in the reference's CSR order, then the host
// all-gathers the owned values: every K_cn / K_c / Euler sum is the
// single-device one, bit for bit, given the same y.
namespace mq {

struct SlabStepHost {
  mq_solver_cfg cfg{};
  int kb = 8;
  int ilo = 0, ihi = 0;
  FamDev *d_fam = nullptr;
  double **d_U[3] = {nullptr, nullptr, nullptr};
  double **d_KU[3] = {nullptr, nullptr, nullptr};
  std::vector<double *> h_U[3], h_KU[3];
  double *last[3] = {nullptr, nullptr, nullptr};
  bool has_last[3] = {false, false, false};
  double *rhs_src = nullptr, *rhs_cpl = nullptr, *y_src = nullptr, *y_cpl = nullptr, *y_cur = nullptr;
  double *w1 = nullptr, *w2 = nullptr, *dvec = nullptr;
  double *d_part = nullptr, *d_tot = nullptr;
  double *h_part = nullptr;  // page-locked landing of partials / owned values
  int64_t h_part_len = 0;
  double *d_red = nullptr;
  unsigned int *d_cnt = nullptr;
  int red_grid = 1;
  int32_t *d_pat_idx = nullptr;
  double *d_pat_val = nullptr;
  int64_t n_pat = 0;
  // conducting block in full-grid compact numbering (replicated)
  CondArgs ca{};
  int64_t n_c = 0, n_cells = 0;
  double *d_ac = nullptr, *d_nu = nullptr;
  // owned conducting edges and their K_cn rows (columns in the slab layout)
  int64_t n_own = 0;
  std::vector<int64_t> h_own;
  int32_t *d_own = nullptr;
  int64_t *d_okcn_ptr = nullptr;
  int32_t *d_okcn_col = nullptr;
  int8_t *d_okcn_sgn = nullptr;
  double *d_own_out = nullptr;
  // K_cn^T rows of the slab's own dofs (slab padded row, full cond sources)
  int64_t n_kt = 0;
  int32_t *d_kt_row = nullptr;
  int64_t *d_kt_ptr = nullptr;
  int32_t *d_kt_src = nullptr;
  int8_t *d_kt_sgn = nullptr;
  unsigned int *d_err = nullptr;
  int64_t solves[3] = {0, 0, 0}, iterations[3] = {0, 0, 0}, pcg_applies = 0;
  std::vector<void *> mem;
};

void slab_step_free(mq_ctx *ctx) {
  SlabStepHost *s = ctx->sstep;
  if (!s) return;
  for (void *p : s->mem) cudaFree(p);
  if (s->h_part) cudaFreeHost(s->h_part);
  delete s;
  ctx->sstep = nullptr;
}

template <class T>
static int ss_up(mq_ctx *ctx, SlabStepHost *s, T **dst, const std::vector<T> &src) {
  *dst = nullptr;
  if (src.empty()) return MQ_OK;
  MQ_CUDA(cudaMalloc((void **)dst, src.size() * sizeof(T)));
  s->mem.push_back(*dst);
  MQ_CUDA(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return MQ_OK;
}

static int ss_zalloc(mq_ctx *ctx, SlabStepHost *s, void **p, size_t bytes) {
  MQ_CUDA(cudaMalloc(p, std::max<size_t>(bytes, 8)));
  s->mem.push_back(*p);
  MQ_CUDA(cudaMemsetAsync(*p, 0, std::max<size_t>(bytes, 8), ctx->stream));
  return MQ_OK;
}

// full padded index -> (component, node plane i, in-plane offset)
struct PadSplit {
  int c;
  int64_t i;
  int64_t jk;
};
static PadSplit split_pad(const Lay &L, int64_t e) {
  PadSplit p;
  p.c = (int)(e / L.C);
  const int64_t rel = e - p.c * L.C;
  const int64_t pp = rel / L.Si;  // padded plane: node plane i sits at i + 1
  p.i = pp - 1;
  p.jk = rel - pp * L.Si;
  return p;
}

__global__ void k_ss_post(FamDev *f, Post post, const double *__restrict__ tot, int n) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int q = 0; q < n; ++q) f->d[q] = tot[q];
  run_post(post);
}

__global__ void k_ss_src(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ val, double s,
                         double *__restrict__ rhs) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    rhs[idx[q]] = mul(val[q], s);
}

// K_cn^T a_c on the slab's rows (csc_matvec order, as k_kcnt)
__global__ void k_ss_kcnt(int64_t n, const int32_t *__restrict__ row, const int64_t *__restrict__ ptr,
                          const int32_t *__restrict__ src, const int8_t *__restrict__ sgn, double of,
                          const double *__restrict__ ac, double *__restrict__ w) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = ptr[r]; q < ptr[r + 1]; ++q) s = add(s, mul(sgn[q] * of, ac[src[q]]));
    w[row[r]] = s;
  }
}

// Euler update of the owned conducting edges (schur.py:392-404, as k_euler):
// dvec = y_cpl - y_src with the neighbours' values in the ghost planes
__global__ void k_ss_euler(CondArgs a, int64_t n_own, const int32_t *__restrict__ own,
                           const int64_t *__restrict__ kptr, const int32_t *__restrict__ kcol,
                           const int8_t *__restrict__ ksgn, const double *__restrict__ nu,
                           const double *__restrict__ ac, const double *__restrict__ dvec, double dt,
                           double *__restrict__ out, unsigned int *err) {
  bool bad = false;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_own; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = own[q];
    double s = 0.0;
    for (int64_t p = kptr[q]; p < kptr[q + 1]; ++p) s = add(s, mul(ksgn[p] * a.of, dvec[kcol[p]]));
    const double rate = sub(s, kc_row(a, e, nu, ac));
    const double v = add(ac[e], mul(dt, mul(a.minv[e], rate)));
    out[q] = v;
    bad |= !isfinite(v);
  }
  if (bad) atomicExch(err, (unsigned)MQ_NONFINITE);
}

static int ss_stream_grid(mq_ctx *ctx) {
  int64_t b = (ctx->topo.L.words + kWarps - 1) / kWarps;
  if (b > (int64_t)ctx->sms * 4) b = ctx->sms * 4;
  return (int)std::max<int64_t>(1, b);
}

static int ss_grid_for(mq_ctx *ctx, int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > (int64_t)ctx->sms * 4) b = ctx->sms * 4;
  return (int)b;
}

static int ss_check(mq_ctx *ctx) {
  if (!ctx) { set_error("NULL context"); return MQ_INVALID; }
  if (!ctx->sstep) { set_error("slab step not initialised (mq_ss_init)"); return MQ_INVALID; }
  return MQ_OK;
}

static double *ss_y(SlabStepHost *s, int fam) {
  return fam == MQ_FAM_SOURCE ? s->y_src : (fam == MQ_FAM_COUPLING_PREVIOUS ? s->y_cpl : s->y_cur);
}

// partials (RQ doubles) of the last reduction -> host
static int ss_fetch(mq_ctx *ctx, double *part, int64_t n) {
  SlabStepHost *s = ctx->sstep;
  MQ_CUDA(cudaMemcpyAsync(s->h_part, s->d_part, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(part, s->h_part, sizeof(double) * n);
  return MQ_OK;
}

static int ss_post(mq_ctx *ctx, int fam, int kind, const double *tot) {
  SlabStepHost *s = ctx->sstep;
  MQ_CUDA(cudaMemcpyAsync(s->d_tot, tot, sizeof(double) * RQ, cudaMemcpyHostToDevice, ctx->stream));
  Post post;
  post.kind = kind;
  post.f = s->d_fam + fam;
  post.max_cols = s->cfg.max_cols;
  post.drop_tol = s->cfg.drop_tol;
  k_ss_post<<<1, 32, 0, ctx->stream>>>(s->d_fam + fam, post, s->d_tot, RQ);
  MQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  return MQ_OK;
}

}  // namespace mq

extern "C" {

int mq_ss_init(mq_ctx *ctx, const mq_solver_cfg *cfg, const double *pattern_local) {
  if (!ctx || !cfg) { set_error("NULL argument"); return MQ_INVALID; }
  if (ctx->slab_hi <= ctx->slab_lo) { set_error("mq_ss_init needs a slab context (mq_ctx_create_slab)"); return MQ_INVALID; }
  if (cfg->strategy == MQ_STRAT_POD) { set_error("the sharded step supports the zero / previous / cspe strategies"); return MQ_INVALID; }
  if (cfg->strategy < 0 || cfg->strategy > 3) { set_error("unknown start-vector strategy"); return MQ_INVALID; }
  if (cfg->strategy == MQ_STRAT_CSPE && (cfg->max_cols < 1 || cfg->max_cols > MAXS)) {
    set_error("max_cols must lie in [1, 32]");
    return MQ_INVALID;
  }
  if (!(cfg->rel_tol > 0.0) || cfg->abs_tol < 0.0 || cfg->max_iter < 1) {
    set_error("invalid PCG configuration");
    return MQ_INVALID;
  }
  MQ_CUDA(cudaSetDevice(ctx->device));
  slab_step_free(ctx);
  SlabStepHost *s = new SlabStepHost();
  ctx->sstep = s;
  s->cfg = *cfg;
  s->ilo = ctx->slab_lo;
  s->ihi = ctx->slab_hi;
  s->kb = cfg->max_cols <= 8 ? 8 : (cfg->max_cols <= 16 ? 16 : 32);
  int rc = MQ_OK;
  const Lay &Ls = ctx->topo.L;
  const size_t vb = sizeof(double) * Ls.total;
  // ---- conducting block of the full grid (host topology, freed below) ----
  {
    Topology full;
    std::string err;
    rc = build_topology(ctx->desc, full, err);
    if (rc) { set_error(err); slab_step_free(ctx); return rc; }
    const Lay &Lf = full.L;
    if (Lf.Si != Ls.Si || Lf.Sj != Ls.Sj) { set_error("internal: slab / grid strides differ"); slab_step_free(ctx); return MQ_INVALID; }
    s->n_c = (int64_t)full.c_pad.size();
    s->n_cells = full.n_cells_c;
    auto to_slab = [&](int64_t e, int64_t *out) -> bool {
      const PadSplit p = split_pad(Lf, e);
      const int64_t li = p.i - s->ilo;
      if (li < -1 || li > s->ihi - s->ilo) return false;
      *out = p.c * Ls.C + (li + 1) * Ls.Si + p.jk;
      return true;
    };
    // owned conducting edges: node plane in [ilo, ihi)
    std::vector<int32_t> own;
    std::vector<int64_t> optr(1, 0);
    std::vector<int32_t> ocol;
    std::vector<int8_t> osgn;
    for (int64_t e = 0; e < s->n_c; ++e) {
      const PadSplit p = split_pad(Lf, full.c_pad[e]);
      if (p.i < s->ilo || p.i >= s->ihi) continue;
      own.push_back((int32_t)e);
      s->h_own.push_back(e);
      for (int64_t q = full.kcn_ptr[e]; q < full.kcn_ptr[e + 1]; ++q) {
        int64_t col;
        if (!to_slab(full.kcn_col[q], &col)) {
          set_error("internal: K_cn row reaches beyond the ghost planes");
          slab_step_free(ctx);
          return MQ_INVALID;
        }
        ocol.push_back((int32_t)col);
        osgn.push_back(full.kcn_sgn[q]);
      }
      optr.push_back((int64_t)ocol.size());
    }
    s->n_own = (int64_t)own.size();
    // K_cn^T rows of owned dofs
    std::vector<int32_t> krow, ksrc;
    std::vector<int64_t> kptr(1, 0);
    std::vector<int8_t> ksgn;
    for (size_t r = 0; r < full.kcnt_row.size(); ++r) {
      const PadSplit p = split_pad(Lf, full.kcnt_row[r]);
      if (p.i < s->ilo || p.i >= s->ihi) continue;
      int64_t row;
      to_slab(full.kcnt_row[r], &row);
      krow.push_back((int32_t)row);
      for (int64_t q = full.kcnt_ptr[r]; q < full.kcnt_ptr[r + 1]; ++q) {
        ksrc.push_back(full.kcnt_src[q]);
        ksgn.push_back(full.kcnt_sgn[q]);
      }
      kptr.push_back((int64_t)ksrc.size());
    }
    s->n_kt = (int64_t)krow.size();
    std::vector<double> minv(full.mc_diag.size());
    for (size_t q = 0; q < minv.size(); ++q) minv[q] = 1.0 / full.mc_diag[q];  // schur.py:212
    CondArgs &a = s->ca;
    a.n_c = s->n_c;
    a.n_cells = s->n_cells;
    a.n_rows_t = 0;
    a.kcn_ptr = nullptr; a.kcn_col = nullptr; a.kcn_sgn = nullptr;
    a.kcnt_row = nullptr; a.kcnt_ptr = nullptr; a.kcnt_src = nullptr; a.kcnt_sgn = nullptr;
    rc = rc ? rc : ss_up(ctx, s, (int32_t **)&a.f_edge, full.f_edge);
    rc = rc ? rc : ss_up(ctx, s, (int8_t **)&a.f_sgn, full.f_sgn);
    rc = rc ? rc : ss_up(ctx, s, (double **)&a.f_base, full.f_base);
    rc = rc ? rc : ss_up(ctx, s, (int32_t **)&a.f_cell, full.f_cell);
    rc = rc ? rc : ss_up(ctx, s, (int32_t **)&a.cell_face, full.cell_face);
    rc = rc ? rc : ss_up(ctx, s, (int32_t **)&a.e_face, full.e_face);
    rc = rc ? rc : ss_up(ctx, s, (int8_t **)&a.e_sgn, full.e_sgn);
    rc = rc ? rc : ss_up(ctx, s, (double **)&a.minv, minv);
    a.of = ctx->kn_off;
    a.h = ctx->desc.h;
    a.two_h4 = 2.0 * std::pow(ctx->desc.h, 4.0);
    a.k1 = ctx->desc.brauer_k1; a.k2 = ctx->desc.brauer_k2; a.k3 = ctx->desc.brauer_k3;
    a.linear = ctx->desc.brauer_k1 == 0.0;
    rc = rc ? rc : ss_up(ctx, s, &s->d_own, own);
    rc = rc ? rc : ss_up(ctx, s, &s->d_okcn_ptr, optr);
    rc = rc ? rc : ss_up(ctx, s, &s->d_okcn_col, ocol);
    rc = rc ? rc : ss_up(ctx, s, &s->d_okcn_sgn, osgn);
    rc = rc ? rc : ss_up(ctx, s, &s->d_kt_row, krow);
    rc = rc ? rc : ss_up(ctx, s, &s->d_kt_ptr, kptr);
    rc = rc ? rc : ss_up(ctx, s, &s->d_kt_src, ksrc);
    rc = rc ? rc : ss_up(ctx, s, &s->d_kt_sgn, ksgn);
    // the host topology must outlive the asynchronous uploads
    if (!rc) {
      cudaError_t e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) rc = cuda_fail(e, "slab step topology upload");
    }
  }
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_ac, sizeof(double) * s->n_c);
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_nu, sizeof(double) * s->n_cells);
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_own_out, sizeof(double) * s->n_own);
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_err, sizeof(unsigned int));
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_fam, sizeof(FamDev) * 3);
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_part, sizeof(double) * RQ);
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_tot, sizeof(double) * RQ);
  auto vec = [&](double **p) { if (!rc) rc = ss_zalloc(ctx, s, (void **)p, vb); };
  auto table = [&](double ***tab, std::vector<double *> &h, int n) {
    if (rc) return;
    h.assign(MAXS, nullptr);
    for (int q = 0; q < n && !rc; ++q) vec(&h[q]);
    if (rc) return;
    rc = ss_zalloc(ctx, s, (void **)tab, sizeof(double *) * MAXS);
    if (!rc) {
      cudaError_t e = cudaMemcpyAsync(*tab, h.data(), sizeof(double *) * MAXS, cudaMemcpyHostToDevice, ctx->stream);
      if (e != cudaSuccess) rc = cuda_fail(e, "slot table");
    }
  };
  for (int fam = 0; fam < 3; ++fam) {
    if (cfg->strategy == MQ_STRAT_CSPE) {
      table(&s->d_U[fam], s->h_U[fam], cfg->max_cols);
      table(&s->d_KU[fam], s->h_KU[fam], cfg->max_cols);
    } else if (cfg->strategy == MQ_STRAT_PREVIOUS) {
      vec(&s->last[fam]);
    }
  }
  vec(&s->rhs_src);
  vec(&s->rhs_cpl);
  vec(&s->y_src);
  vec(&s->y_cpl);
  vec(&s->y_cur);
  vec(&s->w1);
  vec(&s->w2);
  vec(&s->dvec);
  s->red_grid = std::max(1, std::min<int>(ctx->sms * 2, (int)((Ls.words + kWarps - 1) / kWarps)));
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_red, sizeof(double) * RQ * (size_t)s->red_grid);
  rc = rc ? rc : ss_zalloc(ctx, s, (void **)&s->d_cnt, sizeof(unsigned int) * 4);
  if (!rc) {
    s->h_part_len = std::max<int64_t>(RQ, s->n_own);
    cudaError_t e = cudaMallocHost((void **)&s->h_part, sizeof(double) * s->h_part_len);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMallocHost");
  }
  if (!rc && pattern_local) {
    std::vector<int32_t> idx;
    std::vector<double> val;
    const auto &pad = ctx->topo.nc_pad;
    for (size_t q = 0; q < pad.size(); ++q)
      if (pattern_local[q] != 0.0) { idx.push_back(pad[q]); val.push_back(pattern_local[q]); }
    s->n_pat = (int64_t)idx.size();
    rc = ss_up(ctx, s, &s->d_pat_idx, idx);
    rc = rc ? rc : ss_up(ctx, s, &s->d_pat_val, val);
  }
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "slab step init");
  }
  if (rc) slab_step_free(ctx);
  return rc;
}

// out4 = {n_c (full grid), owned conducting edges, conductor cells, K_cn^T rows of the slab}
int mq_ss_info(mq_ctx *ctx, int64_t *out4) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  out4[0] = s->n_c;
  out4[1] = s->n_own;
  out4[2] = s->n_cells;
  out4[3] = s->n_kt;
  return MQ_OK;
}

int mq_ss_owned(mq_ctx *ctx, int64_t *idx) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  std::memcpy(idx, ctx->sstep->h_own.data(), sizeof(int64_t) * ctx->sstep->h_own.size());
  return MQ_OK;
}

// named device vectors of the step (slab layout): 0 rhs_src, 1 rhs_cpl,
// 2 y_src, 3 y_cpl, 4 y_cur, 5 w2 (CGS vector, halo before K u), 6 dvec
// (y_cpl - y_src, halo before the Euler update)
int mq_ss_vec(mq_ctx *ctx, int32_t which, double **out) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  double *v[7] = {s->rhs_src, s->rhs_cpl, s->y_src, s->y_cpl, s->y_cur, s->w2, s->dvec};
  if (which < 0 || which > 6) { set_error("unknown slab step vector"); return MQ_INVALID; }
  *out = v[which];
  return MQ_OK;
}

int mq_ss_state_set(mq_ctx *ctx, const double *a_c) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  MQ_CUDA(cudaMemcpyAsync(s->d_ac, a_c, sizeof(double) * s->n_c, cudaMemcpyHostToDevice, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

int mq_ss_state_get(mq_ctx *ctx, double *a_c) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  MQ_CUDA(cudaMemcpyAsync(a_c, s->d_ac, sizeof(double) * s->n_c, cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

// which = 0: rhs_src = pattern * wave (schur.py:81-82); 1: rhs_cpl = K_cn^T a_c
int mq_ss_rhs(mq_ctx *ctx, int32_t which, double wave) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  if (which == 0) {
    if (s->n_pat) {
      k_ss_src<<<ss_grid_for(ctx, s->n_pat), 256, 0, ctx->stream>>>(s->n_pat, s->d_pat_idx, s->d_pat_val, wave,
                                                                     s->rhs_src);
      LAUNCH_CHECK();
    }
  } else {
    if (s->n_kt) {
      k_ss_kcnt<<<ss_grid_for(ctx, s->n_kt), 256, 0, ctx->stream>>>(s->n_kt, s->d_kt_row, s->d_kt_ptr, s->d_kt_src,
                                                                     s->d_kt_sgn, ctx->kn_off, s->d_ac, s->rhs_cpl);
      LAUNCH_CHECK();
    }
  }
  return MQ_OK;
}

// start vector, part 1 (startvec.py:207-225): this rank's beta = U^T rhs
int mq_ss_project(mq_ctx *ctx, int32_t fam, int32_t rhs_which, double *part) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  if (fam < 0 || fam > 2) { set_error("unknown RHS family"); return MQ_INVALID; }
  std::fill(part, part + RQ, 0.0);
  if (s->cfg.strategy != MQ_STRAT_CSPE) return MQ_OK;
  FamDev *f = s->d_fam + fam;
  const Lay &L = ctx->topo.L;
  const double *rhs = rhs_which == 0 ? s->rhs_src : s->rhs_cpl;
  KB_LAUNCH(s->kb, k_mdot, s->red_grid, kBlock, ctx->stream, L.total / 2, s->d_U[fam], f->order, &f->k, rhs, 0,
            s->d_part, s->d_red, s->d_cnt, Post(), nullptr);
  LAUNCH_CHECK();
  return ss_fetch(ctx, part, RQ);
}

// start vector, part 2: the projected solve on the all-reduced beta (with the
// reference's pivot-drop retry), x0 = U c into x (every entry written)
int mq_ss_start(mq_ctx *ctx, int32_t fam, const double *tot, double *x_dev) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  if (fam < 0 || fam > 2) { set_error("unknown RHS family"); return MQ_INVALID; }
  const Lay &L = ctx->topo.L;
  FamDev *f = s->d_fam + fam;
  switch (s->cfg.strategy) {
    case MQ_STRAT_CSPE:
      rc = ss_post(ctx, fam, POST_PROJECT, tot);
      if (rc) return rc;
      KB_LAUNCH(s->kb, k_comb, s->red_grid, kBlock, ctx->stream, L.total / 2, s->d_U[fam], f->order, &f->k, f->coef,
                x_dev);
      LAUNCH_CHECK();
      break;
    case MQ_STRAT_PREVIOUS:
      MQ_CUDA(cudaMemsetAsync(x_dev, 0, sizeof(double) * L.total, ctx->stream));
      if (s->has_last[fam]) {
        k_copy<<<ss_stream_grid(ctx), kBlock, 0, ctx->stream>>>(L, ctx->d_mask, s->last[fam], x_dev);
        LAUNCH_CHECK();
      }
      break;
    default:
      MQ_CUDA(cudaMemsetAsync(x_dev, 0, sizeof(double) * L.total, ctx->stream));
      break;
  }
  return MQ_OK;
}

// the solve's result x (owned rows) into the family's solution vector; ghost
// planes of the solution vectors stay 0
int mq_ss_store(mq_ctx *ctx, int32_t fam, const double *x_dev, const mq_solve_report *rep) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  if (fam < 0 || fam > 2) { set_error("unknown RHS family"); return MQ_INVALID; }
  k_copy<<<ss_stream_grid(ctx), kBlock, 0, ctx->stream>>>(ctx->topo.L, ctx->d_mask, x_dev, ss_y(s, fam));
  LAUNCH_CHECK();
  if (rep) {
    s->solves[fam] += 1;
    s->iterations[fam] += rep->iterations;
    s->pcg_applies += rep->applies;
  }
  return MQ_OK;
}

// cache update of one family with its last solution (startvec.py:158-199),
// in phases separated by the host's all-reduce of `part` into `tot`:
//   0: part = [U^T y, y.y]
//   1: gate on tot (zero / non-finite), CGS pass 1 -> part = [U^T w1, w1.w1]
//   2: CGS pass 2 -> part = [w2.w2]
//   3: drop test / eviction / slot; *flag = accepted (the host then refreshes
//      the ghost planes of w2 when accepted)
//   4: u = w2/||w2||, K u, part = [U^T K u, u.K u]
//   5: bordered Galerkin commit
// previous strategy: phase 0 stores the solution, nothing else.
int mq_ss_observe(mq_ctx *ctx, int32_t fam, int32_t phase, const double *tot, double *part, int32_t *flag) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  if (fam < 0 || fam > 2) { set_error("unknown RHS family"); return MQ_INVALID; }
  const Lay &L = ctx->topo.L;
  cudaStream_t st = ctx->stream;
  const int G = s->red_grid;
  const double *y = ss_y(s, fam);
  if (part) std::fill(part, part + RQ, 0.0);
  if (flag) *flag = 0;
  if (s->cfg.strategy == MQ_STRAT_PREVIOUS) {
    if (phase == 0) {
      k_copy<<<ss_stream_grid(ctx), kBlock, 0, st>>>(L, ctx->d_mask, y, s->last[fam]);
      LAUNCH_CHECK();
      s->has_last[fam] = true;
    }
    return MQ_OK;
  }
  if (s->cfg.strategy != MQ_STRAT_CSPE) return MQ_OK;
  FamDev *f = s->d_fam + fam;
  switch (phase) {
    case 0:
      KB_LAUNCH(s->kb, k_mdot, G, kBlock, st, L.total / 2, s->d_U[fam], f->order, &f->k, y, 1, s->d_part, s->d_red,
                s->d_cnt, Post(), nullptr);
      LAUNCH_CHECK();
      return ss_fetch(ctx, part, RQ);
    case 1:
      rc = ss_post(ctx, fam, POST_GATE, tot);
      if (rc) return rc;
      KB_LAUNCH(s->kb, k_axpy_dots, G, kBlock, st, L.total / 2, s->d_U[fam], f->order, &f->k, f->coef, y, s->w1, 1,
                s->d_part, s->d_red, s->d_cnt, &f->accept, Post());
      LAUNCH_CHECK();
      return ss_fetch(ctx, part, RQ);
    case 2:
      rc = ss_post(ctx, fam, POST_GATE_C2, tot);
      if (rc) return rc;
      KB_LAUNCH(s->kb, k_axpy_dots, G, kBlock, st, L.total / 2, s->d_U[fam], f->order, &f->k, f->coef, s->w1, s->w2,
                0, s->d_part, s->d_red, s->d_cnt, &f->accept, Post());
      LAUNCH_CHECK();
      return ss_fetch(ctx, part, RQ);
    case 3: {
      rc = ss_post(ctx, fam, POST_DECIDE, tot);
      if (rc) return rc;
      MQ_CUDA(cudaMemcpyAsync(s->h_part, &f->accept, sizeof(int), cudaMemcpyDeviceToHost, st));
      MQ_CUDA(cudaStreamSynchronize(st));
      int acc;
      std::memcpy(&acc, s->h_part, sizeof(int));
      if (flag) *flag = acc;
      return MQ_OK;
    }
    case 4:
      KB_LAUNCH(s->kb, k_cspe_product, G, kBlock, st, L, ctx->d_mask, ctx->kn_diag, ctx->kn_off, f, s->d_U[fam],
                s->d_KU[fam], s->w2, s->d_red, s->d_cnt, Post());
      LAUNCH_CHECK();
      // k_cspe_product reduces into f->d (its fixed output): hand the
      // partials to the host from there
      MQ_CUDA(cudaMemcpyAsync(s->d_part, f->d, sizeof(double) * RQ, cudaMemcpyDeviceToDevice, st));
      return ss_fetch(ctx, part, RQ);
    case 5:
      return ss_post(ctx, fam, POST_COMMIT, tot);
    default:
      set_error("unknown observe phase");
      return MQ_INVALID;
  }
}

// dvec = y_cpl - y_src on the owned rows (the host then refreshes its ghost planes)
int mq_ss_euler_prep(mq_ctx *ctx) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  k_sub<<<ss_stream_grid(ctx), kBlock, 0, ctx->stream>>>(ctx->topo.L, ctx->d_mask, s->y_cpl, s->y_src, s->dvec);
  LAUNCH_CHECK();
  // the halo exchange that follows runs on another stream
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return MQ_OK;
}

// Brauer nu of every conductor cell, then the Euler update of the owned
// conducting edges -> owned_out (n_own values, owned order of mq_ss_owned);
// MQ_NONFINITE when one of them is not finite (schur.py:400-404)
int mq_ss_euler(mq_ctx *ctx, double dt, double *owned_out) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  cudaStream_t st = ctx->stream;
  MQ_CUDA(cudaMemsetAsync(s->d_err, 0, sizeof(unsigned int), st));
  if (s->n_cells) {
    k_cell_nu<<<ss_grid_for(ctx, s->n_cells), 256, 0, st>>>(s->ca, s->d_ac, s->d_nu);
    LAUNCH_CHECK();
  }
  if (s->n_own) {
    k_ss_euler<<<ss_grid_for(ctx, s->n_own), 256, 0, st>>>(s->ca, s->n_own, s->d_own, s->d_okcn_ptr, s->d_okcn_col,
                                                           s->d_okcn_sgn, s->d_nu, s->d_ac, s->dvec, dt, s->d_own_out,
                                                           s->d_err);
    LAUNCH_CHECK();
    MQ_CUDA(cudaMemcpyAsync(s->h_part, s->d_own_out, sizeof(double) * s->n_own, cudaMemcpyDeviceToHost, st));
  }
  MQ_CUDA(cudaStreamSynchronize(st));
  unsigned int err = 0;
  MQ_CUDA(cudaMemcpy(&err, s->d_err, sizeof(unsigned int), cudaMemcpyDeviceToHost));
  if (s->n_own) std::memcpy(owned_out, s->h_part, sizeof(double) * s->n_own);
  if (err) { set_error("non-finite conducting state"); return MQ_NONFINITE; }
  return MQ_OK;
}

// a_n = y_src - y_cur of the last recovery on the slab's own dofs (compact
// slab order, schur.py:408-419)
int mq_ss_an(mq_ctx *ctx, double *a_n_local) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  k_sub<<<ss_stream_grid(ctx), kBlock, 0, ctx->stream>>>(ctx->topo.L, ctx->d_mask, s->y_src, s->y_cur, s->w1);
  LAUNCH_CHECK();
  return mq_vec_download(ctx, s->w1, a_n_local);
}

// CSPE cache of one family on this slab: k, basis / products on the slab's
// own dofs (slab compact order, column-major n_n x k), the Galerkin matrix
int mq_ss_cspe_export(mq_ctx *ctx, int32_t family, int32_t *k, double *basis, double *products, double *galerkin) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  if (s->cfg.strategy != MQ_STRAT_CSPE || family < 0 || family > 2) { set_error("CSPE family expected"); return MQ_INVALID; }
  FamDev f;
  MQ_CUDA(cudaMemcpyAsync(&f, s->d_fam + family, sizeof(FamDev), cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  *k = f.k;
  const int64_t n = (int64_t)ctx->topo.nc_pad.size();
  for (int j = 0; j < f.k; ++j) {
    if (basis && (rc = mq_vec_download(ctx, s->h_U[family][f.order[j]], basis + j * n))) return rc;
    if (products && (rc = mq_vec_download(ctx, s->h_KU[family][f.order[j]], products + j * n))) return rc;
  }
  if (galerkin)
    for (int r = 0; r < f.k; ++r)
      for (int c = 0; c < f.k; ++c) galerkin[r * f.k + c] = f.G[r * MAXS + c];
  return MQ_OK;
}

int mq_ss_diag(mq_ctx *ctx, mq_diag *out) {
  int rc = ss_check(ctx);
  if (rc) return rc;
  SlabStepHost *s = ctx->sstep;
  FamDev h[3];
  MQ_CUDA(cudaMemcpyAsync(h, s->d_fam, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  MQ_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memset(out, 0, sizeof(*out));
  for (int q = 0; q < 3; ++q) {
    out->solves[q] = s->solves[q];
    out->iterations[q] = s->iterations[q];
    out->basis_cols[q] = h[q].k;
    out->columns_accepted[q] = h[q].accepted;
    out->columns_dropped[q] = h[q].dropped;
    out->evictions[q] = h[q].evictions;
    out->maintenance_applies += h[q].products;
  }
  out->pcg_applies = s->pcg_applies;
  out->min_pod_info = 1.0;
  out->pod_info = 1.0;
  return MQ_OK;
}

}  // extern "C"

// Device-resident CSR operator for models given as matrices: the reference's
// manifest path (bench.py:228-313 load_model, model.py:640-689 export_model)
// yields a PartitionedSystem of CSR blocks (K_n, K_cn, K_c, M_c) with no grid
// behind it.  The block is uploaded once; every PCG solve (krylov.py:174-250
// through pcg_csr_kernel, pcg.cu) and SpMV (sparse.py:179-184) reuses it.
// Vectors are host arrays in the block's own row order (one stream, one
// synchronisation per call).
#include <cstring>

#include "mq_ctx.h"
#include "mq_internal.h"

struct mq_csr_op {
  int device = 0;
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int64_t *rp = nullptr;
  int32_t *ci = nullptr;
  double *va = nullptr, *inv = nullptr;
  double *b = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *ap = nullptr;
  double *partials = nullptr;
  mq::GridBar *bar = nullptr;
  mq::PcgOut *out = nullptr, *h_out = nullptr;
  int grid = 1, sms = 148;
  cudaStream_t stream = nullptr;
};

namespace {

using namespace mq;

void op_free(mq_csr_op *op) {
  if (!op) return;
  void *dev[] = {op->rp, op->ci, op->va, op->inv, op->b, op->x, op->r, op->p, op->ap, op->partials, op->bar, op->out};
  for (void *q : dev)
    if (q) cudaFree(q);
  if (op->h_out) cudaFreeHost(op->h_out);
  if (op->stream) cudaStreamDestroy(op->stream);
  delete op;
}

int op_alloc(void **p, size_t bytes) {
  MQ_CUDA(cudaMalloc(p, bytes));
  MQ_CUDA(cudaMemset(*p, 0, bytes));
  return MQ_OK;
}

}  // namespace

extern "C" {

int mq_csr_op_create(int32_t device, int64_t nrows, int64_t ncols, const int64_t *row_ptr, const int32_t *col_idx,
                     const double *values, const double *inv_diag, mq_csr_op **out) {
  if (!out || nrows < 0 || ncols < 0 || !row_ptr) { set_error("invalid CSR operator arguments"); return MQ_INVALID; }
  *out = nullptr;
  const int64_t nnz = row_ptr[nrows];
  if (row_ptr[0] != 0 || nnz < 0 || (nnz > 0 && (!col_idx || !values))) {
    set_error("invalid CSR row pointers");
    return MQ_INVALID;
  }
  for (int64_t i = 0; i < nrows; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) { set_error("CSR row pointers decrease"); return MQ_INVALID; }
  for (int64_t k = 0; k < nnz; ++k)
    if (col_idx[k] < 0 || col_idx[k] >= ncols) { set_error("CSR column index out of range"); return MQ_INVALID; }
  MQ_CUDA(cudaSetDevice(device));
  mq_csr_op *op = new mq_csr_op;
  op->device = device;
  op->nrows = nrows;
  op->ncols = ncols;
  op->nnz = nnz;
  const size_t vr = sizeof(double) * (size_t)std::max<int64_t>(nrows, 1);
  const size_t vc = sizeof(double) * (size_t)std::max<int64_t>(ncols, 1);
  int rc = MQ_OK;
  auto A = [&](void **p, size_t bytes) { if (!rc) rc = op_alloc(p, bytes); };
  A((void **)&op->rp, sizeof(int64_t) * (size_t)(nrows + 1));
  A((void **)&op->ci, sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1));
  A((void **)&op->va, sizeof(double) * (size_t)std::max<int64_t>(nnz, 1));
  A((void **)&op->b, vr);
  A((void **)&op->x, std::max(vr, vc));
  A((void **)&op->r, vr);
  A((void **)&op->p, vr);
  A((void **)&op->ap, vr);
  if (inv_diag) A((void **)&op->inv, vr);
  if (!rc) rc = pcg_csr_grid(std::max<int64_t>(nrows, 1), &op->grid);
  A((void **)&op->partials, sizeof(double) * 8 * (size_t)op->grid);
  A((void **)&op->bar, sizeof(GridBar));
  A((void **)&op->out, sizeof(PcgOut));
  if (!rc) {
    cudaError_t e = cudaMallocHost((void **)&op->h_out, sizeof(PcgOut));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&op->sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaMemcpy(op->rp, row_ptr, sizeof(int64_t) * (size_t)(nrows + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz > 0) e = cudaMemcpy(op->ci, col_idx, sizeof(int32_t) * (size_t)nnz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz > 0) e = cudaMemcpy(op->va, values, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && inv_diag && nrows > 0)
      e = cudaMemcpy(op->inv, inv_diag, sizeof(double) * (size_t)nrows, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) rc = cuda_fail(e, "CSR operator upload");
  }
  if (rc) {
    op_free(op);
    return rc;
  }
  *out = op;
  return MQ_OK;
}

int mq_csr_op_destroy(mq_csr_op *op) {
  op_free(op);
  return MQ_OK;
}

// pcg_solve(a=CsrMatrix, b, x0, config, preconditioner) with the block on the
// device: use_inv selects the Jacobi inverse given at creation.
int mq_csr_op_pcg(mq_csr_op *op, const double *b, const double *x0, double *x, int32_t use_inv, double rel_tol,
                  double abs_tol, int32_t max_iter, mq_solve_report *rep) {
  if (!op || !b || !x) { set_error("invalid CSR PCG arguments"); return MQ_INVALID; }
  if (op->nrows != op->ncols) { set_error("PCG needs a square operator"); return MQ_INVALID; }
  if (!(rel_tol > 0.0) || abs_tol < 0.0 || max_iter < 1) { set_error("invalid PCG configuration"); return MQ_INVALID; }
  if (use_inv && !op->inv) { set_error("no Jacobi inverse was given at creation"); return MQ_INVALID; }
  MQ_CUDA(cudaSetDevice(op->device));
  const int64_t n = op->nrows;
  const size_t vb = sizeof(double) * (size_t)n;
  cudaStream_t s = op->stream;
  if (n > 0) {
    MQ_CUDA(cudaMemcpyAsync(op->b, b, vb, cudaMemcpyHostToDevice, s));
    // pcg_csr_kernel takes x as the start iterate; no x0 means x = 0 (the
    // buffer also carries SpMV inputs)
    if (x0) MQ_CUDA(cudaMemcpyAsync(op->x, x0, vb, cudaMemcpyHostToDevice, s));
    else MQ_CUDA(cudaMemsetAsync(op->x, 0, vb, s));
  }
  CsrPcgArgs a{};
  a.n = n;
  a.rp = op->rp;
  a.ci = op->ci;
  a.va = op->va;
  a.inv = use_inv ? op->inv : nullptr;
  a.has_x0 = x0 != nullptr;
  a.b = op->b;
  a.x = op->x;
  a.r = op->r;
  a.p = op->p;
  a.ap = op->ap;
  a.rel_tol = rel_tol;
  a.abs_tol = abs_tol;
  a.max_iter = max_iter;
  a.partials = op->partials;
  a.bar = op->bar;
  a.out = op->out;
  int rc = launch_pcg_csr(a, op->grid, s);
  if (rc) return rc;
  MQ_CUDA(cudaMemcpyAsync(op->h_out, op->out, sizeof(PcgOut), cudaMemcpyDeviceToHost, s));
  if (n > 0) MQ_CUDA(cudaMemcpyAsync(x, op->x, vb, cudaMemcpyDeviceToHost, s));
  MQ_CUDA(cudaStreamSynchronize(s));
  const PcgOut &o = *op->h_out;
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
  if (o.status == MQ_CUDA_ERROR) { set_error("grid barrier watchdog expired in the CSR PCG kernel"); return MQ_CUDA_ERROR; }
  return o.status;
}

// y = A x (sparse.py:179-184; csr_spmv_kernel sums each row in CSR order)
int mq_csr_op_spmv(mq_csr_op *op, const double *x, double *y) {
  if (!op || (op->ncols > 0 && !x) || (op->nrows > 0 && !y)) { set_error("invalid CSR SpMV arguments"); return MQ_INVALID; }
  MQ_CUDA(cudaSetDevice(op->device));
  cudaStream_t s = op->stream;
  if (op->ncols > 0) MQ_CUDA(cudaMemcpyAsync(op->x, x, sizeof(double) * (size_t)op->ncols, cudaMemcpyHostToDevice, s));
  int rc = launch_csr_spmv(op->nrows, op->rp, op->ci, op->va, op->x, op->ap, op->sms, s);
  if (rc) return rc;
  if (op->nrows > 0) MQ_CUDA(cudaMemcpyAsync(y, op->ap, sizeof(double) * (size_t)op->nrows, cudaMemcpyDeviceToHost, s));
  MQ_CUDA(cudaStreamSynchronize(s));
  return MQ_OK;
}

}  // extern "C"

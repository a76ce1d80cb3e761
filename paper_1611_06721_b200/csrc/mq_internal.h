// Internal declarations of libmq_b200 (not part of the C ABI).
//
// Device layout ("padded edge layout"): the three edge components x, y, z
// each occupy one box of nodes i = -1..nx, j = -1..ny, k = -1..nz(+pad),
// k fastest, the box length rounded up to a multiple of 32 (one 32-bit mask
// word per warp).  Component c starts at c*C; node (i,j,k) sits at
// c*C + off + i*Si + j*Sj + k with Sj = nz+2 rounded up to even and
// Si = (ny+2)*Sj (see topology.cpp).  Within a component the box order is the reference's
// global edge order (model.py:186-207: ids are C-order with k fastest), so the
// compact K_n order (ascending global id, model.py:455-464) is exactly the
// order of active positions in a linear scan of the device layout.  Entries
// that are not K_n dofs (PEC boundary, conducting, box padding) hold 0 in
// every device vector and are never written.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/mq_b200.h"

namespace mq {

struct Lay {
  int64_t C;      // padded component length (multiple of 32)
  int64_t Si, Sj; // strides inside a component
  int64_t off;    // index of node (0,0,0) inside a component (guard layer)
  int64_t total;  // 3*C
  int64_t words;  // total/32 mask words
};

struct GridBar {
  unsigned long long count;  // monotonic arrivals; zeroed before every launch
  unsigned int error;
  unsigned int pad;
};

// Device-side record of one PCG solve (krylov.py:75-79 + counters).
struct PcgOut {
  int32_t iterations;
  int32_t converged;
  int32_t status;      // MQ_OK / MQ_NOT_CONVERGED / MQ_INDEFINITE / MQ_CUDA_ERROR
  int32_t applies;
  double rel;
  double bnorm;
  double alpha, rz;    // last scalars (diagnostics)
};

struct StencilPcgArgs {
  Lay L;
  const uint32_t *mask;
  double dg, of, inv;
  int use_jac;
  int x0_mode;  // 0: x0 == 0 (r = b, one application counted), 1: x holds x0, 2: no x0
  const double *b;
  double *x, *r, *pa, *pb, *ap;
  double rel_tol, abs_tol;
  int max_iter;
  double *partials;  // 6*G: init [0,3G), p.Ap [3G,4G), r.r/r.z [4G,6G)
  GridBar *bar;
  PcgOut *out;
  const int *x0_mode_dev;      // optional: device-chosen start mode
  const unsigned int *err_word;  // optional: skip the solve if set
  unsigned long long *trace;   // optional: %globaltimer stamps (CTA 0) per phase
  double *ap2;                 // second Ap buffer (pcg_resident1_kernel publishes Ap double-buffered)
  double *r2;                  // second r buffer (pcg_tma1_kernel keeps r double-buffered)
  int stress_ns;               // test only (MQ_PCG_STRESS): some CTAs sleep after each grid barrier
};

// Brick decomposition of the node box [0,nx) x [0,ny) x [0,nz) (pcg_brick.cu)
struct BrickGeo {
  int nx, ny, nz;
  int tiles_k, tiles_j, chunks;
  int nbricks;
  // mixed chunking (make_geo, one-barrier kernel): tiles [0, xtiles) are cut
  // into chunks + 1 i-chunks, the others into chunks; bricks [0, nbig) are
  // the longer ones (0 / nbricks: every tile in `chunks`)
  int xtiles, nbig;
};

struct CsrPcgArgs {
  int64_t n;
  const int64_t *rp;
  const int32_t *ci;
  const double *va;
  const double *inv;  // NULL: no preconditioner
  int has_x0;
  const double *b;
  double *x, *r, *p, *ap;
  double rel_tol, abs_tol;
  int max_iter;
  double *partials;
  GridBar *bar;
  PcgOut *out;
};

void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define MQ_CUDA(call)                                     \
  do {                                                    \
    cudaError_t e__ = (call);                             \
    if (e__ != cudaSuccess) return ::mq::cuda_fail(e__, #call); \
  } while (0)

// Host-built topology of the partition and of the conducting block.
struct Topology {
  int nx, ny, nz;
  Lay L;
  std::vector<uint32_t> mask;          // active K_n dofs, bit per padded entry
  std::vector<int32_t> nc_pad;         // compact noncond index -> padded index
  std::vector<int64_t> nc_global;      // compact noncond index -> global edge id
  std::vector<int64_t> c_global;       // compact cond index -> global edge id
  std::vector<int32_t> c_pad;          // compact cond index -> padded index
  // K_cn (n_c rows, columns = padded noncond positions ascending), sign +-1
  std::vector<int64_t> kcn_ptr;
  std::vector<int32_t> kcn_col;
  std::vector<int8_t> kcn_sgn;
  // K_cn^T gather: for every touched noncond padded index, its cond rows
  std::vector<int32_t> kcnt_row;       // padded noncond index per gather row
  std::vector<int64_t> kcnt_ptr;
  std::vector<int32_t> kcnt_src;       // cond compact index (ascending)
  std::vector<int8_t> kcnt_sgn;
  // M_c diagonal (model.py:486-491)
  std::vector<double> mc_diag;
  // Brauer structures (model.py:492-509)
  // faces touching >=1 conducting edge, ascending global face id
  std::vector<int32_t> f_edge;         // 4 per face: cond compact index or -1, ascending
  std::vector<int8_t> f_sgn;           // 4 per face
  std::vector<double> f_base;          // base face weight (air part)
  std::vector<int32_t> f_cell;         // 2 per face: conductor cell list index or -1
  std::vector<int32_t> cell_face;      // 6 per conductor cell: index into faces
  std::vector<int64_t> cell_ids;       // global cell id per conductor cell (ascending)
  std::vector<int32_t> e_face;         // 4 per cond edge: face index, ascending face id
  std::vector<int8_t> e_sgn;           // 4 per cond edge
  int64_t n_faces_c = 0, n_cells_c = 0;
};

int build_topology(const mq_grid_desc &d, Topology &t, std::string &err);
int build_slab_topology(const mq_grid_desc &d, int ilo, int ihi, Topology &t, std::string &err);

}  // namespace mq

// Host-side construction of the partition (bit-exact DoF numbering and region
// masks) and of the conducting-block index structures.
//
// Follows the reference's definitions (paths under pkg/src/mqsolve):
//   edge / face ids, C order with k fastest ........ model.py:186-207
//   curl incidence signs (+,+,-,-) ................. model.py:209-238
//   PEC boundary edges ............................. model.py:240-251
//   conducting rule (edge borders a conductor cell)  model.py:253-272, 460-462
//   edge-averaged conductivity, M_c ................ model.py:274-292, 486-491
//   face/cell averaging and base face weights ...... model.py:294-310, 474-478
//   cell -> six faces .............................. model.py:312-319
// Everything here is integer bookkeeping except M_c and the base face
// weights, which are evaluated in the reference's summation order.
#include <algorithm>
#include <cmath>

#include "mq_internal.h"

namespace mq {

namespace {

struct Dims {
  int nx, ny, nz;
  int64_t n_ex, n_ey, n_ez;
  int64_t n_fx, n_fy, n_fz;
};

inline int64_t gid_x(const Dims &d, int i, int j, int k) {
  return ((int64_t)i * (d.ny + 1) + j) * (d.nz + 1) + k;
}
inline int64_t gid_y(const Dims &d, int i, int j, int k) {
  return d.n_ex + ((int64_t)i * d.ny + j) * (d.nz + 1) + k;
}
inline int64_t gid_z(const Dims &d, int i, int j, int k) {
  return d.n_ex + d.n_ey + ((int64_t)i * (d.ny + 1) + j) * d.nz + k;
}
inline int64_t fid_x(const Dims &d, int i, int j, int k) {  // (nx+1, ny, nz)
  return ((int64_t)i * d.ny + j) * d.nz + k;
}
inline int64_t fid_y(const Dims &d, int i, int j, int k) {  // (nx, ny+1, nz)
  return d.n_fx + ((int64_t)i * (d.ny + 1) + j) * d.nz + k;
}
inline int64_t fid_z(const Dims &d, int i, int j, int k) {  // (nx, ny, nz+1)
  return d.n_fx + d.n_fy + ((int64_t)i * d.ny + j) * (d.nz + 1) + k;
}

}  // namespace

int build_topology(const mq_grid_desc &g, Topology &t, std::string &err) {
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  if (nx < 2 || ny < 2 || nz < 2) {
    err = "grid needs at least two cells per direction";
    return MQ_INVALID;
  }
  if (!(g.h > 0.0)) { err = "grid spacing must be positive"; return MQ_INVALID; }
  if (!g.material) { err = "material map is NULL"; return MQ_INVALID; }
  Dims d{nx, ny, nz, 0, 0, 0, 0, 0, 0};
  d.n_ex = (int64_t)nx * (ny + 1) * (nz + 1);
  d.n_ey = (int64_t)(nx + 1) * ny * (nz + 1);
  d.n_ez = (int64_t)(nx + 1) * (ny + 1) * nz;
  d.n_fx = (int64_t)(nx + 1) * ny * nz;
  d.n_fy = (int64_t)nx * (ny + 1) * nz;
  d.n_fz = (int64_t)nx * ny * (nz + 1);
  t.nx = nx; t.ny = ny; t.nz = nz;
  Lay &L = t.L;
  // One guard node on the low side of every axis (node index -1), so that
  // tile + halo boxes never start at a negative TMA coordinate, and the
  // k-pitch rounded up to even so that every row starts 16-byte aligned (TMA
  // global strides must be multiples of 16 B).  Guard / pad entries are never
  // dofs and hold 0.
  L.Sj = (nz + 3) & ~1;
  L.Si = (int64_t)(ny + 2) * L.Sj;
  L.off = L.Si + L.Sj + 1;
  const int64_t P = (int64_t)(nx + 2) * L.Si;
  L.C = (P + 31) / 32 * 32;
  L.total = 3 * L.C;
  L.words = L.total / 32;
  if (L.total >= ((int64_t)1 << 31)) {
    err = "grid too large for 32-bit device indexing";
    return MQ_INVALID;
  }

  const int8_t *mat = g.material;
  for (int64_t q = 0; q < (int64_t)nx * ny * nz; ++q)
    if (mat[q] < 0 || mat[q] > 2) { err = "material map holds unknown region ids"; return MQ_INVALID; }
  auto cond_cell = [&](int i, int j, int k) -> bool {
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return false;
    return mat[((int64_t)i * ny + j) * nz + k] == 1;
  };
  auto cell_kappa = [&](int i, int j, int k) -> double {
    return cond_cell(i, j, k) ? g.kappa : 0.0;
  };

  t.mask.assign(L.words, 0u);
  t.nc_pad.clear(); t.nc_global.clear(); t.c_global.clear(); t.c_pad.clear();
  t.mc_diag.clear();
  std::vector<int32_t> pad2cond(L.total, -1);
  std::vector<int32_t> pad2nc(L.total, -1);

  // scan components in global-id order; within a component the padded box
  // order (i, j, k) is the global order
  for (int c = 0; c < 3; ++c) {
    for (int i = 0; i <= nx; ++i)
      for (int j = 0; j <= ny; ++j)
        for (int k = 0; k <= nz; ++k) {
          bool exists, boundary, conducting;
          int64_t gid;
          double kap;
          if (c == 0) {
            exists = i < nx;
            if (!exists) continue;
            boundary = (j == 0 || j == ny || k == 0 || k == nz);
            conducting = cond_cell(i, j - 1, k - 1) || cond_cell(i, j - 1, k) ||
                         cond_cell(i, j, k - 1) || cond_cell(i, j, k);
            // edge_cell_mean view order (model.py:284-292): other axes (j,k)
            kap = (((cell_kappa(i, j - 1, k - 1) + cell_kappa(i, j - 1, k)) +
                    cell_kappa(i, j, k - 1)) + cell_kappa(i, j, k)) / 4.0;
            gid = gid_x(d, i, j, k);
          } else if (c == 1) {
            exists = j < ny;
            if (!exists) continue;
            boundary = (i == 0 || i == nx || k == 0 || k == nz);
            conducting = cond_cell(i - 1, j, k - 1) || cond_cell(i - 1, j, k) ||
                         cond_cell(i, j, k - 1) || cond_cell(i, j, k);
            kap = (((cell_kappa(i - 1, j, k - 1) + cell_kappa(i - 1, j, k)) +
                    cell_kappa(i, j, k - 1)) + cell_kappa(i, j, k)) / 4.0;
            gid = gid_y(d, i, j, k);
          } else {
            exists = k < nz;
            if (!exists) continue;
            boundary = (i == 0 || i == nx || j == 0 || j == ny);
            conducting = cond_cell(i - 1, j - 1, k) || cond_cell(i - 1, j, k) ||
                         cond_cell(i, j - 1, k) || cond_cell(i, j, k);
            kap = (((cell_kappa(i - 1, j - 1, k) + cell_kappa(i - 1, j, k)) +
                    cell_kappa(i, j - 1, k)) + cell_kappa(i, j, k)) / 4.0;
            gid = gid_z(d, i, j, k);
          }
          if (boundary) continue;
          const int64_t e = c * L.C + L.off + i * L.Si + j * L.Sj + k;
          if (conducting) {
            pad2cond[e] = (int32_t)t.c_global.size();
            t.c_global.push_back(gid);
            t.c_pad.push_back((int32_t)e);
            t.mc_diag.push_back(kap * g.h);
          } else {
            pad2nc[e] = (int32_t)t.nc_global.size();
            t.nc_global.push_back(gid);
            t.nc_pad.push_back((int32_t)e);
            t.mask[e >> 5] |= (1u << (e & 31));
          }
        }
  }
  if (t.c_global.empty()) { err = "no conducting edges were retained"; return MQ_INVALID; }
  for (double m : t.mc_diag)
    if (!(m > 0.0)) { err = "conducting edge with zero averaged conductivity"; return MQ_INVALID; }

  // ---- faces: four edges each with circulation signs (model.py:213-226) ----
  // Each face is described by padded indices of its 4 edges in the
  // reference's listing order with signs (+,+,-,-).
  const int64_t C = L.C, Si = L.Si, Sj = L.Sj;
  auto pidx = [&](int c, int i, int j, int k) -> int64_t { return c * C + L.off + i * Si + j * Sj + k; };
  auto face_edges = [&](int dir, int i, int j, int k, int64_t out[4]) {
    if (dir == 0) {        // fx(i,j,k): +ey[i,j,k], +ez[i,j+1,k], -ey[i,j,k+1], -ez[i,j,k]
      out[0] = pidx(1, i, j, k); out[1] = pidx(2, i, j + 1, k);
      out[2] = pidx(1, i, j, k + 1); out[3] = pidx(2, i, j, k);
    } else if (dir == 1) { // fy(i,j,k): +ez[i,j,k], +ex[i,j,k+1], -ez[i+1,j,k], -ex[i,j,k]
      out[0] = pidx(2, i, j, k); out[1] = pidx(0, i, j, k + 1);
      out[2] = pidx(2, i + 1, j, k); out[3] = pidx(0, i, j, k);
    } else {               // fz(i,j,k): +ex[i,j,k], +ey[i+1,j,k], -ex[i,j+1,k], -ey[i,j,k]
      out[0] = pidx(0, i, j, k); out[1] = pidx(1, i + 1, j, k);
      out[2] = pidx(0, i, j + 1, k); out[3] = pidx(1, i, j, k);
    }
  };
  const int8_t sgn4[4] = {1, 1, -1, -1};
  auto flat_cell = [&](int i, int j, int k) -> int64_t {
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return -1;
    return ((int64_t)i * ny + j) * nz + k;
  };

  // conductor cell list (ascending flat cell id, model.py:470)
  std::vector<int32_t> cell2list((size_t)nx * ny * nz, -1);
  std::vector<int64_t> cells;
  for (int64_t q = 0; q < (int64_t)nx * ny * nz; ++q)
    if (mat[q] == 1) { cell2list[q] = (int32_t)cells.size(); cells.push_back(q); }

  // faces with at least one conducting edge, ascending face id
  t.f_edge.clear(); t.f_sgn.clear(); t.f_base.clear(); t.f_cell.clear();
  std::vector<int64_t> face_id_of;     // face list -> global face id
  const double nu = g.nu_air;
  for (int dir = 0; dir < 3; ++dir) {
    const int ni = nx + (dir == 0), nj = ny + (dir == 1), nk = nz + (dir == 2);
    for (int i = 0; i < ni; ++i)
      for (int j = 0; j < nj; ++j)
        for (int k = 0; k < nk; ++k) {
          int64_t e[4];
          face_edges(dir, i, j, k, e);
          bool any = false;
          for (int q = 0; q < 4; ++q) any |= (pad2cond[e[q]] >= 0);
          if (!any) continue;
          // cond edges of this face, ascending cond index (csr column order)
          int32_t ce[4]; int8_t cs[4]; int m = 0;
          for (int q = 0; q < 4; ++q)
            if (pad2cond[e[q]] >= 0) { ce[m] = pad2cond[e[q]]; cs[m] = sgn4[q]; ++m; }
          for (int a = 1; a < m; ++a)
            for (int b = a; b > 0 && ce[b - 1] > ce[b]; --b) { std::swap(ce[b - 1], ce[b]); std::swap(cs[b - 1], cs[b]); }
          for (int q = 0; q < 4; ++q) {
            t.f_edge.push_back(q < m ? ce[q] : -1);
            t.f_sgn.push_back(q < m ? cs[q] : 0);
          }
          // adjacent cells (model.py:299-302): lower and upper cell along dir
          int64_t lo, hi;
          if (dir == 0) { lo = flat_cell(i - 1, j, k); hi = flat_cell(i, j, k); }
          else if (dir == 1) { lo = flat_cell(i, j - 1, k); hi = flat_cell(i, j, k); }
          else { lo = flat_cell(i, j, k - 1); hi = flat_cell(i, j, k); }
          // base weight = average @ nu_const_cells: 0.5*nu per non-conductor
          // neighbour (two-term sums are order independent)
          double base = 0.0;
          int32_t cl[2] = {-1, -1}; int nc = 0;
          for (int64_t cc : {lo, hi}) {
            if (cc < 0) continue;
            if (mat[cc] == 1) cl[nc++] = cell2list[cc];
            else base = base + 0.5 * nu;
          }
          t.f_base.push_back(base);
          if (nc == 2 && cl[0] > cl[1]) std::swap(cl[0], cl[1]);
          t.f_cell.push_back(cl[0]);
          t.f_cell.push_back(cl[1]);
          int64_t fid = dir == 0 ? fid_x(d, i, j, k) : dir == 1 ? fid_y(d, i, j, k) : fid_z(d, i, j, k);
          face_id_of.push_back(fid);
        }
  }
  t.n_faces_c = (int64_t)face_id_of.size();
  // global face id -> list index via binary search (ascending by construction)
  auto face_index = [&](int64_t fid) -> int32_t {
    auto it = std::lower_bound(face_id_of.begin(), face_id_of.end(), fid);
    if (it == face_id_of.end() || *it != fid) return -1;
    return (int32_t)(it - face_id_of.begin());
  };
  // cells: six faces [fx_i, fx_i+1, fy_j, fy_j+1, fz_k, fz_k+1] (model.py:312-319)
  t.cell_face.clear();
  for (int64_t q : cells) {
    int i = (int)(q / ((int64_t)ny * nz)), j = (int)((q / nz) % ny), k = (int)(q % nz);
    int64_t f6[6] = {fid_x(d, i, j, k), fid_x(d, i + 1, j, k), fid_y(d, i, j, k),
                     fid_y(d, i, j + 1, k), fid_z(d, i, j, k), fid_z(d, i, j, k + 1)};
    for (int s = 0; s < 6; ++s) {
      // a face with no conducting edge lies in the PEC boundary plane: its
      // row of c_cond is empty, so its flux is 0 (index -1)
      t.cell_face.push_back(face_index(f6[s]));
    }
  }
  t.n_cells_c = (int64_t)cells.size();
  t.cell_ids = cells;
  // per cond edge: its faces ascending face id with the incidence sign
  const int64_t n_c = (int64_t)t.c_global.size();
  std::vector<std::vector<std::pair<int32_t, int8_t>>> ef(n_c);
  for (int64_t f = 0; f < t.n_faces_c; ++f)
    for (int q = 0; q < 4; ++q) {
      int32_t ce = t.f_edge[4 * f + q];
      if (ce >= 0) ef[ce].push_back({(int32_t)f, t.f_sgn[4 * f + q]});
    }
  t.e_face.assign(4 * n_c, -1);
  t.e_sgn.assign(4 * n_c, 0);
  for (int64_t e = 0; e < n_c; ++e) {
    auto &v = ef[e];
    if (v.size() > 4) { err = "internal: edge with more than four faces"; return MQ_INVALID; }
    std::sort(v.begin(), v.end());
    for (size_t q = 0; q < v.size(); ++q) { t.e_face[4 * e + q] = v[q].first; t.e_sgn[4 * e + q] = v[q].second; }
  }

  // ---- K_cn: conducting rows x nonconducting columns --------------------
  // K = C^T diag(w/h) C; an off-diagonal entry couples two edges sharing a
  // face; faces holding a nonconducting edge are air faces (model.py:18-21),
  // so every K_cn entry is +-kn_off.  Sign = product of incidences.
  t.kcn_ptr.assign(n_c + 1, 0);
  t.kcn_col.clear(); t.kcn_sgn.clear();
  std::vector<std::vector<std::pair<int32_t, int8_t>>> rows(n_c);
  for (int dir = 0; dir < 3; ++dir) {
    const int ni = nx + (dir == 0), nj = ny + (dir == 1), nk = nz + (dir == 2);
    for (int i = 0; i < ni; ++i)
      for (int j = 0; j < nj; ++j)
        for (int k = 0; k < nk; ++k) {
          int64_t e[4];
          face_edges(dir, i, j, k, e);
          for (int a = 0; a < 4; ++a) {
            if (pad2cond[e[a]] < 0) continue;
            for (int b = 0; b < 4; ++b) {
              if (pad2nc[e[b]] < 0) continue;
              rows[pad2cond[e[a]]].push_back({(int32_t)e[b], (int8_t)(sgn4[a] * sgn4[b])});
            }
          }
        }
  }
  for (int64_t r = 0; r < n_c; ++r) {
    auto &v = rows[r];
    std::sort(v.begin(), v.end());
    for (size_t q = 0; q + 1 < v.size(); ++q)
      if (v[q].first == v[q + 1].first) { err = "internal: two faces shared by a conducting/nonconducting pair"; return MQ_INVALID; }
    for (auto &pr : v) { t.kcn_col.push_back(pr.first); t.kcn_sgn.push_back(pr.second); }
    t.kcn_ptr[r + 1] = (int64_t)t.kcn_col.size();
  }
  // transpose for K_cn^T a_c: accumulate over cond rows ascending (csc_matvec)
  std::vector<std::vector<std::pair<int32_t, int8_t>>> cols;
  std::vector<int32_t> touched;
  {
    std::vector<int32_t> slot(L.total, -1);
    for (int64_t r = 0; r < n_c; ++r)
      for (int64_t q = t.kcn_ptr[r]; q < t.kcn_ptr[r + 1]; ++q) {
        int32_t col = t.kcn_col[q];
        if (slot[col] < 0) { slot[col] = (int32_t)touched.size(); touched.push_back(col); cols.emplace_back(); }
        cols[slot[col]].push_back({(int32_t)r, t.kcn_sgn[q]});
      }
  }
  std::vector<size_t> order(touched.size());
  for (size_t q = 0; q < order.size(); ++q) order[q] = q;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return touched[a] < touched[b]; });
  t.kcnt_row.clear(); t.kcnt_ptr.assign(1, 0); t.kcnt_src.clear(); t.kcnt_sgn.clear();
  for (size_t q : order) {
    t.kcnt_row.push_back(touched[q]);
    for (auto &pr : cols[q]) { t.kcnt_src.push_back(pr.first); t.kcnt_sgn.push_back(pr.second); }
    t.kcnt_ptr.push_back((int64_t)t.kcnt_src.size());
  }
  return MQ_OK;
}

}  // namespace mq

namespace mq {

// Partition of an i-slab (node planes [ilo, ihi) of the global grid) for the
// distributed K_n solve (BASELINE configs[4]).  Same rules as build_topology
// (global PEC boundary, global conducting rule, global id order); the local
// box holds node planes ilo-1 .. ihi at local plane indices -1 .. n, so the
// two ghost planes sit in the guard plane (-1) and the last plane (n) of a
// box laid out exactly like a full grid with nx = n.  Only owned noncond
// edges are active; ghost planes are filled by the halo exchange.
int build_slab_topology(const mq_grid_desc &g, int ilo, int ihi, Topology &t, std::string &err) {
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  if (nx < 2 || ny < 2 || nz < 2) { err = "grid needs at least two cells per direction"; return MQ_INVALID; }
  if (ilo < 0 || ihi > nx || ihi <= ilo) { err = "invalid slab range"; return MQ_INVALID; }
  if (!g.material) { err = "material map is NULL"; return MQ_INVALID; }
  const int n = ihi - ilo;
  t.nx = n; t.ny = ny; t.nz = nz;
  Lay &L = t.L;
  L.Sj = (nz + 3) & ~1;
  L.Si = (int64_t)(ny + 2) * L.Sj;
  L.off = L.Si + L.Sj + 1;
  const int64_t P = (int64_t)(n + 2) * L.Si;
  L.C = (P + 31) / 32 * 32;
  L.total = 3 * L.C;
  L.words = L.total / 32;
  if (L.total >= ((int64_t)1 << 31)) { err = "slab too large for 32-bit device indexing"; return MQ_INVALID; }
  const int8_t *mat = g.material;
  auto cond_cell = [&](int i, int j, int k) -> bool {
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return false;
    return mat[((int64_t)i * ny + j) * nz + k] == 1;
  };
  const int64_t n_ex = (int64_t)nx * (ny + 1) * (nz + 1), n_ey = (int64_t)(nx + 1) * ny * (nz + 1);
  t.mask.assign(L.words, 0u);
  t.nc_pad.clear(); t.nc_global.clear(); t.c_global.clear(); t.c_pad.clear(); t.mc_diag.clear();
  for (int c = 0; c < 3; ++c)
    for (int i = ilo; i < ihi; ++i)
      for (int j = 0; j <= ny; ++j)
        for (int k = 0; k <= nz; ++k) {
          bool boundary, conducting;
          int64_t gid;
          if (c == 0) {
            if (i >= nx) continue;
            boundary = (j == 0 || j == ny || k == 0 || k == nz);
            conducting = cond_cell(i, j - 1, k - 1) || cond_cell(i, j - 1, k) || cond_cell(i, j, k - 1) ||
                         cond_cell(i, j, k);
            gid = ((int64_t)i * (ny + 1) + j) * (nz + 1) + k;
          } else if (c == 1) {
            if (j >= ny) continue;
            boundary = (i == 0 || i == nx || k == 0 || k == nz);
            conducting = cond_cell(i - 1, j, k - 1) || cond_cell(i - 1, j, k) || cond_cell(i, j, k - 1) ||
                         cond_cell(i, j, k);
            gid = n_ex + ((int64_t)i * ny + j) * (nz + 1) + k;
          } else {
            if (k >= nz) continue;
            boundary = (i == 0 || i == nx || j == 0 || j == ny);
            conducting = cond_cell(i - 1, j - 1, k) || cond_cell(i - 1, j, k) || cond_cell(i, j - 1, k) ||
                         cond_cell(i, j, k);
            gid = n_ex + n_ey + ((int64_t)i * (ny + 1) + j) * nz + k;
          }
          if (boundary || conducting) continue;
          const int64_t e = c * L.C + L.off + (int64_t)(i - ilo) * L.Si + (int64_t)j * L.Sj + k;
          t.nc_global.push_back(gid);
          t.nc_pad.push_back((int32_t)e);
          t.mask[e >> 5] |= (1u << (e & 31));
        }
  // the global id order is component-major, then (i, j, k): re-sort the
  // per-component scans (already ordered) -> nothing to do; keep a check
  for (size_t q = 1; q < t.nc_global.size(); ++q)
    if (t.nc_global[q - 1] >= t.nc_global[q]) { err = "internal: slab order"; return MQ_INVALID; }
  t.n_faces_c = t.n_cells_c = 0;
  return MQ_OK;
}

}  // namespace mq

// Shared-memory-resident fused PCG for grids whose bricks fit on chip
// (krylov.py:174-250).  Two kernels:
//  * pcg_resident1_kernel<LI> (default for li <= 4): one grid reduction per
//    iteration (reduced-synchronisation recurrence, see its comment below);
//  * pcg_resident_kernel<LI> (MQ_PCG_SYNC=2, and li = 5): the reference's two
//    reductions per iteration, same algorithm, stopping rule and bit-level
//    arithmetic as pcg_stencil_kernel / pcg_tma_kernel; described here.
//
// One CTA per SM (512 threads) owns a brick: a 16 (j) x 32 (k) node tile over
// Li <= 5 i-planes, all three edge components.  For the whole solve the
// brick's r, x and search direction p (the latter with a one-node halo ring)
// stay in shared memory, Ap in registers.  Per iteration:
//   K1: own p_new = M^-1 r + beta p (in place); halo p_new = M^-1 r + beta p
//       from the neighbours' published r and the CTA's own halo copy of
//       p_old (computed by the previous K1 from the owner's inputs with the
//       owner's arithmetic, hence bit-identical: p is never published);
//       Ap = K_n p_new from shared memory (plane values cached in registers,
//       all 3*Li row chains interleaved), partial p.Ap
//   K2: x += alpha p and r -= alpha Ap (shared / registers), r published,
//       partials r.r, r.z
// x leaves shared memory once, at the end.  Global traffic per iteration is
// the r halo ring (L2) and the r publication; the two grid barriers
// (~1.2 us each, tools/barrier_bench.cu), the L2 latency of the halo and the
// shared-memory stencil set the iteration time.
#include "mq_device.cuh"

namespace mq {

constexpr int RTJ = 16, RTK = 32, RT = RTJ * RTK;      // 512 threads, one position each
constexpr int RHJ = RTJ + 2, RHK = RTK + 2, RHP = RHJ * RHK;  // 18 x 34 = 612
constexpr int RW = RT / 32;                              // 16 warps
constexpr int RRING = 2 * RHK + 2 * RTJ;                 // 100 ring positions per plane
constexpr int RLI_MAX = 5;                               // planes per brick that fit

struct ResGeo {
  int nx, ny, nz;
  int tiles_k, tiles_j, chunks, nbricks, li_max;
};

struct ResPcgArgs {
  StencilPcgArgs a;
  ResGeo g;
};

__host__ __device__ constexpr size_t res_smem_bytes(int li) {
  return sizeof(double) * ((size_t)(li + 2) * 3 * RHP + (size_t)2 * li * 3 * RT);
}

template <int NV>
__device__ __forceinline__ void block_sum_r(double (&v)[NV], double *smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) smem[q * RW + warp] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
    for (int w = 0; w < RW; ++w) s = add(s, smem[q * RW + w]);
    v[q] = s;
  }
  __syncthreads();
}

// same stencil as stencil3 (pcg_brick.cu), CSR column order
template <class V>
__device__ __forceinline__ double stencil_r(int c, double dg, double of, V v) {
  double s;
  if (c == 0) {
    s = -mul(of, v(0, 0, -1, 0));
    s = sub(s, mul(of, v(0, 0, 0, -1)));
    s = add(s, mul(dg, v(0, 0, 0, 0)));
    s = sub(s, mul(of, v(0, 0, 0, 1)));
    s = sub(s, mul(of, v(0, 0, 1, 0)));
    s = add(s, mul(of, v(1, 0, -1, 0)));
    s = sub(s, mul(of, v(1, 0, 0, 0)));
    s = sub(s, mul(of, v(1, 1, -1, 0)));
    s = add(s, mul(of, v(1, 1, 0, 0)));
    s = add(s, mul(of, v(2, 0, 0, -1)));
    s = sub(s, mul(of, v(2, 0, 0, 0)));
    s = sub(s, mul(of, v(2, 1, 0, -1)));
    s = add(s, mul(of, v(2, 1, 0, 0)));
  } else if (c == 1) {
    s = mul(of, v(0, -1, 0, 0));
    s = sub(s, mul(of, v(0, -1, 1, 0)));
    s = sub(s, mul(of, v(0, 0, 0, 0)));
    s = add(s, mul(of, v(0, 0, 1, 0)));
    s = sub(s, mul(of, v(1, -1, 0, 0)));
    s = sub(s, mul(of, v(1, 0, 0, -1)));
    s = add(s, mul(dg, v(1, 0, 0, 0)));
    s = sub(s, mul(of, v(1, 0, 0, 1)));
    s = sub(s, mul(of, v(1, 1, 0, 0)));
    s = add(s, mul(of, v(2, 0, 0, -1)));
    s = sub(s, mul(of, v(2, 0, 0, 0)));
    s = sub(s, mul(of, v(2, 0, 1, -1)));
    s = add(s, mul(of, v(2, 0, 1, 0)));
  } else {
    s = mul(of, v(0, -1, 0, 0));
    s = sub(s, mul(of, v(0, -1, 0, 1)));
    s = sub(s, mul(of, v(0, 0, 0, 0)));
    s = add(s, mul(of, v(0, 0, 0, 1)));
    s = add(s, mul(of, v(1, 0, -1, 0)));
    s = sub(s, mul(of, v(1, 0, -1, 1)));
    s = sub(s, mul(of, v(1, 0, 0, 0)));
    s = add(s, mul(of, v(1, 0, 0, 1)));
    s = sub(s, mul(of, v(2, -1, 0, 0)));
    s = sub(s, mul(of, v(2, 0, -1, 0)));
    s = add(s, mul(dg, v(2, 0, 0, 0)));
    s = sub(s, mul(of, v(2, 0, 1, 0)));
    s = sub(s, mul(of, v(2, 1, 0, 0)));
  }
  return s;
}

#ifndef MQ_RES_HU
#define MQ_RES_HU 4
#endif
constexpr int HU = MQ_RES_HU;  // halo positions per thread (one round)
static_assert(2 * RHP + RLI_MAX * RRING <= HU * RT, "halo must fit one round");

#ifndef MQ_RES_SLIDE
#define MQ_RES_SLIDE 1
#endif

// The 15 distinct values of one P plane that the three stencil rows of the
// planes i-1, i, i+1 read around the own position (component, dj, dk).
struct PlaneVals {
  double xo, xjm, xjp, xkm, xkp;     // x: own, j-1, j+1, k-1, k+1
  double yo, yjm, ykm, ykp, yjmkp;   // y: own, j-1, k-1, k+1, (j-1,k+1)
  double zo, zjm, zjp, zkm, zjpkm;   // z: own, j-1, j+1, k-1, (j+1,k-1)
};

__device__ __forceinline__ void load_plane(const double *P, int pl, int s, PlaneVals &v) {
  const double *x = P + ((size_t)pl * 3 + 0) * RHP + s;
  const double *y = P + ((size_t)pl * 3 + 1) * RHP + s;
  const double *z = P + ((size_t)pl * 3 + 2) * RHP + s;
  v.xo = x[0]; v.xjm = x[-RHK]; v.xjp = x[RHK]; v.xkm = x[-1]; v.xkp = x[1];
  v.yo = y[0]; v.yjm = y[-RHK]; v.ykm = y[-1]; v.ykp = y[1]; v.yjmkp = y[-RHK + 1];
  v.zo = z[0]; v.zjm = z[-RHK]; v.zjp = z[RHK]; v.zkm = z[-1]; v.zjpkm = z[RHK - 1];
}

// value (component cc, offset dj, dk) of plane q; arguments are literals in
// stencil_r, so the selection folds away
__device__ __forceinline__ double pick(const PlaneVals &q, int cc, int dj, int dk) {
  if (cc == 0) {
    if (dj == -1) return q.xjm;
    if (dj == 1) return q.xjp;
    if (dk == -1) return q.xkm;
    if (dk == 1) return q.xkp;
    return q.xo;
  }
  if (cc == 1) {
    if (dj == -1) return dk == 1 ? q.yjmkp : q.yjm;
    if (dk == -1) return q.ykm;
    if (dk == 1) return q.ykp;
    return q.yo;
  }
  if (dj == 1) return dk == -1 ? q.zjpkm : q.zjp;
  if (dj == -1) return q.zjm;
  if (dk == -1) return q.zkm;
  return q.zo;
}

// LI = planes per brick (compile time, so that every row's stencil chain is
// unrolled and the 3*LI independent chains interleave; bricks of a chunking
// that does not divide nx have li = LI or LI-1 planes).
template <int LI>
__global__ void __launch_bounds__(RT, 1) pcg_resident_kernel(ResPcgArgs A) {
  extern __shared__ __align__(16) double rsm[];
  __shared__ double red[3 * RW];
  __shared__ double tot[4];
  const StencilPcgArgs &a = A.a;
  const ResGeo &g = A.g;
  const Lay &L = a.L;
  const int G = gridDim.x;
  const int tid = threadIdx.x, ty = tid >> 5, tx = tid & 31;
  const double dg = a.dg, of = a.of, inv = a.inv;
  const bool jac = a.use_jac != 0;
  const int x0_mode = a.x0_mode_dev ? *a.x0_mode_dev : a.x0_mode;
  if (a.err_word && *((volatile const unsigned int *)a.err_word)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      PcgOut o{};
      o.status = 99;
      *a.out = o;
    }
    return;
  }
  // brick of this CTA (one per CTA; the launch guarantees nbricks == G)
  const int b = blockIdx.x;
  const int tk = b % g.tiles_k, tj = (b / g.tiles_k) % g.tiles_j, ic = b / (g.tiles_k * g.tiles_j);
  const int k0 = tk * RTK, j0 = tj * RTJ;
  const int i0 = (int)(((int64_t)ic * g.nx) / g.chunks), i1 = (int)(((int64_t)(ic + 1) * g.nx) / g.chunks);
  const int li = i1 - i0;
  double *P = rsm;                                   // [li+2][3][RHP], plane 0 = i0-1
  double *R = P + (size_t)(g.li_max + 2) * 3 * RHP;  // [li][3][RT]
  double *X = R + (size_t)g.li_max * 3 * RT;         // [li][3][RT] own x for the whole solve
  const int j = j0 + ty, k = k0 + tx;
  const bool own_ok = j < g.ny && k < g.nz;
  const int s_own = (ty + 1) * RHK + (tx + 1);
  const int64_t pos_own = L.off + (int64_t)j * L.Sj + k;
  auto Pidx = [&](int l, int c, int s) { return ((size_t)l * 3 + c) * RHP + s; };
  auto Oidx = [&](int l, int c) { return ((size_t)l * 3 + c) * RT + tid; };
  const uint32_t *mask = a.mask;
  // active bits of the own positions, 3 per plane (li <= 5 -> 15 bits)
  uint32_t act = 0u;
  if (own_ok)
    for (int l = 0; l < li; ++l)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t e = c * L.C + (int64_t)(i0 + l) * L.Si + pos_own;
        act |= ((__ldg(mask + (e >> 5)) >> (e & 31)) & 1u) << (3 * l + c);
      }
  auto own_e = [&](int l, int c) { return c * L.C + (int64_t)(i0 + l) * L.Si + pos_own; };
  auto is_act = [&](int l, int c) { return (act >> (3 * l + c)) & 1u; };
  auto V = [&](int l, int c) {
    // neighbourhood accessor of own position at brick plane l (P plane l+1)
    return [=](int cc, int di, int dj, int dk) { return P[Pidx(l + 1 + di, cc, s_own + dj * RHK + dk)]; };
  };
  // halo slots: planes 0 and li+1 in full, ring of the interior planes
  const int nhalo = 2 * RHP + li * RRING;
  auto halo_slot = [&](int h, int &l, int &s) {
    if (h < RHP) { l = 0; s = h; return; }
    if (h < 2 * RHP) { l = li + 1; s = h - RHP; return; }
    h -= 2 * RHP;
    l = 1 + h / RRING;
    const int q = h % RRING;
    int jj, kk;
    if (q < RHK) { jj = 0; kk = q; }
    else if (q < 2 * RHK) { jj = RHJ - 1; kk = q - RHK; }
    else if (q < 2 * RHK + RTJ) { jj = 1 + (q - 2 * RHK); kk = 0; }
    else { jj = 1 + (q - 2 * RHK - RTJ); kk = RHK - 1; }
    s = jj * RHK + kk;
  };
  auto halo_e = [&](int l, int s, int c, bool &ok) {
    const int jj = s / RHK, kk = s % RHK;
    const int gi = i0 - 1 + l, gj = j0 - 1 + jj, gk = k0 - 1 + kk;
    ok = gi >= -1 && gi <= g.nx && gj >= -1 && gj <= g.ny && gk >= -1 && gk <= g.nz;
    return c * L.C + L.off + (int64_t)gi * L.Si + (int64_t)gj * L.Sj + gk;
  };

  unsigned long long *trace = (blockIdx.x == 0 && threadIdx.x == 0) ? a.trace : nullptr;
  auto stamp = [&](int slot) {
    if (trace && slot < 4 * 64 + 1) trace[slot] = globaltimer_ns();
  };
  // fine phase stamps (variant builds with -DMQ_TRACE_FINE): 8 per
  // iteration for the first 32 iterations at trace[320 + 8 (it-1) + k]
  auto fstamp = [&](int it, int k) {
#ifdef MQ_TRACE_FINE
    if (trace && it <= 32) trace[320 + 8 * (it - 1) + k] = globaltimer_ns();
#else
    (void)it;
    (void)k;
#endif
  };
  stamp(0);
  // ---- initial residual (krylov.py:209-218) ----
  double v3[3] = {0.0, 0.0, 0.0};
  {
    // P <- x0 (own + halo) when x0 is given, own r <- b - A x0
    if (x0_mode == 1) {
      for (int h = tid; h < nhalo; h += RT) {
        int l, s;
        halo_slot(h, l, s);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          bool ok;
          const int64_t e = halo_e(l, s, c, ok);
          P[Pidx(l, c, s)] = ok ? __ldcg(a.x + e) : 0.0;
        }
      }
      for (int l = 0; l < li; ++l)
#pragma unroll
        for (int c = 0; c < 3; ++c) P[Pidx(l + 1, c, s_own)] = own_ok ? __ldcg(a.x + own_e(l, c)) : 0.0;
      __syncthreads();
    }
    for (int l = 0; l < li; ++l)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double rv = 0.0;
        if (own_ok && is_act(l, c)) {
          const int64_t e = own_e(l, c);
          const double bv = __ldcg(a.b + e);
          rv = bv;
          if (x0_mode == 1) rv = sub(bv, stencil_r(c, dg, of, V(l, c)));
          else a.x[e] = 0.0;
          const double z = jac ? mul(inv, rv) : rv;
          v3[0] = add(v3[0], mul(bv, bv));
          v3[1] = add(v3[1], mul(rv, rv));
          v3[2] = add(v3[2], mul(rv, z));
          a.r[e] = rv;  // published for the neighbours' first halo
        }
        R[Oidx(l, c)] = rv;
        X[Oidx(l, c)] = (x0_mode == 1 && own_ok) ? P[Pidx(l + 1, c, s_own)] : 0.0;
      }
  }
  block_sum_r<3>(v3, red);
  if (threadIdx.x == 0) {
    a.partials[0 * G + blockIdx.x] = v3[0];
    a.partials[1 * G + blockIdx.x] = v3[1];
    a.partials[2 * G + blockIdx.x] = v3[2];
  }
  int status = MQ_OK, iters = 0, converged = 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  int applies = (x0_mode == 2) ? 0 : 1;
  // the halo r values of K1, loaded in one round (issuing them right after
  // the barrier, ahead of the partial-sum read, measured slower: the partial
  // loads queue behind them)
  double hr[HU][3];
  int hl[HU], hs[HU];
  auto issue_halo = [&]() {
#pragma unroll
    for (int u = 0; u < HU; ++u) {
      const int h = tid + u * RT;
      hl[u] = -1;
      if (h < nhalo) {
        halo_slot(h, hl[u], hs[u]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          bool ok;
          const int64_t e = halo_e(hl[u], hs[u], c, ok);
          hr[u][c] = ok ? __ldcg(a.r + e) : 0.0;
        }
      }
    }
  };
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
    double beta = 0.0;
    bool first = true;
    for (int it = 1; it <= a.max_iter; ++it) {
      fstamp(it, 0);
      // ---- K1: own p_new in place; halo p_new = M^-1 r + beta p_old from the
      // neighbours' published r and this CTA's own copy of the halo p_old
      // (the previous K1 computed it with the owner's inputs and arithmetic,
      // so it equals the owner's value bit for bit: p is never published) ----
#pragma unroll
      for (int l = 0; l < LI; ++l)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (l < li) {
            const double rq = R[Oidx(l, c)];
            const double z = jac ? mul(inv, rq) : rq;
            const size_t pi = Pidx(l + 1, c, s_own);
            P[pi] = first ? z : add(z, mul(beta, P[pi]));
          }
        }
      fstamp(it, 1);
      issue_halo();
#pragma unroll
      for (int u = 0; u < HU; ++u) {
        if (hl[u] < 0) continue;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double z = jac ? mul(inv, hr[u][c]) : hr[u][c];
          const size_t pi = Pidx(hl[u], c, hs[u]);
          P[pi] = first ? z : add(z, mul(beta, P[pi]));
        }
      }
      fstamp(it, 2);
      __syncthreads();
      fstamp(it, 3);
      double v1[1] = {0.0};
      // Ap of the own rows stays in registers until K2
      double av[LI * 3];
      {
        // all LI*3 rows unconditionally (rows past li or inactive read
        // allocated shared memory and are discarded): independent chains
#if MQ_RES_SLIDE
        // march along i keeping the 15 distinct neighbour values of a plane
        // in registers: each value is read from shared memory once instead
        // of once per row that uses it (39 -> ~17 loads per plane)
        PlaneVals pm, p0, pp;
        load_plane(P, 0, s_own, pm);
        load_plane(P, 1, s_own, p0);
#pragma unroll
        for (int l = 0; l < LI; ++l) {
          load_plane(P, l + 2, s_own, pp);
          auto W = [&](int cc, int di, int dj, int dk) { return pick(di < 0 ? pm : (di > 0 ? pp : p0), cc, dj, dk); };
#pragma unroll
          for (int c = 0; c < 3; ++c) av[3 * l + c] = stencil_r(c, dg, of, W);
          pm = p0;
          p0 = pp;
        }
#else
#pragma unroll
        for (int l = 0; l < LI; ++l)
#pragma unroll
          for (int c = 0; c < 3; ++c) av[3 * l + c] = stencil_r(c, dg, of, V(l, c));
#endif
#pragma unroll
        for (int l = 0; l < LI; ++l)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (l < li && own_ok && is_act(l, c)) {
              v1[0] = add(v1[0], mul(P[Pidx(l + 1, c, s_own)], av[3 * l + c]));
            }
          }
      }
      fstamp(it, 4);
      block_sum_r<1>(v1, red);
      fstamp(it, 5);
      if (threadIdx.x == 0) a.partials[3 * G + blockIdx.x] = v1[0];
      ++applies;
      stamp(4 * (it - 1) + 1);
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      stamp(4 * (it - 1) + 2);
      stress_after_barrier(a.stress_ns, 2 * it);
      double s1[1];
      grid_partials_sum_all<1, 5>(a.partials + 3 * G, G, s1, tot);
      const double pap = s1[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; goto done; }
      alpha = rz / pap;
      fstamp(it, 6);
      // ---- K2: x += alpha p (shared), r -= alpha Ap (own), publish r ----
      double v2[2] = {0.0, 0.0};
#pragma unroll
      for (int l = 0; l < LI; ++l)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (!(l < li && own_ok && is_act(l, c))) continue;
          const int64_t e = own_e(l, c);
          X[Oidx(l, c)] = add(X[Oidx(l, c)], mul(alpha, P[Pidx(l + 1, c, s_own)]));
          const double rv = sub(R[Oidx(l, c)], mul(alpha, av[3 * l + c]));
          R[Oidx(l, c)] = rv;
          a.r[e] = rv;
          const double z = jac ? mul(inv, rv) : rv;
          v2[0] = add(v2[0], mul(rv, rv));
          v2[1] = add(v2[1], mul(rv, z));
        }
      fstamp(it, 7);
      block_sum_r<2>(v2, red);
      if (threadIdx.x == 0) {
        a.partials[4 * G + blockIdx.x] = v2[0];
        a.partials[5 * G + blockIdx.x] = v2[1];
      }
      stamp(4 * (it - 1) + 3);
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      stamp(4 * (it - 1) + 4);
      stress_after_barrier(a.stress_ns, 2 * it + 1);
      double s2[2];
      grid_partials_sum_all<2, 5>(a.partials + 4 * G, G, s2, tot);
      rnorm = sqrt(s2[0]);
      iters = it;
      rel = relf(rnorm);
      const double rz_new = jac ? s2[1] : s2[0];
      if (rnorm <= target) { converged = 1; break; }
      if (!isfinite(rz_new)) { status = MQ_INDEFINITE; break; }
      beta = rz_new / rz;
      rz = rz_new;
      first = false;
    }
    if (status == MQ_OK && !converged) status = MQ_NOT_CONVERGED;
    // the iterate leaves shared memory once (converged or budget exhausted)
#pragma unroll
    for (int l = 0; l < LI; ++l)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if (l < li && own_ok && is_act(l, c)) a.x[own_e(l, c)] = X[Oidx(l, c)];
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

// ---------------------------------------------------------------------------
// One grid reduction per iteration (pcg_resident1_kernel).  The reference's
// iteration (krylov.py:231-249) needs p.Ap before alpha and r.z after the
// r update: two reductions, two grid barriers.  With the scalar Jacobi
// preconditioner (z = inv * r) the next r.z follows from scalars of the
// current iteration,
//   |r - alpha Ap|^2 = r.r - 2 alpha r.Ap + alpha^2 Ap.Ap,
// so K1 reduces [p.Ap, r.Ap, Ap.Ap, r.r, r.z] in one barrier (D'Azevedo,
// Eijkhout & Romine's reduced-synchronisation CG).  Only beta uses the
// extrapolated value; alpha uses r.z, and the stopping test |r| <= target
// uses r.r, both summed directly from the vector, one barrier later: the
// test of iteration it is read at the barrier of it+1, whose K1 pass is then
// discarded (x, the iteration count and the reported residual are the
// reference's).  Exact-arithmetic iterates are unchanged; in fp64 they differ
// from the two-barrier kernel in the last bits (PCG parity bar: 1e-8 field,
// +-1 iteration).
// Halo exchange without a second barrier: owners publish Ap (instead of r);
// every CTA keeps the r of its halo ring in shared memory (HR) and advances
// it with alpha and the neighbours' published Ap, bit-identical to the
// owners' own update; halo p follows from HR and the CTA's halo p_old as
// before.  Only for li_max <= 4 (the HR ring needs 39 KB next to the 186 KB
// of P, R and X).
// halo Ap loads issued right after the barrier, ahead of the partial-sum
// read, by warps 1..15 only (2; measured 9.4 us/iteration at 64^3), by all
// warps (1; 9.5 us) or after alpha (0; 10.4 us)
#ifndef MQ_RES1_EARLY
#define MQ_RES1_EARLY 2
#endif
#ifndef MQ_RES1_LH
#define MQ_RES1_LH 1  // planes per batch of the own update's shared-memory loads
#endif
#ifndef MQ_RES1_APSURF
#define MQ_RES1_APSURF 0
#endif
template <int LI>
__global__ void __launch_bounds__(RT, 1) pcg_resident1_kernel(ResPcgArgs A) {
  extern __shared__ __align__(16) double rsm[];
  __shared__ double red[5 * RW];
  __shared__ double tot[5];
  const StencilPcgArgs &a = A.a;
  const ResGeo &g = A.g;
  const Lay &L = a.L;
  const int G = gridDim.x;
  const int tid = threadIdx.x, ty = tid >> 5, tx = tid & 31;
  const double dg = a.dg, of = a.of, inv = a.inv;
  const bool jac = a.use_jac != 0;
  const int x0_mode = a.x0_mode_dev ? *a.x0_mode_dev : a.x0_mode;
  if (a.err_word && *((volatile const unsigned int *)a.err_word)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      PcgOut o{};
      o.status = 99;
      *a.out = o;
    }
    return;
  }
  const int b = blockIdx.x;
  const int tk = b % g.tiles_k, tj = (b / g.tiles_k) % g.tiles_j, ic = b / (g.tiles_k * g.tiles_j);
  const int k0 = tk * RTK, j0 = tj * RTJ;
  const int i0 = (int)(((int64_t)ic * g.nx) / g.chunks), i1 = (int)(((int64_t)(ic + 1) * g.nx) / g.chunks);
  const int li = i1 - i0;
  const int NH = 2 * RHP + g.li_max * RRING;
  double *P = rsm;                                   // [li+2][3][RHP], plane 0 = i0-1
  double *R = P + (size_t)(g.li_max + 2) * 3 * RHP;  // [li][3][RT]
  double *X = R + (size_t)g.li_max * 3 * RT;         // [li][3][RT]
  double *HR = X + (size_t)g.li_max * 3 * RT;        // [3][NH] r of the halo slots
  const int j = j0 + ty, k = k0 + tx;
  const bool own_ok = j < g.ny && k < g.nz;
  const int s_own = (ty + 1) * RHK + (tx + 1);
  const int64_t pos_own = L.off + (int64_t)j * L.Sj + k;
  auto Pidx = [&](int l, int c, int s) { return ((size_t)l * 3 + c) * RHP + s; };
  auto Oidx = [&](int l, int c) { return ((size_t)l * 3 + c) * RT + tid; };
  const uint32_t *mask = a.mask;
  uint32_t act = 0u;
  if (own_ok)
    for (int l = 0; l < li; ++l)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t e = c * L.C + (int64_t)(i0 + l) * L.Si + pos_own;
        act |= ((__ldg(mask + (e >> 5)) >> (e & 31)) & 1u) << (3 * l + c);
      }
  auto own_e = [&](int l, int c) { return c * L.C + (int64_t)(i0 + l) * L.Si + pos_own; };
  auto is_act = [&](int l, int c) { return (act >> (3 * l + c)) & 1u; };
  auto V = [&](int l, int c) {
    return [=](int cc, int di, int dj, int dk) { return P[Pidx(l + 1 + di, cc, s_own + dj * RHK + dk)]; };
  };
  const int nhalo = 2 * RHP + li * RRING;
  auto halo_slot = [&](int h, int &l, int &s) {
    if (h < RHP) { l = 0; s = h; return; }
    if (h < 2 * RHP) { l = li + 1; s = h - RHP; return; }
    h -= 2 * RHP;
    l = 1 + h / RRING;
    const int q = h % RRING;
    int jj, kk;
    if (q < RHK) { jj = 0; kk = q; }
    else if (q < 2 * RHK) { jj = RHJ - 1; kk = q - RHK; }
    else if (q < 2 * RHK + RTJ) { jj = 1 + (q - 2 * RHK); kk = 0; }
    else { jj = 1 + (q - 2 * RHK - RTJ); kk = RHK - 1; }
    s = jj * RHK + kk;
  };
  auto halo_e = [&](int l, int s, int c, bool &ok) {
    const int jj = s / RHK, kk = s % RHK;
    const int gi = i0 - 1 + l, gj = j0 - 1 + jj, gk = k0 - 1 + kk;
    ok = gi >= -1 && gi <= g.nx && gj >= -1 && gj <= g.ny && gk >= -1 && gk <= g.nz;
    return c * L.C + L.off + (int64_t)gi * L.Si + (int64_t)gj * L.Sj + gk;
  };
  unsigned long long *trace = (blockIdx.x == 0 && threadIdx.x == 0) ? a.trace : nullptr;
  auto stamp = [&](int slot) {
    if (trace && slot < 4 * 64 + 1) trace[slot] = globaltimer_ns();
  };
  auto fstamp = [&](int it, int k) {
#ifdef MQ_TRACE_FINE
    if (trace && it <= 32) trace[320 + 8 * (it - 1) + k] = globaltimer_ns();
#else
    (void)it;
    (void)k;
#endif
  };
  stamp(0);
  // ---- initial residual (krylov.py:209-218), as pcg_resident_kernel ----
  double v3[3] = {0.0, 0.0, 0.0};
  {
    if (x0_mode == 1) {
      for (int h = tid; h < nhalo; h += RT) {
        int l, s;
        halo_slot(h, l, s);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          bool ok;
          const int64_t e = halo_e(l, s, c, ok);
          P[Pidx(l, c, s)] = ok ? __ldcg(a.x + e) : 0.0;
        }
      }
      for (int l = 0; l < li; ++l)
#pragma unroll
        for (int c = 0; c < 3; ++c) P[Pidx(l + 1, c, s_own)] = own_ok ? __ldcg(a.x + own_e(l, c)) : 0.0;
      __syncthreads();
    }
    for (int l = 0; l < li; ++l)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double rv = 0.0;
        if (own_ok && is_act(l, c)) {
          const int64_t e = own_e(l, c);
          const double bv = __ldcg(a.b + e);
          rv = bv;
          if (x0_mode == 1) rv = sub(bv, stencil_r(c, dg, of, V(l, c)));
          else a.x[e] = 0.0;
          const double z = jac ? mul(inv, rv) : rv;
          v3[0] = add(v3[0], mul(bv, bv));
          v3[1] = add(v3[1], mul(rv, rv));
          v3[2] = add(v3[2], mul(rv, z));
          a.r[e] = rv;  // the neighbours' initial halo r
        }
        R[Oidx(l, c)] = rv;
        X[Oidx(l, c)] = (x0_mode == 1 && own_ok) ? P[Pidx(l + 1, c, s_own)] : 0.0;
      }
  }
  block_sum_r<3>(v3, red);
  if (threadIdx.x == 0) {
    a.partials[0 * G + blockIdx.x] = v3[0];
    a.partials[1 * G + blockIdx.x] = v3[1];
    a.partials[2 * G + blockIdx.x] = v3[2];
  }
  int status = MQ_OK, iters = 0, converged = 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  const int applies0 = (x0_mode == 2) ? 0 : 1;
  // activity of this thread's halo slots h = hbase + u * hstride (slot u,
  // component c -> bit 3u+c): inactive and out-of-box slots keep r = 0 and
  // never read Ap.  With MQ_RES1_EARLY == 2 warp 0 has no halo slots (it
  // reads the partial sums while the other warps' halo loads are in flight).
  uint32_t hact = 0u;
#if MQ_RES1_EARLY == 2
  const int hbase = tid - 32, hstride = RT - 32;
#else
  const int hbase = tid, hstride = RT;
#endif
  static_assert(2 * RHP + 4 * RRING <= HU * (RT - 32), "halo slots of li <= 4 fit one round");
  if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
  {
    double s3[3];
    grid_partials_sum<3>(a.partials, G, s3, tot);
#pragma unroll
    for (int u = 0; u < HU; ++u) {
      const int h = hbase + u * hstride;
      if (hbase >= 0 && h < nhalo) {
        int l, s;
        halo_slot(h, l, s);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          bool ok;
          const int64_t e = halo_e(l, s, c, ok);
          const bool on = ok && ((__ldg(mask + (e >> 5)) >> (e & 31)) & 1u);
          hact |= (uint32_t)on << (3 * u + c);
          HR[c * NH + h] = on ? __ldcg(a.r + e) : 0.0;
        }
      }
    }
    bnorm = sqrt(s3[0]);
    const double target = fmax(a.rel_tol * bnorm, a.abs_tol);
    double rnorm = sqrt(s3[1]);
    rz = jac ? s3[2] : s3[1];
    auto relf = [&](double res) { return bnorm > 0.0 ? res / bnorm : (res == 0.0 ? 0.0 : INFINITY); };
    rel = relf(rnorm);
    if (rnorm <= target) { converged = 1; goto done; }
    double beta = 0.0;
    bool first = true;
    // this thread's halo slots: P index of component 0 (components are RHP
    // apart) and padded element of component 0 (components L.C apart)
    int hp[HU], he[HU];
#pragma unroll
    for (int u = 0; u < HU; ++u) {
      const int h = hbase + u * hstride;
      hp[u] = -1;
      he[u] = 0;
      if (hbase >= 0 && h < nhalo) {
        int l, s;
        halo_slot(h, l, s);
        bool ok;
        hp[u] = (int)Pidx(l, 0, s);
        he[u] = (int)halo_e(l, s, 0, ok);
      }
    }
    // the neighbours' published Ap at this thread's active halo slots, all
    // loads in flight before the first use (one L2 round trip)
    double hq[HU][3];
    // Ap of iteration it goes to buffer it & 1: a CTA writes Ap_{it+1} before
    // the barrier of it+1, possibly while a slower neighbour is still to load
    // Ap_it after the barrier of it; Ap_{it+2} is written only after every
    // CTA passed the barrier of it+1, i.e. after all loads of Ap_it
    const double *apb = a.ap;
    auto issue_ap_halo = [&]() {
#pragma unroll
      for (int u = 0; u < HU; ++u)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          hq[u][c] = ((hact >> (3 * u + c)) & 1u) ? __ldcg(apb + he[u] + c * L.C) : 0.0;
    };
    // p_0 = z_0 (own and halo); r.r and r.z of r_0 ride on the first
    // reduction (krylov.py:228-230)
    double v5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int l = 0; l < LI; ++l)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (l < li) {
          const double r0 = R[Oidx(l, c)];
          const double z = jac ? mul(inv, r0) : r0;
          P[Pidx(l + 1, c, s_own)] = z;
          if (own_ok && is_act(l, c)) {
            v5[3] = add(v5[3], mul(r0, r0));
            v5[4] = add(v5[4], mul(r0, z));
          }
        }
      }
#pragma unroll
    for (int u = 0; u < HU; ++u)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if (hp[u] >= 0) {
          const double hv = HR[c * NH + hbase + u * hstride];
          P[hp[u] + c * RHP] = jac ? mul(inv, hv) : hv;
        }
    for (int it = 1;; ++it) {
      fstamp(it, 0);
#ifdef MQ_RES1_AP_SINGLE  // the racy single buffer, for the stress test's negative control only
      double *const apw = a.ap;
#else
      double *const apw = (it & 1) ? a.ap2 : a.ap;
#endif
      apb = apw;
      __syncthreads();
      // ---- Ap = K_n p from shared memory; partials p.Ap, r.Ap, Ap.Ap per
      // plane as the march passes it; Ap published for the neighbours' halo
      double av[LI * 3];
      {
        PlaneVals pm, p0, pp;
        load_plane(P, 0, s_own, pm);
        load_plane(P, 1, s_own, p0);
#pragma unroll
        for (int l = 0; l < LI; ++l) {
          load_plane(P, l + 2, s_own, pp);
          auto W = [&](int cc, int di, int dj, int dk) { return pick(di < 0 ? pm : (di > 0 ? pp : p0), cc, dj, dk); };
#pragma unroll
          for (int c = 0; c < 3; ++c) av[3 * l + c] = stencil_r(c, dg, of, W);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (l < li && own_ok && is_act(l, c)) {
              const double apv = av[3 * l + c];
              v5[0] = add(v5[0], mul(pick(p0, c, 0, 0), apv));
              v5[1] = add(v5[1], mul(R[Oidx(l, c)], apv));
              v5[2] = add(v5[2], mul(apv, apv));
              apw[own_e(l, c)] = apv;
            }
          }
          pm = p0;
          p0 = pp;
        }
      }
      fstamp(it, 1);
      // block sums: warp sums to shared memory, lane q of warp 0 adds value
      // q over the 16 warps in order and stores this CTA's partial (only
      // the partials leave the CTA; one CTA barrier)
      double *pt = a.partials + 3 * G + (it & 1) * 5 * G;  // alternating sets: a fast CTA's
#pragma unroll                                              // next partials never race a
      for (int q = 0; q < 5; ++q) v5[q] = warp_sum(v5[q]);  // slow CTA's read of these
      if (tx == 0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) red[q * RW + ty] = v5[q];
      }
      __syncthreads();
      if (ty == 0 && tx < 5) {
        double sacc = 0.0;
        for (int w = 0; w < RW; ++w) sacc = add(sacc, red[tx * RW + w]);
        pt[tx * G + blockIdx.x] = sacc;
      }
      stamp(4 * (it - 1) + 1);
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      stamp(4 * (it - 1) + 2);
      stress_after_barrier(a.stress_ns, it);
      double s5[5];
#if MQ_RES1_EARLY
      issue_ap_halo();
#endif
      {
        // warp q < 5 reads partial row q (G <= 160: five loads per lane in
        // flight), fixed-order lane sums then the warp tree: identical in
        // every CTA
        if (ty < 5) {
          double pv[5];
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            const int bb = tx + 32 * u;
            pv[u] = bb < G ? __ldcg(pt + (int64_t)ty * G + bb) : 0.0;
          }
          double sacc = 0.0;
#pragma unroll
          for (int u = 0; u < 5; ++u)
            if (tx + 32 * u < G) sacc = add(sacc, pv[u]);
          sacc = warp_sum(sacc);
          if (tx == 0) tot[ty] = sacc;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 5; ++q) s5[q] = tot[q];
      }
      fstamp(it, 2);
      if (!first) {
        // the previous iteration's stopping test and r.z (krylov.py:239-246)
        rnorm = sqrt(s5[3]);
        rel = relf(rnorm);
        if (rnorm <= target) { converged = 1; break; }
        const double rz_d = jac ? s5[4] : s5[3];
        if (!isfinite(rz_d)) { status = MQ_INDEFINITE; break; }
        rz = rz_d;
      }
      if (it > a.max_iter) break;  // budget: iters == max_iter, not converged
      const double pap = s5[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; break; }
      alpha = rz / pap;
      // beta from the extrapolated r.z of the updated r
      {
        const double rr_new = add(sub(s5[3], mul(mul(2.0, alpha), s5[1])), mul(mul(alpha, alpha), s5[2]));
        const double rz_new = jac ? mul(inv, rr_new) : rr_new;
        beta = rz_new > 0.0 ? rz_new / rz : 0.0;
      }
#if !MQ_RES1_EARLY
      issue_ap_halo();
#endif
      // ---- own: x += alpha p, r -= alpha Ap, p = z + beta p, and r.r, r.z
      // of the new r for the next reduction (the halo work, which waits on
      // the neighbours' Ap, comes last) ----
#pragma unroll
      for (int q = 0; q < 5; ++q) v5[q] = 0.0;
#pragma unroll
      for (int h2 = 0; h2 < (LI + MQ_RES1_LH - 1) / MQ_RES1_LH; ++h2) {
        constexpr int LH = MQ_RES1_LH;
        double xo[LH * 3], pv[LH * 3], ro[LH * 3];
#pragma unroll
        for (int l2 = 0; l2 < LH; ++l2)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const int l = h2 * LH + l2;
            const bool on = l < LI && l < li;
            xo[3 * l2 + c] = on ? X[Oidx(l, c)] : 0.0;
            pv[3 * l2 + c] = on ? P[Pidx(l + 1, c, s_own)] : 0.0;
            ro[3 * l2 + c] = on ? R[Oidx(l, c)] : 0.0;
          }
#pragma unroll
        for (int l2 = 0; l2 < LH; ++l2)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const int l = h2 * LH + l2;
            if (!(l < LI && l < li && own_ok && is_act(l, c))) continue;
            X[Oidx(l, c)] = add(xo[3 * l2 + c], mul(alpha, pv[3 * l2 + c]));
            const double rn = sub(ro[3 * l2 + c], mul(alpha, av[3 * l + c]));
            R[Oidx(l, c)] = rn;
            const double z = jac ? mul(inv, rn) : rn;
            P[Pidx(l + 1, c, s_own)] = add(z, mul(beta, pv[3 * l2 + c]));
            v5[3] = add(v5[3], mul(rn, rn));
            v5[4] = add(v5[4], mul(rn, z));
          }
      }
      // ---- halo: r -= alpha Ap (the owners' update, bit for bit), p = z + beta p
      {
        double hv[HU][3], ho[HU][3];
#pragma unroll
        for (int u = 0; u < HU; ++u)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const bool on = (hact >> (3 * u + c)) & 1u;
            hv[u][c] = on ? HR[c * NH + hbase + u * hstride] : 0.0;
            ho[u][c] = on ? P[hp[u] + c * RHP] : 0.0;
          }
#pragma unroll
        for (int u = 0; u < HU; ++u)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if ((hact >> (3 * u + c)) & 1u) {
              const double rn = sub(hv[u][c], mul(alpha, hq[u][c]));
              HR[c * NH + hbase + u * hstride] = rn;
              const double z = jac ? mul(inv, rn) : rn;
              P[hp[u] + c * RHP] = add(z, mul(beta, ho[u][c]));
            }
      }
      iters = it;
      first = false;
      fstamp(it, 3);
    }
    if (status == MQ_OK && !converged) status = MQ_NOT_CONVERGED;
#pragma unroll
    for (int l = 0; l < LI; ++l)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if (l < li && own_ok && is_act(l, c)) a.x[own_e(l, c)] = X[Oidx(l, c)];
  }
done:
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    PcgOut o;
    o.iterations = iters;
    o.converged = converged;
    o.status = status;
    o.applies = applies0 + iters;
    o.rel = rel;
    o.bnorm = bnorm;
    o.alpha = alpha;
    o.rz = rz;
    *a.out = o;
  }
}

static const void *resident1_kernel_for(int li_max) {
  switch (li_max) {
    case 1: return (const void *)pcg_resident1_kernel<1>;
    case 2: return (const void *)pcg_resident1_kernel<2>;
    case 3: return (const void *)pcg_resident1_kernel<3>;
    default: return (const void *)pcg_resident1_kernel<4>;
  }
}

__host__ __device__ constexpr size_t res1_smem_bytes(int li) {
  return res_smem_bytes(li) + sizeof(double) * 3 * (size_t)(2 * RHP + li * RRING);
}

// single-reduction kernel unless MQ_PCG_SYNC=2 or the HR ring does not fit
static bool use_resident1(int li_max) {
  const char *v = getenv("MQ_PCG_SYNC");
  return !(v && v[0] == '2') && li_max <= 4;
}

static const void *resident_kernel_for(int li_max) {
  switch (li_max) {
    case 1: return (const void *)pcg_resident_kernel<1>;
    case 2: return (const void *)pcg_resident_kernel<2>;
    case 3: return (const void *)pcg_resident_kernel<3>;
    case 4: return (const void *)pcg_resident_kernel<4>;
    default: return (const void *)pcg_resident_kernel<5>;
  }
}

bool resident_single_reduction(int li_max) { return use_resident1(li_max); }

int pcg_stress_ns() {
  const char *v = getenv("MQ_PCG_STRESS");
  const int ns = v ? atoi(v) : 0;
  return ns > 0 ? (ns < 1000000 ? ns : 1000000) : 0;
}

// Returns 0 with *grid = 0 when the grid does not fit the resident scheme.
int resident_pcg_setup(int nx, int ny, int nz, int *grid, BrickGeo *geo_out) {
  *grid = 0;
  int dev = 0, sms = 0;
  MQ_CUDA(cudaGetDevice(&dev));
  MQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int tiles_k = (nz + RTK - 1) / RTK, tiles_j = (ny + RTJ - 1) / RTJ;
  const int tiles = tiles_k * tiles_j;
  if (tiles > sms) return MQ_OK;
  // smallest number of i-chunks with <= RLI_MAX planes, dividing nx if possible
  int best = 0;
  for (int c = (nx + RLI_MAX - 1) / RLI_MAX; c <= nx && tiles * c <= sms; ++c)
    if (nx % c == 0) { best = c; break; }
  if (!best) {
    const int c = (nx + RLI_MAX - 1) / RLI_MAX;
    if (tiles * c > sms) return MQ_OK;
    best = c;
  }
  // enough CTAs to be worth it (small grids run faster on the TMA brick
  // kernel with one plane per CTA)
  if (2 * tiles * best < sms) return MQ_OK;
  const int li_max = (nx + best - 1) / best;
  const bool one = use_resident1(li_max);
  const size_t smem = one ? res1_smem_bytes(li_max) : res_smem_bytes(li_max);
  const void *fn = one ? resident1_kernel_for(li_max) : resident_kernel_for(li_max);
  // both variants launchable (MQ_PCG_SYNC is read per launch)
  MQ_CUDA(cudaFuncSetAttribute(resident_kernel_for(li_max), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)res_smem_bytes(li_max)));
  if (li_max <= 4)
    MQ_CUDA(cudaFuncSetAttribute(resident1_kernel_for(li_max), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)res1_smem_bytes(li_max)));
  int per = 0;
  MQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, RT, smem));
  if (per < 1 || tiles * best > sms * per) return MQ_OK;
  if (tiles * best > 32 * 5) return MQ_OK;  // grid_partials_sum_all<*, 5>
  geo_out->nx = nx;
  geo_out->ny = ny;
  geo_out->nz = nz;
  geo_out->tiles_k = tiles_k;
  geo_out->tiles_j = tiles_j;
  geo_out->chunks = best;
  geo_out->nbricks = tiles * best;
  geo_out->xtiles = 0;
  geo_out->nbig = tiles * best;
  *grid = tiles * best;
  return MQ_OK;
}

int launch_pcg_resident(const StencilPcgArgs &args, const BrickGeo &geo, int grid, cudaStream_t s) {
  ResPcgArgs A;
  A.a = args;
  A.g.nx = geo.nx;
  A.g.ny = geo.ny;
  A.g.nz = geo.nz;
  A.g.tiles_k = geo.tiles_k;
  A.g.tiles_j = geo.tiles_j;
  A.g.chunks = geo.chunks;
  A.g.nbricks = geo.nbricks;
  A.g.li_max = (geo.nx + geo.chunks - 1) / geo.chunks;
  const bool one = use_resident1(A.g.li_max) && args.ap2 != nullptr;
  const size_t smem = one ? res1_smem_bytes(A.g.li_max) : res_smem_bytes(A.g.li_max);
  MQ_CUDA(cudaMemsetAsync(&args.bar->count, 0, sizeof(unsigned long long), s));
  void *params[] = {&A};
  const void *fn = one ? resident1_kernel_for(A.g.li_max) : resident_kernel_for(A.g.li_max);
  MQ_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(RT), params, smem, s));
  return MQ_OK;
}

}  // namespace mq

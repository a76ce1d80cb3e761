// Brick-tiled fused PCG for the K_n stencil with a TMA pipeline
// (krylov.py:174-250; same algorithm, stopping rule and bit-level arithmetic
// as pcg_stencil_kernel in pcg.cu, different work decomposition).
//
// K1 (the stencil pass).  Every CTA owns bricks: an 8 (j) x 32 (k) tile of
// node positions over a chunk of i planes, all three edge components.  It
// marches along i.  One elected thread streams each plane's (tile + 1-node
// halo) boxes of r and p_old for the three components into a 5-stage shared
// memory ring with 4-D TMA bulk tensor loads (cp.async.bulk.tensor, zero fill
// outside the box = the PEC/grid boundary), two planes ahead of the plane
// being computed, with mbarrier transaction counts for completion.  The raw
// r / p_old of a staged plane are converted in place into
// p_new = M^-1 r + beta p_old; each owner thread writes p_new of its own
// position and applies the deferred x += alpha_prev p_old.  The K_n rows of
// plane i are then evaluated from the three staged planes i-1, i, i+1.
//
// K2, the initial residual and the final x update are elementwise: flat,
// 16-byte vectorised, 4-way unrolled grid-stride passes over the padded
// vectors (entries that are not dofs hold 0 and stay 0).
//
// Streams per iteration (fp64, per dof): K1 reads r, p_old, x and writes
// x, p_new, Ap; K2 reads r, Ap and writes r  ->  9 x 8 B = 72 B.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>
#include <type_traits>

#include "mq_device.cuh"
#include "slab_rank.cuh"

namespace mq {

constexpr int TJ = 8, TK = 32;                 // kBlock = TJ * TK threads
constexpr int HJ = TJ + 2, HK = TK + 2, HP = HJ * HK;  // 10 x 34 box
constexpr int BOXP = HP;                       // one TMA box (34 x 10 x 1 x 3) fills a slot
#ifndef MQ_XDEFER
#define MQ_XDEFER 1
#endif
#ifndef MQ_NAHEAD
#define MQ_NAHEAD 3
#endif
// Two shared-memory rings: the r ring holds planes i-1, i, i+1 (converted
// in place into p_new, read by the stencil) plus NA planes in flight; the
// p_old ring only the NA in-flight planes (p_old is dead once its plane is
// converted).  Same bytes as a 5-stage (r, p) ring, one more plane ahead.
#ifndef MQ_STENCIL_CSE
#define MQ_STENCIL_CSE 1
#endif
// K1 stages of * p_new (the off-diagonal product of every staged value,
// formed once) instead of p_new: stencil3s, bit-identical rows
#ifndef MQ_PRESCALE
#define MQ_PRESCALE 1
#endif
constexpr int NA = MQ_NAHEAD;                  // planes in flight ahead of i+1
constexpr int NR = NA + 3, NP = NA;            // r-ring and p-ring slots
constexpr int NHALO = 2 * HK + 2 * TJ;         // 84 halo positions per plane
static_assert(TJ * TK == kBlock, "one thread per tile position");
static_assert(HP <= BOXP, "box slot");
static_assert(NA >= 1 && NR <= 32, "ring sizes");

// One staged plane of one field, three components packed as the 4-D TMA box
// (k, j, i, c) = (34, 10, 1, 3) lands: one bulk tensor load per field and
// plane (three per plane for r, p_old, Ap instead of nine).
struct __align__(128) Box3 {
  double v[3][BOXP];
};
static_assert(sizeof(Box3) % 128 == 0, "TMA destination alignment");

struct TmaPcgArgs {
  StencilPcgArgs a;
  BrickGeo g;
  CUtensorMap tm_r, tm_pa, tm_pb, tm_x;  // 4-D maps (k, j, i, c), box 34 x 10 x 1 x 3
};

constexpr size_t kTmaSmem = sizeof(Box3) * (NR + NP) + 128;
constexpr int kMaskPlanes = 64;  // MarchCtx::mrow capacity in planes
constexpr int kMaxMultiVec = 32;  // POD basis slots (MAXS)

// ---- PTX helpers ----------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(su32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void brick_of(const BrickGeo &g, int b, int &i0, int &i1, int &j0, int &k0) {
  const int tiles = g.tiles_k * g.tiles_j;
  int tile, ic, nch;
  if (b < g.nbig) {  // tiles [xtiles, tiles) in `chunks` i-chunks
    tile = g.xtiles + b % (tiles - g.xtiles);
    ic = b / (tiles - g.xtiles);
    nch = g.chunks;
  } else {  // tiles [0, xtiles) in chunks + 1
    const int b2 = b - g.nbig;
    tile = b2 % g.xtiles;
    ic = b2 / g.xtiles;
    nch = g.chunks + 1;
  }
  k0 = (tile % g.tiles_k) * TK;
  j0 = (tile / g.tiles_k) * TJ;
  i0 = (int)(((int64_t)ic * g.nx) / nch);
  i1 = (int)(((int64_t)(ic + 1) * g.nx) / nch);
}

// K_n row in CSR column order on a 3-plane neighbourhood:
// v(c', di, dj, dk) is the value of component c' at (i+di, j+dj, k+dk).
// Order and signs are those of stencil_row (mq_device.cuh).
template <class V>
__device__ __forceinline__ double stencil3(int c, double dg, double of, V v) {
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

// stencil3 with every off-diagonal product precomputed: v(c', di, dj, dk)
// returns of * p of that position (formed once per staged value when it is
// converted, the same rounding as forming it in every row that uses it), own
// is the raw p of the row's own position for the diagonal term.  Identical
// bits to stencil3 on the raw values; 13 -> 1 multiplication per row.
template <class V>
__device__ __forceinline__ double stencil3s(int c, double dg, double own, V v) {
  double s;
  if (c == 0) {
    s = -v(0, 0, -1, 0);
    s = sub(s, v(0, 0, 0, -1));
    s = add(s, mul(dg, own));
    s = sub(s, v(0, 0, 0, 1));
    s = sub(s, v(0, 0, 1, 0));
    s = add(s, v(1, 0, -1, 0));
    s = sub(s, v(1, 0, 0, 0));
    s = sub(s, v(1, 1, -1, 0));
    s = add(s, v(1, 1, 0, 0));
    s = add(s, v(2, 0, 0, -1));
    s = sub(s, v(2, 0, 0, 0));
    s = sub(s, v(2, 1, 0, -1));
    s = add(s, v(2, 1, 0, 0));
  } else if (c == 1) {
    s = v(0, -1, 0, 0);
    s = sub(s, v(0, -1, 1, 0));
    s = sub(s, v(0, 0, 0, 0));
    s = add(s, v(0, 0, 1, 0));
    s = sub(s, v(1, -1, 0, 0));
    s = sub(s, v(1, 0, 0, -1));
    s = add(s, mul(dg, own));
    s = sub(s, v(1, 0, 0, 1));
    s = sub(s, v(1, 1, 0, 0));
    s = add(s, v(2, 0, 0, -1));
    s = sub(s, v(2, 0, 0, 0));
    s = sub(s, v(2, 0, 1, -1));
    s = add(s, v(2, 0, 1, 0));
  } else {
    s = v(0, -1, 0, 0);
    s = sub(s, v(0, -1, 0, 1));
    s = sub(s, v(0, 0, 0, 0));
    s = add(s, v(0, 0, 0, 1));
    s = add(s, v(1, 0, -1, 0));
    s = sub(s, v(1, 0, -1, 1));
    s = sub(s, v(1, 0, 0, 0));
    s = add(s, v(1, 0, 0, 1));
    s = sub(s, v(2, -1, 0, 0));
    s = sub(s, v(2, 0, -1, 0));
    s = add(s, mul(dg, own));
    s = sub(s, v(2, 0, 1, 0));
    s = sub(s, v(2, 1, 0, 0));
  }
  return s;
}

// The three K_n rows of one node from pre-scaled staged values (stencil3s),
// each distinct neighbour value loaded once (24 shared-memory loads instead
// of 36, 16 with the thread's own staged values of planes i-1, i, i+1 kept
// in registers;
// identical arithmetic and order per row); own[c] / own[3+c] the raw /
// pre-scaled own p of the row's node.
template <class V, int NPV, int N, int NNV>
__device__ __forceinline__ void stencil3s_rows(double dg, const double (&prev)[NPV], const double (&own)[N],
                                               const double (&next)[NNV], V v, double (&av)[3]) {
  const double v0_0m10 = v(0, 0, -1, 0);
  const double v0_00m1 = v(0, 0, 0, -1);
  const double v0_001 = v(0, 0, 0, 1);
  const double v0_010 = v(0, 0, 1, 0);
  const double v1_0m10 = v(1, 0, -1, 0);
  const double v1_000 = own[4];  // own node, plane i: the value this thread staged
  const double v1_1m10 = v(1, 1, -1, 0);
  const double v1_100 = next[4];  // own node, plane i+1
  const double v2_00m1 = v(2, 0, 0, -1);
  const double v2_000 = own[5];  // own node, plane i: the value this thread staged
  const double v2_10m1 = v(2, 1, 0, -1);
  const double v2_100 = next[5];  // own node, plane i+1
  const double v0_m100 = prev[3];  // own node, plane i-1
  const double v0_m110 = v(0, -1, 1, 0);
  const double v0_000 = own[3];  // own node, plane i: the value this thread staged
  const double v1_m100 = prev[4];  // own node, plane i-1
  const double v1_00m1 = v(1, 0, 0, -1);
  const double v1_001 = v(1, 0, 0, 1);
  const double v2_01m1 = v(2, 0, 1, -1);
  const double v2_010 = v(2, 0, 1, 0);
  const double v0_m101 = v(0, -1, 0, 1);
  const double v1_0m11 = v(1, 0, -1, 1);
  const double v2_m100 = prev[5];  // own node, plane i-1
  const double v2_0m10 = v(2, 0, -1, 0);
  {
    double s;
    s = -v0_0m10;
    s = sub(s, v0_00m1);
    s = add(s, mul(dg, own[0]));
    s = sub(s, v0_001);
    s = sub(s, v0_010);
    s = add(s, v1_0m10);
    s = sub(s, v1_000);
    s = sub(s, v1_1m10);
    s = add(s, v1_100);
    s = add(s, v2_00m1);
    s = sub(s, v2_000);
    s = sub(s, v2_10m1);
    s = add(s, v2_100);
    av[0] = s;
  }
  {
    double s;
    s = v0_m100;
    s = sub(s, v0_m110);
    s = sub(s, v0_000);
    s = add(s, v0_010);
    s = sub(s, v1_m100);
    s = sub(s, v1_00m1);
    s = add(s, mul(dg, own[1]));
    s = sub(s, v1_001);
    s = sub(s, v1_100);
    s = add(s, v2_00m1);
    s = sub(s, v2_000);
    s = sub(s, v2_01m1);
    s = add(s, v2_010);
    av[1] = s;
  }
  {
    double s;
    s = v0_m100;
    s = sub(s, v0_m101);
    s = sub(s, v0_000);
    s = add(s, v0_001);
    s = add(s, v1_0m10);
    s = sub(s, v1_0m11);
    s = sub(s, v1_000);
    s = add(s, v1_001);
    s = sub(s, v2_m100);
    s = sub(s, v2_0m10);
    s = add(s, mul(dg, own[2]));
    s = sub(s, v2_010);
    s = sub(s, v2_100);
    av[2] = s;
  }
}


// stores / own-position loads of the march (experiments: cache operators)
#ifndef MQ_ST_MODE
#define MQ_ST_MODE 0
#endif
#ifndef MQ_LD_MODE
#define MQ_LD_MODE 0
#endif
__device__ __forceinline__ void st_out(double *p, double v) {
#if MQ_ST_MODE == 1
  __stcg(p, v);
#elif MQ_ST_MODE == 2
  __stcs(p, v);
#elif MQ_ST_MODE == 3
  __stwt(p, v);
#else
  *p = v;
#endif
}
__device__ __forceinline__ double ld_own(const double *p) {
#if MQ_LD_MODE == 1
  return __ldcs(p);
#elif MQ_LD_MODE == 2
  return __ldlu(p);
#else
  return __ldcg(p);
#endif
}

__device__ __forceinline__ int rslot(int q) { return (q + NR) % NR; }  // q >= -1
__device__ __forceinline__ int pslot(int q) { return (q + NP) % NP; }

// One brick of K1 (mode kK1) or of the initial residual r = b - A x0 (mode
// kInit: the marched field is x0, staged from tm_x).  Uniform per CTA.
// kK1R: K1 of the one-barrier kernel (pcg_tma1_kernel): the staged r is
// r_{k-2}, advanced to r_{k-1} = r_{k-2} - alpha_{k-1} Ap_{k-1} with the
// staged Ap_{k-1} before the conversion (own and halo positions, the same
// arithmetic as a K2 pass), r_{k-1} stored at the own positions, its r.r and
// r.z summed into mc.crr / mc.crz.
enum { kInit = 0, kK1 = 1, kK1R = 2 };

struct MarchCtx {
  Box3 *sr;        // NR slots of r (-> p_new); bars[] is indexed by r slot
  Box3 *sp;        // NP slots of p_old
  uint64_t *bars;
  uint32_t ph;  // per-slot mbarrier parity (identical in every thread)
  // kK1R only: NP slots of Ap_{k-1}, its map, the r_{k-1} output vector and
  // the own r.r / r.z partial sums
  Box3 *sa = nullptr;
  const CUtensorMap *ma = nullptr;
  double *rout = nullptr;
  double crr = 0.0, crz = 0.0;
  // planes i0-1 .. of the next march's first brick already in flight
  // (tma_preissue), skipped by its prologue
  int pre = 0;
  // one-barrier kernels: the active-dof bits of the brick's own positions,
  // one 32-bit word per (plane, component, tile row) aligned to the tile's
  // k0, kept in shared memory while the CTA stays on the brick (bricks of
  // <= kMaskPlanes planes); nullptr: the mask words are loaded per plane
  uint32_t *mrow = nullptr;
  int mi0 = -1, mj0 = -1, mk0 = -1;  // brick whose bits mrow holds
#ifdef MQ_TRACE_MARCH
  unsigned long long *tr = nullptr;  // CTA 0 thread 0, one iteration: 4 stamps per plane step
#endif
};

struct NoPush {
  __device__ __forceinline__ void operator()(int, int, int64_t, double) const {}
  __device__ __forceinline__ void operator()(int, int, int64_t, double, double) const {}
};

// The TMA loads of one staged plane q of a brick (tile origin j0, k0): the
// r (or x) box, with_p: the p_old box and, kK1R, the Ap box, all on the
// plane's r-slot mbarrier.  One thread.
template <int MODE, int NAT>
__device__ __forceinline__ void tma_issue_plane(MarchCtx &mc, const CUtensorMap *mr, const CUtensorMap *mp,
                                                bool with_p, int q, int j0, int k0) {
  constexpr int NRT = NAT + 3, NPT = NAT;
  const int s = (q + NRT) % NRT, sp = (q + NPT) % NPT;
  const uint32_t bytes = (with_p ? (MODE == kK1R ? 9u : 6u) : 3u) * HP * 8u;
  fence_proxy_async_smem();
  mbar_expect_tx(&mc.bars[s], bytes);
  // box origin (k0-1, j0-1, q) in node coordinates = (k0, j0, q+1) in the
  // guard-shifted map: never negative
  tma_load_4d(mc.sr[s].v[0], mr, &mc.bars[s], k0, j0, q + 1, 0);
  if (with_p) {
    tma_load_4d(mc.sp[sp].v[0], mp, &mc.bars[s], k0, j0, q + 1, 0);
    if (MODE == kK1R) tma_load_4d(mc.sa[sp].v[0], mc.ma, &mc.bars[s], k0, j0, q + 1, 0);
  }
}

// The prologue loads of the next march (planes i0-1 .. i0+NAT-2 of brick
// (i0, i1, j0, k0)) issued ahead, by thread `who`, right after the grid
// barrier that makes their data visible -- their latency then overlaps the
// partial-sum read.  Every thread records the count in mc.pre.
template <int MODE, int NAT, int DIR = 1>
__device__ __forceinline__ void tma_preissue(MarchCtx &mc, const CUtensorMap *mr, const CUtensorMap *mp,
                                             bool with_p, int i0, int i1, int j0, int k0, int who) {
  // the first staged planes of a march in direction DIR: i0-1, i0, .. (DIR > 0) or i1, i1-1, .. (DIR < 0)
  const int n = (NAT < i1 - i0 + 2) ? NAT : i1 - i0 + 2;
  if ((int)threadIdx.x == who) {
    fence_proxy_async_global();
    for (int t = 0; t < n; ++t) tma_issue_plane<MODE, NAT>(mc, mr, mp, with_p, DIR > 0 ? i0 - 1 + t : i1 - t, j0, k0);
  }
  mc.pre = n;
}

// Wait out pre-issued loads that no march will consume (the solve ended at
// this barrier): no bulk copy may still target the CTA's shared memory when
// it exits.
template <int NAT, int DIR = 1>
__device__ __forceinline__ void tma_drain(MarchCtx &mc, int i0, int i1) {
  constexpr int NRT = NAT + 3;
  for (int t = 0; t < mc.pre; ++t) {
    const int q = DIR > 0 ? i0 - 1 + t : i1 - t;
    const int s = (q + NRT) % NRT;
    mbar_wait(&mc.bars[s], (mc.ph >> s) & 1u);
    mc.ph ^= (1u << s);
  }
  mc.pre = 0;
}

// push(q, c, jk, v): p_new of an own active position of plane q (jk = its
// offset inside the padded plane), for the slab kernel's ghost stores;
// kK1R: push(q, c, jk, v, r) with the position's r_{k-1} as well
// XM2 = 0: the instance carries no deferred (two-term) x update: xmode != 0
// means x += a1 p_old (fewer live registers; the slab kernel's short bricks)
// DIR = -1: the brick is marched from plane i1-1 down to i0 (staged planes
// i1 .. i0-1): same rows, same arithmetic per row; the one-barrier kernel
// alternates the direction from pass to pass so that the planes a pass wrote
// last (r, p, Ap around the end of every brick, still in L2) are the first
// the next pass reads.
template <int MODE, int NAT = NA, int MC = 0, int XM2 = 1, int DIR = 1, class ROW, class PUSH = NoPush>
__device__ __forceinline__ void march_tma(MarchCtx &mc, const TmaPcgArgs &A, const CUtensorMap *mr,
                                          const CUtensorMap *mp, bool first, double beta, double alpha_prev,
                                          int xmode, double alpha_prev2, double *pnew, int i0, int i1, int j0,
                                          int k0, ROW row,
                                          PUSH push = PUSH()) {
  const StencilPcgArgs &a = A.a;
  const BrickGeo &g = A.g;
  // 32-bit element indices inside the march (brick_pcg_setup refuses layouts
  // of 2^31 entries or more): one IMAD / IMAD.WIDE per address instead of
  // 64-bit multiply chains, and half the registers per index
  const int LC = (int)a.L.C, LSi = (int)a.L.Si, LSj = (int)a.L.Sj, Loff = (int)a.L.off;
  constexpr int NRT = NAT + 3, NPT = NAT;  // ring slots (the kernel's allocation)
  auto rsl = [](int q) { return (q + NRT) % NRT; };  // q >= -1
  auto psl = [](int q) { return (q + NPT) % NPT; };
  const int tid = threadIdx.x, ty = tid >> 5, tx = tid & 31;
  const int j = j0 + ty, k = k0 + tx;
  const bool own_ok = j < g.ny && k < g.nz;
  const int s_own = (ty + 1) * HK + (tx + 1);
  const int pos_own = Loff + j * LSj + k;
  constexpr bool K1M = MODE == kK1 || MODE == kK1R;
  const bool with_p = K1M && !first;
  // x update of this pass (kK1, !first): 0 none (deferred), 1 x += a1 p_old,
  // 2 x = (x + a2 p_prev2) + a1 p_old with p_prev2 read from the p_new buffer
  // at the own position just before it is overwritten
  const int xm = (K1M && !first) ? (XM2 ? xmode : (xmode ? 1 : 0)) : 0;
  // halo (slot, component) converted by this thread besides its own
  // position: the 84 halo positions x 3 components are spread over threads
  // 0..251, one each, so that no warp carries three times the work
  int hs = -1;
  if (tid < 3 * NHALO) {
    const int h = tid % NHALO;
    const int hc = tid / NHALO;
    int hj, hk;
    if (h < HK) { hj = 0; hk = h; }
    else if (h < 2 * HK) { hj = TJ + 1; hk = h - HK; }
    else if (h < 2 * HK + TJ) { hj = 1 + (h - 2 * HK); hk = 0; }
    else { hj = 1 + (h - 2 * HK - TJ); hk = TK + 1; }
    hs = hc * BOXP + hj * HK + hk;  // offset inside a Box3
  }
  // z = M^-1 r as one product: 1.0 * r is r bit for bit without the
  // preconditioner, so the march carries no select per staged value
  const double invj = a.use_jac != 0 ? a.inv : 1.0;
  const uint32_t *mask = a.mask;
  double *x = a.x;
  // MC: own-position mask bits from shared memory (filled once per brick; the
  // prologue's first __syncthreads orders the fill before any read; the
  // caller guarantees bricks of <= kMaskPlanes planes)
  constexpr bool mcache = MC != 0;
  if (mcache && (mc.mi0 != i0 || mc.mj0 != j0 || mc.mk0 != k0)) {
    for (int w = tid; w < (i1 - i0) * 3 * TJ; w += kBlock) {
      const int q = i0 + w / (3 * TJ), c = (w / TJ) % 3, jj = j0 + w % TJ;
      uint32_t bits = 0u;
      if (jj < g.ny) {
        const int e0 = c * LC + q * LSi + Loff + jj * LSj + k0;
        const uint32_t w0 = __ldg(mask + (e0 >> 5));
        const uint32_t w1 = (e0 & 31) ? __ldg(mask + (e0 >> 5) + 1) : 0u;
        bits = __funnelshift_r(w0, w1, (uint32_t)(e0 & 31));
      }
      mc.mrow[w] = bits;
    }
    mc.mi0 = i0;
    mc.mj0 = j0;
    mc.mk0 = k0;
  }

  auto issue = [&](int q) {
    if (tid == 0) tma_issue_plane<MODE, NAT>(mc, mr, mp, with_p, q, j0, k0);
  };
  // Own-position mask words and x values are software-pipelined ahead in
  // registers: they are loaded while earlier planes are processed, so neither
  // their latency nor the TMA's is exposed.  eq = q * LSi + pos_own is the
  // own-position entry of plane q, component 0, carried along the march.
  struct OwnPre {
    uint32_t mw[3];
    double xo[3], p2[3];
  };
  auto prefetch_own = [&](OwnPre &o, int eq, bool own_plane) {
    if (own_plane && own_ok) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int e = c * LC + eq;
        o.mw[c] = mcache ? 0u : __ldg(mask + (e >> 5));
        if (xm >= 1) o.xo[c] = ld_own(x + e);
        if (XM2 && xm == 2) o.p2[c] = ld_own(pnew + e);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) o.mw[c] = 0u;
    }
  };
  // Ring slots are carried along the march (wrapping increments) instead of
  // q mod ring size at every use.
  auto winc = [](int s, int n) { return DIR > 0 ? (s + 1 == n ? 0 : s + 1) : (s == 0 ? n - 1 : s - 1); };  // next staged plane's slot
  // returns the active-dof bits (bit c = component c) of the own position;
  // s / sp: the r-ring and p-ring slots of plane q
  auto convert = [&](int q, int s, int sp, int eq, bool own_plane, const OwnPre &o, double (&raw)[9]) -> uint32_t {
#ifdef MQ_TRACE_MARCH
    if (mc.tr && q - i0 >= 1 && q - i0 < 33) mc.tr[4 * (q - i0 - 1) + 0] = globaltimer_ns();
#endif
    mbar_wait(&mc.bars[s], (mc.ph >> s) & 1u);
    mc.ph ^= (1u << s);
#ifdef MQ_TRACE_MARCH
    if (mc.tr && q - i0 >= 1 && q - i0 < 33) mc.tr[4 * (q - i0 - 1) + 1] = globaltimer_ns();
#endif
    uint32_t act = 0u;
    if (own_plane && own_ok) {
      if (mcache) {
        const uint32_t *mq = mc.mrow + (q - i0) * (3 * TJ) + ty;
#pragma unroll
        for (int c = 0; c < 3; ++c) act |= ((mq[c * TJ] >> tx) & 1u) << c;
      } else {
        const int sh = eq & 31;  // LC is a multiple of 32: the same bit position in the three words
#pragma unroll
        for (int c = 0; c < 3; ++c) act |= ((o.mw[c] >> sh) & 1u) << c;
      }
    }
    double *Sr = &mc.sr[s].v[0][0];
    if (MODE == kInit) {  // the staged x0 is used as is
#pragma unroll
      for (int c = 0; c < 3; ++c) raw[c] = raw[3 + c] = Sr[c * BOXP + s_own];
      return act;
    }
    const double *Sp = &mc.sp[sp].v[0][0];
    const double *Sa = &mc.sa[MODE == kK1R ? sp : 0].v[0][0];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int e = c * LC + eq;
      const bool on = (act >> c) & 1u;
      double rq = Sr[c * BOXP + s_own];
      if (MODE == kK1R && !first) rq = sub(rq, mul(alpha_prev, Sa[c * BOXP + s_own]));
      const double z = mul(invj, rq);
      double pv = z;
      if (!first) {
        const double po = Sp[c * BOXP + s_own];
        pv = add(z, mul(beta, po));
        if (xm >= 1 && on) {
          const double xv = (XM2 && xm == 2) ? add(o.xo[c], mul(alpha_prev2, o.p2[c])) : o.xo[c];
          st_out(x + e, add(xv, mul(alpha_prev, po)));
        }
      }
      raw[c] = pv;
      raw[3 + c] = (K1M && MQ_PRESCALE) ? mul(a.of, pv) : pv;
      raw[6 + c] = rq;
      Sr[c * BOXP + s_own] = raw[3 + c];
      if (on) {
        st_out(pnew + e, pv);
        if constexpr (MODE == kK1R) push(q, c, pos_own - LSi, pv, rq);
        else push(q, c, pos_own - LSi, pv);
        if (MODE == kK1R) {
          if (!first) st_out(mc.rout + e, rq);
          mc.crr = add(mc.crr, mul(rq, rq));
          mc.crz = add(mc.crz, mul(rq, z));
        }
      }
    }
    if (hs >= 0) {
      double rq = Sr[hs];
      if (MODE == kK1R && !first) rq = sub(rq, mul(alpha_prev, Sa[hs]));
      const double z = mul(invj, rq);
      const double ph = first ? z : add(z, mul(beta, Sp[hs]));
      Sr[hs] = (K1M && MQ_PRESCALE) ? mul(a.of, ph) : ph;
    }
    return act;
  };
  // sm1, s0, sp1: the r-ring slots of planes i-1, i, i+1; pm: the own
  // pre-scaled values of plane i-1
  auto stencil_plane = [&](int i, int sm1, int s0, int sp1, int ei, uint32_t act, const double (&pm)[3],
                           const double (&raw)[9], const double (&next)[9]) {
    if (!act) return;
    const double *bm1 = &mc.sr[sm1].v[0][0] + s_own, *b0 = &mc.sr[s0].v[0][0] + s_own,
                 *bp1 = &mc.sr[sp1].v[0][0] + s_own;
    auto ld = [&](int cc, int di, int dj, int dk) {
      const double *bq = di < 0 ? bm1 : (di == 0 ? b0 : bp1);
      return bq[cc * BOXP + dj * HK + dk];
    };
#if MQ_PRESCALE && MQ_STENCIL_CSE
    if constexpr (K1M) {
      // all three rows from the 24 distinct staged values, each loaded once;
      // the row callback receives the row value (kK1R: and the own r_{k-1})
      double av[3];
      // own pre-scaled values of the actual planes i-1 (prev[3..5]) and i+1
      // (next[4], next[5]): pm holds those of the plane staged before plane
      // i, next those of the plane staged after it
      const double prev[6] = {0.0, 0.0, 0.0, DIR > 0 ? pm[0] : next[3], DIR > 0 ? pm[1] : next[4],
                              DIR > 0 ? pm[2] : next[5]};
      const double nextd[6] = {0.0, 0.0, 0.0, 0.0, DIR > 0 ? next[4] : pm[1], DIR > 0 ? next[5] : pm[2]};
      // the pre-scaled own values of plane i are re-formed from the raw ones
      // (the same product as at the convert step) instead of being carried
      // in registers across the plane step
      const double own2[9] = {raw[0], raw[1], raw[2], mul(a.of, raw[0]), mul(a.of, raw[1]), mul(a.of, raw[2]),
                              raw[6], raw[7], raw[8]};
      stencil3s_rows(a.dg, prev, own2, nextd, ld, av);
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if ((act >> c) & 1u) {
          if constexpr (MODE == kK1R) row(c, c * LC + ei, av[c], raw[c], raw[6 + c], i);
          else row(c, c * LC + ei, av[c], raw[c]);
        }
      return;
    }
#else
    static_assert(MODE != kK1R, "kK1R needs the pre-scaled CSE stencil");
#endif
    if constexpr (MODE != kK1R) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if ((act >> c) & 1u) row(c, c * LC + ei, ld, raw[c]);
      }
    }
  };

  // The march in staging order: t = 0 .. n+1 are the planes i0-1 .. i1
  // (DIR > 0) or i1 .. i0-1 (DIR < 0), qa(t) the plane of step t; the own
  // planes are t = 1 .. n.
  // prologue: staged planes 0 .. NA-1 in flight, then convert 0 and 1, each
  // followed by the issue of the plane that takes over its p slot
  const int n = i1 - i0;
  auto qa = [&](int t) { return DIR > 0 ? i0 - 1 + t : i1 - t; };
  const int dE = DIR > 0 ? LSi : -LSi;
  // Prefetch register sets: two (plane t+2 loaded before plane t+1's set is
  // consumed) where the registers allow it; one, refilled right after the
  // convert step has consumed it (the loads have the barrier and the stencil
  // of plane t to land), in the one-barrier march, which carries r_{k-1} too
  // (two sets spill there: 128^3 97 us per iteration against 76).
  constexpr bool kTwoPre = MODE != kK1R;
  OwnPre oa, ob;
  double pm[3], ra[9], rb[9];  // own staged values: pre-scaled of plane t-1, all of planes t / t+1 (ping-pong)
#ifdef MQ_TRACE_MARCH
  if (mc.tr) mc.tr[128] = globaltimer_ns();  // march entry
#endif
  for (int t = mc.pre; t <= NAT - 1 && t <= n + 1; ++t) issue(qa(t));
  mc.pre = 0;
  int ei = qa(1) * LSi + pos_own;  // own entry of plane t, component 0
  prefetch_own(oa, ei, true);
  // ring slots of planes t-1, t, t+1 (r ring) and t+1 (p ring), carried
  int sl_m = rsl(qa(0)), sl_0 = winc(sl_m, NRT), sl_p = winc(sl_0, NRT), pp1 = psl(qa(2));
  convert(qa(0), sl_m, psl(qa(0)), ei - dE, false, oa, rb);
#pragma unroll
  for (int c = 0; c < 3; ++c) pm[c] = rb[3 + c];
  __syncthreads();
  if (NAT <= n + 1) issue(qa(NAT));
  if (kTwoPre) prefetch_own(ob, ei + dE, 2 <= n);
#ifdef MQ_TRACE_MARCH
  if (mc.tr) mc.tr[129] = globaltimer_ns();  // plane 0 converted
#endif
  uint32_t act = convert(qa(1), sl_0, psl(qa(1)), ei, true, oa, ra);
  if (!kTwoPre) prefetch_own(oa, ei + dE, 2 <= n);
  __syncthreads();
#ifdef MQ_TRACE_MARCH
  if (mc.tr) mc.tr[130] = globaltimer_ns();  // plane 1 converted (prologue done)
#endif
  if (NAT + 1 <= n + 1) issue(qa(NAT + 1));
  // one plane step: own = the staged own values of plane t (from the previous
  // step), nxt receives those of plane t+1; ocur holds the prefetched own
  // words of plane t+1, onxt receives those of plane t+2 (the same set when
  // there is one).  The march calls it with the register sets swapped every
  // plane (no rotation copies).
  auto step = [&](int t, double (&own)[9], double (&nxt)[9], OwnPre &ocur, OwnPre &onxt) {
    if (kTwoPre) prefetch_own(onxt, ei + 2 * dE, t + 2 <= n);
    const uint32_t act_next = convert(qa(t + 1), sl_p, pp1, ei + dE, t + 1 <= n, ocur, nxt);
    if (!kTwoPre) prefetch_own(onxt, ei + 2 * dE, t + 2 <= n);
#ifdef MQ_TRACE_MARCH
    if (mc.tr) mc.tr[4 * (t - 1) + 2] = globaltimer_ns();
#endif
    __syncthreads();
#ifdef MQ_TRACE_MARCH
    if (mc.tr) mc.tr[4 * (t - 1) + 3] = globaltimer_ns();
#endif
    // r slot of plane t-2 (its last stencil was before this barrier), p slot
    // of plane t+1 (converted before this barrier)
    if (t + NAT + 1 <= n + 1) issue(qa(t + NAT + 1));
    // slots of the actual planes i-1, i, i+1
    stencil_plane(qa(t), DIR > 0 ? sl_m : sl_p, sl_0, DIR > 0 ? sl_p : sl_m, ei, act, pm, own, nxt);
    act = act_next;
#pragma unroll
    for (int c = 0; c < 3; ++c) pm[c] = (K1M && MQ_PRESCALE) ? mul(a.of, own[c]) : own[3 + c];
    sl_m = sl_0;
    sl_0 = sl_p;
    sl_p = winc(sl_p, NRT);
    pp1 = winc(pp1, NPT);
    ei += dE;
  };
  {
    int t = 1;
    if (kTwoPre) {
      for (; t + 1 <= n; t += 2) {
        step(t, ra, rb, ob, oa);
        step(t + 1, rb, ra, oa, ob);
      }
      if (t <= n) step(t, ra, rb, ob, oa);
    } else {
      for (; t + 1 <= n; t += 2) {
        step(t, ra, rb, oa, oa);
        step(t + 1, rb, ra, oa, oa);
      }
      if (t <= n) step(t, ra, rb, oa, oa);
    }
  }
  __syncthreads();
#ifdef MQ_TRACE_MARCH
  if (mc.tr) mc.tr[131] = globaltimer_ns();  // march done
#endif
}

// flat 16-byte vectorised grid-stride helper over pairs of padded entries
constexpr int kUnroll = 8;  // 8 x 16 B loads per stream in flight per thread

template <class F>
__device__ __forceinline__ void flat_pairs(int64_t total, F f) {
  const int64_t npair = total >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; p + (kUnroll - 1) * stride < npair; p += kUnroll * stride) f(p, stride, kUnroll);
  for (; p < npair; p += stride) f(p, stride, 1);
}

#ifndef MQ_TMA_MINB
#define MQ_TMA_MINB 2
#endif
__global__ void __launch_bounds__(kBlock, MQ_TMA_MINB) pcg_tma_kernel(const __grid_constant__ TmaPcgArgs A) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bars[NR];
  __shared__ double red[3 * kWarps];
  __shared__ double tot[4];
  const StencilPcgArgs &a = A.a;
  const BrickGeo &g = A.g;
  const int G = gridDim.x;
  const Lay &L = a.L;
  const double dg = a.dg, of = a.of, inv = a.inv;
  const bool jac = a.use_jac != 0;
  double *x = a.x, *r = a.r, *ap = a.ap;
  const double *b = a.b;
  const int x0_mode = a.x0_mode_dev ? *a.x0_mode_dev : a.x0_mode;
  if (a.err_word && *((volatile const unsigned int *)a.err_word)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      PcgOut o{};
      o.status = 99;
      *a.out = o;
    }
    return;
  }
  MarchCtx mc;
  mc.sr = reinterpret_cast<Box3 *>(dsm + ((128u - (su32(dsm) & 127u)) & 127u));  // pointer arithmetic on dsm keeps the shared address space (LDS/STS, not generic LD/ST)
  mc.sp = mc.sr + NR;
  mc.bars = bars;
  mc.ph = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NR; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long *trace = (blockIdx.x == 0 && threadIdx.x == 0) ? a.trace : nullptr;
  auto stamp = [&](int slot) {
    if (trace && slot < 4 * 64 + 1) trace[slot] = globaltimer_ns();
  };
  stamp(0);
  // ---- initial residual (krylov.py:209-218) ----
  double v3[3] = {0.0, 0.0, 0.0};
  if (x0_mode == 1) {
    for (int bi = blockIdx.x; bi < g.nbricks; bi += G) {
      int i0, i1, j0, k0;
      brick_of(g, bi, i0, i1, j0, k0);
      march_tma<kInit>(mc, A, &A.tm_x, nullptr, true, 0.0, 0.0, 0, 0.0, nullptr, i0, i1, j0, k0,
                       [&](int c, int e, auto V, double) {
                         const double bv = __ldcg(b + e);
                         const double rv = sub(bv, stencil3(c, dg, of, V));
                         r[e] = rv;
                         const double z = jac ? mul(inv, rv) : rv;
                         v3[0] = add(v3[0], mul(bv, bv));
                         v3[1] = add(v3[1], mul(rv, rv));
                         v3[2] = add(v3[2], mul(rv, z));
                       });
    }
  } else {
    flat_pairs(L.total, [&](int64_t p, int64_t stride, int n) {
      double2 bv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (u < n) bv[u] = __ldcg(reinterpret_cast<const double2 *>(b) + p + u * stride);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (u < n) {
          reinterpret_cast<double2 *>(x)[p + u * stride] = make_double2(0.0, 0.0);
          reinterpret_cast<double2 *>(r)[p + u * stride] = bv[u];
          const double z0 = jac ? mul(inv, bv[u].x) : bv[u].x, z1 = jac ? mul(inv, bv[u].y) : bv[u].y;
          v3[0] = add(v3[0], mul(bv[u].x, bv[u].x));
          v3[0] = add(v3[0], mul(bv[u].y, bv[u].y));
          v3[2] = add(v3[2], mul(bv[u].x, z0));
          v3[2] = add(v3[2], mul(bv[u].y, z1));
        }
    });
    v3[1] = v3[0];
  }
  block_sum<3>(v3, red);
  if (threadIdx.x == 0) {
    a.partials[0 * G + blockIdx.x] = v3[0];
    a.partials[1 * G + blockIdx.x] = v3[1];
    a.partials[2 * G + blockIdx.x] = v3[2];
  }
  int status = MQ_OK, iters = 0, converged = 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  bool pold_is_a = true;  // pold = pa, pnew = pb
  int applies = (x0_mode == 2) ? 0 : 1;
  if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
  if (threadIdx.x == 0) fence_proxy_async_global();
  {
    double s3[3];
    grid_partials_sum<3>(a.partials, G, s3, tot);
    bnorm = sqrt(s3[0]);
    const double target = fmax(a.rel_tol * bnorm, a.abs_tol);
    double rnorm = sqrt(s3[1]);
    rz = jac ? s3[2] : s3[1];
    auto relf = [&](double res) { return bnorm > 0.0 ? res / bnorm : (res == 0.0 ? 0.0 : INFINITY); };
    if (rnorm <= target) { converged = 1; rel = relf(rnorm); goto done; }
    double beta = 0.0, alpha_prev = 0.0, alpha_prev2 = 0.0;
    bool first = true;
    // deferred x update: x += alpha_{it-1} p_{it-1} is applied every second
    // K1 together with the pending alpha_{it-2} p_{it-2} (same roundings in
    // the same order, one x read/write per two iterations)
    bool pend = false;
    for (int it = 1; it <= a.max_iter; ++it) {
      double *pnew = pold_is_a ? a.pb : a.pa;
      const CUtensorMap *mp = pold_is_a ? &A.tm_pa : &A.tm_pb;
      // ---- K1 ----
      int xmode = 0;
      if (!first) {
#if MQ_XDEFER
        xmode = pend ? 2 : 0;
        pend = !pend;
#else
        xmode = 1;
#endif
      }
      double v1[1] = {0.0};
#ifdef MQ_TRACE_MARCH
      mc.tr = (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && it == 10) ? a.trace + 1300 : nullptr;
#endif
      for (int bi = blockIdx.x; bi < g.nbricks; bi += G) {
        int i0, i1, j0, k0;
        brick_of(g, bi, i0, i1, j0, k0);
        march_tma<kK1>(mc, A, &A.tm_r, mp, first, beta, alpha_prev, xmode, alpha_prev2, pnew, i0, i1, j0, k0,
                       [&](int c, int e, auto V, double own) {
                         double av;
                         if constexpr (std::is_same_v<decltype(V), double>) av = V;  // stencil3s_rows
#if MQ_PRESCALE
                         else av = stencil3s(c, dg, own, V);
#else
                         else av = stencil3(c, dg, of, V);
#endif
                         ap[e] = av;
                         v1[0] = add(v1[0], mul(own, av));
                       });
      }
      block_sum<1>(v1, red);
      if (threadIdx.x == 0) a.partials[3 * G + blockIdx.x] = v1[0];
      ++applies;
      stamp(4 * (it - 1) + 1);
#ifdef MQ_TRACE_SPREAD
      if (a.trace && threadIdx.x == 0 && it == 10 && blockIdx.x < 1024) a.trace[1024 + blockIdx.x] = globaltimer_ns();
#endif
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      stamp(4 * (it - 1) + 2);
      stress_after_barrier(a.stress_ns, 2 * it);
      double s1[1];
      grid_partials_sum<1>(a.partials + 3 * G, G, s1, tot);
      const double pap = s1[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; goto done; }
      alpha = rz / pap;
      // ---- K2: r -= alpha Ap (flat, all padded entries; non-dofs stay 0) ----
      double v2[2] = {0.0, 0.0};
      flat_pairs(L.total, [&](int64_t p, int64_t stride, int n) {
        double2 rv[kUnroll], av[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (u < n) {
            rv[u] = __ldcg(reinterpret_cast<const double2 *>(r) + p + u * stride);
            av[u] = __ldcg(reinterpret_cast<const double2 *>(ap) + p + u * stride);
          }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (u < n) {
            const double r0 = sub(rv[u].x, mul(alpha, av[u].x));
            const double r1 = sub(rv[u].y, mul(alpha, av[u].y));
            reinterpret_cast<double2 *>(r)[p + u * stride] = make_double2(r0, r1);
            const double z0 = jac ? mul(inv, r0) : r0, z1 = jac ? mul(inv, r1) : r1;
            v2[0] = add(v2[0], mul(r0, r0));
            v2[0] = add(v2[0], mul(r1, r1));
            v2[1] = add(v2[1], mul(r0, z0));
            v2[1] = add(v2[1], mul(r1, z1));
          }
      });
      block_sum<2>(v2, red);
      if (threadIdx.x == 0) {
        a.partials[4 * G + blockIdx.x] = v2[0];
        a.partials[5 * G + blockIdx.x] = v2[1];
      }
      stamp(4 * (it - 1) + 3);
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      stamp(4 * (it - 1) + 4);
      stress_after_barrier(a.stress_ns, 2 * it + 1);
      if (threadIdx.x == 0) fence_proxy_async_global();
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
      alpha_prev2 = alpha_prev;
      alpha_prev = alpha;
      first = false;
      pold_is_a = !pold_is_a;
    }
    if (status == MQ_OK) {
      // last direction: p_new of the last iteration (swapped into pold when
      // the budget ran out)
      const double *pdir = converged ? (pold_is_a ? a.pb : a.pa) : (pold_is_a ? a.pa : a.pb);
      // the pending alpha_{K-1} p_{K-1} (deferred x update), applied first
      const double *pdir2 = converged ? (pold_is_a ? a.pa : a.pb) : (pold_is_a ? a.pb : a.pa);
      const double alpha2 = converged ? alpha_prev : alpha_prev2;
      if (pend) {
        flat_pairs(L.total, [&](int64_t p, int64_t stride, int n) {
          double2 xv[kUnroll], pv[kUnroll], qv[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            if (u < n) {
              xv[u] = __ldcg(reinterpret_cast<const double2 *>(x) + p + u * stride);
              qv[u] = __ldcg(reinterpret_cast<const double2 *>(pdir2) + p + u * stride);
              pv[u] = __ldcg(reinterpret_cast<const double2 *>(pdir) + p + u * stride);
            }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            if (u < n)
              reinterpret_cast<double2 *>(x)[p + u * stride] =
                  make_double2(add(add(xv[u].x, mul(alpha2, qv[u].x)), mul(alpha, pv[u].x)),
                               add(add(xv[u].y, mul(alpha2, qv[u].y)), mul(alpha, pv[u].y)));
        });
      } else {
        flat_pairs(L.total, [&](int64_t p, int64_t stride, int n) {
          double2 xv[kUnroll], pv[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            if (u < n) {
              xv[u] = __ldcg(reinterpret_cast<const double2 *>(x) + p + u * stride);
              pv[u] = __ldcg(reinterpret_cast<const double2 *>(pdir) + p + u * stride);
            }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            if (u < n)
              reinterpret_cast<double2 *>(x)[p + u * stride] =
                  make_double2(add(xv[u].x, mul(alpha, pv[u].x)), add(xv[u].y, mul(alpha, pv[u].y)));
        });
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

// ---------------------------------------------------------------------------
// One grid barrier per iteration (pcg_tma1_kernel, the default; MQ_PCG_SYNC=2
// selects pcg_tma_kernel above).  The reference's iteration
// (krylov.py:231-249) needs p.Ap before alpha and r.z after the r update.
// With the scalar Jacobi preconditioner (z = inv * r) the next r.z follows
// from scalars of the current pass,
//   |r - alpha Ap|^2 = r.r - 2 alpha r.Ap + alpha^2 Ap.Ap,
// so the K1 pass of iteration k reduces [p.Ap, r.Ap, Ap.Ap, r.r, r.z] once
// (D'Azevedo, Eijkhout & Romine's reduced-synchronisation CG; the same scheme
// as pcg_resident1_kernel).  The r update moves into the next pass: K1 of
// iteration k stages r_{k-2} and Ap_{k-1} with the TMA next to p_{k-1},
// forms r_{k-1} = r_{k-2} - alpha_{k-1} Ap_{k-1} in shared memory (own and
// halo positions, bit-identical) and stores it, then p_k = z + beta p_{k-1}
// and Ap_k as before; the flat K2 pass and its barrier are gone.  Only beta
// uses the extrapolated r.z; alpha uses r.z and the stopping test |r| <=
// target uses r.r, both summed from r_{k-1} itself, one barrier later: the
// test of iteration k-1 is read at the barrier of k, whose pass is then
// discarded (x, the iteration count, the application count and the reported
// residual are the reference's).  Exact-arithmetic iterates are unchanged; in
// fp64 they differ from the two-barrier kernel in the last bits (PCG parity
// bar: 1e-8 field, +-1 iteration).
// r and Ap are double-buffered (r_j in r / r2, Ap_j in ap / ap2 by the parity
// of j): the pass of k writes r_{k-1} and Ap_k while slower CTAs may still
// stage r_{k-2} and Ap_{k-1} around their bricks; the partial sums alternate
// between two sets for the same reason.
// Streams per iteration: r_{k-2}, Ap_{k-1}, p_{k-1} read, r_{k-1}, p_k, Ap_k
// written, x every second pass (read x, p_{k-2}; write x): 7.5 x 8 B/dof.
// ---------------------------------------------------------------------------
// planes in flight ahead of i+1 (two: the three rings of 9 slots fit the
// smem of the two-ring kernel with three, and leave the same L1 carveout)
#ifndef MQ_NAHEAD1
#define MQ_NAHEAD1 2
#endif
constexpr int NA1 = MQ_NAHEAD1, NR1 = NA1 + 3, NP1 = NA1;
#ifndef MQ_TMA_PREISSUE
#define MQ_TMA_PREISSUE 1
#endif
#ifndef MQ_SLAB_XDEFER
#define MQ_SLAB_XDEFER 1
#endif
// Alternating march direction (odd passes from the top plane of every brick
// down): opt-in.  Measured at 128^3: the L2 reuse is real (DRAM reads 13.22 ->
// 11.12 GB per 60 iterations, 398 -> 364 MB per iteration, L2 hit rate 35.8 ->
// 42.2 %) but an iteration takes 78.4 instead of 76.3 us -- the pass is bound
// by the latency of its staged planes (two in flight per CTA), not by DRAM
// bytes.
#ifndef MQ_SLAB_DEFER_SHORT
#define MQ_SLAB_DEFER_SHORT 0
#endif
#ifndef MQ_TMA_ALTDIR
#define MQ_TMA_ALTDIR 0
#endif
constexpr size_t kTmaSmem1 = sizeof(Box3) * (NR1 + 2 * NP1) + 128;

struct TmaPcg1Args {
  TmaPcgArgs t;
  CUtensorMap tm_r2, tm_a, tm_a2;  // r of odd j (a.r2); Ap of even (a.ap) / odd (a.ap2) j
};

__global__ void __launch_bounds__(kBlock, MQ_TMA_MINB) pcg_tma1_kernel(const __grid_constant__ TmaPcg1Args A1) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bars[NR1];
  __shared__ double red[5 * kWarps];
  __shared__ double tot[5];
  const TmaPcgArgs &A = A1.t;
  const StencilPcgArgs &a = A.a;
  const BrickGeo &g = A.g;
  const int G = gridDim.x;
  const Lay &L = a.L;
  const double dg = a.dg, of = a.of, inv = a.inv;
  const bool jac = a.use_jac != 0;
  double *x = a.x, *r = a.r;
  const double *b = a.b;
  const int x0_mode = a.x0_mode_dev ? *a.x0_mode_dev : a.x0_mode;
  if (a.err_word && *((volatile const unsigned int *)a.err_word)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      PcgOut o{};
      o.status = 99;
      *a.out = o;
    }
    return;
  }
  MarchCtx mc;
  mc.sr = reinterpret_cast<Box3 *>(dsm + ((128u - (su32(dsm) & 127u)) & 127u));  // pointer arithmetic on dsm keeps the shared address space (LDS/STS, not generic LD/ST)
  mc.sp = mc.sr + NR1;
  mc.sa = mc.sp + NP1;
  mc.bars = bars;
  __shared__ uint32_t mrow_s[kMaskPlanes * 3 * TJ];
  mc.mrow = mrow_s;
  mc.ph = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NR1; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long *trace = (blockIdx.x == 0 && threadIdx.x == 0) ? a.trace : nullptr;
  auto stamp = [&](int slot) {
    if (trace && slot < 4 * 64 + 1) trace[slot] = globaltimer_ns();
  };
  stamp(0);
  // ---- initial residual (krylov.py:209-218), as in pcg_tma_kernel ----
  double v3[3] = {0.0, 0.0, 0.0};
  if (x0_mode == 1) {
    for (int bi = blockIdx.x; bi < g.nbricks; bi += G) {
      int i0, i1, j0, k0;
      brick_of(g, bi, i0, i1, j0, k0);
      march_tma<kInit, NA1>(mc, A, &A.tm_x, nullptr, true, 0.0, 0.0, 0, 0.0, nullptr, i0, i1, j0, k0,
                       [&](int c, int e, auto V, double) {
                         const double bv = __ldcg(b + e);
                         const double rv = sub(bv, stencil3(c, dg, of, V));
                         r[e] = rv;
                         const double z = jac ? mul(inv, rv) : rv;
                         v3[0] = add(v3[0], mul(bv, bv));
                         v3[1] = add(v3[1], mul(rv, rv));
                         v3[2] = add(v3[2], mul(rv, z));
                       });
    }
  } else {
    flat_pairs(L.total, [&](int64_t p, int64_t stride, int n) {
      double2 bv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (u < n) bv[u] = __ldcg(reinterpret_cast<const double2 *>(b) + p + u * stride);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (u < n) {
          reinterpret_cast<double2 *>(x)[p + u * stride] = make_double2(0.0, 0.0);
          reinterpret_cast<double2 *>(r)[p + u * stride] = bv[u];
          const double z0 = jac ? mul(inv, bv[u].x) : bv[u].x, z1 = jac ? mul(inv, bv[u].y) : bv[u].y;
          v3[0] = add(v3[0], mul(bv[u].x, bv[u].x));
          v3[0] = add(v3[0], mul(bv[u].y, bv[u].y));
          v3[2] = add(v3[2], mul(bv[u].x, z0));
          v3[2] = add(v3[2], mul(bv[u].y, z1));
        }
    });
    v3[1] = v3[0];
  }
  block_sum<3>(v3, red);
  if (threadIdx.x == 0) {
    a.partials[0 * G + blockIdx.x] = v3[0];
    a.partials[1 * G + blockIdx.x] = v3[1];
    a.partials[2 * G + blockIdx.x] = v3[2];
  }
  int status = MQ_OK, iters = 0, converged = 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  bool pold_is_a = true;  // pold = pa, pnew = pb
  int applies = (x0_mode == 2) ? 0 : 1;
  if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
  if (threadIdx.x == 0) fence_proxy_async_global();
  {
    double s3[3];
    grid_partials_sum<3>(a.partials, G, s3, tot);
    bnorm = sqrt(s3[0]);
    const double target = fmax(a.rel_tol * bnorm, a.abs_tol);
    double rnorm = sqrt(s3[1]);
    rz = jac ? s3[2] : s3[1];
    auto relf = [&](double res) { return bnorm > 0.0 ? res / bnorm : (res == 0.0 ? 0.0 : INFINITY); };
    rel = relf(rnorm);
    if (rnorm <= target) { converged = 1; goto done; }
    if (a.max_iter < 1) { status = MQ_NOT_CONVERGED; goto done; }
    double beta = 0.0, alpha_prev = 0.0, alpha_prev2 = 0.0;
    bool pend = false;  // deferred x update, as in pcg_tma_kernel
    int xmode = 0;
    const int tid = threadIdx.x, ty = tid >> 5, tx = tid & 31;
    int pre_i0 = 0, pre_i1 = 0;  // brick whose prologue is pre-issued
    bool pre_back = false;
    // alternate march direction (odd passes backwards: pass 1 starts where
    // the initial-residual march ended) when every brick is short; long
    // bricks (256^3: vectors far larger than L2) march forwards
    const bool alt = MQ_TMA_ALTDIR && (g.nx + g.chunks - 1) / g.chunks <= kMaskPlanes;
    for (int it = 1;; ++it) {
      const bool first = it == 1;
      double *pnew = pold_is_a ? a.pb : a.pa;
      const CUtensorMap *mp = pold_is_a ? &A.tm_pa : &A.tm_pb;
      // r_j in (r, r2), Ap_j in (ap, ap2) by the parity of j
      const CUtensorMap *mr = (!first && (it & 1)) ? &A1.tm_r2 : &A.tm_r;  // r_{it-2} (r_0 when first)
      mc.ma = ((it - 1) & 1) ? &A1.tm_a2 : &A1.tm_a;                          // Ap_{it-1}
      mc.rout = ((it - 1) & 1) ? a.r2 : a.r;                                   // r_{it-1}
      double *apw = (it & 1) ? a.ap2 : a.ap;                                   // Ap_it
      mc.crr = 0.0;
      mc.crz = 0.0;
      xmode = 0;
      if (!first) {
#if MQ_XDEFER
        xmode = pend ? 2 : 0;
        pend = !pend;
#else
        xmode = 1;
#endif
      }
      double v[3] = {0.0, 0.0, 0.0};
      for (int bi = blockIdx.x; bi < g.nbricks; bi += G) {
        int i0, i1, j0, k0;
        brick_of(g, bi, i0, i1, j0, k0);
        auto rowf = [&](int, int e, double av, double own, double rown, int) {
          st_out(apw + e, av);
          v[0] = add(v[0], mul(own, av));
          v[1] = add(v[1], mul(rown, av));
          v[2] = add(v[2], mul(av, av));
        };
        // bricks of <= kMaskPlanes planes (the default geometry of this kernel):
        // own-position mask bits from shared memory
        if (alt && (it & 1))
          march_tma<kK1R, NA1, 1, 1, -1>(mc, A, mr, mp, first, beta, alpha_prev, xmode, alpha_prev2, pnew, i0, i1, j0, k0,
                                         rowf);
        else if (i1 - i0 <= kMaskPlanes)
          march_tma<kK1R, NA1, 1>(mc, A, mr, mp, first, beta, alpha_prev, xmode, alpha_prev2, pnew, i0, i1, j0, k0, rowf);
        else
          march_tma<kK1R, NA1, 0>(mc, A, mr, mp, first, beta, alpha_prev, xmode, alpha_prev2, pnew, i0, i1, j0, k0, rowf);
      }
      double v5[5] = {v[0], v[1], v[2], mc.crr, mc.crz};
      block_sum<5>(v5, red);
      double *pt = a.partials + 3 * G + (it & 1) * 5 * G;
      if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) pt[q * G + blockIdx.x] = v5[q];
      }
      ++applies;
      stamp(4 * (it - 1) + 1);
#ifdef MQ_TRACE_SPREAD
      if (a.trace && threadIdx.x == 0 && it == 10 && blockIdx.x < 512) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[1024 + blockIdx.x] = globaltimer_ns();
        a.trace[1536 + blockIdx.x] = smid;
      }
#endif
      if (!grid_sync(a.bar)) { status = MQ_CUDA_ERROR; goto done; }
      stamp(4 * (it - 1) + 2);
      stress_after_barrier(a.stress_ns, it);
      if (threadIdx.x == 0) fence_proxy_async_global();
#if MQ_TMA_PREISSUE
      // the next pass's first planes, in flight while the sums are read
      // (its maps depend only on the iteration parity)
      if ((int)blockIdx.x < g.nbricks) {
        int i0, i1, j0, k0;
        brick_of(g, blockIdx.x, i0, i1, j0, k0);
        mc.ma = (it & 1) ? &A1.tm_a2 : &A1.tm_a;
        pre_back = alt && ((it + 1) & 1);
        if (pre_back)
          tma_preissue<kK1R, NA1, -1>(mc, ((it + 1) & 1) ? &A1.tm_r2 : &A.tm_r, pold_is_a ? &A.tm_pb : &A.tm_pa, true,
                                      i0, i1, j0, k0, 5 * 32);
        else
          tma_preissue<kK1R, NA1, 1>(mc, ((it + 1) & 1) ? &A1.tm_r2 : &A.tm_r, pold_is_a ? &A.tm_pb : &A.tm_pa, true,
                                     i0, i1, j0, k0, 5 * 32);
        pre_i0 = i0;
        pre_i1 = i1;
      }
#endif
      double s5[5];
      {
        // warp q < 5 sums partial row q in a fixed order (identical in every CTA)
        if (ty < 5) {
          double pv[kPB];
#pragma unroll
          for (int u = 0; u < kPB; ++u) {
            const int bb = tx + 32 * u;
            pv[u] = bb < G ? __ldcg(pt + (int64_t)ty * G + bb) : 0.0;
          }
          double sacc = 0.0;
#pragma unroll
          for (int u = 0; u < kPB; ++u)
            if (tx + 32 * u < G) sacc = add(sacc, pv[u]);
          for (int bb = tx + 32 * kPB; bb < G; bb += 32) sacc = add(sacc, __ldcg(pt + (int64_t)ty * G + bb));
          sacc = warp_sum(sacc);
          if (tx == 0) tot[ty] = sacc;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 5; ++q) s5[q] = tot[q];
        __syncthreads();
      }
      stamp(4 * (it - 1) + 3);
      stamp(4 * (it - 1) + 4);
      if (!first) {
        // the test of iteration it-1 (krylov.py:239-246) on r_{it-1}; this
        // pass is then discarded
        rnorm = sqrt(s5[3]);
        iters = it - 1;
        rel = relf(rnorm);
        if (rnorm <= target) { converged = 1; --applies; break; }
        const double rz_d = jac ? s5[4] : s5[3];
        if (!isfinite(rz_d)) { status = MQ_INDEFINITE; break; }
        rz = rz_d;
        if (it - 1 >= a.max_iter) { --applies; break; }  // budget spent: iters == max_iter
      }
      const double pap = s5[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; break; }
      alpha = rz / pap;
      {
        // beta from the extrapolated r.z of r_it
        const double rr_new = add(sub(s5[3], mul(mul(2.0, alpha), s5[1])), mul(mul(alpha, alpha), s5[2]));
        const double rz_new = jac ? mul(inv, rr_new) : rr_new;
        beta = rz_new > 0.0 ? rz_new / rz : 0.0;
      }
      alpha_prev2 = alpha_prev;
      alpha_prev = alpha;
      pold_is_a = !pold_is_a;
    }
    if (mc.pre) {
      if (pre_back) tma_drain<NA1, -1>(mc, pre_i0, pre_i1);
      else tma_drain<NA1, 1>(mc, pre_i0, pre_i1);
    }
    if (status == MQ_OK) {
      // the pass that read the final test ran with xmode 2 (x complete) or 0:
      // x += alpha_K p_K pending, p_K = that pass's p_old
      if (xmode == 0) {
        const double *pdir = pold_is_a ? a.pa : a.pb;
        const double aK = alpha;
        flat_pairs(L.total, [&](int64_t p, int64_t stride, int n) {
          double2 xv[kUnroll], pv[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            if (u < n) {
              xv[u] = __ldcg(reinterpret_cast<const double2 *>(x) + p + u * stride);
              pv[u] = __ldcg(reinterpret_cast<const double2 *>(pdir) + p + u * stride);
            }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            if (u < n)
              reinterpret_cast<double2 *>(x)[p + u * stride] =
                  make_double2(add(xv[u].x, mul(aK, pv[u].x)), add(xv[u].y, mul(aK, pv[u].y)));
        });
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

// ---------------------------------------------------------------------------
// Fused slab variant (configs[4]): the kernel above on one i-slab per rank,
// its grid barriers replaced by the rank all-reduce of slab_rank.cuh, and
// the planes 0 / n-1 of r and p_new stored into the neighbour ranks' ghost
// planes (p_new from the TMA march, r after the flat K2 pass by the thread
// that updated it).  Ranks are CTA groups: one group per launch on a GPU of
// its own, or all ranks as the groups of one launch when emulated.
// ---------------------------------------------------------------------------
struct TmaSlabGroup {
  TmaPcgArgs t;
  SlabRank rk;
};

struct TmaSlabArgs {
  TmaSlabGroup grp[kMaxRanks];
  int ngroups, nranks, rank0;
};

// flat pass by the Gr CTAs of one group over the pairs of the OWNED planes
// (padded planes 1..n of each component): the ghost planes are written by
// the neighbour ranks concurrently and must not be touched
template <class F>
__device__ __forceinline__ void flat_pairs_owned(const Lay &L, int n, int lb, int Gr, F f) {
  const int64_t stride = (int64_t)Gr * blockDim.x;
  const int64_t p0 = (int64_t)lb * blockDim.x + threadIdx.x;
  for (int c = 0; c < 3; ++c) {
    const int64_t a = (c * L.C + L.Si) >> 1, b = (c * L.C + (int64_t)(n + 1) * L.Si) >> 1;
    int64_t p = a + p0;
    for (; p + (kUnroll - 1) * stride < b; p += kUnroll * stride) f(p, stride, kUnroll);
    for (; p < b; p += stride) f(p, stride, 1);
  }
}

// the pairs of planes 0 and n-1 (padded planes 1 and n) of vector v owned by
// this thread in flat_pairs_owned's mapping, stored into the neighbours'
// ghost planes
__device__ __forceinline__ void push_planes_group(const SlabRank &me, const double *v, double *lo, double *hi, int lb,
                                                  int Gr) {
  const Lay &L = me.L;
  const int64_t stride = (int64_t)Gr * blockDim.x;
  const int64_t p0 = (int64_t)lb * blockDim.x + threadIdx.x;
  const int64_t half = L.Si >> 1;  // pairs per padded plane (Si is even)
  for (int side = 0; side < 2; ++side) {
    double *dst = side == 0 ? lo : hi;
    if (!dst) continue;
    const int64_t plane = side == 0 ? 1 : me.n;
    for (int c = 0; c < 3; ++c) {
      const int64_t a = (c * L.C + L.Si) >> 1;               // start of the owned pairs
      const int64_t pa = (c * L.C + plane * L.Si) >> 1, pb = pa + half;
      const int64_t d = pa - a - p0;
      int64_t p = a + p0 + (d > 0 ? (d + stride - 1) / stride : 0) * stride;
      const int64_t dbase = side == 0 ? (c * me.lo_C + me.lo_top) : (c * me.hi_C);
      for (; p < pb; p += stride) {
        const double2 w = __ldcg(reinterpret_cast<const double2 *>(v) + p);
        const int64_t jk = 2 * p - (c * L.C + plane * L.Si);
        dst[dbase + jk] = w.x;
        dst[dbase + jk + 1] = w.y;
      }
    }
  }
}

__global__ void __launch_bounds__(kBlock, 2) pcg_tma_slab_kernel(const __grid_constant__ TmaSlabArgs S) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bars[NR];
  __shared__ double red[3 * kWarps];
  __shared__ double tot[4];
  const int Gr = gridDim.x / S.ngroups;
  const int gi = blockIdx.x / Gr, lb = blockIdx.x % Gr;
  const TmaPcgArgs &A = S.grp[gi].t;
  const SlabRank &me = S.grp[gi].rk;
  const int rank = S.rank0 + gi, R = S.nranks;
  const StencilPcgArgs &a = A.a;
  const BrickGeo &g = A.g;
  const Lay &L = a.L;
  const double dg = a.dg, of = a.of, inv = a.inv;
  const bool jac = a.use_jac != 0;
  double *x = a.x, *r = a.r, *ap = a.ap;
  const double *b = a.b;
  const int x0_mode = a.x0_mode;
  MarchCtx mc;
  mc.sr = reinterpret_cast<Box3 *>(dsm + ((128u - (su32(dsm) & 127u)) & 127u));  // pointer arithmetic on dsm keeps the shared address space (LDS/STS, not generic LD/ST)
  mc.sp = mc.sr + NR;
  mc.bars = bars;
  mc.ph = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NR; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long inst = *me.epoch;
  int status = MQ_OK, iters = 0, converged = 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  bool pold_is_a = true;
  int applies = (x0_mode == 2) ? 0 : 1;
  double v3[3] = {0.0, 0.0, 0.0};
  auto push_r = [&](int64_t e, double v) {  // own row e of r (init pass)
    const int c = e < L.C ? 0 : (e < 2 * L.C ? 1 : 2);
    const int64_t rel_e = e - c * L.C, plane = rel_e / L.Si, jk = rel_e - plane * L.Si;
    if (plane == 1 && me.lo_r) me.lo_r[c * me.lo_C + me.lo_top + jk] = v;
    if (plane == me.n && me.hi_r) me.hi_r[c * me.hi_C + jk] = v;
  };
  // ---- initial residual (krylov.py:209-218) ----
  if (x0_mode == 1) {
    // x0 ghost planes first (the march stages planes -1 and n)
    push_planes_group(me, x, me.lo_x, me.hi_x, lb, Gr);
    double v0[1] = {0.0};
    if (!rank_allreduce<1>(me, R, rank, lb, Gr, inst++, v0, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
    if (threadIdx.x == 0) fence_proxy_async_global();
    for (int bi = lb; bi < g.nbricks; bi += Gr) {
      int i0, i1, j0, k0;
      brick_of(g, bi, i0, i1, j0, k0);
      march_tma<kInit>(mc, A, &A.tm_x, nullptr, true, 0.0, 0.0, 0, 0.0, nullptr, i0, i1, j0, k0,
                       [&](int c, int e, auto V, double) {
                         const double bv = __ldcg(b + e);
                         const double rv = sub(bv, stencil3(c, dg, of, V));
                         r[e] = rv;
                         push_r(e, rv);
                         const double z = jac ? mul(inv, rv) : rv;
                         v3[0] = add(v3[0], mul(bv, bv));
                         v3[1] = add(v3[1], mul(rv, rv));
                         v3[2] = add(v3[2], mul(rv, z));
                       });
    }
  } else {
    flat_pairs_owned(L, me.n, lb, Gr, [&](int64_t p, int64_t stride, int n) {
      double2 bv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (u < n) bv[u] = __ldcg(reinterpret_cast<const double2 *>(b) + p + u * stride);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (u < n) {
          reinterpret_cast<double2 *>(x)[p + u * stride] = make_double2(0.0, 0.0);
          reinterpret_cast<double2 *>(r)[p + u * stride] = bv[u];
          const double z0 = jac ? mul(inv, bv[u].x) : bv[u].x, z1 = jac ? mul(inv, bv[u].y) : bv[u].y;
          v3[0] = add(v3[0], mul(bv[u].x, bv[u].x));
          v3[0] = add(v3[0], mul(bv[u].y, bv[u].y));
          v3[2] = add(v3[2], mul(bv[u].x, z0));
          v3[2] = add(v3[2], mul(bv[u].y, z1));
        }
    });
    v3[1] = v3[0];
    push_planes_group(me, r, me.lo_r, me.hi_r, lb, Gr);
  }
  if (!rank_allreduce<3>(me, R, rank, lb, Gr, inst++, v3, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
  if (threadIdx.x == 0) fence_proxy_async_global();
  {
    bnorm = sqrt(v3[0]);
    const double target = fmax(a.rel_tol * bnorm, a.abs_tol);
    double rnorm = sqrt(v3[1]);
    rz = jac ? v3[2] : v3[1];
    auto relf = [&](double res) { return bnorm > 0.0 ? res / bnorm : (res == 0.0 ? 0.0 : INFINITY); };
    if (rnorm <= target) { converged = 1; rel = relf(rnorm); goto done; }
    double beta = 0.0, alpha_prev = 0.0;
    bool first = true;
    for (int it = 1; it <= a.max_iter; ++it) {
      double *pnew = pold_is_a ? a.pb : a.pa;
      double *lo_pn = pold_is_a ? me.lo_pb : me.lo_pa, *hi_pn = pold_is_a ? me.hi_pb : me.hi_pa;
      const CUtensorMap *mp = pold_is_a ? &A.tm_pa : &A.tm_pb;
      const int nmax = me.n - 1;
      auto push_p = [&](int q, int c, int64_t jk, double v) {
        if (q == 0 && lo_pn) lo_pn[c * me.lo_C + me.lo_top + jk] = v;
        if (q == nmax && hi_pn) hi_pn[c * me.hi_C + jk] = v;
      };
      // ---- K1 ----
      double v1[1] = {0.0};
      for (int bi = lb; bi < g.nbricks; bi += Gr) {
        int i0, i1, j0, k0;
        brick_of(g, bi, i0, i1, j0, k0);
        march_tma<kK1>(mc, A, &A.tm_r, mp, first, beta, alpha_prev, 1, 0.0, pnew, i0, i1, j0, k0,
                       [&](int c, int e, auto V, double own) {
                         double av;
                         if constexpr (std::is_same_v<decltype(V), double>) av = V;  // stencil3s_rows
#if MQ_PRESCALE
                         else av = stencil3s(c, dg, own, V);
#else
                         else av = stencil3(c, dg, of, V);
#endif
                         ap[e] = av;
                         v1[0] = add(v1[0], mul(own, av));
                       },
                       push_p);
      }
      ++applies;
      if (!rank_allreduce<1>(me, R, rank, lb, Gr, inst++, v1, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
      stress_after_barrier(a.stress_ns, 2 * it);
      const double pap = v1[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; goto done; }
      alpha = rz / pap;
      // ---- K2 ----
      double v2[2] = {0.0, 0.0};
      flat_pairs_owned(L, me.n, lb, Gr, [&](int64_t p, int64_t stride, int n) {
        double2 rv[kUnroll], av[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (u < n) {
            rv[u] = __ldcg(reinterpret_cast<const double2 *>(r) + p + u * stride);
            av[u] = __ldcg(reinterpret_cast<const double2 *>(ap) + p + u * stride);
          }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (u < n) {
            const double r0 = sub(rv[u].x, mul(alpha, av[u].x));
            const double r1 = sub(rv[u].y, mul(alpha, av[u].y));
            reinterpret_cast<double2 *>(r)[p + u * stride] = make_double2(r0, r1);
            const double z0 = jac ? mul(inv, r0) : r0, z1 = jac ? mul(inv, r1) : r1;
            v2[0] = add(v2[0], mul(r0, r0));
            v2[0] = add(v2[0], mul(r1, r1));
            v2[1] = add(v2[1], mul(r0, z0));
            v2[1] = add(v2[1], mul(r1, z1));
          }
      });
      push_planes_group(me, r, me.lo_r, me.hi_r, lb, Gr);
      if (!rank_allreduce<2>(me, R, rank, lb, Gr, inst++, v2, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
      stress_after_barrier(a.stress_ns, 2 * it + 1);
      if (threadIdx.x == 0) fence_proxy_async_global();
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
      pold_is_a = !pold_is_a;
    }
    if (status == MQ_OK) {
      const double *pdir = converged ? (pold_is_a ? a.pb : a.pa) : (pold_is_a ? a.pa : a.pb);
      flat_pairs_owned(L, me.n, lb, Gr, [&](int64_t p, int64_t stride, int n) {
        double2 xv[kUnroll], pv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (u < n) {
            xv[u] = __ldcg(reinterpret_cast<const double2 *>(x) + p + u * stride);
            pv[u] = __ldcg(reinterpret_cast<const double2 *>(pdir) + p + u * stride);
          }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (u < n)
            reinterpret_cast<double2 *>(x)[p + u * stride] =
                make_double2(add(xv[u].x, mul(alpha, pv[u].x)), add(xv[u].y, mul(alpha, pv[u].y)));
      });
      if (!converged) status = MQ_NOT_CONVERGED;
    }
  }
done:
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
    *a.out = o;
  }
}

// One-barrier slab variant (pcg_tma1_kernel's recurrence on one i-slab per
// rank): one rank all-reduce of [p.Ap, r.Ap, Ap.Ap, r.r, r.z] per iteration
// instead of two.  The march stores r_{k-1} (convert), p_k (convert) and Ap_k
// (row) of the planes 0 / n-1 into the neighbours' ghost planes of the
// buffers of that parity; the next pass stages them through the halo.  x is
// updated in every pass (x += alpha_{k-1} p_{k-1}), so the discarded pass that
// reads the last test leaves x complete.  The default for every slab depth
// (MQ_PCG_SYNC=2 selects pcg_tma_slab_kernel).
struct TmaSlab1Group {
  TmaPcg1Args t1;
  SlabRank rk;
};

struct TmaSlab1Args {
  TmaSlab1Group grp[kMaxRanks];
  int ngroups, nranks, rank0;
};

__global__ void __launch_bounds__(kBlock, MQ_TMA_MINB) pcg_tma1_slab_kernel(const __grid_constant__ TmaSlab1Args S) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bars[NR1];
  __shared__ double red[5 * kWarps];
  __shared__ double tot[5];
  const int Gr = gridDim.x / S.ngroups;
  const int gi = blockIdx.x / Gr, lb = blockIdx.x % Gr;
  const TmaPcg1Args &A1 = S.grp[gi].t1;
  const TmaPcgArgs &A = A1.t;
  const SlabRank &me = S.grp[gi].rk;
  const int rank = S.rank0 + gi, R = S.nranks;
  const StencilPcgArgs &a = A.a;
  const BrickGeo &g = A.g;
  const Lay &L = a.L;
  const double dg = a.dg, of = a.of, inv = a.inv;
  const bool jac = a.use_jac != 0;
  double *x = a.x, *r = a.r;
  const double *b = a.b;
  const int x0_mode = a.x0_mode;
  MarchCtx mc;
  mc.sr = reinterpret_cast<Box3 *>(dsm + ((128u - (su32(dsm) & 127u)) & 127u));  // pointer arithmetic on dsm keeps the shared address space (LDS/STS, not generic LD/ST)
  mc.sp = mc.sr + NR1;
  mc.sa = mc.sp + NP1;
  mc.bars = bars;
  __shared__ uint32_t mrow_s[kMaskPlanes * 3 * TJ];
  mc.mrow = mrow_s;
  mc.ph = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NR1; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long inst = *me.epoch;
  int status = MQ_OK, iters = 0, converged = 0;
  double rel = 0.0, bnorm = 0.0, alpha = 0.0, rz = 0.0;
  bool pold_is_a = true;
  int applies = (x0_mode == 2) ? 0 : 1;
  double v3[3] = {0.0, 0.0, 0.0};
  const int nmax = me.n - 1;
  auto push_r = [&](int64_t e, double v) {  // own row e of r (init pass)
    const int c = e < L.C ? 0 : (e < 2 * L.C ? 1 : 2);
    const int64_t rel_e = e - c * L.C, plane = rel_e / L.Si, jk = rel_e - plane * L.Si;
    if (plane == 1 && me.lo_r) me.lo_r[c * me.lo_C + me.lo_top + jk] = v;
    if (plane == me.n && me.hi_r) me.hi_r[c * me.hi_C + jk] = v;
  };
  // ---- initial residual (krylov.py:209-218), as in pcg_tma_slab_kernel ----
  if (x0_mode == 1) {
    push_planes_group(me, x, me.lo_x, me.hi_x, lb, Gr);
    double v0[1] = {0.0};
    if (!rank_allreduce<1>(me, R, rank, lb, Gr, inst++, v0, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
    if (threadIdx.x == 0) fence_proxy_async_global();
    for (int bi = lb; bi < g.nbricks; bi += Gr) {
      int i0, i1, j0, k0;
      brick_of(g, bi, i0, i1, j0, k0);
      march_tma<kInit, NA1>(mc, A, &A.tm_x, nullptr, true, 0.0, 0.0, 0, 0.0, nullptr, i0, i1, j0, k0,
                            [&](int c, int e, auto V, double) {
                              const double bv = __ldcg(b + e);
                              const double rv = sub(bv, stencil3(c, dg, of, V));
                              r[e] = rv;
                              push_r(e, rv);
                              const double z = jac ? mul(inv, rv) : rv;
                              v3[0] = add(v3[0], mul(bv, bv));
                              v3[1] = add(v3[1], mul(rv, rv));
                              v3[2] = add(v3[2], mul(rv, z));
                            });
    }
  } else {
    flat_pairs_owned(L, me.n, lb, Gr, [&](int64_t p, int64_t stride, int n) {
      double2 bv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (u < n) bv[u] = __ldcg(reinterpret_cast<const double2 *>(b) + p + u * stride);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (u < n) {
          reinterpret_cast<double2 *>(x)[p + u * stride] = make_double2(0.0, 0.0);
          reinterpret_cast<double2 *>(r)[p + u * stride] = bv[u];
          const double z0 = jac ? mul(inv, bv[u].x) : bv[u].x, z1 = jac ? mul(inv, bv[u].y) : bv[u].y;
          v3[0] = add(v3[0], mul(bv[u].x, bv[u].x));
          v3[0] = add(v3[0], mul(bv[u].y, bv[u].y));
          v3[2] = add(v3[2], mul(bv[u].x, z0));
          v3[2] = add(v3[2], mul(bv[u].y, z1));
        }
    });
    v3[1] = v3[0];
    push_planes_group(me, r, me.lo_r, me.hi_r, lb, Gr);
  }
  if (!rank_allreduce<3>(me, R, rank, lb, Gr, inst++, v3, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
  if (threadIdx.x == 0) fence_proxy_async_global();
  {
    bnorm = sqrt(v3[0]);
    const double target = fmax(a.rel_tol * bnorm, a.abs_tol);
    double rnorm = sqrt(v3[1]);
    rz = jac ? v3[2] : v3[1];
    auto relf = [&](double res) { return bnorm > 0.0 ? res / bnorm : (res == 0.0 ? 0.0 : INFINITY); };
    rel = relf(rnorm);
    if (rnorm <= target) { converged = 1; goto done; }
    if (a.max_iter < 1) { status = MQ_NOT_CONVERGED; goto done; }
    double beta = 0.0, alpha_prev = 0.0, alpha_prev2 = 0.0;
    // deferred x update as in pcg_tma1_kernel (MQ_SLAB_XDEFER) for long
    // bricks (> kMaskPlanes planes: slabs of 128 / 256 planes, 671 -> 625 us
    // per iteration at one rank); short bricks (slabs of <= 64 planes) update
    // x every pass: the two-term update's extra registers spill in this
    // kernel (32-plane slab 89.8 -> 91.4 us).  Uniform per launch.
    const bool defer = MQ_SLAB_XDEFER && (MQ_SLAB_DEFER_SHORT || (g.nx + g.chunks - 1) / g.chunks > kMaskPlanes);
    bool pend = false;
    int xmode = 0;
    for (int it = 1;; ++it) {
      const bool first = it == 1;
      xmode = 0;
      if (!first) {
        if (defer) {
          xmode = pend ? 2 : 0;
          pend = !pend;
        } else {
          xmode = 1;
        }
      }
      double *pnew = pold_is_a ? a.pb : a.pa;
      const CUtensorMap *mp = pold_is_a ? &A.tm_pa : &A.tm_pb;
      const bool odd_r = (it - 1) & 1;  // r_{it-1} goes to r2 when odd
      const bool odd_a = it & 1;        // Ap_it goes to ap2 when odd
      const CUtensorMap *mr = (!first && (it & 1)) ? &A1.tm_r2 : &A.tm_r;
      mc.ma = odd_r ? &A1.tm_a2 : &A1.tm_a;
      mc.rout = odd_r ? a.r2 : a.r;
      double *apw = odd_a ? a.ap2 : a.ap;
      mc.crr = 0.0;
      mc.crz = 0.0;
      // Ghost stores: after the march of a brick that holds the slab's first
      // or last plane, every thread re-reads the p_new, r_{k-1} and Ap_k it
      // stored itself at its own position of that plane (L1/L2 hits) and
      // stores them into the neighbour ranks' ghost planes -- the plane loop
      // itself carries no ghost logic (it is the march of pcg_tma1_kernel: 395
      // instead of ~ 880 instructions per plane step).  Neighbour pointers are
      // read from the kernel parameters where they are used.
      auto push_edges = [&](int i0, int i1, int j0, int k0) {
        const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
        const int j = j0 + ty, kk = k0 + tx;
        if (j >= g.ny || kk >= g.nz) return;
        const int64_t pos = L.off + (int64_t)j * L.Sj + kk, jk = pos - L.Si;
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const int q = side == 0 ? 0 : nmax;
          if (q < i0 || q >= i1) continue;
          double *dp = side == 0 ? (pold_is_a ? me.lo_pb : me.lo_pa) : (pold_is_a ? me.hi_pb : me.hi_pa);
          if (!dp) continue;
          double *dr = side == 0 ? (odd_r ? me.lo_r2 : me.lo_r) : (odd_r ? me.hi_r2 : me.hi_r);
          double *da = side == 0 ? (odd_a ? me.lo_a2 : me.lo_a) : (odd_a ? me.hi_a2 : me.hi_a);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const int64_t e = c * L.C + (int64_t)q * L.Si + pos;
            if (!((__ldg(a.mask + (e >> 5)) >> (e & 31)) & 1u)) continue;
            const int64_t d = side == 0 ? c * me.lo_C + me.lo_top + jk : c * me.hi_C + jk;
            dp[d] = pnew[e];
            if (!first) dr[d] = mc.rout[e];
            da[d] = apw[e];
          }
        }
      };
      double v[3] = {0.0, 0.0, 0.0};
      for (int bi = lb; bi < g.nbricks; bi += Gr) {
        int i0, i1, j0, k0;
        brick_of(g, bi, i0, i1, j0, k0);
        auto rowf = [&](int, int e, double av, double own, double rown, int) {
          apw[e] = av;
          v[0] = add(v[0], mul(own, av));
          v[1] = add(v[1], mul(rown, av));
          v[2] = add(v[2], mul(av, av));
        };
#if MQ_SLAB_DEFER_SHORT
        if (i1 - i0 <= kMaskPlanes)
          march_tma<kK1R, NA1, 1, 1>(mc, A, mr, mp, first, beta, alpha_prev, xmode, alpha_prev2, pnew, i0, i1, j0, k0,
                                     rowf);
#else
        if (!defer && i1 - i0 <= kMaskPlanes)
          march_tma<kK1R, NA1, 1, 0>(mc, A, mr, mp, first, beta, alpha_prev, xmode, 0.0, pnew, i0, i1, j0, k0, rowf);
#endif
        else
          march_tma<kK1R, NA1, 0, 1>(mc, A, mr, mp, first, beta, alpha_prev, xmode, alpha_prev2, pnew, i0, i1, j0, k0,
                                     rowf);
        push_edges(i0, i1, j0, k0);
      }
      ++applies;
      double v5[5] = {v[0], v[1], v[2], mc.crr, mc.crz};
      if (!rank_allreduce<5>(me, R, rank, lb, Gr, inst++, v5, red, tot)) { status = MQ_CUDA_ERROR; goto done; }
      stress_after_barrier(a.stress_ns, it);
      if (threadIdx.x == 0) fence_proxy_async_global();
      if (!first) {
        // the test of iteration it-1 on r_{it-1}; this pass is then discarded
        rnorm = sqrt(v5[3]);
        iters = it - 1;
        rel = relf(rnorm);
        if (rnorm <= target) { converged = 1; --applies; break; }
        const double rz_d = jac ? v5[4] : v5[3];
        if (!isfinite(rz_d)) { status = MQ_INDEFINITE; break; }
        rz = rz_d;
        if (it - 1 >= a.max_iter) { --applies; break; }
      }
      const double pap = v5[0];
      if (!isfinite(pap) || pap <= 0.0) { status = MQ_INDEFINITE; iters = it; break; }
      alpha = rz / pap;
      {
        const double rr_new = add(sub(v5[3], mul(mul(2.0, alpha), v5[1])), mul(mul(alpha, alpha), v5[2]));
        const double rz_new = jac ? mul(inv, rr_new) : rr_new;
        beta = rz_new > 0.0 ? rz_new / rz : 0.0;
      }
      alpha_prev2 = alpha_prev;
      alpha_prev = alpha;
      pold_is_a = !pold_is_a;
    }
    if (status == MQ_OK && defer && xmode == 0) {
      // the pass that read the final test left x += alpha_K p_K pending
      // (p_K = that pass's p_old); with xmode 2 x is complete
      const double *pdir = pold_is_a ? a.pa : a.pb;
      const double aK = alpha;
      flat_pairs_owned(L, me.n, lb, Gr, [&](int64_t p, int64_t stride, int n) {
        double2 xv[kUnroll], pv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (u < n) {
            xv[u] = __ldcg(reinterpret_cast<const double2 *>(x) + p + u * stride);
            pv[u] = __ldcg(reinterpret_cast<const double2 *>(pdir) + p + u * stride);
          }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (u < n)
            reinterpret_cast<double2 *>(x)[p + u * stride] =
                make_double2(add(xv[u].x, mul(aK, pv[u].x)), add(xv[u].y, mul(aK, pv[u].y)));
      });
    }
    if (status == MQ_OK && !converged) status = MQ_NOT_CONVERGED;
  }
done:
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
    *a.out = o;
  }
}

// K_n SpMV through the same TMA march (y on active rows only).
__global__ void __launch_bounds__(kBlock, 2) kn_apply_tma_kernel(const __grid_constant__ TmaPcgArgs A,
                                                                 double *__restrict__ y) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bars[NR];
  MarchCtx mc;
  mc.sr = reinterpret_cast<Box3 *>(dsm + ((128u - (su32(dsm) & 127u)) & 127u));  // pointer arithmetic on dsm keeps the shared address space (LDS/STS, not generic LD/ST)
  mc.sp = mc.sr + NR;
  mc.bars = bars;
  mc.ph = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NR; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int bi = blockIdx.x; bi < A.g.nbricks; bi += gridDim.x) {
    int i0, i1, j0, k0;
    brick_of(A.g, bi, i0, i1, j0, k0);
    march_tma<kInit>(mc, A, &A.tm_x, nullptr, true, 0.0, 0.0, 0, 0.0, nullptr, i0, i1, j0, k0,
                     [&](int c, int e, auto V, double own) { y[e] = stencil3(c, A.a.dg, A.a.of, V); });
  }
}

// K_n applied to the POD basis vectors B_j, j < *kptr (the k SpMVs of
// pod_start_vector, startvec.py:296): blockIdx.y = j, the same TMA march as
// kn_apply_tma_kernel with one tensor map per basis slot.
struct KnMultiArgs {
  TmaPcgArgs A;
  const int *kptr;
  double *y[kMaxMultiVec];
  CUtensorMap tm[kMaxMultiVec];
};

__global__ void __launch_bounds__(kBlock, 2) kn_apply_tma_multi_kernel(const __grid_constant__ KnMultiArgs M) {
  const int j = blockIdx.y;
  if (j >= *M.kptr) return;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bars[NR];
  MarchCtx mc;
  mc.sr = reinterpret_cast<Box3 *>(dsm + ((128u - (su32(dsm) & 127u)) & 127u));  // pointer arithmetic on dsm keeps the shared address space (LDS/STS, not generic LD/ST)
  mc.sp = mc.sr + NR;
  mc.bars = bars;
  mc.ph = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NR; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double *y = M.y[j];
  for (int bi = blockIdx.x; bi < M.A.g.nbricks; bi += gridDim.x) {
    int i0, i1, j0, k0;
    brick_of(M.A.g, bi, i0, i1, j0, k0);
    march_tma<kInit>(mc, M.A, &M.tm[j], nullptr, true, 0.0, 0.0, 0, 0.0, nullptr, i0, i1, j0, k0,
                     [&](int c, int e, auto V, double) { y[e] = stencil3(c, M.A.a.dg, M.A.a.of, V); });
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encoder() {
  if (g_encode) return MQ_OK;
  cudaDriverEntryPointQueryResult q;
  void *fn = nullptr;
  MQ_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return MQ_CUDA_ERROR;
  }
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  return MQ_OK;
}

// 4-D view (k, j, i, c) of a padded device vector including the guard layer
// (coordinate 0 = node -1); box = tile + 1-node halo, all three components.
int make_vec_map(const Lay &L, int nx, int ny, int nz, const double *base, CUtensorMap *map, int bk = HK, int bj = HJ) {
  int rc = get_encoder();
  if (rc) return rc;
  cuuint64_t dims[4] = {(cuuint64_t)nz + 2, (cuuint64_t)ny + 2, (cuuint64_t)nx + 2, 3};
  cuuint64_t strides[3] = {(cuuint64_t)L.Sj * 8, (cuuint64_t)L.Si * 8, (cuuint64_t)L.C * 8};
  cuuint32_t box[4] = {(cuuint32_t)bk, (cuuint32_t)bj, 1, 3};  // all three components
  cuuint32_t estr[4] = {1, 1, 1, 1};
  // the map starts at node (-1,-1,-1) of component 0: index off - Si - Sj - 1 = 0
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void *)base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return MQ_CUDA_ERROR;
  }
  return MQ_OK;
}

static BrickGeo make_geo(int nx, int ny, int nz, int resident) {
  BrickGeo g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  g.tiles_k = (nz + TK - 1) / TK;
  g.tiles_j = (ny + TJ - 1) / TJ;
  const int tiles = g.tiles_k * g.tiles_j;
  int chunks = resident / tiles;
  if (chunks < 1) chunks = 1;
  if (chunks > nx) chunks = nx;
  // equal bricks: the largest chunk count <= the budget that divides nx (the
  // grid barrier waits for the longest brick)
  for (int c = chunks; c >= 1; --c)
    if (nx % c == 0) {
      if (2 * c >= chunks) chunks = c;
      break;
    }
  if (const char *v = getenv("MQ_BRICK_CHUNKS")) {  // experiments: fixed i-chunk count
    const int c = atoi(v);
    if (c >= 1 && c <= nx) chunks = c;
  }
  g.chunks = chunks;
  g.nbricks = tiles * chunks;
  g.xtiles = 0;
  g.nbig = g.nbricks;
  return g;
}

// Mixed chunking for the one-barrier kernel (opt-in, MQ_BRICK_MIX=1; measured
// slower at 128^3: 81.2 -> 84.4 us per iteration, the pass of CTA 0 69.6 ->
// 74.7 us with every SM carrying two CTAs -- the SMs are not the bound, see
// DESIGN.md §3).  When
// the co-resident CTA count R is not a multiple of the tile count, the first
// x = R mod tiles tiles (whole rows of tiles along j, so that the i-chunk
// boundaries of neighbouring tiles coincide everywhere but at one row
// boundary: the halo rows a brick stages are then rows its neighbour streamed
// a moment earlier, read from L2) are cut into chunks + 1 i-chunks, the rest
// into chunks, so that all R slots hold a brick.  The longer bricks take CTA
// indices [0, nbig), the shorter ones the rest: with two CTAs per SM, CTA b
// and CTA b + R/2 share an SM (%smid census), so every long brick shares its
// SM with a short one.  At 128^3: 96 bricks of 32 planes + 200 of 25-26 on
// 296 slots (the equal split: 256 bricks of 32 planes, 40 SMs with one CTA).
// The split depends only on the grid, never on the CTA placement: the
// partial sums, hence the iterates, stay run-to-run deterministic.
static BrickGeo make_geo_mixed(int nx, int ny, int nz, int resident) {
  BrickGeo g = make_geo(nx, ny, nz, resident);
  const char *v = getenv("MQ_BRICK_MIX");
  if (!v || atoi(v) != 1) return g;
  const int tiles = g.tiles_k * g.tiles_j;
  const int c = resident / tiles, x = resident - c * tiles;
  if (c < 1 || x == 0 || c + 1 > nx) return g;
  if ((nx + c - 1) / c > 64) return g;  // two-barrier bricks: keep equal
  if (x % g.tiles_k != 0) return g;     // whole tile rows only
  const int nbig = (tiles - x) * c;
  if (nbig > resident / 2) return g;    // every long brick paired with a short one
  g.chunks = c;
  g.xtiles = x;
  g.nbig = nbig;
  g.nbricks = resident;
  return g;
}

// Shared-memory carveout of the TMA kernels: the smallest preference at which
// the occupancy calculator places two CTAs per SM, so the rest stays L1.  The
// L1 share matters: with the largest carveout (28 KB L1) the global loads and
// stores of K1 throttle (ncu stall_lg 0.61 -> 1.53 per issue) and an iteration
// at 128^3 takes 104 instead of 94 us; left to the driver the carveout
// sometimes fits only one CTA per SM (118 us).  MQ_PCG_CARVEOUT overrides.
//
// One grid barrier per iteration (pcg_tma1_kernel) at every brick length.
// Before the march's instruction diet the one-barrier pass lost at 256^3
// (256-plane bricks: 657 vs 642 us per iteration -- the single pass carried
// the whole iteration's CTA imbalance) and the two-barrier kernel was kept
// for bricks of more than 64 planes; with the leaner march the pass is
// DRAM-bound and the imbalance small: 128^3 75.8 vs 85.5, 256^3 551.5 vs
// 612.8 us per iteration.  MQ_PCG_SYNC=1|2 forces either (pcg_tma_kernel stays
// as the two-barrier reference variant); read per launch.
static bool tma_one_barrier(const BrickGeo &g) {
  (void)g;
  if (const char *v = getenv("MQ_PCG_SYNC")) {
    const int k = atoi(v);
    if (k == 1 || k == 2) return k == 1;
  }
  return true;
}
bool tma_single_reduction(const BrickGeo &g) { return tma_one_barrier(g); }

static cudaError_t two_cta_carveout(const void *fn, int want = 2, size_t smem = kTmaSmem) {
  int pct = 100;
  for (int c = 50; c <= 100; ++c) {
    int per2 = 0;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, c);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, fn, kBlock, smem);
    if (e != cudaSuccess) return e;
    if (per2 >= want) { pct = c; break; }
  }
  if (const char *v = getenv("MQ_PCG_CARVEOUT")) pct = atoi(v);
  if (getenv("MQ_PCG_VERBOSE")) fprintf(stderr, "TMA kernel carveout preference %d %%\n", pct);
  return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct < 100 ? pct : 100);
}

int brick_pcg_setup(const Lay &L, int nx, int ny, int nz, int sm_cap, int *grid, BrickGeo *geo) {
  // the march indexes entries with 32-bit integers
  if (L.total >= (int64_t)1 << 31) { set_error("TMA PCG kernels: padded vector of 2^31 entries or more"); return MQ_INVALID; }
  int dev = 0, sms = 0, per = 0;
  MQ_CUDA(cudaGetDevice(&dev));
  MQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (sm_cap > 0 && sm_cap < sms) sms = sm_cap;
  MQ_CUDA(cudaFuncSetAttribute(pcg_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
  MQ_CUDA(cudaFuncSetAttribute(pcg_tma1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem1));
  MQ_CUDA(cudaFuncSetAttribute(kn_apply_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
  MQ_CUDA(two_cta_carveout((const void *)pcg_tma_kernel, MQ_TMA_MINB));
  MQ_CUDA(two_cta_carveout((const void *)pcg_tma1_kernel, MQ_TMA_MINB, kTmaSmem1));
  MQ_CUDA(two_cta_carveout((const void *)kn_apply_tma_kernel));
  MQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, pcg_tma_kernel, kBlock, kTmaSmem));
  static_assert(kTmaSmem1 <= kTmaSmem || 2 * (kTmaSmem1 + 8 * 1024) <= 227 * 1024, "both TMA PCG kernels place two CTAs per SM");
  if (getenv("MQ_PCG_VERBOSE")) fprintf(stderr, "pcg_tma_kernel: %d CTAs per SM, %zu B smem\n", per, kTmaSmem);
  if (per < 1) { set_error("TMA PCG kernel cannot be resident"); return MQ_CUDA_ERROR; }
  if (const char *v = getenv("MQ_BRICK_CTAS_PER_SM")) {
    const int want = atoi(v);
    if (want >= 1 && want < per) per = want;
  }
  const int resident = sms * per;
  *geo = make_geo_mixed(nx, ny, nz, resident);
  *grid = geo->nbricks < resident ? geo->nbricks : resident;
  return MQ_OK;
}

int launch_pcg_brick(const StencilPcgArgs &args, const BrickGeo &geo, int grid, cudaStream_t s) {
  TmaPcgArgs A;
  std::memset(&A, 0, sizeof(A));
  A.a = args;
  A.g = geo;
  const Lay &L = args.L;
  int rc = make_vec_map(L, geo.nx, geo.ny, geo.nz, args.r, &A.tm_r);
  rc = rc ? rc : make_vec_map(L, geo.nx, geo.ny, geo.nz, args.pa, &A.tm_pa);
  rc = rc ? rc : make_vec_map(L, geo.nx, geo.ny, geo.nz, args.pb, &A.tm_pb);
  rc = rc ? rc : make_vec_map(L, geo.nx, geo.ny, geo.nz, args.x, &A.tm_x);
  if (rc) return rc;
  MQ_CUDA(cudaMemsetAsync(&args.bar->count, 0, sizeof(unsigned long long), s));
  if (tma_one_barrier(geo) && args.r2 && args.ap2) {
    TmaPcg1Args A1;
    std::memset(&A1, 0, sizeof(A1));
    A1.t = A;
    rc = make_vec_map(L, geo.nx, geo.ny, geo.nz, args.r2, &A1.tm_r2);
    rc = rc ? rc : make_vec_map(L, geo.nx, geo.ny, geo.nz, args.ap, &A1.tm_a);
    rc = rc ? rc : make_vec_map(L, geo.nx, geo.ny, geo.nz, args.ap2, &A1.tm_a2);
    if (rc) return rc;
    void *params[] = {&A1};
    MQ_CUDA(cudaLaunchCooperativeKernel((const void *)pcg_tma1_kernel, dim3(grid), dim3(kBlock), params, kTmaSmem1, s));
    return MQ_OK;
  }
  void *params[] = {&A};
  MQ_CUDA(cudaLaunchCooperativeKernel((const void *)pcg_tma_kernel, dim3(grid), dim3(kBlock), params, kTmaSmem, s));
  return MQ_OK;
}

// groups[q] = (PCG arguments, rank description) of the q-th group of this
// launch; nplanes[q] its owned planes.  Tensor maps and brick geometry are
// built here; grid = the co-resident CTA count split evenly over the groups.
int launch_pcg_tma_slab(const StencilPcgArgs *args, const SlabRank *ranks, const int *nplanes, int ngroups,
                        int nranks, int rank0, int ny, int nz, cudaStream_t s) {
  if (ngroups < 1 || ngroups > kMaxRanks) { set_error("1..8 rank groups per launch"); return MQ_INVALID; }
  for (int q = 0; q < ngroups; ++q)
    if (args[q].L.total >= (int64_t)1 << 31) { set_error("TMA PCG kernels: padded vector of 2^31 entries or more"); return MQ_INVALID; }
  int dev = 0, sms = 0, per = 0;
  MQ_CUDA(cudaGetDevice(&dev));
  MQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  MQ_CUDA(cudaFuncSetAttribute(pcg_tma_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
  MQ_CUDA(two_cta_carveout((const void *)pcg_tma_slab_kernel));
  MQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, pcg_tma_slab_kernel, kBlock, kTmaSmem));
  if (per < 1) { set_error("TMA slab PCG kernel cannot be resident"); return MQ_CUDA_ERROR; }
  const int Gr = (sms * per) / ngroups;
  if (Gr < 1) { set_error("too many rank groups for one GPU"); return MQ_INVALID; }
  TmaSlabArgs *S = new TmaSlabArgs;
  std::memset(S, 0, sizeof(TmaSlabArgs));
  S->ngroups = ngroups;
  S->nranks = nranks;
  S->rank0 = rank0;
  int rc = MQ_OK;
  for (int q = 0; q < ngroups && rc == MQ_OK; ++q) {
    TmaPcgArgs &t = S->grp[q].t;
    t.a = args[q];
    t.g = make_geo(nplanes[q], ny, nz, Gr);
    const Lay &L = args[q].L;
    rc = make_vec_map(L, nplanes[q], ny, nz, args[q].r, &t.tm_r);
    rc = rc ? rc : make_vec_map(L, nplanes[q], ny, nz, args[q].pa, &t.tm_pa);
    rc = rc ? rc : make_vec_map(L, nplanes[q], ny, nz, args[q].pb, &t.tm_pb);
    rc = rc ? rc : make_vec_map(L, nplanes[q], ny, nz, args[q].x, &t.tm_x);
    S->grp[q].rk = ranks[q];
  }
  if (rc == MQ_OK) {
    for (int q = 0; q < ngroups; ++q) {
      cudaError_t e = cudaMemsetAsync(&args[q].bar->count, 0, sizeof(unsigned long long), s);
      if (e != cudaSuccess) { rc = cuda_fail(e, "slab barrier reset"); break; }
    }
  }
  // one rank all-reduce per iteration unless MQ_PCG_SYNC=2 (measured faster
  // at every slab depth: one GPU's slab of configs[4] split 1/2/4/8 ways,
  // 687/343/181/100 -> 660/327/169/92 us per iteration), when the contexts
  // carry the double buffers
  const char *sv = getenv("MQ_PCG_SYNC");
  bool one = !(sv && atoi(sv) == 2);
  for (int q = 0; q < ngroups; ++q) one = one && args[q].r2 && args[q].ap2;
  if (rc == MQ_OK && one) {
    TmaSlab1Args *S1 = new TmaSlab1Args;
    std::memset(S1, 0, sizeof(TmaSlab1Args));
    S1->ngroups = ngroups;
    S1->nranks = nranks;
    S1->rank0 = rank0;
    for (int q = 0; q < ngroups && rc == MQ_OK; ++q) {
      TmaPcg1Args &t1 = S1->grp[q].t1;
      t1.t = S->grp[q].t;
      const Lay &L = args[q].L;
      rc = make_vec_map(L, nplanes[q], ny, nz, args[q].r2, &t1.tm_r2);
      rc = rc ? rc : make_vec_map(L, nplanes[q], ny, nz, args[q].ap, &t1.tm_a);
      rc = rc ? rc : make_vec_map(L, nplanes[q], ny, nz, args[q].ap2, &t1.tm_a2);
      S1->grp[q].rk = S->grp[q].rk;
    }
    if (rc == MQ_OK) {
      MQ_CUDA(cudaFuncSetAttribute(pcg_tma1_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem1));
      MQ_CUDA(two_cta_carveout((const void *)pcg_tma1_slab_kernel, 2, kTmaSmem1));
      void *params[] = {S1};
      cudaError_t e = cudaLaunchCooperativeKernel((const void *)pcg_tma1_slab_kernel, dim3(Gr * ngroups),
                                                  dim3(kBlock), params, kTmaSmem1, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "TMA slab PCG launch");
    }
    delete S1;
    delete S;
    return rc;
  }
  if (rc == MQ_OK) {
    void *params[] = {S};
    cudaError_t e = cudaLaunchCooperativeKernel((const void *)pcg_tma_slab_kernel, dim3(Gr * ngroups), dim3(kBlock),
                                                params, kTmaSmem, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "TMA slab PCG launch");
  }
  delete S;
  return rc;
}

int launch_kn_apply_brick(const Lay &L, const BrickGeo &geo, const uint32_t *mask, double dg, double of,
                          const double *x, double *y, int sms, cudaStream_t s) {
  TmaPcgArgs A;
  std::memset(&A, 0, sizeof(A));
  A.a.L = L;
  A.a.mask = mask;
  A.a.dg = dg;
  A.a.of = of;
  A.g = geo;
  int rc = make_vec_map(L, geo.nx, geo.ny, geo.nz, x, &A.tm_x);
  if (rc) return rc;
  const int grid = geo.nbricks < sms * 2 ? geo.nbricks : sms * 2;
  kn_apply_tma_kernel<<<grid, kBlock, kTmaSmem, s>>>(A, y);
  MQ_CUDA(cudaGetLastError());
  return MQ_OK;
}

// prepared once per solver (tensor maps of the basis slots), launched inside
// the captured POD start vector
struct KnMulti {
  KnMultiArgs M;
  int grid = 0, nvec = 0;
};

int kn_multi_prepare(const Lay &L, const BrickGeo &geo, const uint32_t *mask, double dg, double of,
                     double *const *x, double *const *y, int nvec, const int *kptr, int sms, KnMulti **out) {
  if (nvec < 1 || nvec > kMaxMultiVec) { set_error("1..32 vectors per multi-SpMV"); return MQ_INVALID; }
  KnMulti *k = new KnMulti();
  std::memset(&k->M, 0, sizeof(k->M));
  k->M.A.a.L = L;
  k->M.A.a.mask = mask;
  k->M.A.a.dg = dg;
  k->M.A.a.of = of;
  k->M.A.g = geo;
  k->M.kptr = kptr;
  for (int j = 0; j < nvec; ++j) {
    int rc = make_vec_map(L, geo.nx, geo.ny, geo.nz, x[j], &k->M.tm[j]);
    if (rc) { delete k; return rc; }
    k->M.y[j] = y[j];
  }
  MQ_CUDA(cudaFuncSetAttribute(kn_apply_tma_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
  MQ_CUDA(two_cta_carveout((const void *)kn_apply_tma_multi_kernel));
  k->grid = geo.nbricks < sms * 2 ? geo.nbricks : sms * 2;
  k->nvec = nvec;
  *out = k;
  return MQ_OK;
}

int kn_multi_launch(const KnMulti *k, cudaStream_t s) {
  kn_apply_tma_multi_kernel<<<dim3(k->grid, k->nvec), kBlock, kTmaSmem, s>>>(k->M);
  MQ_CUDA(cudaGetLastError());
  return MQ_OK;
}

void kn_multi_free(KnMulti *k) { delete k; }

}  // namespace mq

// Cross-rank pieces of the fused slab PCG kernels (slab_fused.cu, and the
// TMA variant in pcg_brick.cu): per-rank slab description, the group barrier
// of a rank's CTAs and the rank all-reduce through device mailboxes.  See
// slab_fused.cu for the protocol.
#pragma once

#include "mq_device.cuh"

namespace mq {

constexpr int kMaxRanks = 8;
constexpr int kRing = 8;
constexpr int kMbW = 8;  // mailbox values per rank and slot (all-reduces of up to 8 sums)

struct SlabRank {
  Lay L;
  const uint32_t *mask;
  const double *b;
  double *x, *r, *pa, *pb, *ap;
  int n;  // owned planes
  // neighbour below (rank - 1): our plane 0 -> its top ghost plane (n_lo)
  double *lo_x, *lo_r, *lo_pa, *lo_pb;
  double *lo_r2, *lo_a, *lo_a2;  // one-barrier kernel: r of odd, Ap of even / odd iterations
  int64_t lo_C, lo_top;
  // neighbour above (rank + 1): our plane n - 1 -> its bottom ghost plane (-1)
  double *hi_x, *hi_r, *hi_pa, *hi_pb;
  double *hi_r2, *hi_a, *hi_a2;
  int64_t hi_C;
  // all-reduce: every rank's mailbox [kRing][kMaxRanks][kMbW] and counter
  double *mbox[kMaxRanks];
  unsigned long long *mcount[kMaxRanks];
  unsigned long long *epoch;  // this rank's instances of earlier solves
  double *partials;           // group partials, 2 sets x NV x group size
  GridBar *bar;               // group barrier
  PcgOut *out;
};

struct SlabFusedArgs {
  SlabRank rk[kMaxRanks];
  int ngroups, nranks, rank0;
  double dg, of, inv;
  int use_jac, x0_mode, max_iter;
  double rel_tol, abs_tol;
};

__device__ __forceinline__ void red_add_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_f64(double *p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys_f64(const double *p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// barrier of the Gr CTAs of one group (the group's own counter)
__device__ __forceinline__ bool group_sync(GridBar *bar, int Gr) {
  __shared__ int s_fail;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_fail = 0;
    const unsigned long long G = (unsigned long long)Gr;
    const unsigned long long old = atom_add_release_gpu(&bar->count, 1ull);
    const unsigned long long target = (old / G + 1ull) * G;
    const uint64_t t0 = globaltimer_ns();
    unsigned spins = 0;
    while (ld_acquire_gpu(&bar->count) < target) {
      if ((++spins & 1023u) == 0u && globaltimer_ns() - t0 > 5000000000ull) {
        atomicExch(&bar->error, 1u);
        s_fail = 1;
        break;
      }
    }
  }
  __syncthreads();
  return s_fail == 0;
}

// v: this CTA's partial sums; returns the global (all ranks) totals in v
template <int NV>
__device__ bool rank_allreduce(const SlabRank &me, int nranks, int rank, int lb, int Gr, unsigned long long inst,
                               double (&v)[NV], double *red, double *tot) {
  static_assert(NV <= kMbW, "mailbox width");
  block_sum<NV>(v, red);
  // two alternating partial sets: a CTA that is already in the next
  // all-reduce never overwrites values a slower CTA of the group still reads
  double *pt = me.partials + (int64_t)(inst & 1ull) * NV * Gr;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) pt[(int64_t)q * Gr + lb] = v[q];
  }
  if (!group_sync(me.bar, Gr)) return false;
  grid_partials_sum<NV>(pt, Gr, v, tot);  // rank total, identical in the group
  const int R = nranks;
  if (R == 1) return true;  // a single rank: the group total is the total
  const int slot = (int)(inst % kRing);
  if (lb == 0 && threadIdx.x == 0) {
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int k = 0; k < NV; ++k) st_relaxed_sys_f64(me.mbox[q] + ((int64_t)slot * kMaxRanks + rank) * kMbW + k, v[k]);
    for (int q = 0; q < R; ++q) red_add_release_sys(me.mcount[q], 1ull);
  }
  __shared__ int s_fail;
  if (threadIdx.x == 0) {
    s_fail = 0;
    const unsigned long long target = (unsigned long long)R * (inst + 1ull);
    const uint64_t t0 = globaltimer_ns();
    unsigned spins = 0;
    while (ld_acquire_sys(me.mcount[rank]) < target) {
      if ((++spins & 1023u) == 0u && globaltimer_ns() - t0 > 5000000000ull) {
        atomicExch(&me.bar->error, 1u);
        s_fail = 1;
        break;
      }
    }
  }
  __syncthreads();
  if (s_fail) return false;
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    const double *box = me.mbox[rank] + (int64_t)slot * kMaxRanks * kMbW;
    double val[kMaxRanks][NV];  // all loads in flight, then the rank-order sums
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q)
#pragma unroll
      for (int k = 0; k < NV; ++k) val[q][k] = q < R ? ld_relaxed_sys_f64(box + q * kMbW + k) : 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q)
        if (q < R) s = add(s, val[q][k]);
      tot[k] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = tot[k];
  __syncthreads();
  return true;
}

}  // namespace mq

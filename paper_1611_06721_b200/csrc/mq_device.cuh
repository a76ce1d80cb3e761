// Device helpers shared by the libmq_b200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mq_internal.h"

namespace mq {

constexpr int kBlock = 256;            // threads per CTA for streaming kernels
constexpr int kWarps = kBlock / 32;

// IEEE round-to-nearest without FMA contraction: numpy evaluates a*x + y as
// a rounded multiply followed by a rounded add (krylov.py:238-248,
// schur.py:400), so every update below spells out the two roundings.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ bool active(const uint32_t *mask, int64_t e) {
  return (mask[e >> 5] >> (e & 31)) & 1u;
}

// ---- deterministic reductions -------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum of NV values per thread; result valid in every thread.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *smem /* NV*kWarps */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) smem[q * kWarps + warp] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s = add(s, smem[q * kWarps + w]);
    v[q] = s;
  }
  __syncthreads();
}

// Sum partials[q*G + 0..G) in a fixed order; identical in every CTA.  Lane l
// adds b = l, l+32, ... in order; the first kPB loads per lane are issued
// back to back so the read costs one L2 round trip.
#ifndef MQ_PSUM_BATCH
#define MQ_PSUM_BATCH 10
#endif
constexpr int kPB = MQ_PSUM_BATCH;  // G <= 32 * kPB in one batch
template <int NV>
__device__ __forceinline__ void grid_partials_sum(const double *partials, int G, double (&out)[NV],
                                                  double *smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double v[kPB > 0 ? kPB : 1];
#pragma unroll
      for (int u = 0; u < kPB; ++u) {
        const int b = lane + 32 * u;
        v[u] = b < G ? __ldcg(partials + (int64_t)q * G + b) : 0.0;
      }
      double s = 0.0;
#pragma unroll
      for (int u = 0; u < kPB; ++u)
        if (lane + 32 * u < G) s = add(s, v[u]);
      for (int b = lane + 32 * kPB; b < G; b += 32) s = add(s, __ldcg(partials + (int64_t)q * G + b));
      s = warp_sum(s);
      if (lane == 0) smem[q] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = smem[q];
  __syncthreads();
}

// grid_partials_sum_all split in two: warp 0 issues its loads, other work
// (other warps' loads) can be issued before warp 0 consumes them.
template <int NV, int PB>
__device__ __forceinline__ void psum_issue(const double *partials, int G, double (&v)[NV][PB]) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int b = lane + 32 * u;
        v[q][u] = b < G ? __ldcg(partials + (int64_t)q * G + b) : 0.0;
      }
  }
}

template <int NV, int PB>
__device__ __forceinline__ void psum_finish(const double (&v)[NV][PB], int G, double (&out)[NV], double *smem) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
#pragma unroll
      for (int u = 0; u < PB; ++u)
        if (lane + 32 * u < G) s = add(s, v[q][u]);
      s = warp_sum(s);
      if (lane == 0) smem[q] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = smem[q];
  __syncthreads();
}

// Same sums with every load of all NV rows issued before the first add (one
// L2 round trip for all NV values); G <= 32 * PB.  Used by kernels with
// registers to spare.
template <int NV, int PB>
__device__ __forceinline__ void grid_partials_sum_all(const double *partials, int G, double (&out)[NV],
                                                      double *smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    double v[NV][PB];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int b = lane + 32 * u;
        v[q][u] = b < G ? __ldcg(partials + (int64_t)q * G + b) : 0.0;
      }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
#pragma unroll
      for (int u = 0; u < PB; ++u)
        if (lane + 32 * u < G) s = add(s, v[q][u]);
      s = warp_sum(s);
      if (lane == 0) smem[q] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = smem[q];
  __syncthreads();
}

// ---- grid-wide barrier (cooperative launch guarantees co-residency) -------
// One release-atomic arrival per CTA on a monotonic 64-bit counter (zeroed
// before every launch), then acquire-polling until all G CTAs of this
// barrier instance arrived: barrier k completes when the counter reaches
// (k+1)*G.  Cumulativity of the release (after the CTA barrier) publishes
// every thread's writes; the acquire + CTA barrier makes them visible to the
// whole CTA.  Data produced by other CTAs is read with L2-only loads (ldcg)
// or TMA, never through a possibly stale L1 line.  A watchdog (5 s on
// %globaltimer) turns a lost arrival into an error instead of a hang.
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long atom_add_release_gpu(unsigned long long *p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.release.gpu.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// (An acq_rel arrival that lets the last CTA skip polling, and a failure bit
// folded into the counter, measured no faster at 64^3 and made the TMA brick
// kernel's K1 ~30 % slower at 128^3 through its register allocation; kept
// as is.)
__device__ __forceinline__ bool grid_sync(GridBar *bar) {
  __shared__ int s_fail;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_fail = 0;
    const unsigned long long G = gridDim.x;
    const unsigned long long old = atom_add_release_gpu(&bar->count, 1ull);
    const unsigned long long target = (old / G + 1ull) * G;
    if (ld_acquire_gpu(&bar->count) < target) {
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
    if (*((volatile unsigned int *)&bar->error)) s_fail = 1;
  }
  __syncthreads();
  return s_fail == 0;
}

// test-only: a pseudo-random subset of CTAs sleeps right after a grid barrier
// (MQ_PCG_STRESS; the results depend on no timing and must not change)
__device__ __forceinline__ void stress_after_barrier(int ns, int it) {
  if (ns && ((blockIdx.x * 37 + it * 11) % 29 == 0)) __nanosleep((unsigned)ns);
}

// ---- the K_n stencil -------------------------------------------------------
// Row of K_n = (nu0/h) * S at padded index e of component c, evaluated as the
// CSR row sum in ascending column order with separately rounded products and
// sums, which reproduces scipy's csr_matvec (sum starts at 0, += a_ij*x_j)
// bit for bit: columns sorted by global id are the padded offsets below in
// ascending order, and absent (masked) neighbours hold exact zeros.
// Coefficients: SURVEY Appendix A, derived from C^T diag(w/h) C with the
// curl incidence of model.py:213-226.
template <class Ld>
__device__ __forceinline__ double stencil_row(int c, int64_t e, const Lay &L, double dg, double of,
                                              Ld ld) {
  const int64_t C = L.C, Si = L.Si, Sj = L.Sj;
  double s;
  if (c == 0) {
    s = -mul(of, ld(e - Sj));
    s = sub(s, mul(of, ld(e - 1)));
    s = add(s, mul(dg, ld(e)));
    s = sub(s, mul(of, ld(e + 1)));
    s = sub(s, mul(of, ld(e + Sj)));
    s = add(s, mul(of, ld(e + C - Sj)));
    s = sub(s, mul(of, ld(e + C)));
    s = sub(s, mul(of, ld(e + C + Si - Sj)));
    s = add(s, mul(of, ld(e + C + Si)));
    s = add(s, mul(of, ld(e + 2 * C - 1)));
    s = sub(s, mul(of, ld(e + 2 * C)));
    s = sub(s, mul(of, ld(e + 2 * C + Si - 1)));
    s = add(s, mul(of, ld(e + 2 * C + Si)));
  } else if (c == 1) {
    s = mul(of, ld(e - C - Si));
    s = sub(s, mul(of, ld(e - C - Si + Sj)));
    s = sub(s, mul(of, ld(e - C)));
    s = add(s, mul(of, ld(e - C + Sj)));
    s = sub(s, mul(of, ld(e - Si)));
    s = sub(s, mul(of, ld(e - 1)));
    s = add(s, mul(dg, ld(e)));
    s = sub(s, mul(of, ld(e + 1)));
    s = sub(s, mul(of, ld(e + Si)));
    s = add(s, mul(of, ld(e + C - 1)));
    s = sub(s, mul(of, ld(e + C)));
    s = sub(s, mul(of, ld(e + C + Sj - 1)));
    s = add(s, mul(of, ld(e + C + Sj)));
  } else {
    s = mul(of, ld(e - 2 * C - Si));
    s = sub(s, mul(of, ld(e - 2 * C - Si + 1)));
    s = sub(s, mul(of, ld(e - 2 * C)));
    s = add(s, mul(of, ld(e - 2 * C + 1)));
    s = add(s, mul(of, ld(e - C - Sj)));
    s = sub(s, mul(of, ld(e - C - Sj + 1)));
    s = sub(s, mul(of, ld(e - C)));
    s = add(s, mul(of, ld(e - C + 1)));
    s = sub(s, mul(of, ld(e - Si)));
    s = sub(s, mul(of, ld(e - Sj)));
    s = add(s, mul(dg, ld(e)));
    s = sub(s, mul(of, ld(e + Sj)));
    s = sub(s, mul(of, ld(e + Si)));
  }
  return s;
}

}  // namespace mq

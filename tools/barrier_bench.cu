// Grid-barrier microbenchmark: ns per barrier for the PCG kernels' barrier
// (release atomic + acquire polling) and a cluster-hierarchical variant.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/barrier_bench.cu -o /tmp/bb && /tmp/bb
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

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
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// flat: every CTA arrives on one counter
__global__ void k_flat(unsigned long long *cnt, int iters, double *sink) {
  const unsigned long long G = gridDim.x;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long old = atom_add_release_gpu(cnt, 1ull);
      const unsigned long long target = (old / G + 1ull) * G;
      while (ld_acquire_gpu(cnt) < target) {
      }
    }
    __syncthreads();
    acc += 1.0;
  }
  if (threadIdx.x == 0 && acc < 0) *sink = acc;
}

// flat, relaxed polling then one acquire
__global__ void k_flat_relaxed(unsigned long long *cnt, int iters, double *sink) {
  const unsigned long long G = gridDim.x;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long old = atom_add_release_gpu(cnt, 1ull);
      const unsigned long long target = (old / G + 1ull) * G;
      while (ld_relaxed_gpu(cnt) < target) {
      }
      (void)ld_acquire_gpu(cnt);
    }
    __syncthreads();
    acc += 1.0;
  }
  if (threadIdx.x == 0 && acc < 0) *sink = acc;
}

// fire-and-forget release reduction; the target is known from the barrier count
__global__ void k_red(unsigned long long *cnt, int iters, double *sink) {
  const unsigned long long G = gridDim.x;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(cnt), "l"(1ull) : "memory");
      const unsigned long long target = (unsigned long long)(it + 1) * G;
      while (ld_acquire_gpu(cnt) < target) {
      }
    }
    __syncthreads();
    acc += 1.0;
  }
  if (threadIdx.x == 0 && acc < 0) *sink = acc;
}

__global__ void k_red_relaxed(unsigned long long *cnt, int iters, double *sink) {
  const unsigned long long G = gridDim.x;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(cnt), "l"(1ull) : "memory");
      const unsigned long long target = (unsigned long long)(it + 1) * G;
      while (ld_relaxed_gpu(cnt) < target) {
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    acc += 1.0;
  }
  if (threadIdx.x == 0 && acc < 0) *sink = acc;
}

// cluster-hierarchical: cluster barrier, rank-0 CTA of each cluster arrives
// globally and polls, cluster barrier again
__global__ void k_cluster(unsigned long long *cnt, int iters, double *sink) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned long long NC = gridDim.x / cl.num_blocks();
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
      const unsigned long long old = atom_add_release_gpu(cnt, 1ull);
      const unsigned long long target = (old / NC + 1ull) * NC;
      while (ld_acquire_gpu(cnt) < target) {
      }
    }
    cl.sync();
    acc += 1.0;
  }
  if (threadIdx.x == 0 && acc < 0) *sink = acc;
}

// spread arrivals: 8 counters (one per group), group leaders' last arriver
// bumps the top counter
__global__ void k_tree(unsigned long long *cnt, int iters, double *sink) {
  const int G = gridDim.x;
  const int NG = 8;
  const int grp = blockIdx.x % NG;
  const unsigned long long gsz = (G - grp + NG - 1) / NG;  // CTAs in my group
  unsigned long long *top = cnt;
  unsigned long long *mine = cnt + 32 * (1 + grp);  // separate 256-B lines
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long old = atom_add_release_gpu(mine, 1ull);
      if ((old + 1) % gsz == 0) atom_add_release_gpu(top, 1ull);
      const unsigned long long target = (unsigned long long)(it + 1) * NG;
      while (ld_acquire_gpu(top) < target) {
      }
    }
    __syncthreads();
    acc += 1.0;
  }
  if (threadIdx.x == 0 && acc < 0) *sink = acc;
}

int main() {
  unsigned long long *cnt;
  double *sink;
  cudaMalloc(&cnt, 4096);
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  auto run = [&](const char *name, void *fn, int grid, int cluster, int threads) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cnt, 0, 4096);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = 0;
      cudaLaunchAttribute attr[2];
      int na = 0;
      if (cluster > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
      } else {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
      }
      cfg.attrs = attr;
      cfg.numAttrs = na;
      int it = iters;
      void *args[] = {&cnt, &it, &sink};
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
      cudaEventRecord(e1);
      cudaError_t e2 = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1)
        printf("%-14s grid %3d cluster %d threads %d: %7.1f ns/barrier  (%s %s)\n", name, grid, cluster, threads,
               1e6 * ms / iters, cudaGetErrorString(e), cudaGetErrorString(e2));
    }
  };
  for (int grid : {128, sms}) {
    for (int threads : {256, 512}) {
      run("flat", (void *)k_flat, grid, 1, threads);
      run("flat_relaxed", (void *)k_flat_relaxed, grid, 1, threads);
      run("red", (void *)k_red, grid, 1, threads);
      run("red_relaxed", (void *)k_red_relaxed, grid, 1, threads);
      run("cluster4", (void *)k_cluster, grid / 4 * 4, 4, threads);
      run("cluster8", (void *)k_cluster, grid / 8 * 8, 8, threads);
    }
  }
  return 0;
}

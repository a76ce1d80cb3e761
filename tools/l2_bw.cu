// L2 (LTS) throughput of this GPU, to put the fused PCG pass's L2-side
// traffic (ncu lts__t_sectors x 32 B per second) against: repeated reads of
// an L2-resident buffer with 16-byte .cg loads, a read+write copy inside L2,
// and the same two kernels on buffers far larger than L2 (DRAM).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2_bw.cu -o tools/l2_bw.bin && tools/l2_bw.bin
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const double2 *__restrict__ src, size_t n, int reps, double *out) {
  double acc = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; p + 3 * stride < n; p += 4 * stride) {
      const double2 a = __ldcg(src + p), b = __ldcg(src + p + stride), c = __ldcg(src + p + 2 * stride),
                    d = __ldcg(src + p + 3 * stride);
      acc += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
    }
    for (; p < n; p += stride) {
      const double2 a = __ldcg(src + p);
      acc += a.x + a.y;
    }
  }
  if (acc == 1.2345e300) out[0] = acc;
}

__global__ void k_copy(const double2 *__restrict__ src, double2 *__restrict__ dst, size_t n, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; p + 3 * stride < n; p += 4 * stride) {
      const double2 a = __ldcg(src + p), b = __ldcg(src + p + stride), c = __ldcg(src + p + 2 * stride),
                    d = __ldcg(src + p + 3 * stride);
      dst[p] = a;
      dst[p + stride] = b;
      dst[p + 2 * stride] = c;
      dst[p + 3 * stride] = d;
    }
    for (; p < n; p += stride) dst[p] = __ldcg(src + p);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = (size_t)2 << 30;
  double2 *a, *b;
  double *out;
  cudaMalloc(&a, big);
  cudaMalloc(&b, big);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, big);
  cudaMemset(b, 0, big);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = sms * 4, block = 256;
  const size_t sizes[] = {(size_t)16 << 20, (size_t)32 << 20, (size_t)48 << 20, (size_t)2 << 30};
  for (size_t bytes : sizes) {
    const size_t n = bytes / 16;
    const int reps = bytes > ((size_t)1 << 30) ? 4 : 200;
    for (int kind = 0; kind < 2; ++kind) {
      float best = 1e30f;
      for (int t = 0; t < 4; ++t) {
        cudaEventRecord(e0);
        if (kind == 0) k_read<<<grid, block>>>(a, n, reps, out);
        else k_copy<<<grid, block>>>(a, b, n / 2, reps);  // half the bytes read, half written: same footprint
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (t > 0 && ms < best) best = ms;
      }
      const double moved = (double)bytes * reps;  // read: bytes; copy: bytes/2 read + bytes/2 written
      printf("%s footprint %7.1f MB  %8.1f GB/s\n", kind == 0 ? "read " : "copy ", bytes / 1048576.0,
             moved / (best * 1e-3) / 1e9);
    }
  }
  printf("cudaGetLastError: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

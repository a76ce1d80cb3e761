// Launch cost of an empty kernel shaped like the resident PCG kernel (128
// CTAs x 512 threads, 225 KB dynamic shared memory, cooperative) against a
// small plain kernel, back to back on one stream and as CUDA-graph nodes.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/launch_probe tools/launch_probe.cu
//   tools/launch_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int *p) {
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}

__global__ void __launch_bounds__(512, 1) big_kernel(int *p) {
  extern __shared__ double sm[];
  if (threadIdx.x == 0) sm[0] = 1.0;
  __syncthreads();
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += (int)sm[0];
}

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e = (x);                                               \
    if (e != cudaSuccess) {                                            \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                   \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main() {
  int *d = nullptr;
  CK(cudaMalloc(&d, sizeof(int)));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t smem = 225408;
  CK(cudaFuncSetAttribute(big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int N = 200;
  auto timeit = [&](const char *name, auto launch) -> int {
    for (int i = 0; i < 10; ++i) launch();
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(a, s));
    for (int i = 0; i < N; ++i) launch();
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-48s %7.2f us per launch\n", name, 1000.f * ms / N);
    return 0;
  };
  void *args[] = {&d};
  if (timeit("plain 1x32", [&] { empty_kernel<<<1, 32, 0, s>>>(d); })) return 1;
  if (timeit("plain 128x512, 225 KB smem", [&] { big_kernel<<<128, 512, smem, s>>>(d); })) return 1;
  if (timeit("cooperative 128x512, 225 KB smem", [&] {
        cudaLaunchCooperativeKernel((const void *)big_kernel, dim3(128), dim3(512), args, smem, s);
      }))
    return 1;
  if (timeit("cooperative 128x512 + 8-byte memset", [&] {
        cudaMemsetAsync(d, 0, 8, s);
        cudaLaunchCooperativeKernel((const void *)big_kernel, dim3(128), dim3(512), args, smem, s);
      }))
    return 1;
  if (timeit("alternating plain 148x256 / cooperative big", [&] {
        empty_kernel<<<148, 256, 0, s>>>(d);
        cudaLaunchCooperativeKernel((const void *)big_kernel, dim3(128), dim3(512), args, smem, s);
      }))
    return 1;
  // the same sequences as graph nodes (N per graph)
  for (int variant = 0; variant < 2; ++variant) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < N; ++i) {
      if (variant == 1) empty_kernel<<<148, 256, 0, s>>>(d);
      cudaLaunchCooperativeKernel((const void *)big_kernel, dim3(128), dim3(512), args, smem, s);
    }
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(a, s));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-48s %7.2f us per %s\n", variant ? "graph: plain + cooperative big" : "graph: cooperative big",
           1000.f * ms / N, variant ? "pair" : "launch");
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  return 0;
}

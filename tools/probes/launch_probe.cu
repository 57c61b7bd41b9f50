// Dev probe: launch-to-completion time of an empty kernel vs its launch shape
// (CTAs x threads, dynamic shared memory), after an L2-flushing write, with
// CUDA events on the stream.   nvcc -gencode arch=compute_100a,code=sm_100a launch_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* out) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && out != nullptr) out[0] = s[0];
}
__global__ void k_fill(unsigned char* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = 1;
}

int main() {
  unsigned char* buf;
  size_t n = size_t(256) << 20;
  cudaMalloc(&buf, n);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Shape { int ctas, threads, smem_kb; } shapes[] = {{1, 32, 0}, {148, 32, 0}, {147, 1024, 0}, {147, 1024, 123}, {148, 256, 18},
                                                             {147, 1024, 123}, {592, 256, 18}, {129, 512, 17}};
  for (int flush = 0; flush < 2; ++flush)
    for (auto sh : shapes) {
      float tot = 0;
      for (int r = 0; r < 20; ++r) {
        if (flush) k_fill<<<148 * 8, 256>>>(buf, n);
        cudaEventRecord(a);
        k_empty<<<sh.ctas, sh.threads, sh.smem_kb * 1024>>>(nullptr);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        float ms = 0;
        cudaError_t e2 = cudaEventElapsedTime(&ms, a, b);
        if (e != cudaSuccess || e2 != cudaSuccess || cudaGetLastError() != cudaSuccess) {
          printf("error: %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
          return 1;
        }
        if (r >= 5) tot += ms;
      }
      printf("flush=%d ctas=%d threads=%d smem=%dKB: %.2f us\n", flush, sh.ctas, sh.threads, sh.smem_kb,
             tot / 15 * 1e3);
    }
  return 0;
}

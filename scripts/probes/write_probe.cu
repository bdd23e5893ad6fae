// Diagnostic: HBM write-only and write-dominated (1 read : 8 writes, the
// direct AllGather's mix) rates on this B200, 16-byte vector stores from all
// SMs, CUDA events, best of 10.  The roofline of K6.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_write(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
// read one vector, store it to 8 destinations (the AllGather fan-out)
__global__ void __launch_bounds__(512) k_fanout(const uint4* src, uint4* dst, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
#pragma unroll
    for (int k = 0; k < 8; k++) dst[(size_t)k * n + i] = v;
  }
}
__global__ void __launch_bounds__(512) k_copy(const uint4* src, uint4* dst, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}

template <typename F>
float best_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = (size_t)2 << 30, n = bytes / 16;
  uint4 *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes + (bytes / 8) * 8);
  for (int per : {1, 2, 4}) {
    const int g = sms * per;
    float t = best_ms([&] { k_write<<<g, 512>>>(a, n); });
    printf("write-only   %d CTA/SM: %.0f GB/s\n", per, bytes / (t * 1e-3) / 1e9);
    t = best_ms([&] { k_copy<<<g, 512>>>(a, b, n); });
    printf("copy         %d CTA/SM: %.0f GB/s\n", per, 2 * bytes / (t * 1e-3) / 1e9);
    const size_t m = n / 8;   // 256 MiB read, 2 GiB written
    t = best_ms([&] { k_fanout<<<g, 512>>>(a, b, m); });
    printf("1:8 fan-out  %d CTA/SM: %.0f GB/s\n", per, 9 * (m * 16) / (t * 1e-3) / 1e9);
  }
  return 0;
}

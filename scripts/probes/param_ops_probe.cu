// Diagnostic: can the plan interpreter take its (host-resolved) op array in
// the kernel parameter space?  Graph-replayed launch cost vs parameter size,
// and the in-kernel latency of reading one 512-byte op at a dynamic index from
// the parameter space vs from global memory (L2 flushed), %globaltimer stamps.
#include <cstdio>
#include <cuda_runtime.h>

template <int B> struct P { uint4 d[B / 16]; };

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int B>
__global__ void k_empty(const __grid_constant__ P<B> p, int* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.d[B / 16 - 1].x == 42) out[0] = 1;
}

// one thread per 16-byte word of op `idx`: param space (dynamic index)
template <int B>
__global__ void k_param(const __grid_constant__ P<B> p, int idx, uint4* out, unsigned long long* ts) {
  unsigned long long t0 = gt();
  __shared__ uint4 s[32];
  if (threadIdx.x < 32) s[threadIdx.x] = p.d[idx * 32 + threadIdx.x];
  __syncthreads();
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) { out[blockIdx.x] = s[5]; if (blockIdx.x == 0) { ts[0] = t1 - t0; } }
}
__global__ void k_global(const uint4* ops, int idx, uint4* out, unsigned long long* ts) {
  unsigned long long t0 = gt();
  __shared__ uint4 s[32];
  if (threadIdx.x < 32) s[threadIdx.x] = ops[idx * 32 + threadIdx.x];
  __syncthreads();
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) { out[blockIdx.x] = s[5]; if (blockIdx.x == 0) { ts[0] = t1 - t0; } }
}

template <int B>
static float launch_cost(int blocks, int* out) {
  P<B> p{};
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 200; i++) k_empty<B><<<blocks, 512, 0, s>>>(p, out);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best * 1000.f / 200.f;
}

int main() {
  int* out;
  cudaMalloc(&out, 4);
  printf("param bytes -> us per graph-replayed launch (8 CTAs / 144 CTAs of 512)\n");
#define LC(B) printf("  %6d %.3f %.3f\n", B, launch_cost<B>(8, out), launch_cost<B>(144, out));
  LC(64) LC(4096) LC(8192) LC(16384) LC(24576) LC(32000)
  // op read latency
  constexpr int B = 24576;
  P<B>* hp = new P<B>();
  for (int i = 0; i < B / 16; i++) hp->d[i] = make_uint4(i, i + 1, i + 2, i + 3);
  uint4 *dops, *dout;
  unsigned long long* dts;
  cudaMalloc(&dops, B);
  cudaMemcpy(dops, hp, B, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, 1024 * 16);
  cudaMalloc(&dts, 8);
  char* flush;
  const size_t FL = 256u << 20;
  cudaMalloc(&flush, FL);
  for (int rep = 0; rep < 5; rep++) {
    unsigned long long tp = 0, tg = 0;
    cudaMemset(flush, rep, FL);
    k_param<B><<<8, 512>>>(*hp, rep % 40, dout, dts);
    cudaMemcpy(&tp, dts, 8, cudaMemcpyDeviceToHost);
    cudaMemset(flush, rep + 1, FL);
    k_global<<<8, 512>>>(dops, rep % 40, dout, dts);
    cudaMemcpy(&tg, dts, 8, cudaMemcpyDeviceToHost);
    printf("op read (L2 flushed): param %llu ns, global %llu ns\n", tp, tg);
  }
  return 0;
}

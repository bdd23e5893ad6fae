// Diagnostic: graph-replayed launch cost of an (almost) empty kernel vs the
// size of its __grid_constant__ parameter struct.
#include <cstdio>
#include <cuda_runtime.h>

template <int B> struct P { char d[B]; };

template <int B>
__global__ void k(const __grid_constant__ P<B> p, int* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.d[B - 1] == 42) out[0] = 1;
}

template <int B>
static float run(int blocks, int threads, int* out) {
  P<B> p{};
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 200; i++) k<B><<<blocks, threads, 0, s>>>(p, out);
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

extern "C" void probe() {
  int* out;
  cudaMalloc(&out, 4);
  printf("param bytes -> us per launch (8 CTAs x 512 / 144 CTAs x 512)\n");
  printf("  64   %.3f %.3f\n", run<64>(8, 512, out), run<64>(144, 512, out));
  printf("  1024 %.3f %.3f\n", run<1024>(8, 512, out), run<1024>(144, 512, out));
  printf("  2048 %.3f %.3f\n", run<2048>(8, 512, out), run<2048>(144, 512, out));
  printf("  4000 %.3f %.3f\n", run<4000>(8, 512, out), run<4000>(144, 512, out));
  printf("  8192 %.3f %.3f\n", run<8192>(8, 512, out), run<8192>(144, 512, out));
  printf("  16384 %.3f %.3f\n", run<16384>(8, 512, out), run<16384>(144, 512, out));
}

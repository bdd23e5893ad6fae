// Diagnostic: one-way flag latency between two CTAs of one GPU (the
// co-resident-rank hop every LL / semaphore kernel pays), per load/store
// flavour.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pp pingpong_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) {
  uint32_t v; asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ uint32_t ld_rlx_gpu(const uint32_t* p) {
  uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ uint32_t ld_acq_gpu(const uint32_t* p) {
  uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) {
  uint32_t v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ uint32_t ld_v4vol(const uint32_t* p) {   // LL16-style 16-byte poll, flag in .y
  uint32_t a, b, c, d;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
  return b == d ? b : 0;
}
__device__ __forceinline__ void st_plain(uint32_t* p, uint32_t v) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_vol(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_v4vol(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(7u), "r"(v), "r"(9u), "r"(v) : "memory");
}
__device__ __forceinline__ void st_v4(uint32_t* p, uint32_t v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(7u), "r"(v), "r"(9u), "r"(v) : "memory");
}

template <int L, int S>
__device__ __forceinline__ uint32_t LD(const uint32_t* p) {
  if (L == 0) return ld_vol(p);
  if (L == 1) return ld_rlx_gpu(p);
  if (L == 2) return ld_acq_gpu(p);
  if (L == 3) return ld_acq_sys(p);
  return ld_v4vol(p);
}
template <int L, int S>
__device__ __forceinline__ void ST(uint32_t* p, uint32_t v) {
  if (S == 0) st_plain(p, v);
  else if (S == 1) st_vol(p, v);
  else if (S == 2) st_rel_gpu(p, v);
  else if (S == 3) st_rel_sys(p, v);
  else if (S == 4) st_v4vol(p, v);
  else st_v4(p, v);
}

template <int L, int S>
__global__ void pp(uint32_t* a, uint32_t* b, int iters, unsigned long long* out) {
  if (threadIdx.x) return;
  uint64_t t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (blockIdx.x == 0) {
    for (int i = 1; i <= iters; i++) {
      ST<L, S>(a, i);
      while (LD<L, S>(b) != (uint32_t)i) {}
    }
  } else {
    for (int i = 1; i <= iters; i++) {
      while (LD<L, S>(a) != (uint32_t)i) {}
      ST<L, S>(b, i);
    }
  }
  uint64_t t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0) *out = t1 - t0;
}

template <int L, int S>
void run(const char* name, int blocks_apart) {
  uint32_t *a, *b;
  unsigned long long* o;
  cudaMalloc(&a, 4096); cudaMalloc(&b, 4096); cudaMalloc(&o, 8);
  cudaMemset(a, 0, 4096); cudaMemset(b, 0, 4096);
  const int iters = 2000;
  pp<L, S><<<2, 32>>>(a, b + 256, iters, o);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long ns = 0;
  cudaMemcpy(&ns, o, 8, cudaMemcpyDeviceToHost);
  printf("%-34s one-way hop %7.1f ns  (%s)\n", name, ns / (2.0 * iters), cudaGetErrorString(e));
  cudaFree(a); cudaFree(b); cudaFree(o);
  (void)blocks_apart;
}

int main() {
  run<0, 0>("ld.volatile / st plain", 0);
  run<0, 1>("ld.volatile / st.volatile", 0);
  run<1, 0>("ld.relaxed.gpu / st plain", 0);
  run<1, 2>("ld.relaxed.gpu / st.release.gpu", 0);
  run<2, 2>("ld.acquire.gpu / st.release.gpu", 0);
  run<3, 3>("ld.acquire.sys / st.release.sys", 0);
  run<4, 4>("LL16 ld.v4.volatile / st.v4.volatile", 0);
  run<4, 5>("LL16 ld.v4.volatile / st.v4 plain", 0);
  return 0;
}

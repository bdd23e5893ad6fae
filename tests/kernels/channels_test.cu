// Test kernels for the device Primitive API (cf_device.cuh / cf_proxy.h):
// a ring pass where rank r sends its buffer to rank r+1 through a user
// channel.  All ranks are co-resident CTAs of one launch (blockIdx.y = rank).
// Test infrastructure: built into tests/kernels/ by __graft_entry__.build().
#include <cuda_runtime.h>
#include "cf_proxy.h"
#include "device/cf_device.cuh"

using namespace cf;

__global__ void mem_ring(const MemoryChannelDevice* tx, const MemoryChannelDevice* rx, size_t bytes, int ll,
                         uint32_t flag, char* const* outs, int rounds) {
  const int r = blockIdx.y, tid = threadIdx.x, nt = blockDim.x;
  const MemoryChannelDevice& t = tx[r];
  const MemoryChannelDevice& x = rx[r];
  for (int k = 0; k < rounds; k++) {
    if (!ll) {
      t.put(0, 0, bytes, tid, nt);
      __syncthreads();
      if (tid == 0) t.signal();
      if (tid == 0) x.wait();
      __syncthreads();
      for (size_t i = tid; i < bytes; i += nt) outs[r][i] = x.dst_local[i];
      __syncthreads();
    } else {
      t.put_packets(2 * bytes * k, 0, bytes, flag + k, tid, nt);   // fresh packet area per round
      x.read_packets(outs[r], 2 * bytes * k, bytes, flag + k, tid, nt);
      __syncthreads();
    }
  }
}

__global__ void port_ring(const PortChannelDevice* tx, const PortChannelDevice* rx, size_t bytes,
                          char* const* outs, int rounds) {
  const int r = blockIdx.y, tid = threadIdx.x;
  for (int k = 0; k < rounds; k++) {
    if (tid == 0) {
      if (k & 1) {
        tx[r].put(0, 0, bytes);
        tx[r].signal();
      } else {
        tx[r].put_with_signal(0, 0, bytes);
      }
      tx[r].flush();
      rx[r].wait();
    }
    __syncthreads();
    for (size_t i = tid; i < bytes; i += blockDim.x) outs[r][i] = rx[r].dst_buf[i];
    __syncthreads();
  }
}

template <typename H>
static int upload(const void* host, int n, H** dev) {
  if (cudaMalloc((void**)dev, sizeof(H) * n) != cudaSuccess) return 1;
  return cudaMemcpy(*dev, host, sizeof(H) * n, cudaMemcpyHostToDevice) != cudaSuccess;
}

extern "C" int cftest_mem_ring(const void* tx, const void* rx, int n, size_t bytes, int ll, unsigned flag,
                               void* const* outs, int rounds) {
  MemoryChannelDevice *dtx, *drx;
  char** douts;
  if (upload(tx, n, &dtx) || upload(rx, n, &drx)) return 1;
  if (cudaMalloc((void**)&douts, sizeof(char*) * n) != cudaSuccess) return 1;
  cudaMemcpy(douts, outs, sizeof(char*) * n, cudaMemcpyHostToDevice);
  mem_ring<<<dim3(1, n), 256>>>(dtx, drx, bytes, ll, flag, douts, rounds);
  int rc = cudaDeviceSynchronize() != cudaSuccess;
  cudaFree(dtx);
  cudaFree(drx);
  cudaFree(douts);
  return rc;
}

extern "C" int cftest_port_ring(const void* tx, const void* rx, int n, size_t bytes, void* const* outs, int rounds) {
  PortChannelDevice *dtx, *drx;
  char** douts;
  if (upload(tx, n, &dtx) || upload(rx, n, &drx)) return 1;
  if (cudaMalloc((void**)&douts, sizeof(char*) * n) != cudaSuccess) return 1;
  cudaMemcpy(douts, outs, sizeof(char*) * n, cudaMemcpyHostToDevice);
  port_ring<<<dim3(1, n), 64>>>(dtx, drx, bytes, douts, rounds);
  int rc = cudaDeviceSynchronize() != cudaSuccess;
  cudaFree(dtx);
  cudaFree(drx);
  cudaFree(douts);
  return rc;
}

// NVLS AllReduce written against the SwitchChannel primitive: rank r (blockIdx.y)
// reduces chunk r of every member's heap range [off_in, off_in + bytes) and
// broadcasts the sums to [off_out, ...) of every member.  One co-resident
// launch: inputs are complete before it, each output chunk has one writer.
__global__ void switch_allreduce(const SwitchChannelDevice* sw, size_t off_in, size_t off_out, size_t bytes) {
  const int r = blockIdx.y;
  const SwitchChannelDevice& s = sw[r];
  const size_t chunk = bytes / s.n;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  s.reduce_broadcast<float>(off_out + r * chunk, off_in + r * chunk, chunk, tid, nt);
}

extern "C" int cftest_switch_allreduce(const void* handles, int n, size_t off_in, size_t off_out, size_t bytes) {
  SwitchChannelDevice* d;
  if (upload(handles, n, &d)) return 1;
  switch_allreduce<<<dim3(8, n), 256>>>(d, off_in, off_out, bytes);
  int rc = cudaDeviceSynchronize() != cudaSuccess;
  cudaFree(d);
  return rc;
}

// A compute stand-in that holds `nctas` SMs (one CTA per SM through its
// shared-memory request) until the host raises a flag, or a 30 s safety
// timeout: the collectives of the partial-residency test run beside it.
__global__ void spin_hold(volatile int* flag, unsigned long long timeout_ns, int* timed_out) {
  extern __shared__ char smem[];
  if (threadIdx.x == 0) {
    smem[0] = 1;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      if (*flag) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) { atomicExch(timed_out, 1); break; }
      __nanosleep(2000);
    }
  }
  __syncthreads();
}

static int* g_flag = nullptr;
static int* g_timed_out = nullptr;
static cudaStream_t g_spin = nullptr;

extern "C" int cftest_spin_start(int nctas, int smem_bytes) {
  if (!g_flag && cudaHostAlloc((void**)&g_flag, 2 * sizeof(int), cudaHostAllocMapped) != cudaSuccess) return 1;
  g_timed_out = g_flag + 1;
  g_flag[0] = 0;
  g_flag[1] = 0;
  if (!g_spin && cudaStreamCreateWithFlags(&g_spin, cudaStreamNonBlocking) != cudaSuccess) return 2;
  if (cudaFuncSetAttribute(spin_hold, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess)
    return 3;
  int *dflag, *dto;
  cudaHostGetDevicePointer((void**)&dflag, g_flag, 0);
  cudaHostGetDevicePointer((void**)&dto, g_timed_out, 0);
  spin_hold<<<nctas, 32, smem_bytes, g_spin>>>(dflag, 30ull * 1000000000ull, dto);
  return cudaGetLastError() != cudaSuccess ? 4 : 0;
}

// 0: released by the flag; 1: the hold hit its timeout; >1: CUDA error
extern "C" int cftest_spin_stop(void) {
  *(volatile int*)g_flag = 1;
  if (cudaStreamSynchronize(g_spin) != cudaSuccess) return 2;
  return g_flag[1] ? 1 : 0;
}

// Message-passing litmus test (MP): a producer CTA writes a 64 KiB payload
// stamped with round i, then publishes flag = i; a consumer CTA on another SM
// waits for the flag, reads the payload and counts words older than i.
// `ordered` = 1: every producer thread fences before the barrier and the
// flag is a release store, the consumer's flag load is an acquire (the
// handshake of the collective kernels); 0: relaxed stores / loads only (the
// CF_DROP_FENCE=1/2/3 mutations).  Returns the stale words seen.
__global__ void mp_litmus(uint32_t* data, uint64_t* flag, uint64_t* ack, int rounds, int ordered, int consumer,
                          unsigned long long* stale) {
  const int words = 16384;
  if (blockIdx.x != 0 && blockIdx.x != consumer) return;
  unsigned long long bad = 0;
  for (int i = 1; i <= rounds; i++) {
    if (blockIdx.x == 0) {   // producer
      if (threadIdx.x == 0)
        while (ld_acquire_gpu(ack) < (uint64_t)(i - 1)) {}
      __syncthreads();
      for (int k = threadIdx.x; k < words; k += blockDim.x) data[k] = (uint32_t)i;
      if (ordered) __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        if (ordered) st_release_gpu(flag, (uint64_t)i);
        else st_relaxed(flag, (uint64_t)i, true);
      }
    } else {                 // consumer
      if (threadIdx.x == 0)
        while ((ordered ? ld_acquire_gpu(flag) : ld_relaxed(flag, true)) < (uint64_t)i) {}
      __syncthreads();
      for (int k = threadIdx.x; k < words; k += blockDim.x) {
        uint32_t v;
        asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(data + k));
        bad += v < (uint32_t)i;
      }
      __syncthreads();
      if (threadIdx.x == 0) st_release_gpu(ack, (uint64_t)i);
    }
  }
  if (blockIdx.x == consumer && bad) atomicAdd(stale, bad);
}

extern "C" long long cftest_mp_litmus(int rounds, int ordered, int consumer) {
  uint32_t* data;
  uint64_t* sync;
  unsigned long long* stale;
  if (cudaMalloc((void**)&data, 16384 * 4) || cudaMalloc((void**)&sync, 256) || cudaMalloc((void**)&stale, 8))
    return -1;
  cudaMemset(data, 0, 16384 * 4);
  cudaMemset(sync, 0, 256);
  cudaMemset(stale, 0, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  mp_litmus<<<sms, 512>>>(data, sync, sync + 8, rounds, ordered, consumer, stale);
  unsigned long long h = 0;
  if (cudaMemcpy(&h, stale, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
  cudaFree(data);
  cudaFree(sync);
  cudaFree(stale);
  return (long long)h;
}

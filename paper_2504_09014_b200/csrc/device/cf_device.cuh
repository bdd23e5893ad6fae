// cf_device.cuh -- device-side primitive API for sm_100a (the paper's Primitive
// API), re-designed for B200 NVLink 5 / NVSwitch.
//
// Reference semantics (commforge 0.1.0, cf/):
//   MemoryChannel HB  put / signal / wait / flush     cf/channels.py:181-240
//   MemoryChannel LL  put_packets / read_packets      cf/channels.py:244-330
//   SwitchChannel     reduce / broadcast (multimem)   cf/channels.py:333-409
//   Semaphore         monotonic u64, release/acquire  cf/world.py:148-181
//
// B200 mapping
//   - peer memory is plain global memory mapped into this GPU's VA (cudaIpc /
//     P2P / same device); 16-byte vector loads and stores.
//   - signal  = fence + st.release.sys of a monotonically increasing value on
//               the receiver's slot (one writer per slot, so a value store is
//               equivalent to the reference's +1 counter).
//   - wait    = ld.acquire.sys spin until value >= target, bounded by a
//               %globaltimer timeout that raises the rank's error word
//               (-> CF_E_DEADLOCK on the host).
//   - LL16    = one 16-byte st.volatile {d0, flag, d1, flag}: two reference
//               packets ([u32 data | u32 flag], cf/channels.py:36-37) in one
//               single-copy-atomic transaction, byte-identical layout.
//   - multimem.ld_reduce / multimem.st on NVLS multicast addresses.
#pragma once
#include <cstdint>
#ifdef CF_WAIT_DEBUG
#include <cstdio>
#endif
#include <cuda_fp16.h>
#include <cuda_bf16.h>

#ifndef CF_MAX_RANKS
#define CF_MAX_RANKS 8
#endif
#ifndef CF_MAX_BLOCKS
#define CF_MAX_BLOCKS 1024
#endif

namespace cf {

enum DevError : uint32_t { kDevOk = 0, kDevTimeout = 6 /* == CF_E_DEADLOCK */ };

// Per-rank device state (lives in the rank's symmetric heap).
struct RankState {
  uint64_t epoch;      // completed collective calls on this rank
  uint32_t arrive;     // CTAs of the current launch that finished (last-CTA-done)
  uint32_t error;      // DevError
  uint64_t timeout_ns;
  uint64_t pad[5];
};

// LL flag of call `e`: never 0 (cf/channels.py:254-255), distinct for
// 2^32-1 consecutive calls, so stale packets of earlier calls never match.
__host__ __device__ __forceinline__ uint32_t ll_flag(uint64_t e) {
  return (uint32_t)(e % 0xffffffffull) + 1u;
}

// ---------------------------------------------------------------- memory model

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Scope-selected release/acquire: `gpu` when every rank of the communicator
// lives on this device (co-resident ranks), `sys` across GPUs (NVLink peers).
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v, bool gpu) {
  if (gpu) st_release_gpu(p, v); else st_release_sys(p, v);
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p, bool gpu) {
  return gpu ? ld_acquire_gpu(p) : ld_acquire_sys(p);
}
__device__ __forceinline__ void fence_publish(bool gpu) {
  if (gpu) __threadfence(); else __threadfence_system();
}
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// 16-byte vector global access (.v4.u32), plain and volatile (LL packets).
__device__ __forceinline__ uint4 ld16(const void* p) {
  uint4 v;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// L2-only load (no L1 allocation): data another SM or GPU rewrites between
// this CTA's reads of the same address (staging halves, piece after piece).
__device__ __forceinline__ uint4 ld16_cg(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld16_nc(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// L2 cache policies (createpolicy): streaming data read once marked
// evict_first so it does not push reused lines (ring slots) out of L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld16_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st16(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld16_volatile(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st16_volatile(void* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint2 ld8(const void* p) {
  uint2 v;
  asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st8(void* p, uint2 v) {
  asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ uint2 ld8_volatile(const void* p) {
  uint2 v;
  asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st8_volatile(void* p, uint2 v) {
  asm volatile("st.volatile.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}

// Partial 16-byte vectors (ragged heads/tails) in registers only: the loops
// unroll, so every word index is a compile-time constant (a union or array
// with a runtime index would live in local memory).
template <int ES>
__device__ __forceinline__ uint4 ld_partial16(const char* p, int nbytes) {
  uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int b = 0; b < 16; b += ES) {
    if (b < nbytes) {
      const uint32_t v = ES == 4 ? *reinterpret_cast<const uint32_t*>(p + b)
                                 : (uint32_t)*reinterpret_cast<const uint16_t*>(p + b);
      w[b / 4] |= v << ((b % 4) * 8);
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
// Store elements [jlo, jhi) of a 16-byte vector at base + j*ES.
template <int ES>
__device__ __forceinline__ void st_masked16(char* base, uint4 v, int jlo, int jhi) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int b = 0; b < 16; b += ES) {
    const int jj = b / ES;
    if (jj >= jlo && jj < jhi) {
      if (ES == 4) *reinterpret_cast<uint32_t*>(base + b) = w[b / 4];
      else *reinterpret_cast<uint16_t*>(base + b) = (uint16_t)(w[b / 4] >> ((b % 4) * 8));
    }
  }
}

// ---------------------------------------------------------------- robustness builds
//
// -DCF_STRESS=<ns>: a pseudo-random __nanosleep of up to <ns> at one in four
// visits of every synchronization site (before LL packet stores and before
// handshake / ring releases, after acquires), widening every race window --
// the GPU counterpart of the reference's adversarial schedules
// (pkg/tests/test_acceptance.py:115-202).
// -DCF_DROP_FENCE=<site>: mutation builds, each removing one ordering
// guarantee; tests/test_gpu_stress.py requires the stress run to fail on them:
//   1  handshake release: no publishing fence, relaxed signal store
//   2  every semaphore wait: relaxed instead of acquire load
//   3  ring data release: no publishing fence, relaxed store
//   4  LL packets: flags stored before (and apart from) the payload words
//   5  exit / phase handshakes: signal without waiting for the peers
//   6  ring credits: the sender does not wait for the receiver's ack
//   7  K13 two-shot: phase 2 does not wait for the owners' arrivals
#ifndef CF_DROP_FENCE
#define CF_DROP_FENCE 0
#endif
#ifdef CF_STRESS
__device__ __forceinline__ void cf_stress(uint32_t site) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  uint32_t h = (uint32_t)t ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu) ^
               (blockIdx.y * 0xC2B2AE35u) ^ (site * 0x27D4EB2Fu);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0) __nanosleep(h % (uint32_t)(CF_STRESS));
}
#define CF_STRESS_AT(site) ::cf::cf_stress(site)
#else
#define CF_STRESS_AT(site) ((void)0)
#endif

__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v, bool gpu) {
  if (gpu) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p, bool gpu) {
  uint64_t v;
  if (gpu) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// the load of a semaphore wait (mutation 2 drops its acquire)
__device__ __forceinline__ uint64_t ld_wait(const uint64_t* p, bool gpu) {
#if CF_DROP_FENCE == 2
  return ld_relaxed(p, gpu);
#else
  return ld_acquire(p, gpu);
#endif
}

// ---------------------------------------------------------------- spin waits

// Spin until *sem >= target (acquire).  Returns false on timeout or when the
// rank's error word is already set (so one stuck wait does not cascade into a
// full-timeout per wait).
__device__ __forceinline__ bool wait_geq(const uint64_t* sem, uint64_t target, RankState* st,
                                         bool gpu = false) {
  if (ld_wait(sem, gpu) >= target) {
    CF_STRESS_AT(1);
    return true;
  }
  const uint64_t t0 = globaltimer();
  const uint64_t limit = st->timeout_ns;
  for (uint32_t it = 1;; ++it) {
    if (ld_wait(sem, gpu) >= target) {
      CF_STRESS_AT(2);
      return true;
    }
    if ((it & 255u) == 0) {
      if (*(volatile uint32_t*)&st->error != kDevOk) return false;
      if (globaltimer() - t0 > limit) {
#ifdef CF_WAIT_DEBUG
        printf("wait timeout: block %d thread %d sem %p target %llu value %llu\n", (int)blockIdx.x,
               (int)threadIdx.x, (const void*)sem, (unsigned long long)target,
               (unsigned long long)ld_wait(sem, gpu));
#endif
        atomicExch(&st->error, (uint32_t)kDevTimeout);
        return false;
      }
    }
  }
}

#if CF_DROP_FENCE == 4
// mutation 4: a torn packet -- both flags land first, the payload later
__device__ __forceinline__ void ll16_torn(void* dst, uint2 data, uint32_t flag) {
  volatile uint32_t* w = reinterpret_cast<volatile uint32_t*>(dst);
  w[1] = flag;
  w[3] = flag;
  CF_STRESS_AT(4);
  w[0] = data.x;
  w[2] = data.y;
}
#endif
// LL16: two reference packets {d0, flag, d1, flag} in one 16-byte store.
__device__ __forceinline__ void ll16_put(void* dst, uint2 data, uint32_t flag) {
  CF_STRESS_AT(3);
#if CF_DROP_FENCE == 4
  ll16_torn(dst, data, flag);
#else
  st16_volatile(dst, make_uint4(data.x, flag, data.y, flag));
#endif
}
// LL16 put choosing the store by scope: ranks on one GPU meet in its L2, where
// a plain 16-byte store is already one transaction; across GPUs the store is
// volatile (not cached, not merged) like the reference's packet writes.
__device__ __forceinline__ void ll16_put_scoped(void* dst, uint2 data, uint32_t flag, bool gpu) {
  CF_STRESS_AT(3);
#if CF_DROP_FENCE == 4
  ll16_torn(dst, data, flag);
#else
  if (gpu) st16(dst, make_uint4(data.x, flag, data.y, flag));
  else st16_volatile(dst, make_uint4(data.x, flag, data.y, flag));
#endif
}
// Poll one LL16 packet until both flag words equal `flag`.
__device__ __forceinline__ uint2 ll16_get(const void* src, uint32_t flag, RankState* st) {
  uint4 v = ld16_volatile(src);
  if (v.y == flag && v.w == flag) return make_uint2(v.x, v.z);
  const uint64_t t0 = globaltimer();
  for (uint32_t it = 1;; ++it) {
    v = ld16_volatile(src);
    if (v.y == flag && v.w == flag) break;
    if ((it & 255u) == 0) {
      if (*(volatile uint32_t*)&st->error != kDevOk) break;
      if (globaltimer() - t0 > st->timeout_ns) {
        atomicExch(&st->error, (uint32_t)kDevTimeout);
        break;
      }
    }
  }
  return make_uint2(v.x, v.z);
}

// Address of 32-byte LL16 unit i of a batch: slot i of `base` (slots
// `stride` bytes apart), skipping slot `skip` (the reader's own rank).
__device__ __forceinline__ const char* ll_unit(const char* base, size_t stride, int skip, int i) {
  return base + (size_t)(i + (i >= skip ? 1 : 0)) * stride;
}

// Batched poll of K 32-byte LL16 units (two packets each, at ll_unit(i) and
// ll_unit(i) + 16) whose first loads r0/r1 the caller already issued.  Every
// round re-issues the loads of ALL units still unstamped before checking any
// of them, so waiting for K peers costs one local round trip per round, not
// one per peer.  `pend` selects the participating units.
template <int K>
__device__ __forceinline__ void ll16x2_poll(const char* base, size_t stride, int skip, uint4 (&r0)[K],
                                            uint4 (&r1)[K], uint32_t pend, uint32_t flag, RankState* st) {
  auto stamped = [&](int i) {
    return r0[i].y == flag && r0[i].w == flag && r1[i].y == flag && r1[i].w == flag;
  };
#pragma unroll
  for (int i = 0; i < K; i++)
    if (((pend >> i) & 1u) && stamped(i)) pend &= ~(1u << i);
  if (!pend) return;
  const uint64_t t0 = globaltimer();
  for (uint32_t it = 1; pend; ++it) {
#pragma unroll
    for (int i = 0; i < K; i++) {
      if ((pend >> i) & 1u) {
        const char* u = ll_unit(base, stride, skip, i);
        r0[i] = ld16_volatile(u);
        r1[i] = ld16_volatile(u + 16);
      }
    }
#pragma unroll
    for (int i = 0; i < K; i++)
      if (((pend >> i) & 1u) && stamped(i)) pend &= ~(1u << i);
    if ((it & 255u) == 0 && pend) {
      if (*(volatile uint32_t*)&st->error != kDevOk) return;
      if (globaltimer() - t0 > st->timeout_ns) {
        atomicExch(&st->error, (uint32_t)kDevTimeout);
        return;
      }
    }
  }
}

// Batched poll of K single LL16 packets (8 payload bytes each) at
// ll_unit(base, stride, skip, i); same round structure as ll16x2_poll.
template <int K>
__device__ __forceinline__ void ll16_poll(const char* base, size_t stride, int skip, uint4 (&pk)[K],
                                          uint32_t pend, uint32_t flag, RankState* st) {
#pragma unroll
  for (int i = 0; i < K; i++)
    if (((pend >> i) & 1u) && pk[i].y == flag && pk[i].w == flag) pend &= ~(1u << i);
  if (!pend) return;
  const uint64_t t0 = globaltimer();
  for (uint32_t it = 1; pend; ++it) {
#pragma unroll
    for (int i = 0; i < K; i++)
      if ((pend >> i) & 1u) pk[i] = ld16_volatile(ll_unit(base, stride, skip, i));
#pragma unroll
    for (int i = 0; i < K; i++)
      if (((pend >> i) & 1u) && pk[i].y == flag && pk[i].w == flag) pend &= ~(1u << i);
    if ((it & 255u) == 0 && pend) {
      if (*(volatile uint32_t*)&st->error != kDevOk) return;
      if (globaltimer() - t0 > st->timeout_ns) {
        atomicExch(&st->error, (uint32_t)kDevTimeout);
        return;
      }
    }
  }
}

// Payload of a stamped LL16 unit.
__device__ __forceinline__ uint4 ll16x2_payload(uint4 r0, uint4 r1) {
  return make_uint4(r0.x, r0.z, r1.x, r1.z);
}

// ---------------------------------------------------------------- element math

template <typename T> struct Vec;  // 16-byte vector of T <-> f32/i32 accumulators
template <> struct Vec<float> {
  static constexpr int N = 4;
  using Acc = float;
  __device__ static void load(uint4 v, float* a) {
    a[0] = __uint_as_float(v.x); a[1] = __uint_as_float(v.y);
    a[2] = __uint_as_float(v.z); a[3] = __uint_as_float(v.w);
  }
  __device__ static uint4 store(const float* a) {
    return make_uint4(__float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]),
                      __float_as_uint(a[3]));
  }
  __device__ static float round(float x) { return x; }
};
template <> struct Vec<int32_t> {
  static constexpr int N = 4;
  using Acc = int32_t;
  __device__ static void load(uint4 v, int32_t* a) {
    a[0] = (int32_t)v.x; a[1] = (int32_t)v.y; a[2] = (int32_t)v.z; a[3] = (int32_t)v.w;
  }
  __device__ static uint4 store(const int32_t* a) {
    return make_uint4((uint32_t)a[0], (uint32_t)a[1], (uint32_t)a[2], (uint32_t)a[3]);
  }
  __device__ static int32_t round(int32_t x) { return x; }
};
template <> struct Vec<__half> {
  static constexpr int N = 8;
  using Acc = float;
  __device__ static void load(uint4 v, float* a) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; i++) {
      __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      float2 f = __half22float2(h);
      a[2 * i] = f.x; a[2 * i + 1] = f.y;
    }
  }
  __device__ static uint4 store(const float* a) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      __half2 h = __floats2half2_rn(a[2 * i], a[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ static float round(float x) { return __half2float(__float2half_rn(x)); }
};
template <> struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  using Acc = float;
  __device__ static void load(uint4 v, float* a) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; i++) {
      a[2 * i] = __uint_as_float(w[i] << 16);
      a[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ static uint4 store(const float* a) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      __nv_bfloat162 h = __floats2bfloat162_rn(a[2 * i], a[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ static float round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
};

// Scalar element access for ragged heads/tails.
template <typename T> __device__ __forceinline__ typename Vec<T>::Acc to_acc(T x);
template <> __device__ __forceinline__ float to_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ int32_t to_acc<int32_t>(int32_t x) { return x; }
template <> __device__ __forceinline__ float to_acc<__half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ float to_acc<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <typename T> __device__ __forceinline__ T from_acc(typename Vec<T>::Acc x);
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ int32_t from_acc<int32_t>(int32_t x) { return x; }
template <> __device__ __forceinline__ __half from_acc<__half>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// i32 adds wrap like numpy int32 (two's complement); use unsigned math.
__device__ __forceinline__ int32_t acc_add(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a + (uint32_t)b);
}
__device__ __forceinline__ float acc_add(float a, float b) { return __fadd_rn(a, b); }

// ---------------------------------------------------------------- reduction orders
//
// The reference accumulates each element chunk in an algorithm-specific order
// (probed, pinned by tests/golden):
//   kLead   : x[lead], then every other rank ascending   (1pa: lead = own rank,
//             2pa: lead = chunk owner)          cf/collectives.py:156-161, 187-231
//   kAscZero: 0 + x[0] + ... + x[n-1]          switch_reduce, cf/channels.py:380-388
//   kRingZero: 0 + x[c] + x[c+1] + ... (mod n) ring_rs / 2pr, cf/collectives.py:52-79
enum Order : int { kLead = 0, kAscZero = 1, kRingZero = 2 };

// k-th source rank of the order.
__device__ __forceinline__ int order_src(int mode, int k, int lead, int n) {
  if (mode == kLead) return k == 0 ? lead : (k - 1 + (k - 1 >= lead ? 1 : 0));
  if (mode == kRingZero) { int q = lead + k; return q >= n ? q - n : q; }
  return k;
}

// ---------------------------------------------------------------- channels
//
// The Primitive API for user kernels.  A channel handle is
// built on the host (cfMemoryChannelCreate / cfPortChannelCreate) and passed
// by value to the kernels of BOTH endpoints: put / signal / put_packets /
// flush run on the source rank, wait / read_packets on the destination rank
// (cf/channels.py:54-330).  Semaphores count (signal = +1, wait = expected+1
// then spin), so k signals satisfy k waits (reference test_channels.py:185-229).

struct MemoryChannelDevice {
  char* src_buf;            // source rank's buffer (source device)
  char* dst_buf;            // destination rank's buffer as mapped on the source device
  char* dst_local;          // destination rank's buffer on the destination device
  uint64_t* sem;            // semaphore slot in the destination heap
  uint64_t* expected;       // destination-side wait counter
  RankState* src_st;
  RankState* dst_st;
  int gpu_scope;            // both endpoints on one device
  int pad_;

  // put (HB): cooperative 16-byte copy src_buf[src_off..] -> dst_buf[dst_off..]
  // by threads tid of nthreads; visible to the peer after signal().
  __device__ void put(size_t dst_off, size_t src_off, size_t bytes, int tid, int nthreads) const {
    const size_t nv = bytes / 16;
    for (size_t i = tid; i < nv; i += nthreads) st16(dst_buf + dst_off + i * 16, ld16(src_buf + src_off + i * 16));
    for (size_t i = nv * 16 + tid; i < bytes; i += nthreads) dst_buf[dst_off + i] = src_buf[src_off + i];
  }
  // signal (one thread, after a block barrier covering the puts it publishes)
  __device__ void signal() const {
    fence_publish(gpu_scope);
    if (gpu_scope) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(sem) : "memory");
    else asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(sem) : "memory");
  }
  // wait (one thread on the destination rank): false on timeout (E_DEADLOCK)
  __device__ bool wait() const {
    const uint64_t target = ++*expected;
    return wait_geq(sem, target, dst_st, gpu_scope);
  }
  __device__ void flush() const {}   // memory channel: the put completed in place
  // put_packets (LL): `bytes` (multiple of 8) as LL16 packets at packet offset
  // pkt_off of the destination buffer; no semaphore needed.
  __device__ void put_packets(size_t pkt_off, size_t src_off, size_t bytes, uint32_t flag, int tid,
                              int nthreads) const {
    for (size_t u = tid; u < bytes / 8; u += nthreads)
      ll16_put(dst_buf + pkt_off + u * 16, *reinterpret_cast<const uint2*>(src_buf + src_off + u * 8), flag);
  }
  // read_packets (destination rank): decode packets at pkt_off of the local
  // destination buffer into out, spinning until every flag is stamped.
  __device__ void read_packets(char* out, size_t pkt_off, size_t bytes, uint32_t flag, int tid, int nthreads) const {
    for (size_t u = tid; u < bytes / 8; u += nthreads)
      *reinterpret_cast<uint2*>(out + u * 8) = ll16_get(dst_local + pkt_off + u * 16, flag, dst_st);
  }
};


// ---------------------------------------------------------------- NVLS switch
//
// multimem.ld_reduce sums the same address over every member of a multicast
// object inside the NVSwitch (f16/bf16 accumulate in f32); multimem.st
// broadcasts one store to every member.  Both need a multicast mapping
// (cuMulticastCreate + cuMulticastBindMem + cuMemMap of the multicast handle).
template <typename T>
__device__ __forceinline__ uint4 multimem_ld_reduce(const void* p);
template <>
__device__ __forceinline__ uint4 multimem_ld_reduce<float>(const void* p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 multimem_ld_reduce<__nv_bfloat16>(const void* p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 multimem_ld_reduce<__half>(const void* p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 multimem_ld_reduce<int32_t>(const void* p) {
  uint4 v;
  const char* c = (const char*)p;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(v.x) : "l"(c) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(v.y) : "l"(c + 4) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(v.z) : "l"(c + 8) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(v.w) : "l"(c + 12) : "memory");
  return v;
}
__device__ __forceinline__ void multimem_st16(void* p, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w) : "memory");
}

// 0 + x_0 + x_1 + ... + x_{n-1} of one 16-byte vector read from every
// member's unicast mapping (the reference switch order, cf/channels.py:380-388)
template <typename T>
__device__ __forceinline__ uint4 switch_sum_unicast(char* const* uc, int n, size_t off) {
  using A = typename Vec<T>::Acc;
  constexpr int V = Vec<T>::N;
  A acc[V], t[V];
#pragma unroll
  for (int j = 0; j < V; j++) acc[j] = A(0);
#pragma unroll
  for (int q = 0; q < CF_MAX_RANKS; q++)
    if (q < n) {
      Vec<T>::load(ld16_cg(uc[q] + off), t);
#pragma unroll
      for (int j = 0; j < V; j++) acc[j] = acc_add(acc[j], t[j]);
    }
  return Vec<T>::store(acc);
}

// SwitchChannel (cf/channels.py:333-409) for user kernels: the members'
// symmetric heaps bound to one multicast object.  Offsets are heap offsets
// (cfMemAlloc returns the same offset on every rank).  `mc` is null on boxes
// without multicast when the communicator emulates the switch
// (cfConfig.use_multicast = 2): the same calls then run as per-member
// unicast loads / stores through `uc`.  Built by cfSwitchChannelCreate.
struct SwitchChannelDevice {
  char* mc;                  // multicast mapping of the heap (null: emulated)
  char* uc[CF_MAX_RANKS];    // every member's heap, as mapped on this rank's device
  char* local;               // this rank's heap
  int n;                     // members
  int rank;

  // switch_reduce (cf/channels.py:367-389): local dst[v] = sum over members of
  // their heap at src_off, for the 16-byte vectors v = tid, tid+nthreads, ...
  // of `bytes` (multiple of 16).
  template <typename T>
  __device__ void reduce(char* dst, size_t src_off, size_t bytes, int tid, int nthreads) const {
    size_t v = tid;
    if (mc)   // four switch reductions in flight per thread
      for (; v + 3 * (size_t)nthreads < bytes / 16; v += 4 * (size_t)nthreads) {
        uint4 x[4];
#pragma unroll
        for (int u = 0; u < 4; u++) x[u] = multimem_ld_reduce<T>(mc + src_off + (v + u * nthreads) * 16);
#pragma unroll
        for (int u = 0; u < 4; u++) st16(dst + (v + u * nthreads) * 16, x[u]);
      }
    for (; v < bytes / 16; v += nthreads)
      st16(dst + v * 16, mc ? multimem_ld_reduce<T>(mc + src_off + v * 16)
                            : switch_sum_unicast<T>(uc, n, src_off + v * 16));
  }
  // switch_broadcast (cf/channels.py:392-409): every member's heap at dst_off
  // receives src[v].
  __device__ void broadcast(size_t dst_off, const char* src, size_t bytes, int tid, int nthreads) const {
    for (size_t v = tid; v < bytes / 16; v += nthreads) {
      const uint4 x = ld16(src + v * 16);
      if (mc) {
        multimem_st16(mc + dst_off + v * 16, x);
      } else {
        for (int q = 0; q < n; q++) st16(uc[q] + dst_off + v * 16, x);
      }
    }
  }
  // fused reduce + broadcast of heap range [off, off + bytes) from src_off
  // (one pass, the NVLS AllReduce of one chunk)
  template <typename T>
  __device__ void reduce_broadcast(size_t dst_off, size_t src_off, size_t bytes, int tid, int nthreads) const {
    size_t v = tid;
    if (mc)
      for (; v + 3 * (size_t)nthreads < bytes / 16; v += 4 * (size_t)nthreads) {
        uint4 x[4];
#pragma unroll
        for (int u = 0; u < 4; u++) x[u] = multimem_ld_reduce<T>(mc + src_off + (v + u * nthreads) * 16);
#pragma unroll
        for (int u = 0; u < 4; u++) multimem_st16(mc + dst_off + (v + u * nthreads) * 16, x[u]);
      }
    for (; v < bytes / 16; v += nthreads) {
      if (mc) {
        multimem_st16(mc + dst_off + v * 16, multimem_ld_reduce<T>(mc + src_off + v * 16));
      } else {
        const uint4 x = switch_sum_unicast<T>(uc, n, src_off + v * 16);
        for (int q = 0; q < n; q++) st16(uc[q] + dst_off + v * 16, x);
      }
    }
  }
};

}  // namespace cf

// cf_proxy.h -- PortChannel request FIFO shared by device producers and the
// host proxy thread (cf/channels.py:54-150 PortChannel, cf/fifo.py:19-108).
//
// Device side: any thread reserves a ticket with an atomic on device memory,
// writes the request into a slot of a host-mapped pinned ring, and publishes
// it by storing ticket+1 last.  Host side: one proxy thread per communicator
// consumes tickets in order, issues the copy on the copy engine
// (cudaMemcpyAsync, peer DMA over NVLink) and then, in the same stream, the
// semaphore write (signal ordered after the put, cf/channels.py:124-150) and
// the producer's completion value (flush waits for it, cf/fifo.py:92-108).
#pragma once
#include <cstdint>
#include "device/cf_device.cuh"

namespace cf {

struct PortRequest {
  uint64_t src;        // device address (0 bytes: no copy)
  uint64_t dst;
  uint64_t bytes;
  uint64_t sem;        // device address written after the copy (0: none)
  uint64_t sem_value;
  uint64_t done;       // producer's completion counter (device address; 0: none)
  uint64_t ticket;     // ticket + 1 once the entry is complete
  uint64_t pad;
};

constexpr uint32_t kPortFifoCap = 1024;

struct PortFifo {                    // pinned host memory, mapped into the device
  PortRequest slots[kPortFifoCap];
  uint64_t tail;                     // entries consumed by the proxy
  uint64_t pad[7];
};

// What a kernel needs to post requests for one rank.
struct PortQueue {
  PortRequest* slots;                // device pointer of the mapped slots
  const uint64_t* tail;              // device pointer of the mapped tail
  uint64_t* head;                    // device memory: next ticket
};

}  // namespace cf

struct cfComm;
namespace cf {
// Device handle of local rank li's request ring (the proxy must be running).
PortQueue proxy_queue(const cfComm* c, int li);

#ifdef __CUDACC__
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Post one request (single thread).  Returns the ticket.
__device__ __forceinline__ uint64_t port_post(const PortQueue& q, uint64_t src, uint64_t dst, uint64_t bytes,
                                              uint64_t sem, uint64_t sem_value, uint64_t done, RankState* st) {
  const uint64_t t = atomicAdd((unsigned long long*)q.head, 1ull);
  if (t >= kPortFifoCap) {           // ring full: wait until the proxy consumed slot t - cap
    const uint64_t t0 = globaltimer();
    for (uint32_t it = 0;; ++it) {
      const uint64_t tail = *(volatile const uint64_t*)q.tail;
      if (t - tail < kPortFifoCap) break;
      if ((it & 63u) == 0) {
        if (*(volatile uint32_t*)&st->error != kDevOk) return t;
        if (globaltimer() - t0 > st->timeout_ns) { atomicExch(&st->error, (uint32_t)kDevTimeout); return t; }
      }
    }
  }
  PortRequest* s = q.slots + (t % kPortFifoCap);
  st_volatile_u64(&s->src, src);
  st_volatile_u64(&s->dst, dst);
  st_volatile_u64(&s->bytes, bytes);
  st_volatile_u64(&s->sem, sem);
  st_volatile_u64(&s->sem_value, sem_value);
  st_volatile_u64(&s->done, done);
  __threadfence_system();
  st_volatile_u64(&s->ticket, t + 1);
  return t;
}

// Wait until the proxy completed ticket t of this producer.
__device__ __forceinline__ void port_flush(const uint64_t* done, uint64_t t, RankState* st) {
  wait_geq(done, t + 1, st, false);
}
#endif

// PortChannel handle for user kernels (Primitive API, cf/channels.py:54-150):
// put / signal / put_with_signal / flush on the source rank (one thread per
// channel), wait on the destination rank.  Requests go to the source rank's
// proxy, which copies with the copy engine and then writes the semaphore.
struct PortChannelDevice {
  PortQueue q;
  char* src_buf;            // source rank's buffer
  char* dst_buf;            // destination rank's buffer (UVA address for the DMA engine)
  uint64_t* sem;            // destination semaphore slot
  uint64_t* sent;           // source side: signals issued (absolute count)
  uint64_t* done;           // source side: completion counter written by the proxy
  uint64_t* last;           // source side: last ticket + 1 (0: nothing issued)
  uint64_t* expected;       // destination side: waits issued
  RankState* src_st;
  RankState* dst_st;
#ifdef __CUDACC__
  __device__ void put(size_t dst_off, size_t src_off, size_t bytes) const {
    *last = port_post(q, (uint64_t)(src_buf + src_off), (uint64_t)(dst_buf + dst_off), bytes, 0, 0,
                      (uint64_t)done, src_st) + 1;
  }
  __device__ void signal() const {
    const uint64_t v = ++*sent;
    *last = port_post(q, 0, 0, 0, (uint64_t)sem, v, (uint64_t)done, src_st) + 1;
  }
  __device__ void put_with_signal(size_t dst_off, size_t src_off, size_t bytes) const {
    const uint64_t v = ++*sent;
    *last = port_post(q, (uint64_t)(src_buf + src_off), (uint64_t)(dst_buf + dst_off), bytes, (uint64_t)sem, v,
                      (uint64_t)done, src_st) + 1;
  }
  // every request issued so far completed (the source may be reused)
  __device__ void flush() const {
    if (*last) port_flush(done, *last - 1, src_st);
  }
  __device__ bool wait() const {
    const uint64_t target = ++*expected;
    return wait_geq(sem, target, dst_st, false);
  }
#endif
};

}  // namespace cf

// cf_proxy.cu -- the host proxy serving PortChannel requests (cf/channels.py:
// 54-150, cf/fifo.py:19-108) with copy-engine DMA.
//
// One thread per communicator polls the request ring of every local rank in
// ticket order.  Per request, on the rank's proxy stream: cudaMemcpyAsync
// (peer DMA over NVLink / same-device copy engine), then the semaphore value
// (the signal is ordered after the put because the stream is FIFO), then the
// producer's completion value (what flush waits for).  The device never waits
// for the host except in flush / when the ring is full.
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <cuda.h>
#include "cf_proxy.h"
#include "cf_runtime.h"

namespace cf {

struct Proxy {
  std::thread thread;
  std::atomic<bool> stop{false};
  std::atomic<bool> alive{false};
  std::atomic<bool> failed{false};
  std::vector<PortFifo*> fifo;         // host pointers, per local rank
  std::vector<PortFifo*> fifo_dev;     // device pointers of the same memory
  std::vector<uint64_t*> head;         // device memory, per local rank
  std::vector<cudaStream_t> stream;    // proxy streams, per local rank
};

namespace {

using WriteValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

void proxy_main(cfComm* c, Proxy* p) {
  auto write64 = (WriteValue64)driver_fn("cuStreamWriteValue64");
  if (!write64) { p->failed = true; p->alive = false; return; }
  const size_t nl = p->fifo.size();
  std::vector<uint64_t> tail(nl, 0);
  int cur_dev = -1;
  uint32_t idle = 0;
  while (!p->stop.load(std::memory_order_relaxed)) {
    bool busy = false;
    for (size_t li = 0; li < nl; li++) {
      PortFifo* f = p->fifo[li];
      const uint64_t t = tail[li];
      PortRequest* s = &f->slots[t % kPortFifoCap];
      if (__atomic_load_n(&s->ticket, __ATOMIC_ACQUIRE) != t + 1) continue;
      PortRequest r;
      memcpy(&r, (const void*)s, sizeof(r));
      if (cur_dev != c->local[li].dev) {
        cudaSetDevice(c->local[li].dev);
        cur_dev = c->local[li].dev;
      }
      bool ok = true;
      if (r.bytes)
        ok &= cudaMemcpyAsync((void*)r.dst, (const void*)r.src, r.bytes, cudaMemcpyDeviceToDevice,
                              p->stream[li]) == cudaSuccess;
      if (r.sem) ok &= write64((CUstream)p->stream[li], (CUdeviceptr)r.sem, r.sem_value, 0) == CUDA_SUCCESS;
      if (r.done) ok &= write64((CUstream)p->stream[li], (CUdeviceptr)r.done, t + 1, 0) == CUDA_SUCCESS;
      if (!ok) {
        fprintf(stderr, "libcf proxy: request %llu failed\n", (unsigned long long)t);
        p->failed = true;
        p->alive = false;
        return;
      }
      tail[li] = t + 1;
      __atomic_store_n(&f->tail, t + 1, __ATOMIC_RELEASE);
      busy = true;
    }
    if (busy) {
      idle = 0;
    } else if (++idle > 4096) {
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    } else {
      std::this_thread::yield();
    }
  }
  p->alive = false;
}

}  // namespace

cfStatus proxy_start(cfComm* c) {
  if (c->proxy && c->proxy->alive) return CF_OK;
  if (c->proxy && c->proxy->failed) return fail(CF_E_PROXY_DOWN, "the port-channel proxy stopped after a failed request");
  Proxy* p = new Proxy();
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto& lr : c->local) {
    cudaSetDevice(lr.dev);
    PortFifo* f = nullptr;
    if (cudaHostAlloc((void**)&f, sizeof(PortFifo), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
      cudaSetDevice(prev);
      return fail(CF_E_CUDA, "pinned FIFO allocation failed");
    }
    memset((void*)f, 0, sizeof(PortFifo));
    PortFifo* fd = nullptr;
    cudaHostGetDevicePointer((void**)&fd, f, 0);
    uint64_t* head = nullptr;
    cudaMalloc((void**)&head, 256);
    cudaMemset(head, 0, 256);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    p->fifo.push_back(f);
    p->fifo_dev.push_back(fd);
    p->head.push_back(head);
    p->stream.push_back(s);
  }
  cudaDeviceSynchronize();
  cudaSetDevice(prev);
  p->alive = true;
  p->thread = std::thread(proxy_main, c, p);
  c->proxy = p;
  return CF_OK;
}

void proxy_stop(cfComm* c) {
  Proxy* p = c->proxy;
  if (!p) return;
  p->stop = true;
  if (p->thread.joinable()) p->thread.join();
  for (size_t li = 0; li < p->fifo.size(); li++) {
    cudaSetDevice(c->local[li].dev);
    cudaStreamSynchronize(p->stream[li]);
    cudaStreamDestroy(p->stream[li]);
    cudaFree(p->head[li]);
    cudaFreeHost(p->fifo[li]);
  }
  delete p;
  c->proxy = nullptr;
}

bool proxy_alive(const cfComm* c) { return c->proxy && c->proxy->alive; }

PortQueue proxy_queue(const cfComm* c, int li) {
  PortQueue q;
  q.slots = c->proxy->fifo_dev[li]->slots;
  q.tail = &c->proxy->fifo_dev[li]->tail;
  q.head = c->proxy->head[li];
  return q;
}

}  // namespace cf

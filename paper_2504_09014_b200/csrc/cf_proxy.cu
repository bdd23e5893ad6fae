// cf_proxy.cu -- the host proxy serving PortChannel requests (cf/channels.py:
// 54-150, cf/fifo.py:19-108) with copy-engine DMA.
//
// One thread per communicator polls the request ring of every local rank in
// ticket order and serves the ready requests in batches, on the rank's proxy
// stream: their copies (peer DMA over NVLink / same-device copy engine), then
// their semaphore values and the producer's
// completion values in one cuStreamBatchMemOp -- every signal is ordered
// after its put because the stream is FIFO, and flush waits for completion,
// not for the pop.  The device never waits for the host except in flush /
// when the ring is full.
#include <algorithm>
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

using BatchMemOp = CUresult (*)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

// Requests taken per batch: one cudaMemcpyAsync per copy, then all their
// semaphore / completion writes in one cuStreamBatchMemOp (the host cost per
// API call, not the copy engine, bounds a request-at-a-time proxy: a 2pa port
// plan posts one request per CTA slice and put).
constexpr int kProxyBatch = 64;

bool overlap(uint64_t a, uint64_t na, uint64_t b, uint64_t nb) { return na && nb && a < b + nb && b < a + na; }

// A batch may not hold two requests whose copies touch each other's ranges
// (kept conservative: the batch's signals all follow all of its copies).
bool conflicts(const std::vector<PortRequest>& batch, const PortRequest& r) {
  for (const auto& q : batch)
    if (overlap(q.dst, q.bytes, r.dst, r.bytes) || overlap(q.dst, q.bytes, r.src, r.bytes) ||
        overlap(q.src, q.bytes, r.dst, r.bytes))
      return true;
  return false;
}

// A stream capture in progress elsewhere in the process (global capture mode)
// makes these calls fail without harm: retry the batch once it ends.
bool capture_blocked(cudaError_t e) {
  return e == cudaErrorStreamCaptureImplicit || e == cudaErrorStreamCaptureUnsupported ||
         e == cudaErrorStreamCaptureWrongThread;
}
bool capture_blocked(CUresult e) {
  return e == CUDA_ERROR_STREAM_CAPTURE_IMPLICIT || e == CUDA_ERROR_STREAM_CAPTURE_UNSUPPORTED ||
         e == CUDA_ERROR_STREAM_CAPTURE_WRONG_THREAD;
}

void proxy_main(cfComm* c, Proxy* p) {
  auto mem_ops = (BatchMemOp)driver_fn("cuStreamBatchMemOp_v2");
  if (!mem_ops) mem_ops = (BatchMemOp)driver_fn("cuStreamBatchMemOp");
  if (!mem_ops) { p->failed = true; p->alive = false; return; }
  const size_t nl = p->fifo.size();
  std::vector<uint64_t> tail(nl, 0);
  int cur_dev = -1;
  uint32_t idle = 0;
  std::vector<PortRequest> batch;
  std::vector<void*> dsts, srcs, mdst, msrc;
  std::vector<size_t> sizes, msz, idx;
  std::vector<CUstreamBatchMemOpParams> ops;
  batch.reserve(kProxyBatch);
  while (!p->stop.load(std::memory_order_relaxed)) {
    bool busy = false;
    for (size_t li = 0; li < nl; li++) {
      PortFifo* f = p->fifo[li];
      batch.clear();
      for (uint64_t t = tail[li]; batch.size() < (size_t)kProxyBatch; t++) {
        PortRequest* s = &f->slots[t % kPortFifoCap];
        if (__atomic_load_n(&s->ticket, __ATOMIC_ACQUIRE) != t + 1) break;
        PortRequest r;
        memcpy(&r, (const void*)s, sizeof(r));
        if (conflicts(batch, r)) break;
        batch.push_back(r);
      }
      if (batch.empty()) continue;
      if (cur_dev != c->local[li].dev) {
        cudaSetDevice(c->local[li].dev);
        cur_dev = c->local[li].dev;
      }
      const uint64_t t0 = tail[li];
      dsts.clear(), srcs.clear(), sizes.clear(), ops.clear();
      for (size_t i = 0; i < batch.size(); i++) {
        const PortRequest& r = batch[i];
        if (r.bytes) {
          dsts.push_back((void*)r.dst);
          srcs.push_back((void*)r.src);
          sizes.push_back(r.bytes);
        }
        auto write = [&](uint64_t addr, uint64_t v) {
          CUstreamBatchMemOpParams o;
          memset(&o, 0, sizeof(o));
          o.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
          o.writeValue.address = (CUdeviceptr)addr;
          o.writeValue.value64 = v;
          ops.push_back(o);
        };
        if (r.sem) write(r.sem, r.sem_value);
        if (r.done) write(r.done, t0 + i + 1);
      }
      // the CTA slices of one put arrive as adjacent ranges: merge them into
      // one copy (copies of a batch never overlap, and every signal of the
      // batch follows all of its copies, so their order is free)
      idx.resize(sizes.size());
      for (size_t i = 0; i < idx.size(); i++) idx[i] = i;
      std::sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return dsts[x] < dsts[y]; });
      size_t ncopy = 0;
      for (size_t k = 0; k < idx.size(); k++) {
        const size_t i = idx[k];
        if (ncopy && (char*)mdst[ncopy - 1] + msz[ncopy - 1] == (char*)dsts[i] &&
            (char*)msrc[ncopy - 1] + msz[ncopy - 1] == (char*)srcs[i]) {
          msz[ncopy - 1] += sizes[i];
          continue;
        }
        if (mdst.size() <= ncopy) mdst.resize(ncopy + 1), msrc.resize(ncopy + 1), msz.resize(ncopy + 1);
        mdst[ncopy] = dsts[i], msrc[ncopy] = srcs[i], msz[ncopy] = sizes[i];
        ncopy++;
      }
      // copies first (stream order), then every signal / completion of the batch
      cudaError_t ce = cudaSuccess;
      for (size_t i = 0; i < ncopy && ce == cudaSuccess; i++)
        ce = cudaMemcpyAsync(mdst[i], msrc[i], msz[i], cudaMemcpyDeviceToDevice, p->stream[li]);
      CUresult me = CUDA_SUCCESS;
      if (ce == cudaSuccess && !ops.empty())
        me = mem_ops((CUstream)p->stream[li], (unsigned)ops.size(), ops.data(), 0);
      if (ce != cudaSuccess || me != CUDA_SUCCESS) {
        if (capture_blocked(ce) || capture_blocked(me)) {   // retried (copies and writes are idempotent)
          cudaGetLastError();
          std::this_thread::sleep_for(std::chrono::microseconds(20));
          continue;
        }
        fprintf(stderr, "libcf proxy: requests %llu..%llu failed (%s, CUresult %d)\n", (unsigned long long)t0,
                (unsigned long long)(t0 + batch.size() - 1), cudaGetErrorString(ce), (int)me);
        p->failed = true;
        p->alive = false;
        return;
      }
      tail[li] = t0 + batch.size();
      __atomic_store_n(&f->tail, tail[li], __ATOMIC_RELEASE);
      busy = true;
    }
    if (busy) {
      idle = 0;
    } else if (++idle > 4096) {
      std::this_thread::sleep_for(std::chrono::microseconds(5));
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

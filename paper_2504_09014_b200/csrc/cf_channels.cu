// cf_channels.cu -- host construction of channel handles for user kernels
// (MemoryChannel cf/channels.py:153-300, PortChannel cf/channels.py:54-150).
//
// Per channel (src, dst, tag) the heaps hold five u64 words:
//   dst heap  sem[src][tag]       the semaphore the source increments
//   dst heap  expected[src][tag]  the destination's wait counter
//   src heap  sent[dst][tag]      port: signals issued (absolute semaphore value)
//   src heap  done[dst][tag]      port: proxy completion counter
//   src heap  last[dst][tag]      port: last ticket + 1
#include <cstring>
#include "cf_proxy.h"
#include "cf_runtime.h"

namespace cf {
namespace {

enum ChanWord { kSem = 0, kExpected = 1, kSent = 2, kDone = 3, kLast = 4 };

uint64_t* chan_word(cfComm* c, int li_view, int owner_rank, int word, int other_rank, int tag) {
  char* heap = c->peer_heap[li_view][owner_rank];
  uint64_t* base = (uint64_t*)(heap + c->lay.chan_off);
  return base + ((size_t)word * CF_MAX_RANKS + other_rank) * CF_MAX_CHANNEL_TAGS + tag;
}

cfStatus check_args(cfComm* c, int src, int dst, int tag, void* sbuf, void* dbuf, void* handle, size_t* bytes,
                    size_t need) {
  if (!c || !handle || !bytes || !sbuf || !dbuf) return fail(CF_E_CONFIG, "null argument");
  if (c->multiprocess) return fail(CF_E_TOPOLOGY, "user channels need a one-process communicator in this version");
  if (src < 0 || src >= c->nranks || dst < 0 || dst >= c->nranks) return fail(CF_E_OOB, "rank out of range");
  if (src == dst) return fail(CF_E_SHAPE, "channel has src == dst");
  if (tag < 0 || tag >= CF_MAX_CHANNEL_TAGS) return fail(CF_E_OOB, "tag %d outside [0, %d)", tag, CF_MAX_CHANNEL_TAGS);
  if (*bytes < need) {
    *bytes = need;
    return fail(CF_E_BAD_SIZE, "handle buffer needs %zu bytes", need);
  }
  *bytes = need;
  return CF_OK;
}

}  // namespace
}  // namespace cf

using namespace cf;

extern "C" cfStatus cfMemoryChannelCreate(cfComm_t c, int src, int dst, int tag, void* sbuf, void* dbuf,
                                          void* handle, size_t* bytes) {
  static_assert(sizeof(MemoryChannelDevice) <= CF_CHANNEL_HANDLE_BYTES, "handle too large");
  CF_TRY(check_args(c, src, dst, tag, sbuf, dbuf, handle, bytes, sizeof(MemoryChannelDevice)));
  MemoryChannelDevice h;
  memset(&h, 0, sizeof(h));
  h.src_buf = (char*)sbuf;
  h.dst_buf = (char*)dbuf;     // one process: UVA address valid on both devices
  h.dst_local = (char*)dbuf;
  h.sem = chan_word(c, src, dst, kSem, src, tag);
  h.expected = chan_word(c, dst, dst, kExpected, src, tag);
  h.src_st = c->state(src);
  h.dst_st = c->state(dst);
  h.gpu_scope = c->local[src].dev == c->local[dst].dev;
  memcpy(handle, &h, sizeof(h));
  return CF_OK;
}

extern "C" cfStatus cfPortChannelCreate(cfComm_t c, int src, int dst, int tag, void* sbuf, void* dbuf,
                                        void* handle, size_t* bytes) {
  static_assert(sizeof(PortChannelDevice) <= CF_CHANNEL_HANDLE_BYTES, "handle too large");
  CF_TRY(check_args(c, src, dst, tag, sbuf, dbuf, handle, bytes, sizeof(PortChannelDevice)));
  CF_TRY(proxy_start(c));
  PortChannelDevice h;
  memset(&h, 0, sizeof(h));
  h.q = proxy_queue(c, src);
  h.src_buf = (char*)sbuf;
  h.dst_buf = (char*)dbuf;
  h.sem = chan_word(c, src, dst, kSem, src, tag);
  h.sent = chan_word(c, src, src, kSent, dst, tag);
  h.done = chan_word(c, src, src, kDone, dst, tag);
  h.last = chan_word(c, src, src, kLast, dst, tag);
  h.expected = chan_word(c, dst, dst, kExpected, src, tag);
  h.src_st = c->state(src);
  h.dst_st = c->state(dst);
  memcpy(handle, &h, sizeof(h));
  return CF_OK;
}

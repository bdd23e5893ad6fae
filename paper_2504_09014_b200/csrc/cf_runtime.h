// cf_runtime.h -- host-side communicator internals shared by the collective
// API (cf_runtime.cu) and the plan executor (cf_plan.cu).  Not part of the ABI.
#pragma once
#include <array>
#include <cstdarg>
#include <cstddef>
#include <cstdint>
#include <map>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "cf.h"
#include "cf_kernels.cuh"

namespace cf {

struct Proxy;
cfStatus fail(cfStatus s, const char* fmt, ...);

#define CF_CUDA(call)                                                                \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return ::cf::fail(CF_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));  \
  } while (0)

#define CF_TRY(call)                     \
  do {                                   \
    cfStatus s_ = (call);                \
    if (s_ != CF_OK) return s_;          \
  } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline size_t ceil_div(size_t x, size_t a) { return (x + a - 1) / a; }
inline int dtype_size(int dt) { return dt <= 1 ? 4 : 2; }

// Symmetric heap of one rank:
// [RankState | semaphore slab | ack slab | ring slots | LL scratch (2 parities)]
struct HeapLayout {
  size_t state_off = 0;
  size_t sem_off = 256;
  size_t sem_bytes = (size_t)CF_MAX_RANKS * CF_MAX_BLOCKS * sizeof(uint64_t);
  size_t ack_off = 0;
  size_t chan_off = 0;      // user channels: 5 arrays [CF_MAX_RANKS][CF_MAX_CHANNEL_TAGS] u64
  size_t ring_off = 0;
  size_t scr_off = 0, scr_bytes = 0;
  size_t slot = 0, half = 0;
  size_t total = 0;
  void compute(int nranks, size_t ll_max);
};

struct LocalRank {
  int rank = -1;
  int dev = -1;
  char* heap = nullptr;
  cudaEvent_t ev = nullptr;   // stream joins for co-resident ranks
  char* stage_in = nullptr;   // cfAllReduceHost device staging (grown on demand)
  char* stage_out = nullptr;
  size_t stage_bytes = 0;
};

// cfAllReduceHost: per-device copy streams and the events of one pipelined call.
constexpr int kHostPieces = 32;
struct HostPipe {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t fork = nullptr, done = nullptr;
  cudaEvent_t in[kHostPieces] = {}, ar[kHostPieces] = {};
};

// A registered buffer range (one-process-per-GPU mode) and the peers' mapped
// counterparts.
struct Registration {
  const char* ptr = nullptr;
  size_t bytes = 0;
  std::array<char*, CF_MAX_RANKS> peer{};
  std::vector<std::string> keys;   // ipc cache keys held by this registration
};

struct IpcMapping {
  void* base = nullptr;
  int refs = 0;
};

// NVLS multicast staging of one local rank: physical memory bound to the
// communicator's multicast object, mapped twice (unicast for the local
// copy-in/out, multicast for multimem.ld_reduce / multimem.st).
struct NvlsRank {
  unsigned long long mem = 0;   // CUmemGenericAllocationHandle
  char* uc = nullptr;           // [input half | output half], unicast
  char* mc = nullptr;           // same layout, multicast
};

struct Nvls {
  bool enabled = false;
  bool emul = false;            // emulated switch: unicast staging, no multicast object
  std::vector<char*> peer_uc;   // emulated switch, one process per rank: every rank's staging (mapped)
  size_t half = 0;              // bytes of each half (input, output)
  size_t size = 0;              // 2*half rounded to the multicast granularity
  size_t gran = 0;
  unsigned long long mc = 0;    // CUmemGenericAllocationHandle of the multicast object
  bool added = false;
  std::vector<NvlsRank> ranks;  // per local rank
};

// Symmetric heap (cfSymHeapCreate / cfMemAlloc): per rank one cuMem
// allocation of `bytes`, mapped unicast on every local device and -- one
// process per GPU -- imported into every peer by POSIX fd; with a multicast
// object the heap is also bound and mapped multicast.  cfMemAlloc carves
// the same offset out of every rank's heap, so a buffer's peers are
// base[p] + offset: no per-buffer registration.
struct SymRank {
  unsigned long long mem = 0;   // CUmemGenericAllocationHandle (own allocation)
  char* uc = nullptr;           // own heap, unicast
  char* mc = nullptr;           // own heap, multicast mapping (mode 1)
};

struct SymHeap {
  int mode = 0;                 // 0 none, 1 multicast (NVLS), 2 emulated switch (unicast)
  size_t bytes = 0, gran = 0;
  unsigned long long mc = 0;    // multicast object (mode 1)
  bool mc_added = false;
  std::vector<SymRank> ranks;   // per local rank
  std::vector<std::array<char*, CF_MAX_RANKS>> peer;   // [li][p]: rank p's heap as seen from li
  std::vector<std::pair<unsigned long long, char*>> imported;   // (handle, va) of mapped peers
  std::map<size_t, size_t> used;  // allocations: offset -> bytes
  bool on() const { return bytes != 0; }
  // offset of p inside local rank li's heap, or -1
  long long offset(int li, const void* p) const {
    if (!bytes || li >= (int)ranks.size() || !ranks[li].uc) return -1;
    const char* q = (const char*)p;
    return (q >= ranks[li].uc && q < ranks[li].uc + bytes) ? (long long)(q - ranks[li].uc) : -1;
  }
};

}  // namespace cf

struct cfComm {
  int nranks = 0;
  bool multiprocess = false;
  bool connected = false;
  cfConfig cfg{};
  cf::HeapLayout lay;
  std::vector<cf::LocalRank> local;
  // peer_heap[li][p]: heap base of rank p as addressable from local rank li's device
  std::vector<std::array<char*, CF_MAX_RANKS>> peer_heap;
  // local-rank indices grouped by device (one launch per group)
  std::vector<std::vector<int>> groups;
  std::vector<void*> ipc_opened;       // cudaIpcOpenMemHandle mappings to close
  std::vector<cf::Registration> regs;  // registered user buffers (multi-process)
  std::map<std::string, cf::IpcMapping> ipc_cache;  // peer allocation -> mapping
  std::map<int, int> sm_count;         // device -> SMs
  std::map<std::pair<const void*, int>, int> occ;  // (kernel, device) -> CTAs/SM
  bool multicast_supported = false;
  // CTA budget per rank and algorithm (cfCommSetCtaBudget; index CF_ALGO_COUNT =
  // the fused K13 kernel; budget_all applies to every algorithm without its own)
  int budget[CF_ALGO_COUNT + 1] = {};
  int budget_all = 0;
  // measured selection tables (cfCommSetSelection) per (collective, dtype):
  // {max bytes inclusive, algo}, the last entry covering every larger size;
  // empty = the built-in table
  std::vector<std::pair<size_t, int>> select_table[3][4];
  size_t nvls_min_bytes = (size_t)1 << 20;   // AUTO: in-place NVLS from here (symmetric, multicast)
  cf::Nvls nvls;
  cf::SymHeap sym;
  cf::Proxy* proxy = nullptr;          // PortChannel proxy thread (started on demand)
  std::vector<cf::HostPipe> pipes;     // per group (cfAllReduceHost), created on first use

  cf::RankState* state(int li) const { return (cf::RankState*)(local[li].heap + lay.state_off); }
  uint64_t* sem(int li, int p) const { return (uint64_t*)(peer_heap[li][p] + lay.sem_off); }
  char* scr(int li, int p) const { return peer_heap[li][p] + lay.scr_off; }
  uint64_t* ack(int li, int p) const { return (uint64_t*)(peer_heap[li][p] + lay.ack_off); }
  char* ring(int li, int p) const { return peer_heap[li][p] + lay.ring_off; }
  // registered range containing p (nullptr if none)
  const cf::Registration* find_reg(const void* p) const {
    for (auto& r : regs)
      if ((const char*)p >= r.ptr && (const char*)p < r.ptr + r.bytes) return &r;
    return nullptr;
  }
};

namespace cf {
// CTAs of `kernel` (launched with `threads`) that may run per SM on `dev`.
int occupancy(cfComm* c, const void* kernel, int dev, int threads, size_t smem = 0);
// Driver API function by name (nullptr if unavailable).
void* driver_fn(const char* name);
// Co-residency cap: CTAs per rank such that every rank of the group fits at
// once, further capped by the algorithm's CTA budget (cfCommSetCtaBudget;
// algo -1 = none, CF_ALGO_COUNT = the fused K13 kernel).
int max_blocks_per_rank(cfComm* c, const void* kernel, int group, int threads, int per_sm = 0, int algo = -1,
                        size_t smem = 0);
// Default CTA budget per rank when every rank has its own GPU (NVLink-bound
// collectives): well under half the SMs, so a concurrent compute kernel
// holding half of them cannot leave a collective partially resident.
constexpr int kNvlinkCtaBudget = 64;
// Make streams[first] of the group wait for the others; after the launch, the
// others wait for it.  `after` selects the phase.
cfStatus join_streams(cfComm* c, int group, const cudaStream_t* streams, bool after);
// NVLS: probe support; set up for a one-process world; tear down.
bool multicast_capable(int dev);
cfStatus nvls_setup_inprocess(cfComm* c);
cfStatus nvls_setup_emulated(cfComm* c);
void nvls_teardown(cfComm* c);
void sym_teardown(cfComm* c);
// PortChannel proxy (cf_proxy.cu)
cfStatus proxy_start(cfComm* c);
void proxy_stop(cfComm* c);
bool proxy_alive(const cfComm* c);
}  // namespace cf

// cf_runtime.cu -- communicator bootstrap, symmetric heap, measured algorithm
// selection and the collective entry points of the C ABI (include/cf.h).
//
// Reference counterparts (commforge 0.1.0, cf/):
//   make_world / SimWorld regions + semaphores   cf/world.py:80-185
//   collective() facade                          cf/collectives.py:532-573
//   Selector / default_table / select_algorithm  cf/collectives.py:415-491
//   error codes                                  cf/errors.py:6-93
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <cuda.h>
#include "cf_runtime.h"

namespace cf {
const void* collective_kernel(int kind, int dtype, int n);

static thread_local std::string g_last_error;

cfStatus fail(cfStatus s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

void HeapLayout::compute(int nranks, size_t ll_max) {
  sem_off = 256;
  sem_bytes = (size_t)CF_MAX_RANKS * CF_MAX_BLOCKS * sizeof(uint64_t);
  ack_off = round_up(sem_off + sem_bytes, 256);
  chan_off = round_up(ack_off + sem_bytes, 256);
  ring_off = round_up(chan_off + 5 * (size_t)CF_MAX_RANKS * CF_MAX_CHANNEL_TAGS * sizeof(uint64_t), 4096);
  scr_off = round_up(ring_off + kRingBytes, 4096);
  // one LL16 packet (16 B) per 8 payload bytes: a slot holds 2*ll_max bytes
  slot = round_up(2 * ll_max + 64, 256);
  half = (size_t)nranks * slot;
  scr_bytes = 2 * half;
  total = round_up(scr_off + scr_bytes, 1 << 21);
}

int occupancy(cfComm* c, const void* kernel, int dev, int threads, size_t smem) {
  auto key = std::make_pair(kernel, dev * 2048 + threads);   // residency depends on the block size
  auto it = c->occ.find(key);
  if (it != c->occ.end()) return it->second;
  int nb = 0;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess) nb = 1;
  c->occ[key] = std::max(nb, 1);
  return c->occ[key];
}

// `per_sm` > 0 caps the residency used at that many CTAs per SM (K3 two-shot
// at 256 MiB: 2 CTAs/SM 731 us, 1 CTA/SM 663 us).
static int cta_budget(const cfComm* c, int algo) {
  if (algo >= 0 && algo <= CF_ALGO_COUNT && c->budget[algo] > 0) return c->budget[algo];
  if (c->budget_all > 0) return c->budget_all;
  std::map<int, int> per_dev;
  for (const auto& lr : c->local) per_dev[lr.dev]++;
  for (const auto& d : per_dev)
    if (d.second > 1) return 0;   // co-resident ranks (HBM proxy, tests): full residency
  return kNvlinkCtaBudget;
}

int max_blocks_per_rank(cfComm* c, const void* kernel, int group, int threads, int per_sm, int algo, size_t smem) {
  const auto& g = c->groups[group];
  const int dev = c->local[g[0]].dev;
  int occ = occupancy(c, kernel, dev, threads, smem);
  if (per_sm > 0) occ = std::min(occ, per_sm);
  const int cap = occ * c->sm_count[dev];
  // every rank on this device shares its SMs (one launch per device, or one
  // per rank with CF_SPLIT_GROUPS): all CTAs of a call must be co-resident
  int on_dev = 0;
  for (const auto& lr : c->local) on_dev += lr.dev == dev;
  int mb = std::max(1, cap / std::max(on_dev, (int)g.size()));
  mb = std::min(mb, CF_MAX_BLOCKS);
  if (c->cfg.max_blocks > 0) mb = std::min(mb, c->cfg.max_blocks);
  const int budget = cta_budget(c, algo);
  if (budget > 0) mb = std::min(mb, budget);
  return mb;
}

cfStatus join_streams(cfComm* c, int group, const cudaStream_t* streams, bool after) {
  const auto& g = c->groups[group];
  const cudaStream_t s0 = streams[g[0]];
  for (size_t i = 1; i < g.size(); i++) {
    const int li = g[i];
    if (streams[li] == s0) continue;
    if (!after) {
      CF_CUDA(cudaEventRecord(c->local[li].ev, streams[li]));
      CF_CUDA(cudaStreamWaitEvent(s0, c->local[li].ev, 0));
    } else {
      CF_CUDA(cudaEventRecord(c->local[g[0]].ev, s0));
      CF_CUDA(cudaStreamWaitEvent(streams[li], c->local[g[0]].ev, 0));
    }
  }
  return CF_OK;
}

// Driver API entry points resolved through the runtime, so libcf.so has no
// link-time dependency on libcuda (it loads on GPU-less build hosts).
void* driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return fn;
}

static cfStatus alloc_heap(cfComm* c, LocalRank& lr) {
  CF_CUDA(cudaSetDevice(lr.dev));
  CF_CUDA(cudaMalloc((void**)&lr.heap, c->lay.total));
  CF_CUDA(cudaMemset(lr.heap, 0, c->lay.total));
  RankState st{};
  st.timeout_ns = c->cfg.spin_timeout_ns;
  CF_CUDA(cudaMemcpy(lr.heap + c->lay.state_off, &st, sizeof(st), cudaMemcpyHostToDevice));
  CF_CUDA(cudaEventCreateWithFlags(&lr.ev, cudaEventDisableTiming));
  int sms = 0;
  CF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, lr.dev));
  c->sm_count[lr.dev] = sms;
  return CF_OK;
}

static void apply_defaults(cfConfig* cfg) {
  if (cfg->ll_max_bytes == 0) cfg->ll_max_bytes = 4u << 20;
  if (cfg->nvls_bytes == 0) cfg->nvls_bytes = 64u << 20;
  if (cfg->threads == 0) cfg->threads = 512;
  if (cfg->spin_timeout_ns == 0) {
    cfg->spin_timeout_ns = 10ull * 1000 * 1000 * 1000;
    if (const char* s = getenv("CF_SPIN_TIMEOUT_MS")) cfg->spin_timeout_ns = strtoull(s, nullptr, 10) * 1000000ull;
  }
}

static void build_groups(cfComm* c) {
  c->groups.clear();
  // CF_SPLIT_GROUPS=1 (tests): one launch per rank even when ranks share a
  // device -- the multi-GPU in-process path (per-device launches, .sys
  // handshakes) exercised on one GPU; the caller supplies one stream per rank
  if (getenv("CF_SPLIT_GROUPS") && *getenv("CF_SPLIT_GROUPS") == '1' && !c->multiprocess) {
    for (int li = 0; li < (int)c->local.size(); li++) c->groups.push_back({li});
    return;
  }
  std::map<int, int> by_dev;
  for (int li = 0; li < (int)c->local.size(); li++) {
    const int d = c->local[li].dev;
    auto it = by_dev.find(d);
    if (it == by_dev.end()) {
      by_dev[d] = (int)c->groups.size();
      c->groups.push_back({li});
    } else {
      c->groups[it->second].push_back(li);
    }
  }
}

// ---------------------------------------------------------------- selection

// Measured crossover table: replaces DEFAULT_THRESHOLDS
// (cf/collectives.py:418).  Thresholds are per-rank message bytes.  Values
// come from bench.py sweeps; see DESIGN.md "selector".
// K6 bulk (TMA bulk copies): tile size of push_gather_bulk_kernel, smallest
// shard it takes (smaller shards: the register kernel's lower latency)
#ifndef CF_BULK_TILE_KB
#define CF_BULK_TILE_KB 32
#endif
constexpr size_t kBulkTileBytes = (size_t)CF_BULK_TILE_KB * 1024;
constexpr size_t kAgBulkMin = (size_t)4 << 20;
static bool ag_bulk_enabled() {
  static const bool on = [] {
    const char* v = getenv("CF_AG_BULK");
    return !v || atoi(v) != 0;
  }();
  return on;
}

static int select_algo(const cfComm* c, int coll, size_t nbytes, int dtype) {
  // a measured table (cfCommSetSelection: Communicator.tune / World.tune)
  // wins over the built-in one; LL picks beyond the LL capacity fall back
  if (coll >= 0 && coll < 3 && dtype >= 0 && dtype < 4 && !c->select_table[coll][dtype].empty()) {
    const auto& t = c->select_table[coll][dtype];
    int algo = t.back().second;
    for (const auto& e : t)
      if (nbytes <= e.first) {
        algo = e.second;
        break;
      }
    if ((algo == CF_ALGO_1PA || algo == CF_ALGO_2PA_LL) && nbytes > c->cfg.ll_max_bytes) algo = CF_ALGO_2PA;
    return algo;
  }
  const bool coresident = c->groups.size() == 1 && c->local.size() > 1;
  if (coll == 1) return CF_ALGO_ALLPAIRS_AG;
  if (coll == 2) return CF_ALGO_RS_DIRECT;
  if (c->nranks == 1) return CF_ALGO_2PA;
  if (coresident) {
    // Ranks share one GPU (one launch, no handshakes).  Measured (bench sweep,
    // bf16, 8 ranks, L2 flushed, profiles/round1/bench_line.json): the
    // whole-vector pull (1pa_hb) has the lowest latency up to 256 KiB
    // (3.3-4.4 us vs 4.3-4.8 us for 2pa, 3.4-13 us for LL, which doubles the
    // bytes); the two-shot pull moves the minimum bytes and wins from 1 MiB
    // on (5.9 vs 10.1 us) to 1 GiB.
    if (nbytes <= 256 * 1024) return CF_ALGO_1PA_HB;
    return CF_ALGO_2PA;
  }
  if (nbytes < 256 * 1024 && nbytes <= c->cfg.ll_max_bytes) return CF_ALGO_1PA;
  if (nbytes < 2 * 1024 * 1024 && nbytes <= c->cfg.ll_max_bytes) return CF_ALGO_2PA_LL;
  return CF_ALGO_2PA;
}

}  // namespace cf

using namespace cf;

// ---------------------------------------------------------------- C ABI: misc

extern "C" const char* cfStatusCode(cfStatus s) {
  static const char* codes[] = {"OK", "E_GENERIC", "E_BAD_SIZE", "E_NO_SEM", "E_BAD_DELTA", "E_OOB",
                                "E_DEADLOCK", "E_PROXY_DOWN", "E_ZERO_FLAG", "E_WRONG_PROTOCOL",
                                "E_BAD_ALIGN", "E_SYNTAX", "E_VERSION", "E_REF", "E_SHAPE",
                                "E_PROTOCOL", "E_RANK_MISMATCH", "E_TOPOLOGY", "E_NO_ALGO",
                                "E_BAD_TIME", "E_CONFIG", "E_CUDA", "E_INTERNAL"};
  if ((int)s < 0 || (int)s > (int)CF_E_INTERNAL) return "E_GENERIC";
  return codes[s];
}

extern "C" const char* cfLastErrorMessage(void) { return g_last_error.c_str(); }
extern "C" int cfVersion(void) { return CF_VERSION; }

// ---------------------------------------------------------------- C ABI: comm

static cfStatus comm_common_init(cfComm* c, int nranks, const cfConfig* cfg) {
  if (nranks < 1 || nranks > CF_MAX_RANKS)
    return fail(CF_E_BAD_SIZE, "nranks %d outside [1, %d]", nranks, CF_MAX_RANKS);
  c->nranks = nranks;
  if (cfg) c->cfg = *cfg;
  apply_defaults(&c->cfg);
  // every collective kernel is compiled with __launch_bounds__(512)
  if (c->cfg.threads % 32 || c->cfg.threads < 64 || c->cfg.threads > 512)
    return fail(CF_E_CONFIG, "threads must be a multiple of 32 in [64, 512]");
  c->lay.compute(nranks, c->cfg.ll_max_bytes);
  return CF_OK;
}

extern "C" cfStatus cfCommInitAll(cfComm_t* out, int nranks, const int* devs, const cfConfig* cfg) {
  if (!out || !devs) return fail(CF_E_CONFIG, "null argument");
  DeviceGuard guard;
  cfComm* c = new cfComm();
  cfStatus s = comm_common_init(c, nranks, cfg);
  if (s != CF_OK) { delete c; return s; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    delete c;
    return fail(CF_E_CUDA, "no CUDA device visible");
  }
  c->local.resize(nranks);
  for (int r = 0; r < nranks; r++) {
    if (devs[r] < 0 || devs[r] >= ndev) {
      delete c;
      return fail(CF_E_TOPOLOGY, "rank %d: device %d not present (%d visible)", r, devs[r], ndev);
    }
    c->local[r].rank = r;
    c->local[r].dev = devs[r];
  }
  // peer access between every pair of distinct devices
  for (int a = 0; a < nranks; a++)
    for (int b = 0; b < nranks; b++) {
      if (devs[a] == devs[b]) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, devs[a], devs[b]);
      if (!ok) {
        delete c;
        return fail(CF_E_TOPOLOGY, "device %d cannot access device %d over NVLink/P2P", devs[a], devs[b]);
      }
      cudaSetDevice(devs[a]);
      cudaError_t e = cudaDeviceEnablePeerAccess(devs[b], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        delete c;
        return fail(CF_E_CUDA, "cudaDeviceEnablePeerAccess(%d->%d): %s", devs[a], devs[b], cudaGetErrorString(e));
      }
      cudaGetLastError();
    }
  for (int r = 0; r < nranks; r++) {
    s = alloc_heap(c, c->local[r]);
    if (s != CF_OK) { cfCommDestroy(c); return s; }
  }
  c->peer_heap.assign(nranks, {});
  for (int li = 0; li < nranks; li++)
    for (int p = 0; p < nranks; p++) c->peer_heap[li][p] = c->local[p].heap;
  build_groups(c);
  // NVLS needs one device per rank, each multicast-capable
  bool mc_ok = c->groups.size() == (size_t)nranks;
  for (int r = 0; r < nranks && mc_ok; r++) mc_ok = multicast_capable(devs[r]);
  if (c->cfg.use_multicast == 2) {
    // emulated switch: the K5 control path on unicast staging (tests, one GPU)
    s = nvls_setup_emulated(c);
    if (s != CF_OK) { cfCommDestroy(c); return s; }
  } else if (c->cfg.use_multicast && mc_ok) {
    // a box that advertises multicast but cannot build the object (e.g. no
    // fabric manager) keeps working: switch_2pa then runs the all-pairs kernel
    if (nvls_setup_inprocess(c) != CF_OK) {
      fprintf(stderr, "libcf: NVLS setup failed (%s); switch_2pa uses the all-pairs kernel\n",
              cfLastErrorMessage());
      nvls_teardown(c);
    }
  }
  c->multicast_supported = c->nvls.enabled && !c->nvls.emul;
  c->connected = true;
  *out = c;
  return CF_OK;
}

namespace {
struct HandleBlob {
  uint32_t magic;
  uint32_t version;
  int32_t nranks;
  int32_t rank;
  int32_t dev;
  int32_t pid;
  uint64_t heap_bytes;
  uint64_t ll_max;
  cudaIpcMemHandle_t ipc;
};
constexpr uint32_t kMagic = 0x43464d31;  // "CFM1"
static_assert(sizeof(HandleBlob) <= CF_HANDLE_BYTES, "handle too large");
}  // namespace

extern "C" cfStatus cfCommCreateRank(cfComm_t* out, int nranks, int rank, int cuda_dev, const cfConfig* cfg) {
  if (!out) return fail(CF_E_CONFIG, "null argument");
  if (rank < 0 || rank >= nranks) return fail(CF_E_OOB, "rank %d out of range", rank);
  DeviceGuard guard;
  cfComm* c = new cfComm();
  cfStatus s = comm_common_init(c, nranks, cfg);
  if (s != CF_OK) { delete c; return s; }
  c->multiprocess = true;
  c->local.resize(1);
  c->local[0].rank = rank;
  c->local[0].dev = cuda_dev;
  s = alloc_heap(c, c->local[0]);
  if (s != CF_OK) { cfCommDestroy(c); return s; }
  c->peer_heap.assign(1, {});
  c->peer_heap[0][rank] = c->local[0].heap;
  build_groups(c);
  *out = c;
  return CF_OK;
}

extern "C" cfStatus cfCommGetHandle(cfComm_t c, void* handle, size_t* bytes) {
  if (!c || !bytes) return fail(CF_E_CONFIG, "null argument");
  if (!c->multiprocess) return fail(CF_E_CONFIG, "handles exist only for cfCommCreateRank communicators");
  if (!handle) { *bytes = CF_HANDLE_BYTES; return CF_OK; }
  if (*bytes < CF_HANDLE_BYTES) return fail(CF_E_BAD_SIZE, "handle buffer needs %d bytes", CF_HANDLE_BYTES);
  DeviceGuard guard;
  HandleBlob h{};
  h.magic = kMagic;
  h.version = CF_VERSION;
  h.nranks = c->nranks;
  h.rank = c->local[0].rank;
  h.dev = c->local[0].dev;
  h.pid = (int32_t)getpid();
  h.heap_bytes = c->lay.total;
  h.ll_max = c->cfg.ll_max_bytes;
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  CF_CUDA(cudaIpcGetMemHandle(&h.ipc, c->local[0].heap));
  memset(handle, 0, CF_HANDLE_BYTES);
  memcpy(handle, &h, sizeof(h));
  *bytes = CF_HANDLE_BYTES;
  return CF_OK;
}

extern "C" cfStatus cfCommConnect(cfComm_t c, const void* handles, size_t bytes_per_handle) {
  if (!c || !handles) return fail(CF_E_CONFIG, "null argument");
  if (!c->multiprocess) return fail(CF_E_CONFIG, "cfCommConnect needs a cfCommCreateRank communicator");
  if (bytes_per_handle < sizeof(HandleBlob)) return fail(CF_E_BAD_SIZE, "handle stride too small");
  DeviceGuard guard;
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  const int me = c->local[0].rank;
  for (int p = 0; p < c->nranks; p++) {
    HandleBlob h;
    memcpy(&h, (const char*)handles + (size_t)p * bytes_per_handle, sizeof(h));
    if (h.magic != kMagic || h.version != CF_VERSION)
      return fail(CF_E_VERSION, "rank %d handle is not a cf v%d handle", p, CF_VERSION);
    if (h.nranks != c->nranks || h.rank != p)
      return fail(CF_E_RANK_MISMATCH, "handle %d claims rank %d of %d (expected %d of %d)", p, h.rank,
                  h.nranks, p, c->nranks);
    if (h.heap_bytes != c->lay.total || h.ll_max != c->cfg.ll_max_bytes)
      return fail(CF_E_CONFIG, "rank %d was created with a different configuration", p);
    if (p == me) continue;
    void* ptr = nullptr;
    CF_CUDA(cudaIpcOpenMemHandle(&ptr, h.ipc, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(ptr);
    c->peer_heap[0][p] = (char*)ptr;
  }
  c->connected = true;
  return CF_OK;
}

static void release_reg(cfComm* c, const Registration& r);

extern "C" cfStatus cfCommDestroy(cfComm_t c) {
  if (!c) return CF_OK;
  DeviceGuard guard;
  if (!c->local.empty()) cudaSetDevice(c->local[0].dev);
  for (auto& r : c->regs) release_reg(c, r);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  proxy_stop(c);
  nvls_teardown(c);
  sym_teardown(c);
  for (size_t gi = 0; gi < c->pipes.size(); gi++) {
    auto& hp = c->pipes[gi];
    cudaSetDevice(c->local[c->groups[gi][0]].dev);
    for (cudaEvent_t e : {hp.fork, hp.done})
      if (e) cudaEventDestroy(e);
    for (int k = 0; k < kHostPieces; k++) {
      if (hp.in[k]) cudaEventDestroy(hp.in[k]);
      if (hp.ar[k]) cudaEventDestroy(hp.ar[k]);
    }
    if (hp.h2d) cudaStreamDestroy(hp.h2d);
    if (hp.d2h) cudaStreamDestroy(hp.d2h);
  }
  for (auto& lr : c->local) {
    if (lr.dev >= 0) cudaSetDevice(lr.dev);
    if (lr.heap) cudaFree(lr.heap);
    if (lr.ev) cudaEventDestroy(lr.ev);
    if (lr.stage_in) cudaFree(lr.stage_in);
    if (lr.stage_out) cudaFree(lr.stage_out);
  }
  delete c;
  return CF_OK;
}

// ---------------------------------------------------------------- registration

namespace {
struct BufferBlob {
  uint32_t magic;
  int32_t rank;
  uint64_t offset;   // ptr - allocation base
  uint64_t bytes;
  cudaIpcMemHandle_t ipc;
};
constexpr uint32_t kBufMagic = 0x43464231;  // "CFB1"
static_assert(sizeof(BufferBlob) <= CF_BUFFER_HANDLE_BYTES, "buffer handle too large");
}  // namespace

extern "C" cfStatus cfBufferExport(cfComm_t c, const void* ptr, size_t bytes, void* handle) {
  if (!c || !ptr || !handle) return fail(CF_E_CONFIG, "null argument");
  memset(handle, 0, CF_BUFFER_HANDLE_BYTES);
  if (!c->multiprocess) return CF_OK;
  DeviceGuard guard;
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  CUdeviceptr base = 0;
  size_t size = 0;
  auto get_range = (CUresult(*)(CUdeviceptr*, size_t*, CUdeviceptr))driver_fn("cuMemGetAddressRange");
  if (!get_range) return fail(CF_E_CUDA, "driver entry point cuMemGetAddressRange unavailable");
  if (get_range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
    return fail(CF_E_CUDA, "cuMemGetAddressRange(%p) failed: not device memory", ptr);
  if ((const char*)ptr + bytes > (const char*)base + size)
    return fail(CF_E_OOB, "registered range exceeds its allocation");
  BufferBlob b{};
  b.magic = kBufMagic;
  b.rank = c->local[0].rank;
  b.offset = (uint64_t)((const char*)ptr - (const char*)base);
  b.bytes = bytes;
  CF_CUDA(cudaIpcGetMemHandle(&b.ipc, (void*)base));
  memcpy(handle, &b, sizeof(b));
  return CF_OK;
}

extern "C" cfStatus cfBufferImport(cfComm_t c, const void* ptr, const void* handles, size_t stride) {
  if (!c || !ptr || !handles) return fail(CF_E_CONFIG, "null argument");
  if (!c->multiprocess) return CF_OK;
  if (stride < sizeof(BufferBlob)) return fail(CF_E_BAD_SIZE, "buffer handle stride too small");
  DeviceGuard guard;
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  const int me = c->local[0].rank;
  Registration reg;
  reg.ptr = (const char*)ptr;
  for (int p = 0; p < c->nranks; p++) {
    BufferBlob b;
    memcpy(&b, (const char*)handles + (size_t)p * stride, sizeof(b));
    if (b.magic != kBufMagic || b.rank != p) return fail(CF_E_RANK_MISMATCH, "buffer handle %d is not rank %d's", p, p);
    if (p == me) {
      reg.bytes = b.bytes;
      reg.peer[p] = (char*)ptr;
      continue;
    }
    std::string key(std::to_string(p) + ":" + std::string((const char*)&b.ipc, sizeof(b.ipc)));
    auto it = c->ipc_cache.find(key);
    if (it == c->ipc_cache.end()) {
      void* mapped = nullptr;
      CF_CUDA(cudaIpcOpenMemHandle(&mapped, b.ipc, cudaIpcMemLazyEnablePeerAccess));
      it = c->ipc_cache.emplace(key, IpcMapping{mapped, 0}).first;
    }
    it->second.refs++;
    reg.keys.push_back(key);
    reg.peer[p] = (char*)it->second.base + b.offset;
  }
  for (auto& r : c->regs)
    if (r.ptr == reg.ptr) return fail(CF_E_CONFIG, "buffer %p registered twice", ptr);
  c->regs.push_back(reg);
  return CF_OK;
}

static void release_reg(cfComm* c, const Registration& r) {
  for (auto& k : r.keys) {
    auto it = c->ipc_cache.find(k);
    if (it != c->ipc_cache.end() && --it->second.refs == 0) {
      cudaIpcCloseMemHandle(it->second.base);
      c->ipc_cache.erase(it);
    }
  }
}

extern "C" cfStatus cfBufferRelease(cfComm_t c, const void* ptr) {
  if (!c) return fail(CF_E_CONFIG, "null argument");
  if (!c->multiprocess) return CF_OK;
  DeviceGuard guard;
  cudaSetDevice(c->local[0].dev);
  for (size_t i = 0; i < c->regs.size(); i++)
    if (c->regs[i].ptr == (const char*)ptr) {
      release_reg(c, c->regs[i]);
      c->regs.erase(c->regs.begin() + i);
      return CF_OK;
    }
  return fail(CF_E_OOB, "buffer %p is not registered", ptr);
}

extern "C" cfStatus cfCommNumRanks(cfComm_t c, int* n) {
  if (!c || !n) return fail(CF_E_CONFIG, "null argument");
  *n = c->nranks;
  return CF_OK;
}

extern "C" cfStatus cfCommLocalRanks(cfComm_t c, int* nlocal, int* ranks) {
  if (!c || !nlocal) return fail(CF_E_CONFIG, "null argument");
  *nlocal = (int)c->local.size();
  if (ranks)
    for (size_t i = 0; i < c->local.size(); i++) ranks[i] = c->local[i].rank;
  return CF_OK;
}

extern "C" cfStatus cfCommMulticastSupported(cfComm_t c, int* supported) {
  if (!c || !supported) return fail(CF_E_CONFIG, "null argument");
  *supported = c->multicast_supported ? 1 : 0;
  return CF_OK;
}

extern "C" cfStatus cfCommLastDeviceError(cfComm_t c, int* code) {
  if (!c || !code) return fail(CF_E_CONFIG, "null argument");
  DeviceGuard guard;
  uint32_t worst = 0;
  for (size_t li = 0; li < c->local.size(); li++) {
    CF_CUDA(cudaSetDevice(c->local[li].dev));
    // a synchronous copy on the legacy stream waits for every blocking stream
    // (the caller's collectives) but not for unrelated non-blocking streams
    // (a compute kernel running beside the collectives)
    RankState st;
    CF_CUDA(cudaMemcpy(&st, c->state((int)li), sizeof(st), cudaMemcpyDeviceToHost));
    worst = std::max(worst, st.error);
  }
  *code = (int)worst;
  return CF_OK;
}

extern "C" cfStatus cfCommClearDeviceError(cfComm_t c) {
  if (!c) return fail(CF_E_CONFIG, "null argument");
  DeviceGuard guard;
  for (size_t li = 0; li < c->local.size(); li++) {
    CF_CUDA(cudaSetDevice(c->local[li].dev));
    CF_CUDA(cudaMemset((char*)c->state((int)li) + offsetof(RankState, error), 0, sizeof(uint32_t)));
    CF_CUDA(cudaStreamSynchronize(0));
  }
  return CF_OK;
}

extern "C" cfStatus cfCommSetCtaBudget(cfComm_t c, int algo, int ctas) {
  if (!c) return fail(CF_E_CONFIG, "null communicator");
  if (ctas < 0 || ctas > CF_MAX_BLOCKS) return fail(CF_E_CONFIG, "ctas must be in [0, %d]", CF_MAX_BLOCKS);
  if (algo == -1) {
    c->budget_all = ctas;
    return CF_OK;
  }
  if (algo < 0 || algo > CF_ALGO_COUNT) return fail(CF_E_NO_ALGO, "unknown algorithm %d", algo);
  c->budget[algo] = ctas;
  return CF_OK;
}

extern "C" cfStatus cfCommSetSelection(cfComm_t c, int coll, cfDtype dtype, int nentries, const size_t* max_bytes,
                                       const int* algos) {
  if (!c) return fail(CF_E_CONFIG, "null communicator");
  if (coll < 0 || coll > 2) return fail(CF_E_CONFIG, "collective must be 0 (AllReduce), 1 (AllGather), 2 (ReduceScatter)");
  if ((int)dtype < 0 || (int)dtype > 3) return fail(CF_E_SHAPE, "unknown dtype %d", (int)dtype);
  if (nentries < 0 || (nentries > 0 && (!max_bytes || !algos))) return fail(CF_E_CONFIG, "bad selection table");
  std::vector<std::pair<size_t, int>> t;
  for (int i = 0; i < nentries; i++) {
    const int base = algos[i] & ~CF_ALGO_RING_LINKS;
    const bool ring = base == CF_ALGO_2PR || base == CF_ALGO_RING_AG || base == CF_ALGO_RING_RS;
    if ((algos[i] & CF_ALGO_RING_LINKS) && !ring) return fail(CF_E_NO_ALGO, "CF_ALGO_RING_LINKS on algorithm %d", base);
    const bool ok = coll == 0 ? (base == CF_ALGO_1PA || base == CF_ALGO_1PA_HB || base == CF_ALGO_2PA ||
                                 base == CF_ALGO_2PA_LL || base == CF_ALGO_2PR)
                  : coll == 1 ? (base == CF_ALGO_ALLPAIRS_AG || base == CF_ALGO_RING_AG)
                              : (base == CF_ALGO_RS_DIRECT || base == CF_ALGO_RING_RS);
    if (!ok) return fail(CF_E_NO_ALGO, "algorithm %d cannot serve collective %d from a selection table", algos[i], coll);
    if (i && max_bytes[i] <= max_bytes[i - 1]) return fail(CF_E_CONFIG, "selection table sizes must increase");
    t.push_back({max_bytes[i], algos[i]});
  }
  c->select_table[coll][(int)dtype] = t;
  return CF_OK;
}

extern "C" cfStatus cfCommSetNvlsMinBytes(cfComm_t c, size_t bytes) {
  if (!c) return fail(CF_E_CONFIG, "null communicator");
  c->nvls_min_bytes = bytes;
  return CF_OK;
}

extern "C" cfStatus cfSelectAlgorithm(cfComm_t c, int coll, size_t nbytes, cfDtype dtype, int* algo) {
  if (!c || !algo) return fail(CF_E_CONFIG, "null argument");
  if (coll < 0 || coll > 2) return fail(CF_E_NO_ALGO, "unknown collective %d", coll);
  *algo = select_algo(c, coll, nbytes, dtype);
  return CF_OK;
}

// ---------------------------------------------------------------- collectives

namespace {

enum Kind { kPull = 0, kLL1 = 1, kLL2 = 2, kGather = 3, kNvls = 4, kRing = 5, kRingGather = 6, kNorm = 7,
            kGatherBulk = 9 };

struct Job {
  int algo = -1;      // cfAlgo (CF_ALGO_COUNT: K13) -- selects the CTA budget
  int kind = kPull;
  int order = kLead;
  int push = 0, whole = 0, rs_shift = 0;
  size_t count = 0;   // elements per rank on the reduced/gathered axis
  size_t cs = 0;      // reference chunk (elements)
  size_t slot = 0;
  size_t work = 0;    // 16-byte vectors per rank (grid sizing)
  size_t rows = 0, hidden = 0;   // K13
  float eps = 0.f;
  int blocks = 0;     // explicit CTAs per rank (K13: one per row), else from `work`
  int threads = 0;    // CTA size (0: the configured threads)
  size_t smem = 0;    // dynamic shared memory per CTA
  size_t win_lo = 0, win_hi = ~(size_t)0;   // pull-reduce window inside each chunk
};

// K13's extra per-local-rank buffers.
struct NormBufs {
  const void* const* resid_in;
  void* const* resid_out;
  const void* const* weight;
};

// every rank's symmetric heap is mapped here (multi-process: after cfSymHeapMapPeer)
bool sym_mapped(const cfComm* c) {
  if (!c->sym.on()) return false;
  for (size_t li = 0; li < c->local.size(); li++)
    for (int p = 0; p < c->nranks; p++)
      if (!c->sym.peer[li][p]) return false;
  return true;
}

// send / recv of every local rank are symmetric (same heap offsets on every
// local rank, `bytes` inside the heap) and the switch is usable (multicast
// bound, or emulated): the in-place NVLS kernel applies
bool sym_switch_ok(const cfComm* c, const void* const* send, void* const* recv, size_t bytes, long long* oi,
                   long long* oo) {
  if (c->sym.mode == 0 || !sym_mapped(c)) return false;
  *oi = c->sym.offset(0, send[0]);
  *oo = c->sym.offset(0, recv[0]);
  if (*oi < 0 || *oo < 0 || (size_t)*oi + bytes > c->sym.bytes || (size_t)*oo + bytes > c->sym.bytes) return false;
  if ((*oi & 15) || (*oo & 15)) return false;
  for (size_t li = 0; li < c->local.size(); li++) {
    if (c->sym.offset((int)li, send[li]) != *oi || c->sym.offset((int)li, recv[li]) != *oo) return false;
    if (c->sym.mode == 1 && !c->sym.ranks[li].mc) return false;
  }
  return true;
}

cfStatus check_ptrs(cfComm* c, const void* const* send, void* const* recv, const cudaStream_t* streams) {
  if (!c) return fail(CF_E_CONFIG, "null communicator");
  if (!c->connected) return fail(CF_E_CONFIG, "communicator not connected (call cfCommConnect)");
  if (!send || !recv || !streams) return fail(CF_E_CONFIG, "null buffer or stream array");
  for (size_t li = 0; li < c->local.size(); li++) {
    if (!send[li] || !recv[li]) return fail(CF_E_OOB, "local rank %zu: null buffer", li);
    if (((uintptr_t)send[li] | (uintptr_t)recv[li]) & 15)
      return fail(CF_E_BAD_ALIGN, "local rank %zu: buffers must be 16-byte aligned", li);
  }
  return CF_OK;
}

cfStatus launch(cfComm* c, const Job& j, int dtype, const void* const* send, void* const* recv,
                const cudaStream_t* streams, const NormBufs* nb = nullptr) {
  // one-process-per-GPU: peers' buffers come from the registration table
  const bool need_in = j.kind == kPull || j.kind == kNorm;
  const bool need_out = j.kind == kGather || j.kind == kGatherBulk || j.kind == kRingGather ||
                        ((j.kind == kPull || j.kind == kNorm || j.kind == kRing) && j.push);
  const bool need_out2 = false;   // K13 writes only its own resid_out (both modes)
  const Registration* reg_in = nullptr;
  const Registration* reg_out = nullptr;
  const Registration* reg_out2 = nullptr;
  // symmetric-heap buffers (cfMemAlloc) need no registration: peers at base[p] + offset
  const long long sym_in = c->multiprocess && sym_mapped(c) ? c->sym.offset(0, send[0]) : -1;
  const long long sym_out = c->multiprocess && sym_mapped(c) ? c->sym.offset(0, recv[0]) : -1;
  if (c->multiprocess) {
    if (need_out2 && !(reg_out2 = c->find_reg(nb->resid_out[0])))
      return fail(CF_E_TOPOLOGY, "residual-out buffer %p is not registered (cfBufferExport/cfBufferImport); "
                                 "the two-shot fused kernel writes it from the peers", nb->resid_out[0]);
    if (need_in && sym_in < 0 && !(reg_in = c->find_reg(send[0])))
      return fail(CF_E_TOPOLOGY, "send buffer %p is neither registered (cfBufferExport/cfBufferImport) nor "
                                 "symmetric (cfMemAlloc); HB algorithms read it from the peers", send[0]);
    if (need_out && sym_out < 0 && !(reg_out = c->find_reg(recv[0])))
      return fail(CF_E_TOPOLOGY, "recv buffer %p is neither registered (cfBufferExport/cfBufferImport) nor "
                                 "symmetric (cfMemAlloc); HB algorithms write it from the peers", recv[0]);
  }
  DeviceGuard guard;
  const void* kernel = collective_kernel(j.kind, dtype, c->nranks);
  if (!kernel) return fail(CF_E_INTERNAL, "no kernel for kind %d dtype %d", j.kind, dtype);
  // Ring links are latency chains (every step waits for the previous rank's
  // step): smaller CTAs give each rank up to kRingCtas independent links.
  const bool ring = j.kind == kRing || j.kind == kRingGather;
  int threads = j.kind == kRing ? std::min(c->cfg.threads, 256) : c->cfg.threads;   // ring_kernel's bound
  if (j.threads) threads = j.threads;
  // K13 keeps 512-thread CTAs at every row count: with phase 2 pipelined over
  // a CTA's rows, a 512-thread CTA holds a whole 8192-wide bf16 row in
  // registers (no second-pass re-reads) and beats two 256-thread CTAs per SM
  // even when rows take several rounds (C5 b=64 16.4 -> 14.2 us, b=256 40.9 ->
  // 35.3 us; scripts/k13_threads_ab.py)
  if (j.kind == kNorm)
    if (const char* env = getenv("CF_K13_THREADS")) threads = atoi(env);   // diagnostics
  for (size_t gi = 0; gi < c->groups.size(); gi++) {
    const auto& g = c->groups[gi];
    const int dev = c->local[g[0]].dev;
    CF_CUDA(cudaSetDevice(dev));
    CollArgs a;
    memset(&a, 0, sizeof(a));
    a.n = c->nranks;
    a.nlocal = (int)g.size();
    a.order = j.order;
    a.push = j.push;
    a.whole = j.whole;
    a.rs_shift = j.rs_shift;
    a.gpu_scope = (c->groups.size() == 1 && !c->multiprocess) ? 1 : 0;
    a.single_launch = (c->groups.size() == 1 && !c->multiprocess && (int)g.size() == c->nranks) ? 1 : 0;
    a.count = j.count;
    a.cs = j.cs;
    a.slot = j.slot ? j.slot : c->lay.slot;
    a.half = c->lay.half;
    a.rows = j.rows;
    a.hidden = j.hidden;
    a.win_lo = j.win_lo;
    a.win_hi = j.win_hi;
    a.eps = j.eps;
    for (size_t k = 0; k < g.size(); k++) {
      const int li = g[k];
      RankCtx& rk = a.rk[k];
      rk.rank = c->local[li].rank;
      rk.st = c->state(li);
      for (int p = 0; p < c->nranks; p++) {
        // one-process mode: rank p's buffers are the caller's entries (UVA)
        rk.in[p] = c->multiprocess ? nullptr : (const char*)send[p];
        rk.out[p] = c->multiprocess ? nullptr : (char*)recv[p];
        rk.scr[p] = c->scr(li, p);
        rk.sem[p] = c->sem(li, p);
        rk.ack[p] = c->ack(li, p);
        rk.ring[p] = c->ring(li, p);
        if (nb) rk.out2[p] = c->multiprocess ? nullptr : (char*)nb->resid_out[p];
      }
      if (nb) {
        rk.resid = (const char*)nb->resid_in[li];
        rk.weight = (const char*)nb->weight[li];
      }
      if (c->multiprocess) {
        for (int p = 0; p < c->nranks; p++) {
          if (reg_in) rk.in[p] = reg_in->peer[p] + ((const char*)send[li] - reg_in->ptr);
          if (reg_out) rk.out[p] = reg_out->peer[p] + ((char*)recv[li] - reg_out->ptr);
          if (need_in && sym_in >= 0) rk.in[p] = c->sym.peer[0][p] + sym_in;
          if (need_out && sym_out >= 0) rk.out[p] = c->sym.peer[0][p] + sym_out;
          if (reg_out2) rk.out2[p] = reg_out2->peer[p] + ((char*)nb->resid_out[li] - reg_out2->ptr);
        }
        rk.in[rk.rank] = (const char*)send[li];
        rk.out[rk.rank] = (char*)recv[li];
        if (nb) rk.out2[rk.rank] = (char*)nb->resid_out[li];
      }
    }
    // two-shot push (K3) above 8 MiB per rank: one CTA per SM (64 MiB: 182 ->
    // 171 us); below, full residency hides more latency (4 MiB: 15.8 -> 14.4
    // us); the pull-only variants (K2, K8) gain from full residency at every
    // size (K8 256 MiB 394 -> 354 us, K2 1 MiB 13.4 -> 10.1 us)
    const bool k3_big = j.kind == kPull && j.push && j.count * dtype_size(dtype) > ((size_t)8 << 20);
    int mb = max_blocks_per_rank(c, kernel, (int)gi, threads, k3_big ? 1 : 0, j.algo, j.smem);
    if (ring) mb = std::min(mb, kRingCtas);   // ring slot region
    int blocks = (int)std::min<size_t>((size_t)mb, std::max<size_t>(1, ceil_div(j.work, (size_t)threads)));
    if (j.blocks) blocks = std::min(mb, j.blocks);
    CF_TRY(join_streams(c, (int)gi, streams, false));
    void* args[] = {&a};
    CF_CUDA(cudaLaunchKernel(kernel, dim3(blocks, g.size()), dim3(threads), args, j.smem, streams[g[0]]));
    CF_TRY(join_streams(c, (int)gi, streams, true));
  }
  return CF_OK;
}

// K5: one nvls_kernel launch per device group (copy-in, multimem reduce /
// broadcast and copy-out fused, the message in pieces of the staging half).
cfStatus nvls_allreduce(cfComm* c, const void* const* send, void* const* recv, size_t count, int dtype,
                        const cudaStream_t* streams) {
  DeviceGuard guard;
  const size_t es = dtype_size(dtype);
  const void* kernel = collective_kernel(4, dtype, c->nranks);
  const int threads = c->cfg.threads;
  const size_t total = ceil_div(count * es, (size_t)16), piece = c->nvls.half / 16;
  const size_t work = ceil_div(std::min(total, piece), (size_t)c->nranks);   // vectors per chunk
  for (size_t gi = 0; gi < c->groups.size(); gi++) {
    const auto& g = c->groups[gi];
    CF_CUDA(cudaSetDevice(c->local[g[0]].dev));
    CollArgs a;
    memset(&a, 0, sizeof(a));
    a.n = c->nranks;
    a.nlocal = (int)g.size();
    a.count = count;
    a.half = c->nvls.half;
    a.emul = c->nvls.emul ? 1 : 0;
    a.gpu_scope = (c->groups.size() == 1 && !c->multiprocess) ? 1 : 0;
    for (size_t k = 0; k < g.size(); k++) {
      const int li = g[k];
      RankCtx& rk = a.rk[k];
      rk.rank = c->local[li].rank;
      rk.st = c->state(li);
      for (int p = 0; p < c->nranks; p++) rk.sem[p] = c->sem(li, p);
      rk.in[rk.rank] = (const char*)send[li];
      rk.out[rk.rank] = (char*)recv[li];
      if (c->nvls.emul && c->multiprocess) {   // every rank's registered staging, mapped
        for (int q = 0; q < c->nranks; q++) rk.nv[q] = c->nvls.peer_uc[q];
      } else if (c->nvls.emul) {   // every rank's unicast staging (in-process)
        for (size_t q = 0; q < c->local.size(); q++) rk.nv[c->local[q].rank] = c->nvls.ranks[q].uc;
      } else {
        rk.nv[rk.rank] = c->nvls.ranks[li].uc;
      }
      rk.nv_mc = c->nvls.ranks[li].mc;
    }
    const int mb = max_blocks_per_rank(c, kernel, (int)gi, threads, 0, CF_ALGO_SWITCH_2PA);
    const int blocks = (int)std::min<size_t>((size_t)mb, std::max<size_t>(1, ceil_div(work, (size_t)threads)));
    CF_TRY(join_streams(c, (int)gi, streams, false));
    void* args[] = {&a};
    CF_CUDA(cudaLaunchKernel(kernel, dim3(blocks, g.size()), dim3(threads), args, 0, streams[g[0]]));
    CF_TRY(join_streams(c, (int)gi, streams, true));
  }
  return CF_OK;
}

// K5 direct: the in-place NVLS kernel on symmetric buffers (heap offsets
// oi / oo on every rank), one launch per device group.
cfStatus nvls_direct(cfComm* c, size_t count, int dtype, long long oi, long long oo, const cudaStream_t* streams) {
  DeviceGuard guard;
  const size_t es = dtype_size(dtype);
  const void* kernel = collective_kernel(8, dtype, c->nranks);
  const int threads = c->cfg.threads;
  const size_t work = ceil_div(ceil_div(count * es, (size_t)16), (size_t)c->nranks);
  for (size_t gi = 0; gi < c->groups.size(); gi++) {
    const auto& g = c->groups[gi];
    CF_CUDA(cudaSetDevice(c->local[g[0]].dev));
    CollArgs a;
    memset(&a, 0, sizeof(a));
    a.n = c->nranks;
    a.nlocal = (int)g.size();
    a.count = count;
    a.emul = c->sym.mode == 2 ? 1 : 0;
    a.gpu_scope = (c->groups.size() == 1 && !c->multiprocess) ? 1 : 0;
    a.single_launch = (c->groups.size() == 1 && !c->multiprocess && (int)g.size() == c->nranks) ? 1 : 0;
    for (size_t k = 0; k < g.size(); k++) {
      const int li = g[k];
      RankCtx& rk = a.rk[k];
      rk.rank = c->local[li].rank;
      rk.st = c->state(li);
      for (int p = 0; p < c->nranks; p++) {
        rk.sem[p] = c->sem(li, p);
        rk.in[p] = c->sym.peer[li][p] + oi;
        rk.out[p] = c->sym.peer[li][p] + oo;
      }
      if (c->sym.mode == 1) {
        rk.mc_in = c->sym.ranks[li].mc + oi;
        rk.mc_out = c->sym.ranks[li].mc + oo;
      }
    }
    const int mb = max_blocks_per_rank(c, kernel, (int)gi, threads, 0, CF_ALGO_SWITCH_2PA);
    const int blocks = (int)std::min<size_t>((size_t)mb, std::max<size_t>(1, ceil_div(work, (size_t)threads)));
    CF_TRY(join_streams(c, (int)gi, streams, false));
    void* args[] = {&a};
    CF_CUDA(cudaLaunchKernel(kernel, dim3(blocks, g.size()), dim3(threads), args, 0, streams[g[0]]));
    CF_TRY(join_streams(c, (int)gi, streams, true));
  }
  return CF_OK;
}

// Strip CF_ALGO_RING_LINKS off `algo`: true when the caller asked for the
// literal ring transport (only meaningful for the three ring algorithms).
cfStatus split_links(int& algo, bool& links) {
  links = algo != CF_ALGO_AUTO && (algo & CF_ALGO_RING_LINKS);
  if (links) {
    algo &= ~CF_ALGO_RING_LINKS;
    if (algo != CF_ALGO_2PR && algo != CF_ALGO_RING_RS && algo != CF_ALGO_RING_AG)
      return fail(CF_E_NO_ALGO, "CF_ALGO_RING_LINKS applies to 2pr / ring_rs / ring_ag only (algo %d)", algo);
  }
  return CF_OK;
}

}  // namespace

extern "C" cfStatus cfAllReduce(cfComm_t c, const void* const* send, void* const* recv, size_t count,
                                cfDtype dtype, int algo, const cudaStream_t* streams) {
  CF_TRY(check_ptrs(c, send, recv, streams));
  if ((int)dtype < 0 || (int)dtype > 3) return fail(CF_E_SHAPE, "unknown dtype %d", (int)dtype);
  if (count == 0) return CF_OK;
  const int n = c->nranks;
  const size_t es = dtype_size(dtype), V = 16 / es;
  const size_t bytes = count * es;
  bool links = false;
  CF_TRY(split_links(algo, links));
  long long oi = -1, oo = -1;
  const bool sym_switch = sym_switch_ok(c, send, recv, bytes, &oi, &oo);
  if (algo == CF_ALGO_AUTO) {
    algo = select_algo(c, 0, bytes, dtype);
    // 1pa_hb cannot run in place.  In one process every rank is local, so the
    // in-place test is rank-uniform; one process per GPU cannot see the
    // peers' pointers, so AUTO there never picks 1pa_hb (ranks running in
    // place and out of place would launch different kernels on the same
    // handshake slots): the LL one-shot (in-place safe) when it fits, else
    // the two-shot pull.  An explicit CF_ALGO_1PA_HB is still honoured.
    if (algo == CF_ALGO_1PA_HB && c->multiprocess)
      algo = bytes <= c->cfg.ll_max_bytes ? CF_ALGO_1PA : CF_ALGO_2PA;
    if (algo == CF_ALGO_1PA_HB)
      for (size_t li = 0; li < c->local.size(); li++)
        if (send[li] == recv[li]) algo = CF_ALGO_2PA;
    // symmetric buffers on a real multicast heap: the in-place NVLS kernel
    // moves S per rank per direction on NVLink instead of 2(n-1)/n S
    // (provisional crossover until an NVLink sweep measures it)
    if (sym_switch && c->sym.mode == 1 && bytes >= c->nvls_min_bytes) algo = CF_ALGO_SWITCH_2PA;
  }
  if (algo == CF_ALGO_SWITCH_2PA && sym_switch) return nvls_direct(c, count, dtype, oi, oo, streams);
  if (algo == CF_ALGO_SWITCH_2PA && c->nvls.enabled) return nvls_allreduce(c, send, recv, count, dtype, streams);
  Job j;
  j.algo = algo;
  j.count = count;
  switch (algo) {
    case CF_ALGO_1PA:
      if (bytes > c->cfg.ll_max_bytes)
        return fail(CF_E_BAD_SIZE, "1pa: %zu bytes exceed the LL capacity %zu", bytes, c->cfg.ll_max_bytes);
      j.kind = kLL1;
      j.order = kLead;
      j.work = ceil_div(bytes, (size_t)8);   // one thread per 8-byte packet unit
      break;
    case CF_ALGO_1PA_HB:
      for (size_t li = 0; li < c->local.size(); li++)
        if (send[li] == recv[li]) return fail(CF_E_SHAPE, "1pa_hb cannot run in place");
      j.kind = kPull;
      j.whole = 1;
      j.order = kLead;
      j.work = ceil_div(count, V);
      break;
    case CF_ALGO_2PA:
    case CF_ALGO_SWITCH_2PA: {
      // switch_2pa without a multicast object: the all-pairs pull in the
      // switch's reference order (0 + ranks ascending)
      j.kind = kPull;
      j.push = 1;
      j.order = algo == CF_ALGO_2PA ? kLead : kAscZero;
      j.cs = round_up(count, n) / n;   // cf/collectives.py:497-504
      j.work = ceil_div(j.cs, V) + 1;
      break;
    }
    case CF_ALGO_2PR:
      // ring order (0 + x_c + x_{c+1} + ...) on the reference's 2n-padded
      // chunks; all-pairs by default (see CF_ALGO_RING_LINKS)
      j.kind = links ? kRing : kPull;
      j.order = kRingZero;
      j.push = 1;
      j.cs = round_up(count, 2 * n) / n;
      j.work = ceil_div(j.cs, V) + 1;
      break;
    case CF_ALGO_2PA_LL: {
      if (bytes > c->cfg.ll_max_bytes)   // cfConfig.ll_max_bytes bounds every LL algorithm
        return fail(CF_E_BAD_SIZE, "2pa_ll: %zu bytes exceed the LL capacity %zu", bytes, c->cfg.ll_max_bytes);
      j.kind = kLL2;
      j.cs = round_up(count, n) / n;
      j.slot = c->lay.half / (2 * n) / 256 * 256;
      if (32 * (ceil_div(j.cs, V) + 1) > j.slot)
        return fail(CF_E_BAD_SIZE, "2pa_ll: %zu bytes exceed the LL capacity", bytes);
      j.work = ceil_div(bytes, (size_t)8);    // phases 1 / 2: one thread per 8-byte packet unit
      break;
    }
    default:
      return fail(CF_E_NO_ALGO, "algorithm %d is not an AllReduce algorithm", algo);
  }
  return launch(c, j, dtype, send, recv, streams);
}

extern "C" cfStatus cfAllGather(cfComm_t c, const void* const* send, void* const* recv, size_t sendcount,
                                cfDtype dtype, int algo, const cudaStream_t* streams) {
  CF_TRY(check_ptrs(c, send, recv, streams));
  if ((int)dtype < 0 || (int)dtype > 3) return fail(CF_E_SHAPE, "unknown dtype %d", (int)dtype);
  if (sendcount == 0) return CF_OK;
  bool links = false;
  CF_TRY(split_links(algo, links));
  if (algo == CF_ALGO_AUTO) algo = select_algo(c, 1, sendcount * dtype_size(dtype) * c->nranks, dtype);
  if (algo != CF_ALGO_ALLPAIRS_AG && algo != CF_ALGO_RING_AG)
    return fail(CF_E_NO_ALGO, "algorithm %d is not an AllGather algorithm", algo);
  Job j;
  j.algo = algo;
  // ring_ag: the same bytes land in the same places either way; direct
  // stores by default (see CF_ALGO_RING_LINKS)
  j.kind = links ? kRingGather : kGather;
  j.count = sendcount;
  j.work = ceil_div(sendcount * dtype_size(dtype), 16);
  const size_t sb = sendcount * dtype_size(dtype);
  if (j.kind == kGather && sb % 16 == 0 && sb >= kAgBulkMin && ag_bulk_enabled()) {
    // whole 16-byte shard of at least kAgBulkMin: the TMA bulk-copy kernel
    j.kind = kGatherBulk;
    j.threads = 32;
    j.smem = 2 * kBulkTileBytes;
    j.work = ceil_div(sb, kBulkTileBytes) * 32;   // one tile per CTA (32 threads)
  }
  return launch(c, j, dtype, send, recv, streams);
}

extern "C" cfStatus cfReduceScatter(cfComm_t c, const void* const* send, void* const* recv,
                                    size_t recvcount, cfDtype dtype, int algo, const cudaStream_t* streams) {
  CF_TRY(check_ptrs(c, send, recv, streams));
  if ((int)dtype < 0 || (int)dtype > 3) return fail(CF_E_SHAPE, "unknown dtype %d", (int)dtype);
  if (recvcount == 0) return CF_OK;
  const int n = c->nranks;
  const size_t es = dtype_size(dtype);
  bool links = false;
  CF_TRY(split_links(algo, links));
  if (algo == CF_ALGO_AUTO) algo = select_algo(c, 2, recvcount * es * n, dtype);
  if (algo != CF_ALGO_RS_DIRECT && algo != CF_ALGO_RING_RS)
    return fail(CF_E_NO_ALGO, "algorithm %d is not a ReduceScatter algorithm", algo);
  Job j;
  j.algo = algo;
  // ring_rs: rank r pulls chunk r from every peer in ring order (0 + x_r +
  // x_{r+1} + ...) unless the literal ring was asked for
  j.kind = links ? kRing : kPull;
  j.rs_shift = 1;
  j.order = algo == CF_ALGO_RING_RS ? kRingZero : kLead;
  j.count = recvcount * n;
  j.cs = recvcount;
  j.work = ceil_div(recvcount, 16 / es) + 1;
  return launch(c, j, dtype, send, recv, streams);
}

// K13: AllReduce + residual add + RMSNorm (see cf.h).
extern "C" cfStatus cfAllReduceAddRMSNorm(cfComm_t c, const void* const* send, const void* const* resid_in,
                                          void* const* resid_out, void* const* norm_out,
                                          const void* const* weight, size_t rows, size_t hidden, float eps,
                                          cfDtype dtype, int algo, const cudaStream_t* streams) {
  CF_TRY(check_ptrs(c, send, norm_out, streams));
  if (!resid_in || !resid_out || !weight) return fail(CF_E_CONFIG, "null buffer array");
  if (dtype != CF_F32 && dtype != CF_F16 && dtype != CF_BF16)
    return fail(CF_E_SHAPE, "RMSNorm needs a floating-point dtype (got %d)", (int)dtype);
  if (rows == 0 || hidden == 0) return CF_OK;
  const int n = c->nranks;
  const size_t es = dtype_size(dtype);
  if ((hidden * es) % 16)
    return fail(CF_E_BAD_ALIGN, "hidden=%zu: rows must be whole 16-byte vectors (hidden * %zu %% 16 != 0)",
                hidden, es);
  if (!(eps >= 0.f)) return fail(CF_E_CONFIG, "eps must be >= 0");
  for (size_t li = 0; li < c->local.size(); li++) {
    if (!resid_in[li] || !resid_out[li] || !weight[li]) return fail(CF_E_OOB, "local rank %zu: null buffer", li);
    if (((uintptr_t)resid_in[li] | (uintptr_t)resid_out[li] | (uintptr_t)weight[li]) & 15)
      return fail(CF_E_BAD_ALIGN, "local rank %zu: buffers must be 16-byte aligned", li);
  }
  if (algo == CF_ALGO_AUTO) {
    // two-shot once every rank owns at least one row and the rows are large
    // enough for the (n-1)x smaller reads to beat the extra pushes (measured,
    // [b, 8192] bf16, 8 ranks: one-shot 7.0 vs 9.4 us at 256 KiB, 9.7 vs 9.9
    // at 512 KiB, 16.6 vs 10.6 at 1 MiB)
    // The pick depends only on rank-uniform arguments (rows, hidden, dtype,
    // n), so every rank of a one-process-per-GPU communicator launches the
    // same kernel.  In place (send == norm_out) needs two-shot: in one
    // process every rank is local, so the in-place test is uniform too; one
    // process per GPU cannot see the peers' pointers and reports it instead.
    algo = (rows >= (size_t)n && rows * hidden * es > ((size_t)512 << 10)) ? CF_ALGO_2PA : CF_ALGO_1PA_HB;
    if (algo == CF_ALGO_1PA_HB)
      for (size_t li = 0; li < c->local.size(); li++)
        if (send[li] == norm_out[li]) {
          if (c->multiprocess)
            return fail(CF_E_SHAPE, "in-place fused AllReduce with algo=auto: pass CF_ALGO_2PA explicitly in "
                                    "the one-process-per-GPU mode (AUTO must pick the same kernel on every rank)");
          algo = CF_ALGO_2PA;
        }
  }
  Job j;
  j.algo = CF_ALGO_COUNT;
  j.kind = kNorm;
  j.order = kLead;
  j.rows = rows;
  j.hidden = hidden;
  j.eps = eps;
  j.count = rows * hidden;
  switch (algo) {
    case CF_ALGO_1PA_HB:
      for (size_t li = 0; li < c->local.size(); li++)
        if (send[li] == norm_out[li]) return fail(CF_E_SHAPE, "one-shot fused AllReduce cannot run in place");
      j.blocks = (int)std::min<size_t>(rows, CF_MAX_BLOCKS);
      break;
    case CF_ALGO_2PA:
      j.push = 1;
      j.blocks = (int)std::min<size_t>(rows, CF_MAX_BLOCKS);   // phase 2 finishes every row
      break;
    default:
      return fail(CF_E_NO_ALGO, "algorithm %d: the fused AllReduce+RMSNorm runs as 1pa_hb or 2pa", algo);
  }
  NormBufs nb{resid_in, resid_out, weight};
  return launch(c, j, dtype, send, norm_out, streams, &nb);
}

// ---------------------------------------------------------------- host-buffer AllReduce

namespace {

// Copy window [w0, w1) of every n-row chunk (row pitch cs elements) of a
// count-element message between host and a device buffer of the same layout.
cudaError_t copy_window(char* dst, const char* src, size_t count, size_t cs, int n, size_t w0, size_t w1,
                        size_t es, cudaMemcpyKind kind, cudaStream_t st) {
  // rows whose whole window lies inside the message: one 2-D copy
  size_t full = 0;
  while ((int)full < n && full * cs + w1 <= count) full++;
  if (full)
    if (cudaError_t e = cudaMemcpy2DAsync(dst + w0 * es, cs * es, src + w0 * es, cs * es, (w1 - w0) * es, full,
                                          kind, st))
      return e;
  // at most one ragged row (the padded tail lies beyond `count`)
  if ((int)full < n && full * cs + w0 < count) {
    const size_t o = full * cs + w0;
    return cudaMemcpyAsync(dst + o * es, src + o * es, (count - o) * es, kind, st);
  }
  return cudaSuccess;
}

}  // namespace

// AllReduce of HOST buffers (the reference's own calling convention:
// collective() takes host arrays, cf/collectives.py:532-573).  Large two-shot
// messages run as a pipeline of up to kHostPieces windows per chunk: the
// H2D copy of window p+1, the K3 kernel on window p and the D2H copy of
// window p-1 overlap (copy engines in both directions + SMs).  Windowing
// keeps each element's owner chunk, so results are bit-identical to
// cfAllReduce.  Completion is ordered on streams[] like every other call.
static cfStatus host_allreduce(cfComm* c, const void* const* hsend, void* const* hrecv, const void* const* dsend,
                               void* const* drecv, size_t count, cfDtype dtype, int algo,
                               const cudaStream_t* streams);

extern "C" cfStatus cfAllReduceHost(cfComm_t c, const void* const* hsend, void* const* hrecv, size_t count,
                                    cfDtype dtype, int algo, const cudaStream_t* streams) {
  CF_TRY(check_ptrs(c, hsend, hrecv, streams));
  if (c->multiprocess)
    return fail(CF_E_TOPOLOGY, "cfAllReduceHost serves one-process worlds; in the one-process-per-GPU mode "
                               "pass registered device staging buffers to cfAllReduceHostStaged");
  if ((int)dtype < 0 || (int)dtype > 3) return fail(CF_E_SHAPE, "unknown dtype %d", (int)dtype);
  if (count == 0) return CF_OK;
  const size_t padded = round_up(count, (size_t)c->nranks);
  const size_t need = round_up(padded * dtype_size(dtype), 256);
  DeviceGuard guard;
  for (size_t li = 0; li < c->local.size(); li++) {
    LocalRank& lr = c->local[li];
    if (lr.stage_bytes >= need) continue;
    CF_CUDA(cudaSetDevice(lr.dev));
    CF_CUDA(cudaDeviceSynchronize());   // earlier calls may still read the old staging
    if (lr.stage_in) cudaFree(lr.stage_in);
    if (lr.stage_out) cudaFree(lr.stage_out);
    lr.stage_in = lr.stage_out = nullptr;
    lr.stage_bytes = 0;
    CF_CUDA(cudaMalloc(&lr.stage_in, need));
    CF_CUDA(cudaMalloc(&lr.stage_out, need));
    lr.stage_bytes = need;
  }
  std::vector<const void*> din(c->local.size());
  std::vector<void*> dout(c->local.size());
  for (size_t li = 0; li < c->local.size(); li++) {
    din[li] = c->local[li].stage_in;
    dout[li] = c->local[li].stage_out;
  }
  return host_allreduce(c, hsend, hrecv, din.data(), dout.data(), count, dtype, algo, streams);
}

extern "C" cfStatus cfAllReduceHostStaged(cfComm_t c, const void* const* hsend, void* const* hrecv,
                                          const void* const* dsend, void* const* drecv, size_t count,
                                          cfDtype dtype, int algo, const cudaStream_t* streams) {
  CF_TRY(check_ptrs(c, hsend, hrecv, streams));
  CF_TRY(check_ptrs(c, dsend, drecv, streams));
  if ((int)dtype < 0 || (int)dtype > 3) return fail(CF_E_SHAPE, "unknown dtype %d", (int)dtype);
  if (count == 0) return CF_OK;
  for (size_t li = 0; li < c->local.size(); li++)
    if (dsend[li] == drecv[li]) return fail(CF_E_SHAPE, "staging send and recv must differ");
  DeviceGuard guard;
  return host_allreduce(c, hsend, hrecv, dsend, drecv, count, dtype, algo, streams);
}

static cfStatus host_allreduce(cfComm* c, const void* const* hsend, void* const* hrecv, const void* const* dsend,
                               void* const* drecv, size_t count, cfDtype dtype, int algo,
                               const cudaStream_t* streams) {
  const int n = c->nranks;
  const size_t es = dtype_size(dtype), V = 16 / es;
  const size_t bytes = count * es;
  if (algo == CF_ALGO_AUTO) algo = select_algo(c, 0, bytes, dtype);
  // the two-shot pulls (2pa, all-pairs 2pr) pipeline: windows keep each
  // element's owner and accumulation order
  const bool pull2 = algo == CF_ALGO_2PA || algo == CF_ALGO_2PR;
  const size_t padded = round_up(count, (size_t)(algo == CF_ALGO_2PR ? 2 * n : n));
  if (c->pipes.empty()) {
    c->pipes.resize(c->groups.size());
    for (size_t gi = 0; gi < c->groups.size(); gi++) {
      auto& hp = c->pipes[gi];
      CF_CUDA(cudaSetDevice(c->local[c->groups[gi][0]].dev));
      CF_CUDA(cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking));
      CF_CUDA(cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking));
      CF_CUDA(cudaEventCreateWithFlags(&hp.fork, cudaEventDisableTiming));
      CF_CUDA(cudaEventCreateWithFlags(&hp.done, cudaEventDisableTiming));
      for (int k = 0; k < kHostPieces; k++) {
        CF_CUDA(cudaEventCreateWithFlags(&hp.in[k], cudaEventDisableTiming));
        CF_CUDA(cudaEventCreateWithFlags(&hp.ar[k], cudaEventDisableTiming));
      }
    }
  }
  // pipeline only the two-shot HB kernel (windows keep each element's owner)
  const bool pipelined = pull2 && bytes >= ((size_t)32 << 20);
  const size_t cs = padded / n;
  size_t pieces = 1, q = cs;
  if (pipelined) {
    pieces = std::min<size_t>(kHostPieces, bytes / ((size_t)8 << 20));
    if (const char* env = getenv("CF_HOST_PIECES")) pieces = std::max<size_t>(1, std::min<size_t>(kHostPieces, atoi(env)));
    q = round_up(ceil_div(cs, pieces), V);
    pieces = ceil_div(cs, q);
  }
  const size_t G = c->groups.size();
  auto s0 = [&](size_t gi) { return streams[c->groups[gi][0]]; };
  // fork the copy streams off the callers' streams
  for (size_t gi = 0; gi < G; gi++) {
    auto& hp = c->pipes[gi];
    CF_CUDA(cudaSetDevice(c->local[c->groups[gi][0]].dev));
    CF_TRY(join_streams(c, (int)gi, streams, false));
    CF_CUDA(cudaEventRecord(hp.fork, s0(gi)));
    CF_CUDA(cudaStreamWaitEvent(hp.h2d, hp.fork, 0));
    CF_CUDA(cudaStreamWaitEvent(hp.d2h, hp.fork, 0));
  }
  for (size_t p = 0; p < pieces; p++) {
    const size_t w0 = p * q, w1 = std::min(cs, w0 + q);
    for (size_t gi = 0; gi < G; gi++) {
      auto& hp = c->pipes[gi];
      CF_CUDA(cudaSetDevice(c->local[c->groups[gi][0]].dev));
      for (int li : c->groups[gi]) {
        if (pipelined)
          CF_CUDA(copy_window((char*)dsend[li], (const char*)hsend[li], count, cs, n, w0, w1, es,
                              cudaMemcpyHostToDevice, hp.h2d));
        else
          CF_CUDA(cudaMemcpyAsync((void*)dsend[li], hsend[li], bytes, cudaMemcpyHostToDevice, hp.h2d));
      }
      CF_CUDA(cudaEventRecord(hp.in[p], hp.h2d));
    }
    for (size_t gi = 0; gi < G; gi++) {   // every rank's window is read by every rank
      CF_CUDA(cudaSetDevice(c->local[c->groups[gi][0]].dev));
      for (size_t g2 = 0; g2 < G; g2++) CF_CUDA(cudaStreamWaitEvent(s0(gi), c->pipes[g2].in[p], 0));
    }
    if (pipelined) {
      Job j;
      j.algo = algo;
      j.kind = kPull;
      j.push = 1;
      j.order = algo == CF_ALGO_2PA ? kLead : kRingZero;
      j.count = count;
      j.cs = cs;
      j.win_lo = w0;
      j.win_hi = w1;
      j.work = ceil_div(w1 - w0, V) + 1;
      CF_TRY(launch(c, j, dtype, dsend, drecv, streams));
    } else {
      CF_TRY(cfAllReduce(c, dsend, drecv, count, dtype, algo, streams));
    }
    for (size_t gi = 0; gi < G; gi++) {
      CF_CUDA(cudaSetDevice(c->local[c->groups[gi][0]].dev));
      CF_CUDA(cudaEventRecord(c->pipes[gi].ar[p], s0(gi)));
    }
    for (size_t gi = 0; gi < G; gi++) {   // two-shot pushes: window p is final once every rank ran it
      auto& hp = c->pipes[gi];
      CF_CUDA(cudaSetDevice(c->local[c->groups[gi][0]].dev));
      for (size_t g2 = 0; g2 < G; g2++) CF_CUDA(cudaStreamWaitEvent(hp.d2h, c->pipes[g2].ar[p], 0));
      for (int li : c->groups[gi]) {
        if (pipelined)
          CF_CUDA(copy_window((char*)hrecv[li], (const char*)drecv[li], count, cs, n, w0, w1, es,
                              cudaMemcpyDeviceToHost, hp.d2h));
        else
          CF_CUDA(cudaMemcpyAsync(hrecv[li], drecv[li], bytes, cudaMemcpyDeviceToHost, hp.d2h));
      }
    }
  }
  // join: the callers' streams complete after the last D2H copy
  for (size_t gi = 0; gi < G; gi++) {
    auto& hp = c->pipes[gi];
    CF_CUDA(cudaSetDevice(c->local[c->groups[gi][0]].dev));
    CF_CUDA(cudaEventRecord(hp.done, hp.d2h));
    CF_CUDA(cudaStreamWaitEvent(s0(gi), hp.done, 0));
    CF_CUDA(cudaEventRecord(hp.fork, hp.h2d));   // h2d idle before the next call's fork
    CF_CUDA(cudaStreamWaitEvent(s0(gi), hp.fork, 0));
    CF_TRY(join_streams(c, (int)gi, streams, true));
  }
  return CF_OK;
}

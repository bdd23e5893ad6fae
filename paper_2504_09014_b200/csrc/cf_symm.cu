// cf_symm.cu -- symmetric heap, cfMemAlloc / cfMemFree, SwitchChannel handles.
//
// SURVEY §8(b) cfMemAlloc: symmetric, peer-mapped (+ multicast) memory.  The
// reference's SimWorld gives every rank the same named regions
// (cf/world.py:113-138) and its SwitchChannel reduces / broadcasts one offset
// across members (cf/channels.py:333-409).  Here each rank owns one cuMem
// allocation (POSIX-fd shareable); every rank's heap is mapped into every
// other rank (unicast, for the HB kernels) and, where the box builds a
// multicast object, bound to it (multicast mapping, for multimem).  Buffers
// carved at the same offset of every heap are symmetric: a collective on them
// needs no registration, and the NVLS AllReduce runs on them in place
// (multimem.ld_reduce from the send buffer, multimem.st into the recv buffer,
// no staging copies).
#include <algorithm>
#include <cstring>
#include <cuda.h>
#include "cf_runtime.h"

namespace cf {
namespace {

template <typename F>
F drv(const char* name) {
  return (F)driver_fn(name);
}
#define CF_DRV(name) auto p_##name = drv<decltype(&name)>(#name)

cfStatus dchk(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return CF_OK;
  return fail(CF_E_CUDA, "%s failed (CUresult %d)", what, (int)r);
}

constexpr size_t kSymAlign = 512;   // allocation granularity inside a heap

CUmemAllocationProp phys_prop(int dev) {
  CUmemAllocationProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  mp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  mp.location.id = dev;
  mp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return mp;
}

// map `mem` (bytes) at a fresh VA readable/writable from every device in `devs`
cfStatus map_va(unsigned long long mem, size_t bytes, size_t gran, const std::vector<int>& devs, char** va) {
  CF_DRV(cuMemAddressReserve);
  CF_DRV(cuMemMap);
  CF_DRV(cuMemSetAccess);
  CUdeviceptr p = 0;
  CF_TRY(dchk(p_cuMemAddressReserve(&p, bytes, gran, 0, 0), "cuMemAddressReserve"));
  CF_TRY(dchk(p_cuMemMap(p, bytes, 0, (CUmemGenericAllocationHandle)mem, 0), "cuMemMap"));
  std::vector<CUmemAccessDesc> acc(devs.size());
  for (size_t i = 0; i < devs.size(); i++) {
    memset(&acc[i], 0, sizeof(acc[i]));
    acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[i].location.id = devs[i];
    acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  CF_TRY(dchk(p_cuMemSetAccess(p, bytes, acc.data(), acc.size()), "cuMemSetAccess"));
  *va = (char*)p;
  return CF_OK;
}

void unmap_va(char* va, size_t bytes) {
  CF_DRV(cuMemUnmap);
  CF_DRV(cuMemAddressFree);
  if (!va) return;
  p_cuMemUnmap((CUdeviceptr)va, bytes);
  p_cuMemAddressFree((CUdeviceptr)va, bytes);
}

// heap size rounded to the allocation (and, for NVLS, multicast) granularity
cfStatus sym_size(cfComm* c, size_t bytes, bool multicast) {
  CF_DRV(cuMemGetAllocationGranularity);
  CF_DRV(cuMulticastGetGranularity);
  CUmemAllocationProp mp = phys_prop(c->local[0].dev);
  size_t g = 0;
  CF_TRY(dchk(p_cuMemGetAllocationGranularity(&g, &mp, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
              "cuMemGetAllocationGranularity"));
  if (multicast && p_cuMulticastGetGranularity) {
    CUmulticastObjectProp p;
    memset(&p, 0, sizeof(p));
    p.numDevices = (unsigned)c->nranks;
    p.size = bytes;
    p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t mg = 0;
    if (p_cuMulticastGetGranularity(&mg, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && mg > g) g = mg;
  }
  c->sym.gran = g;
  c->sym.bytes = round_up(bytes, g);
  return CF_OK;
}

cfStatus create_own(cfComm* c, int li, const std::vector<int>& devs) {
  CF_DRV(cuMemCreate);
  CUmemAllocationProp mp = phys_prop(c->local[li].dev);
  CUmemGenericAllocationHandle mem;
  CF_CUDA(cudaSetDevice(c->local[li].dev));
  CF_TRY(dchk(p_cuMemCreate(&mem, c->sym.bytes, &mp, 0), "cuMemCreate"));
  c->sym.ranks[li].mem = (unsigned long long)mem;
  CF_TRY(map_va(c->sym.ranks[li].mem, c->sym.bytes, c->sym.gran, devs, &c->sym.ranks[li].uc));
  CF_CUDA(cudaMemset(c->sym.ranks[li].uc, 0, c->sym.bytes));
  return CF_OK;
}

cfStatus mc_add(cfComm* c, int dev) {
  CF_DRV(cuMulticastAddDevice);
  CF_DRV(cuDeviceGet);
  CUdevice d;
  CF_TRY(dchk(p_cuDeviceGet(&d, dev), "cuDeviceGet"));
  return dchk(p_cuMulticastAddDevice((CUmemGenericAllocationHandle)c->sym.mc, d), "cuMulticastAddDevice");
}

cfStatus mc_bind(cfComm* c, int li) {
  CF_DRV(cuMulticastBindMem);
  CF_CUDA(cudaSetDevice(c->local[li].dev));
  CF_TRY(dchk(p_cuMulticastBindMem((CUmemGenericAllocationHandle)c->sym.mc, 0,
                                   (CUmemGenericAllocationHandle)c->sym.ranks[li].mem, 0, c->sym.bytes, 0),
              "cuMulticastBindMem"));
  return map_va(c->sym.mc, c->sym.bytes, c->sym.gran, {c->local[li].dev}, &c->sym.ranks[li].mc);
}

cfStatus mc_create(cfComm* c, unsigned ndev) {
  CF_DRV(cuMulticastCreate);
  if (!p_cuMulticastCreate) return fail(CF_E_TOPOLOGY, "driver lacks cuMulticastCreate");
  CUmulticastObjectProp p;
  memset(&p, 0, sizeof(p));
  p.numDevices = ndev;
  p.size = c->sym.bytes;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mc;
  CF_TRY(dchk(p_cuMulticastCreate(&mc, &p), "cuMulticastCreate"));
  c->sym.mc = (unsigned long long)mc;
  return CF_OK;
}

}  // namespace

void sym_teardown(cfComm* c) {
  SymHeap& h = c->sym;
  if (!h.on() && h.ranks.empty()) return;
  CF_DRV(cuMemRelease);
  CF_DRV(cuMulticastUnbind);
  CF_DRV(cuDeviceGet);
  for (size_t li = 0; li < h.ranks.size(); li++) {
    cudaSetDevice(c->local[li].dev);
    cudaDeviceSynchronize();
  }
  for (auto& im : h.imported) {
    unmap_va(im.second, h.bytes);
    p_cuMemRelease((CUmemGenericAllocationHandle)im.first);
  }
  for (size_t li = 0; li < h.ranks.size(); li++) {
    SymRank& sr = h.ranks[li];
    unmap_va(sr.mc, h.bytes);
    unmap_va(sr.uc, h.bytes);
    if (sr.mem) {
      CUdevice d;
      if (h.mc && sr.mc && p_cuDeviceGet(&d, c->local[li].dev) == CUDA_SUCCESS)
        p_cuMulticastUnbind((CUmemGenericAllocationHandle)h.mc, d, 0, h.bytes);
      p_cuMemRelease((CUmemGenericAllocationHandle)sr.mem);
    }
  }
  if (h.mc) p_cuMemRelease((CUmemGenericAllocationHandle)h.mc);
  c->sym = SymHeap();
}

}  // namespace cf

using namespace cf;

// In-process communicators: every local rank's heap, unicast-mapped on every
// local device; mode 1 binds them to one multicast object (distinct devices
// that all support multicast, else CF_E_TOPOLOGY); mode 2 is the emulated
// switch (unicast only).  One process per GPU: this rank's heap only; `fd`
// receives its POSIX handle for the peers' cfSymHeapMapPeer.
extern "C" cfStatus cfSymHeapCreate(cfComm_t c, size_t bytes, int mode, int* fd) {
  if (!c) return fail(CF_E_CONFIG, "null communicator");
  if (c->sym.on()) return fail(CF_E_CONFIG, "the communicator already has a symmetric heap");
  if (bytes == 0) return fail(CF_E_BAD_SIZE, "symmetric heap of 0 bytes");
  if (mode < 0 || mode > 2) return fail(CF_E_CONFIG, "mode must be 0 (none), 1 (multicast) or 2 (emulated)");
  if (c->multiprocess && !fd) return fail(CF_E_CONFIG, "one process per GPU: pass fd to export the heap");
  DeviceGuard guard;
  std::vector<int> devs;
  for (auto& lr : c->local)
    if (std::find(devs.begin(), devs.end(), lr.dev) == devs.end()) devs.push_back(lr.dev);
  if (mode == 1) {
    if (!c->multiprocess && devs.size() != c->local.size())
      return fail(CF_E_TOPOLOGY, "NVLS needs one device per rank (%zu devices for %zu ranks)", devs.size(),
                  c->local.size());
    for (int d : devs)
      if (!multicast_capable(d)) return fail(CF_E_TOPOLOGY, "device %d does not support multicast", d);
  }
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  CF_TRY(sym_size(c, bytes, mode == 1));
  c->sym.mode = mode;
  c->sym.ranks.assign(c->local.size(), SymRank());
  c->sym.peer.assign(c->local.size(), {});
  cfStatus s = CF_OK;
  for (size_t li = 0; li < c->local.size() && s == CF_OK; li++) s = create_own(c, (int)li, devs);
  if (s == CF_OK && mode == 1 && !c->multiprocess) {
    s = mc_create(c, (unsigned)c->local.size());
    for (size_t li = 0; li < c->local.size() && s == CF_OK; li++) s = mc_add(c, c->local[li].dev);
    for (size_t li = 0; li < c->local.size() && s == CF_OK; li++) s = mc_bind(c, (int)li);
  }
  if (s != CF_OK) {
    sym_teardown(c);
    return s;
  }
  for (size_t li = 0; li < c->local.size(); li++)
    for (size_t q = 0; q < c->local.size(); q++) c->sym.peer[li][c->local[q].rank] = c->sym.ranks[q].uc;
  if (c->multiprocess) {
    CF_DRV(cuMemExportToShareableHandle);
    int f = -1;
    s = dchk(p_cuMemExportToShareableHandle(&f, (CUmemGenericAllocationHandle)c->sym.ranks[0].mem,
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
             "cuMemExportToShareableHandle");
    if (s != CF_OK) {
      sym_teardown(c);
      return s;
    }
    *fd = f;
  }
  return CF_OK;
}

// One process per GPU: map rank `peer`'s heap from its exported fd.
extern "C" cfStatus cfSymHeapMapPeer(cfComm_t c, int peer, int fd) {
  if (!c) return fail(CF_E_CONFIG, "null communicator");
  if (!c->multiprocess) return fail(CF_E_CONFIG, "cfSymHeapMapPeer is for cfCommCreateRank communicators");
  if (!c->sym.on()) return fail(CF_E_CONFIG, "cfSymHeapCreate first");
  if (peer < 0 || peer >= c->nranks || peer == c->local[0].rank) return fail(CF_E_RANK_MISMATCH, "bad peer %d", peer);
  CF_DRV(cuMemImportFromShareableHandle);
  DeviceGuard guard;
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  CUmemGenericAllocationHandle mem;
  CF_TRY(dchk(p_cuMemImportFromShareableHandle(&mem, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
              "cuMemImportFromShareableHandle"));
  char* va = nullptr;
  CF_TRY(map_va((unsigned long long)mem, c->sym.bytes, c->sym.gran, {c->local[0].dev}, &va));
  c->sym.imported.push_back({(unsigned long long)mem, va});
  c->sym.peer[0][peer] = va;
  return CF_OK;
}

// One process per GPU, mode 1, in phases the caller separates with bootstrap
// barriers: phase 0 on rank 0 creates the multicast object and returns its fd
// (send it to every rank); phase 1 on the others imports it (*fd in); phase 2
// on every rank binds and maps its heap; phase 3 (every rank, when any rank
// failed a phase) turns the switch off for this heap.
extern "C" cfStatus cfSymHeapMulticast(cfComm_t c, int phase, int* fd) {
  if (!c || !fd) return fail(CF_E_CONFIG, "null argument");
  if (!c->multiprocess) return fail(CF_E_CONFIG, "in-process communicators bind in cfSymHeapCreate");
  if (!c->sym.on() || c->sym.mode != 1) return fail(CF_E_CONFIG, "cfSymHeapCreate(mode = 1) first");
  DeviceGuard guard;
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  if (phase == 0) {
    if (c->local[0].rank != 0) return fail(CF_E_RANK_MISMATCH, "rank 0 creates the multicast object");
    CF_DRV(cuMemExportToShareableHandle);
    CF_TRY(mc_create(c, (unsigned)c->nranks));
    CF_TRY(dchk(p_cuMemExportToShareableHandle(fd, (CUmemGenericAllocationHandle)c->sym.mc,
                                               CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                "cuMemExportToShareableHandle"));
    CF_TRY(mc_add(c, c->local[0].dev));
    c->sym.mc_added = true;
    return CF_OK;
  }
  if (phase == 1) {
    CF_DRV(cuMemImportFromShareableHandle);
    CUmemGenericAllocationHandle mc;
    CF_TRY(dchk(p_cuMemImportFromShareableHandle(&mc, (void*)(uintptr_t)*fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                "cuMemImportFromShareableHandle"));
    c->sym.mc = (unsigned long long)mc;
    CF_TRY(mc_add(c, c->local[0].dev));
    c->sym.mc_added = true;
    return CF_OK;
  }
  if (phase == 2) {
    if (!c->sym.mc_added) return fail(CF_E_CONFIG, "multicast phase 0 / 1 first");
    return mc_bind(c, 0);
  }
  if (phase == 3) {
    // some rank failed a phase: every rank stops using the switch (the heap
    // stays usable for the HB algorithms), so no rank's AUTO picks NVLS
    // while a peer picks another kernel
    c->sym.mode = 0;
    return CF_OK;
  }
  return fail(CF_E_CONFIG, "phase must be 0, 1, 2 or 3");
}

// Collective: every rank asks for the same sizes in the same order, so the
// first-fit allocator hands out the same offset everywhere.  ptrs[li] =
// local rank li's buffer.
extern "C" cfStatus cfMemAlloc(cfComm_t c, size_t bytes, void** ptrs) {
  if (!c || !ptrs) return fail(CF_E_CONFIG, "null argument");
  if (!c->sym.on()) return fail(CF_E_CONFIG, "no symmetric heap (cfSymHeapCreate)");
  const size_t need = round_up(std::max<size_t>(bytes, 1), kSymAlign);
  size_t at = 0;
  bool found = false;
  for (auto& u : c->sym.used) {   // first gap that fits
    if (u.first - at >= need) { found = true; break; }
    at = u.first + u.second;
  }
  if (!found && c->sym.bytes - at >= need) found = true;
  if (!found || at + need > c->sym.bytes)
    return fail(CF_E_BAD_SIZE, "symmetric heap exhausted: %zu bytes requested, heap %zu bytes", bytes, c->sym.bytes);
  c->sym.used[at] = need;
  for (size_t li = 0; li < c->local.size(); li++) ptrs[li] = c->sym.ranks[li].uc + at;
  return CF_OK;
}

extern "C" cfStatus cfMemFree(cfComm_t c, const void* ptr) {
  if (!c) return fail(CF_E_CONFIG, "null communicator");
  for (size_t li = 0; li < c->local.size(); li++) {
    const long long off = c->sym.offset((int)li, ptr);
    if (off < 0) continue;
    auto it = c->sym.used.find((size_t)off);
    if (it == c->sym.used.end()) return fail(CF_E_OOB, "%p is not the start of a cfMemAlloc buffer", ptr);
    c->sym.used.erase(it);
    return CF_OK;
  }
  return fail(CF_E_OOB, "%p is not in the symmetric heap", ptr);
}

// Heap base of every rank as seen from local rank `li` (peer mappings; the
// caller's own rank included) and the mode; `bases` holds nranks entries.
extern "C" cfStatus cfSymHeapInfo(cfComm_t c, int li, void** bases, size_t* bytes, int* mode) {
  if (!c) return fail(CF_E_CONFIG, "null communicator");
  if (li < 0 || li >= (int)c->local.size()) return fail(CF_E_RANK_MISMATCH, "bad local rank %d", li);
  if (bytes) *bytes = c->sym.bytes;
  if (mode) *mode = c->sym.mode;
  if (bases)
    for (int p = 0; p < c->nranks; p++) bases[p] = c->sym.on() ? c->sym.peer[li][p] : nullptr;
  return CF_OK;
}

// SwitchChannel handle (cf::SwitchChannelDevice) for local rank `li`'s kernels.
extern "C" cfStatus cfSwitchChannelCreate(cfComm_t c, int li, void* handle, size_t* handle_bytes) {
  if (!c || !handle || !handle_bytes) return fail(CF_E_CONFIG, "null argument");
  if (*handle_bytes < sizeof(SwitchChannelDevice)) return fail(CF_E_BAD_SIZE, "handle buffer too small");
  if (li < 0 || li >= (int)c->local.size()) return fail(CF_E_RANK_MISMATCH, "bad local rank %d", li);
  if (!c->sym.on() || c->sym.mode == 0)
    return fail(CF_E_TOPOLOGY, "no switch: the symmetric heap has neither a multicast object nor emulation");
  for (int p = 0; p < c->nranks; p++)
    if (!c->sym.peer[li][p]) return fail(CF_E_CONFIG, "rank %d's heap is not mapped (cfSymHeapMapPeer)", p);
  SwitchChannelDevice d;
  memset(&d, 0, sizeof(d));
  d.mc = c->sym.mode == 1 ? c->sym.ranks[li].mc : nullptr;
  if (c->sym.mode == 1 && !d.mc) return fail(CF_E_CONFIG, "multicast not bound (cfSymHeapMulticast phase 2)");
  for (int p = 0; p < c->nranks; p++) d.uc[p] = c->sym.peer[li][p];
  d.local = c->sym.ranks[li].uc;
  d.n = c->nranks;
  d.rank = c->local[li].rank;
  memcpy(handle, &d, sizeof(d));
  *handle_bytes = sizeof(d);
  return CF_OK;
}

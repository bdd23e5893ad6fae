// cf_nvls.cu -- NVLS multicast objects for SwitchChannel-style collectives
// (cf/channels.py:333-409 SwitchChannel / switch_reduce / switch_broadcast).
//
// Every rank binds CF-owned physical memory to one multicast object; the
// memory is mapped twice: unicast (local copy-in / copy-out) and multicast
// (multimem.ld_reduce sums the same offset across all members inside the
// NVSwitch, multimem.st broadcasts).  Driver entry points are resolved through
// the runtime (driver_fn), so libcf keeps no link-time libcuda dependency.
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

cfStatus drv_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return CF_OK;
  return fail(CF_E_CUDA, "%s failed (CUresult %d)", what, (int)r);
}

CUmulticastObjectProp mc_prop(const cfComm* c, size_t size) {
  CUmulticastObjectProp p;
  memset(&p, 0, sizeof(p));
  p.numDevices = (unsigned)c->nranks;
  p.size = size;
  // the driver rejects multicast objects without a shareable handle type
  // (CUDA_ERROR_INVALID_VALUE, measured on B200), even in one process
  (void)c;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  p.flags = 0;
  return p;
}

// granularity and rounded size for the configured staging region
cfStatus nvls_size(cfComm* c) {
  CF_DRV(cuMulticastGetGranularity);
  if (!p_cuMulticastGetGranularity) return fail(CF_E_TOPOLOGY, "driver lacks multicast entry points");
  c->nvls.half = c->cfg.nvls_bytes;
  CUmulticastObjectProp p = mc_prop(c, 2 * c->nvls.half);
  size_t g = 0;
  CF_TRY(drv_check(p_cuMulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED),
                   "cuMulticastGetGranularity"));
  c->nvls.gran = g;
  c->nvls.half = round_up(c->nvls.half, g);
  c->nvls.size = 2 * c->nvls.half;
  return CF_OK;
}

cfStatus add_device(cfComm* c, int dev) {
  CF_DRV(cuMulticastAddDevice);
  CF_DRV(cuDeviceGet);
  CUdevice d;
  CF_TRY(drv_check(p_cuDeviceGet(&d, dev), "cuDeviceGet"));
  return drv_check(p_cuMulticastAddDevice((CUmemGenericAllocationHandle)c->nvls.mc, d), "cuMulticastAddDevice");
}

// bind this local rank's physical memory and map unicast + multicast
cfStatus bind_rank(cfComm* c, int li) {
  CF_DRV(cuMemCreate);
  CF_DRV(cuMulticastBindMem);
  CF_DRV(cuMemAddressReserve);
  CF_DRV(cuMemMap);
  CF_DRV(cuMemSetAccess);
  const int dev = c->local[li].dev;
  CF_CUDA(cudaSetDevice(dev));
  CUmemAllocationProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  mp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  mp.location.id = dev;
  mp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  NvlsRank& nr = c->nvls.ranks[li];
  CUmemGenericAllocationHandle mem;
  CF_TRY(drv_check(p_cuMemCreate(&mem, c->nvls.size, &mp, 0), "cuMemCreate"));
  nr.mem = (unsigned long long)mem;
  CF_TRY(drv_check(p_cuMulticastBindMem((CUmemGenericAllocationHandle)c->nvls.mc, 0, mem, 0, c->nvls.size, 0),
                   "cuMulticastBindMem"));
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mc = 0;
  CF_TRY(drv_check(p_cuMemAddressReserve(&uc, c->nvls.size, c->nvls.gran, 0, 0), "cuMemAddressReserve"));
  CF_TRY(drv_check(p_cuMemMap(uc, c->nvls.size, 0, mem, 0), "cuMemMap(unicast)"));
  CF_TRY(drv_check(p_cuMemSetAccess(uc, c->nvls.size, &acc, 1), "cuMemSetAccess(unicast)"));
  nr.uc = (char*)uc;
  CF_TRY(drv_check(p_cuMemAddressReserve(&mc, c->nvls.size, c->nvls.gran, 0, 0), "cuMemAddressReserve"));
  CF_TRY(drv_check(p_cuMemMap(mc, c->nvls.size, 0, (CUmemGenericAllocationHandle)c->nvls.mc, 0),
                   "cuMemMap(multicast)"));
  CF_TRY(drv_check(p_cuMemSetAccess(mc, c->nvls.size, &acc, 1), "cuMemSetAccess(multicast)"));
  nr.mc = (char*)mc;
  CF_CUDA(cudaMemset(nr.uc, 0, c->nvls.size));
  return CF_OK;
}

}  // namespace

bool multicast_capable(int dev) {
  CF_DRV(cuDeviceGetAttribute);
  CF_DRV(cuDeviceGet);
  if (!p_cuDeviceGetAttribute || !p_cuDeviceGet) return false;
  CUdevice d;
  if (p_cuDeviceGet(&d, dev) != CUDA_SUCCESS) return false;
  int v = 0;
  if (p_cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d) != CUDA_SUCCESS) return false;
  return v != 0;
}

cfStatus nvls_setup_inprocess(cfComm* c) {
  CF_DRV(cuMulticastCreate);
  if (!p_cuMulticastCreate) return fail(CF_E_TOPOLOGY, "driver lacks cuMulticastCreate");
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  CF_TRY(nvls_size(c));
  CUmulticastObjectProp p = mc_prop(c, c->nvls.size);
  CUmemGenericAllocationHandle mc;
  CF_TRY(drv_check(p_cuMulticastCreate(&mc, &p), "cuMulticastCreate"));
  c->nvls.mc = (unsigned long long)mc;
  c->nvls.ranks.assign(c->local.size(), NvlsRank());
  for (auto& lr : c->local) CF_TRY(add_device(c, lr.dev));   // every device before any bind
  c->nvls.added = true;
  for (size_t li = 0; li < c->local.size(); li++) CF_TRY(bind_rank(c, (int)li));
  c->nvls.enabled = true;
  return CF_OK;
}

// Emulated switch (cfConfig.use_multicast = 2): plain per-rank staging, the
// kernel replaces multimem by per-rank loads / stores (in-process worlds).
cfStatus nvls_setup_emulated(cfComm* c) {
  if (c->multiprocess) return fail(CF_E_CONFIG, "the emulated switch needs every rank in this process");
  c->nvls.half = round_up(c->cfg.nvls_bytes ? c->cfg.nvls_bytes : (size_t)64 << 20, (size_t)4096);
  c->nvls.size = 2 * c->nvls.half;
  c->nvls.ranks.assign(c->local.size(), NvlsRank());
  for (size_t li = 0; li < c->local.size(); li++) {
    CF_CUDA(cudaSetDevice(c->local[li].dev));
    CF_CUDA(cudaMalloc((void**)&c->nvls.ranks[li].uc, c->nvls.size));
    CF_CUDA(cudaMemset(c->nvls.ranks[li].uc, 0, c->nvls.size));
  }
  c->nvls.emul = true;
  c->nvls.enabled = true;
  return CF_OK;
}

void nvls_teardown(cfComm* c) {
  if (c->nvls.emul && c->multiprocess) {   // staging is the caller's registered buffer
    c->nvls = Nvls();
    return;
  }
  if (c->nvls.emul) {
    for (size_t li = 0; li < c->nvls.ranks.size(); li++) {
      cudaSetDevice(c->local[li].dev);
      cudaDeviceSynchronize();
      cudaFree(c->nvls.ranks[li].uc);
    }
    c->nvls = Nvls();
    return;
  }
  if (!c->nvls.mc && c->nvls.ranks.empty()) return;
  CF_DRV(cuMemUnmap);
  CF_DRV(cuMemAddressFree);
  CF_DRV(cuMemRelease);
  CF_DRV(cuMulticastUnbind);
  CF_DRV(cuDeviceGet);
  for (size_t li = 0; li < c->nvls.ranks.size(); li++) {
    NvlsRank& nr = c->nvls.ranks[li];
    cudaSetDevice(c->local[li].dev);
    cudaDeviceSynchronize();
    if (nr.mc) { p_cuMemUnmap((CUdeviceptr)nr.mc, c->nvls.size); p_cuMemAddressFree((CUdeviceptr)nr.mc, c->nvls.size); }
    if (nr.uc) { p_cuMemUnmap((CUdeviceptr)nr.uc, c->nvls.size); p_cuMemAddressFree((CUdeviceptr)nr.uc, c->nvls.size); }
    if (nr.mem) {
      CUdevice d;
      if (c->nvls.mc && p_cuDeviceGet(&d, c->local[li].dev) == CUDA_SUCCESS)
        p_cuMulticastUnbind((CUmemGenericAllocationHandle)c->nvls.mc, d, 0, c->nvls.size);
      p_cuMemRelease((CUmemGenericAllocationHandle)nr.mem);
    }
  }
  if (c->nvls.mc) p_cuMemRelease((CUmemGenericAllocationHandle)c->nvls.mc);
  c->nvls = Nvls();
}

}  // namespace cf

using namespace cf;

extern "C" cfStatus cfDeviceMulticastSupported(int cuda_dev, int* supported) {
  if (!supported) return fail(CF_E_CONFIG, "null argument");
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(cuda_dev) != cudaSuccess) return fail(CF_E_TOPOLOGY, "no device %d", cuda_dev);
  *supported = multicast_capable(cuda_dev) ? 1 : 0;
  if (prev >= 0) cudaSetDevice(prev);
  return CF_OK;
}

extern "C" cfStatus cfNvlsCreate(cfComm_t c, int* fd) {
  if (!c || !fd) return fail(CF_E_CONFIG, "null argument");
  if (!c->multiprocess) return fail(CF_E_CONFIG, "cfNvlsCreate is for cfCommCreateRank communicators");
  if (c->local[0].rank != 0) return fail(CF_E_RANK_MISMATCH, "rank 0 creates the multicast object");
  if (!multicast_capable(c->local[0].dev)) return fail(CF_E_TOPOLOGY, "device does not support multicast");
  CF_DRV(cuMulticastCreate);
  CF_DRV(cuMemExportToShareableHandle);
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  if (c->cfg.nvls_bytes == 0) c->cfg.nvls_bytes = 64u << 20;
  CF_TRY(nvls_size(c));
  CUmulticastObjectProp p = mc_prop(c, c->nvls.size);
  CUmemGenericAllocationHandle mc;
  CF_TRY(drv_check(p_cuMulticastCreate(&mc, &p), "cuMulticastCreate"));
  c->nvls.mc = (unsigned long long)mc;
  int f = -1;
  CF_TRY(drv_check(p_cuMemExportToShareableHandle(&f, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                   "cuMemExportToShareableHandle"));
  c->nvls.ranks.assign(1, NvlsRank());
  CF_TRY(add_device(c, c->local[0].dev));
  c->nvls.added = true;
  *fd = f;
  return CF_OK;
}

extern "C" cfStatus cfNvlsImport(cfComm_t c, int fd) {
  if (!c) return fail(CF_E_CONFIG, "null argument");
  if (!c->multiprocess) return fail(CF_E_CONFIG, "cfNvlsImport is for cfCommCreateRank communicators");
  if (!multicast_capable(c->local[0].dev)) return fail(CF_E_TOPOLOGY, "device does not support multicast");
  CF_DRV(cuMemImportFromShareableHandle);
  CF_CUDA(cudaSetDevice(c->local[0].dev));
  if (c->cfg.nvls_bytes == 0) c->cfg.nvls_bytes = 64u << 20;
  CF_TRY(nvls_size(c));
  CUmemGenericAllocationHandle mc;
  CF_TRY(drv_check(p_cuMemImportFromShareableHandle(&mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                   "cuMemImportFromShareableHandle"));
  c->nvls.mc = (unsigned long long)mc;
  c->nvls.ranks.assign(1, NvlsRank());
  CF_TRY(add_device(c, c->local[0].dev));
  c->nvls.added = true;
  return CF_OK;
}

extern "C" cfStatus cfNvlsBind(cfComm_t c) {
  if (!c) return fail(CF_E_CONFIG, "null argument");
  if (!c->nvls.added) return fail(CF_E_CONFIG, "cfNvlsCreate/cfNvlsImport first");
  CF_TRY(bind_rank(c, 0));
  c->nvls.enabled = true;
  c->multicast_supported = true;
  return CF_OK;
}

extern "C" cfStatus cfNvlsEmulate(cfComm_t c, void* staging, size_t bytes) {
  if (!c || !staging) return fail(CF_E_CONFIG, "null argument");
  if (!c->multiprocess) return fail(CF_E_CONFIG, "cfNvlsEmulate is for cfCommCreateRank communicators "
                                                 "(in-process worlds: cfConfig.use_multicast = 2)");
  if (c->nvls.enabled && !c->nvls.emul) return fail(CF_E_CONFIG, "a real multicast object is already bound");
  const Registration* reg = c->find_reg(staging);
  if (!reg) return fail(CF_E_TOPOLOGY, "staging %p is not registered (cfBufferExport/cfBufferImport)", staging);
  const size_t off = (const char*)staging - reg->ptr;
  if (off + bytes > reg->bytes) return fail(CF_E_OOB, "staging range exceeds its registration");
  const size_t half = bytes / 2 / 16 * 16;
  if (half == 0 || ((uintptr_t)staging & 15)) return fail(CF_E_BAD_ALIGN, "staging must be 16-byte aligned, >= 32 B");
  c->nvls = Nvls();
  c->nvls.half = half;
  c->nvls.size = 2 * half;
  c->nvls.ranks.assign(1, NvlsRank());
  c->nvls.ranks[0].uc = (char*)staging;
  c->nvls.peer_uc.assign(c->nranks, nullptr);
  for (int q = 0; q < c->nranks; q++) c->nvls.peer_uc[q] = reg->peer[q] + off;
  c->nvls.peer_uc[c->local[0].rank] = (char*)staging;
  c->nvls.emul = true;
  c->nvls.enabled = true;
  return CF_OK;
}

"""Probe NVLS multicast object creation on this box (diagnostic only)."""
from cuda.bindings import driver as d


def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    return err, (r[1:] if isinstance(r, tuple) else ())


print("init", d.cuInit(0))
err, (dev,) = chk(d.cuDeviceGet(0))
err, (ctx,) = chk(d.cuDevicePrimaryCtxRetain(dev))
print("ctx", d.cuCtxSetCurrent(ctx))
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    a = getattr(d.CUdevice_attribute, attr, None)
    if a is not None:
        print(attr, d.cuDeviceGetAttribute(a, dev))
for ht_name in ("CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC",
                "CU_MEM_HANDLE_TYPE_NONE"):
    for ndev in (1, 2):
        p = d.CUmulticastObjectProp()
        p.numDevices = ndev
        p.handleTypes = getattr(d.CUmemAllocationHandleType, ht_name)
        p.size = 2 << 20
        p.flags = 0
        err, rest = chk(d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        gran = rest[0] if rest else None
        err2, rest2 = chk(d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM))
        if gran:
            p.size = max(gran, 2 << 20)
        err3, rest3 = chk(d.cuMulticastCreate(p))
        print(ht_name, "ndev", ndev, "gran", err, gran, "min", err2, rest2[0] if rest2 else None,
              "create", err3)
        if err3 == d.CUresult.CUDA_SUCCESS:
            print("  add", d.cuMulticastAddDevice(rest3[0], dev))

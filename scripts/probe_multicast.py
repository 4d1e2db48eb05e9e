"""Probe the multicast (NVLS) API on the GPU box: attributes, granularities,
and which cuMulticastCreate property combinations are accepted."""
from cuda.bindings import driver as d

d.cuInit(0)
_, dev = d.cuDeviceGet(0)
_, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"]:
    print(name, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, name), dev))
for nd in (1, 2):
    for ht in (d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE,
               d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
               d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC):
        p = d.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = int(ht)
        p.size = 2 << 20
        e1, gmin = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        e2, grec = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        for size in (gmin if isinstance(gmin, int) else 0, grec if isinstance(grec, int) else 0):
            if not size:
                continue
            p.size = size
            err, h = d.cuMulticastCreate(p)
            print(f"numDevices={nd} handle={ht.name} gran_min={gmin} gran_rec={grec} size={size} -> {err}")
            if err == d.CUresult.CUDA_SUCCESS:
                if nd == 1:
                    print("  addDevice:", d.cuMulticastAddDevice(h, dev))
                d.cuMemRelease(h)

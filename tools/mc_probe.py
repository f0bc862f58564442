"""Probe: can this box create a CUDA multicast object (NVLS)? Prints the driver's answers."""
from cuda.bindings import driver as d

d.cuInit(0)
_, dev = d.cuDeviceGet(0)
_, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"]:
    print(name, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, name), dev))
for ht in [d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE,
           d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
           d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC]:
    for n in (1, 2):
        p = d.CUmulticastObjectProp()
        p.numDevices = n
        p.handleTypes = int(ht)
        p.size = 2 << 20
        g = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        if g[0] == 0:
            p.size = max(p.size, g[1])
        r = d.cuMulticastCreate(p)
        print("handle", ht.name, "numDevices", n, "gran", g, "create", r[0])

"""Is NVLink SHARP multicast (multimem) usable on this box's GPU?  Queries the
device attribute and tries to create + bind a one-device multicast object
(cuMulticastCreate / cuMulticastAddDevice / cuMulticastBindMem)."""
from cuda.bindings import driver as d


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) and len(r) == 2 else None)


ck(d.cuInit(0))
dev = ck(d.cuDeviceGet(0))
ctx = ck(d.cuDevicePrimaryCtxRetain(dev))
ck(d.cuCtxSetCurrent(ctx))
sup = ck(d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
print("MULTICAST_SUPPORTED", sup)
try:
    prop = d.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 2 << 20
    prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE
    gran = ck(d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
    print("granularity", gran)
    prop.size = max(prop.size, gran)
    mc = ck(d.cuMulticastCreate(prop))
    ck(d.cuMulticastAddDevice(mc, dev))
    ap = d.CUmemAllocationProp()
    ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    ap.location.id = 0
    mem = ck(d.cuMemCreate(prop.size, ap, 0))
    ck(d.cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0))
    print("one-device multicast object created and bound: OK")
except Exception as exc:
    print("multicast create/bind failed:", exc)

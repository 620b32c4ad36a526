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
def attempt(handle):
    prop = d.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 2 << 20
    prop.handleTypes = handle
    prop.flags = 0
    step = "granularity"
    try:
        gran = ck(d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        prop.size = max(prop.size, gran)
        step = "create"
        mc = ck(d.cuMulticastCreate(prop))
        step = "add device"
        ck(d.cuMulticastAddDevice(mc, dev))
        ap = d.CUmemAllocationProp()
        ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = 0
        ap.requestedHandleTypes = handle
        step = "mem create"
        mem = ck(d.cuMemCreate(prop.size, ap, 0))
        step = "bind"
        ck(d.cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0))
        print(handle, "one-device multicast object created and bound: OK (granularity %d)" % gran)
        return True
    except Exception as exc:
        print(handle, "failed at", step, exc)
        return False


for h in (d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
          d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC,
          d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE):
    if attempt(h):
        break

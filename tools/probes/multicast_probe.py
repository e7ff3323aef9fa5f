"""Probe CUDA multicast (NVLS) object creation on this box: which
(numDevices, size, handleTypes) cuMulticastCreate accepts."""
import json
from cuda.bindings import driver as cu

cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
err, ctx = cu.cuDevicePrimaryCtxRetain(dev)
cu.cuCtxSetCurrent(ctx)
out = {}
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    try:
        e, v = cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, attr), dev)
        out[attr] = (int(e), v)
    except Exception as x:
        out[attr] = str(x)
for nd in (1, 2):
    for ht in ("CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_FABRIC"):
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.handleTypes = getattr(cu.CUmemAllocationHandleType, ht)
        prop.size = 2 << 20
        e, g = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        e2, gmin = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        res = {"gran_rec": (int(e), g), "gran_min": (int(e2), gmin)}
        for size in sorted({gmin or (2 << 20), g or (2 << 20), 512 << 20}):
            prop.size = size
            e3, h = cu.cuMulticastCreate(prop)
            res[f"create_{size}"] = int(e3)
            if int(e3) == 0:
                e4, = cu.cuMulticastAddDevice(h, dev)
                res[f"add_{size}"] = int(e4)
                cu.cuMemRelease(h)
        out[f"nd{nd}_{ht}"] = res
print(json.dumps(out, indent=1))

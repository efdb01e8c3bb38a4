
import torch
torch.zeros(1, device="cuda")
from cuda.bindings import driver as cu
cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
err, ctx = cu.cuDevicePrimaryCtxRetain(dev); cu.cuCtxSetCurrent(ctx)
H = cu.CUmemAllocationHandleType
for nd in (1, 2):
    for ht in (H.CU_MEM_HANDLE_TYPE_NONE, H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, H.CU_MEM_HANDLE_TYPE_FABRIC):
        p = cu.CUmulticastObjectProp(); p.numDevices = nd; p.handleTypes = ht; p.size = 2 << 20
        e, gmin = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        e2, grec = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        p.size = max(int(grec), 2 << 20)
        r = cu.cuMulticastCreate(p)
        print("numDevices", nd, ht.name, "gran", e, gmin, e2, grec, "create:", r[0])

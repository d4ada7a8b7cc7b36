"""Probe cuMulticastCreate variants on this device (development helper)."""
import torch
import cuda.bindings.driver as d
torch.cuda.init(); torch.zeros(1, device="cuda")
print(d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0))
print("fabric", d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, 0))
print("posix", d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, 0))
for ht in [d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE, d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
           d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC]:
    for nd in (1, 2):
        p = d.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = ht
        p.size = 2 << 20
        e1, gmin = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        e2, grec = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        for size in (gmin, grec, 16 << 20):
            p.size = size
            e, h = d.cuMulticastCreate(p)
            print(ht.name, nd, "gran", e1, gmin, e2, grec, "size", size, "->", e)
            if e == d.CUresult.CUDA_SUCCESS:
                print("  add", d.cuMulticastAddDevice(h, 0))
                d.cuMemRelease(h)

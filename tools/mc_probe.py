#!/usr/bin/env python
"""Probe: can this box create an NVLS multicast object (driver API) and
torch symmetric memory with a multicast pointer at world size 1?"""
import os
import torch

from cuda.bindings import driver as cu

cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"]:
    a = getattr(cu.CUdevice_attribute, name, None)
    if a is None:
        print(name, "n/a")
        continue
    print(name, cu.cuDeviceGetAttribute(a, dev))
torch.cuda.init()
prop = cu.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 2 << 20
prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
print("granularity", cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
r = cu.cuMulticastCreate(prop)
print("cuMulticastCreate", r[0])
if r[0] == cu.CUresult.CUDA_SUCCESS:
    print("add device", cu.cuMulticastAddDevice(r[1], dev))
try:
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    t = symm.empty(1 << 20, dtype=torch.float32, device="cuda:0")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("symm ok; multicast_ptr", getattr(h, "multicast_ptr", None), "buffer_ptrs", getattr(h, "buffer_ptrs", None))
except Exception as ex:  # noqa: BLE001
    print("symm failed:", repr(ex)[:300])

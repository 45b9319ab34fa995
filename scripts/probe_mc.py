"""Probe (GPU box, torchrun): multicast / NVLS support for the K5 design."""
import os
import torch
import torch.distributed as dist

rank = int(os.environ.get("RANK", 0)); ws = int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
try:
    from cuda.bindings import driver as drv
except Exception:
    from cuda import cuda as drv
drv.cuInit(0)
err, dev = drv.cuDeviceGet(rank)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"]:
    a = getattr(drv.CUdevice_attribute, name, None)
    if a is None:
        print(rank, name, "n/a"); continue
    print(rank, name, drv.cuDeviceGetAttribute(a, dev))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1 << 20, dtype=torch.float32, device=f"cuda:{rank}")
    h = symm.rendezvous(t, dist.group.WORLD)
    print(rank, "symm ok multicast_ptr", hex(h.multicast_ptr), "buffer_ptrs", [hex(x) for x in h.buffer_ptrs])
except Exception as e:
    print(rank, "symm failed:", repr(e)[:300])
dist.barrier()
dist.destroy_process_group()

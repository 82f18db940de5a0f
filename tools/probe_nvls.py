"""Probe: multicast (NVLS) support per GPU and whether NCCL picks NVLS for AllReduce."""
import os
import sys

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
try:
    from cuda.bindings import driver as drv
except ImportError:
    from cuda import cuda as drv
drv.cuInit(0)
err, dev = drv.cuDeviceGet(rank)
err, mc = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
err2, fab = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
print(f"rank {rank}: multicast_supported={mc} (err {err}) fabric_handle={fab}", flush=True)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
x = torch.ones(1 << 20, device="cuda")
for _ in range(3):
    dist.all_reduce(x)
torch.cuda.synchronize()
print(f"rank {rank}: allreduce ok {x[0].item()}", flush=True)
dist.destroy_process_group()

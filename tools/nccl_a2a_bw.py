"""NCCL all_to_all_single bus bandwidth (nccl-tests convention busbw = algbw * (W-1)/W), one process
per GPU; the same bytes per peer as tools/p2p_bench.cu."""
import os
import sys

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
for mb in (20.0, 40.0, 80.0):
    n = int(mb * 1e6 / 4) * world
    x = torch.ones(n, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        dist.all_to_all_single(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    e0.record()
    for _ in range(10):
        dist.all_to_all_single(y, x)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e-3
    sent = 4 * n * (world - 1) / world  # bytes to remote peers
    if rank == 0:
        print(f"nccl all_to_all_single W={world} {mb:.0f} MB/peer: {t * 1e6:.1f} us, "
              f"{sent / t / 1e9:.0f} GB/s per GPU per direction (busbw)", flush=True)
dist.destroy_process_group()

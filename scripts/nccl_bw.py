"""NCCL bandwidth between the ranks of one node (torchrun): all_to_all_single
and paired P2P of bench-sized buffers."""
import os
import time

import torch
import torch.distributed as dist

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
P, me = dist.get_world_size(), dist.get_rank()
for mb in (96, 384, 1536):
    n = mb * (1 << 20) // 4
    a = torch.randn(n * P // P, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        dist.all_to_all_single(b, a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dist.all_to_all_single(b, a)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    sent = a.numel() * 4 * (P - 1) / P
    if me == 0:
        print(f"all_to_all_single {mb} MB/rank: {ms:.3f} ms  {sent / ms / 1e6:.0f} GB/s sent per rank", flush=True)
    peer = (me + 1) % P
    src = (me - 1) % P
    for _ in range(3):
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, a, peer), dist.P2POp(dist.irecv, b, src)]):
            w.wait()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, a, peer), dist.P2POp(dist.irecv, b, src)]):
            w.wait()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    if me == 0:
        print(f"p2p shift {mb} MB: {ms:.3f} ms  {a.numel() * 4 / ms / 1e6:.0f} GB/s per direction", flush=True)
dist.destroy_process_group()

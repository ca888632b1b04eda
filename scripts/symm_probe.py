"""Probe: torch symmetric memory on this box -- rendezvous, copy-engine push
into a peer buffer + put_signal / wait_signal, push bandwidth.
    torchrun --nproc-per-node 2 scripts/symm_probe.py"""
import os
import time
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
group = dist.group.WORLD.group_name
symm.enable_symm_mem_for_group(group)
n = 48 * 1024 * 1024            # 192 MB fp32 per peer slot
buf = symm.empty(world * n, dtype=torch.float32, device="cuda")
hdl = symm.rendezvous(buf, group)
print(rank, "rendezvous ok, signal pad", hdl.signal_pad_size, flush=True)
src = torch.full((n,), float(rank + 1), device="cuda")
cs = torch.cuda.Stream()
torch.cuda.synchronize()
dist.barrier()
for it in range(4):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        e0.record(cs)
        for k in range(1, world):
            q = (rank + k) % world
            peer = hdl.get_buffer(q, (n,), torch.float32, rank * n)
            peer.copy_(src)
            hdl.put_signal(q, channel=rank)
        e1.record(cs)
    for k in range(1, world):
        p = (rank - k) % world
        hdl.wait_signal(p, channel=p)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ok = all(float(buf[p * n:(p + 1) * n].min()) == p + 1 == float(buf[p * n:(p + 1) * n].max())
             for p in range(world) if p != rank)
    print(f"rank {rank} it {it}: pushed {(world - 1) * n * 4 / 1e9:.2f} GB in {ms:.2f} ms = "
          f"{(world - 1) * n * 4 / ms / 1e6:.0f} GB/s, data ok {ok}", flush=True)
    dist.barrier()
dist.destroy_process_group()

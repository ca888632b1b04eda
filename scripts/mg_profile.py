"""torch.profiler view of one multi-GPU bench epoch (torchrun, every rank):
how much of the step is compute, NCCL, and NCCL not hidden under compute.

    torchrun --nproc-per-node 2 scripts/mg_profile.py
"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P, me = dist.get_world_size(), dist.get_rank()
    from paper_2109_07893_b200.engine import Engine, NcclFabric
    cfg, g, data, train, params = bench.make_workload(P)
    eng = Engine(cfg, g, P, bench.NBLK, resident=True, fabric=NcclFabric())
    eng.set_labels(train.by_time, None)
    eng.params.load(params)
    count = train.total_pairs()

    def step():
        eng.epoch(None, None, None, count, "mean")
        eng.params.adam(0.01)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    iv = [(e.time_range.start, e.time_range.end, e.name) for e in ev]
    t0 = min(a for a, _, _ in iv)
    t1 = max(b for _, b, _ in iv)
    nccl = sorted((a, b) for a, b, n in iv if "nccl" in n.lower())
    comp = sorted((a, b) for a, b, n in iv if "nccl" not in n.lower() and "Memcpy" not in n and "Memset" not in n)

    def union(xs):
        out = []
        for a, b in xs:
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        return out

    uc, un = union(comp), union(nccl)
    tot = lambda u: sum(b - a for a, b in u)
    # NCCL time not overlapped by compute
    i = j = 0
    ov = 0.0
    while i < len(uc) and j < len(un):
        a, b = max(uc[i][0], un[j][0]), min(uc[i][1], un[j][1])
        if a < b:
            ov += b - a
        if uc[i][1] < un[j][1]:
            i += 1
        else:
            j += 1
    print(f"rank {me}: span {(t1 - t0) / 1e3:.1f} ms, compute busy {tot(uc) / 1e3:.1f} ms, "
          f"nccl busy {tot(un) / 1e3:.1f} ms, nccl overlapped {ov / 1e3:.1f} ms, "
          f"idle {((t1 - t0) - tot(union(sorted(comp + nccl)))) / 1e3:.1f} ms", flush=True)
    if me == 0:
        names = {}
        for a, b, n in iv:
            if "nccl" in n.lower():
                names[n[:60]] = names.get(n[:60], 0) + (b - a)
        for n, t in sorted(names.items(), key=lambda kv: -kv[1])[:5]:
            print(f"  {n}: {t / 1e3:.1f} ms")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

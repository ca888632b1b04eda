"""Multi-GPU (NCCL) parity check of the snapshot-partitioned epoch.

    python scripts/nccl_check.py --ref                 # 1 process: P emulated ranks (LocalFabric)
    torchrun --nproc-per-node P scripts/nccl_check.py  # P processes over NCCL

The first writes gpurun_out/nccl_ref_P.npz; the second runs the same epoch
with one rank per GPU (NcclFabric: all_to_all_single + all_reduce) and
compares loss, gradients and the communication ledger with it.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2109_07893_b200 as pk  # noqa: E402
from paper_2109_07893_b200.synth import churn_graph  # noqa: E402


def problem():
    g = churn_graph(20_000, 8, 30_000, 0.10, seed=5)
    cfg = pk.ModelConfig("cd-gcn", hidden_features=64, embed_features=64)
    data = pk.prepare_training_data(cfg, g)
    train, _ = pk.sample_link_prediction_sets(g, 0.1, 9)
    params = pk.init_params(cfg, 4)
    rng = np.random.default_rng(1)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    return cfg, data, train, params


def main():
    ref = "--ref" in sys.argv
    world = int(os.environ.get("WORLD_SIZE", "1"))
    P = int(sys.argv[sys.argv.index("--ref") + 1]) if ref and len(sys.argv) > sys.argv.index("--ref") + 1 else world
    out = ROOT / "gpurun_out" / f"nccl_ref_{P}.npz"
    if not ref:
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, data, train, params = problem()
    loss, grads, comm, tr = pk.distributed_epoch(cfg, data, train, params, P, 2)
    keys = sorted(grads)
    if ref:
        np.savez(out, loss=loss, units=comm.redistribution_units, events=len(comm.events),
                 **{"g_" + k: grads[k] for k in keys})
        print(f"ref P={P}: loss {loss!r} units {comm.redistribution_units}")
        return
    rank = torch.distributed.get_rank()
    r = np.load(out)
    worst = max(float(np.max(np.abs(grads[k] - r["g_" + k]))) / max(float(np.max(np.abs(r["g_" + k]))), 1e-30)
                for k in keys)
    # rank-local ledger: this process counts its own sends; the sum over ranks
    # is the emulated total
    units = torch.tensor([comm.redistribution_units], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(units)
    ok_loss = abs(loss - float(r["loss"])) <= 1e-12 * max(1.0, abs(float(r["loss"])))
    print(f"rank {rank}: loss {loss!r} (ref {float(r['loss'])!r}) worst grad rel diff {worst:.3e} "
          f"units {int(units.item())} (ref {int(r['units'])})", flush=True)
    ok = ok_loss and worst <= 1e-12 and int(units.item()) in (int(r["units"]), int(r["units"]) * P)
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()
    if not ok:
        raise SystemExit(f"rank {rank}: NCCL epoch differs from the emulated-rank epoch")
    if rank == 0:
        print("NCCL parity OK")


if __name__ == "__main__":
    main()

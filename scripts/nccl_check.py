"""Multi-GPU parity check of the snapshot-partitioned epoch: one process
per GPU vs the same P ranks emulated in one process.

    python scripts/nccl_check.py --ref P                 # 1 process: P emulated ranks (LocalFabric)
    torchrun --nproc-per-node P scripts/nccl_check.py    # P processes (peer pushes or NCCL)

The first writes gpurun_out/nccl_ref_P_<case>.npz for every case; the
second runs the same two epochs (host Adam in between, so the second epoch
reuses the kept snapshots, the head chain and the label cache) with one rank
per GPU and compares loss, gradients and the communication ledger.  Cases:
hidden = embed = 64 (the bench widths) and hidden 32 / embed 64 (layer 1's
input narrower than its output: the seed buffers of the two layers differ
in width), cd-gcn; tm-gcn and egcn-o at hidden 32.  Transport: DGNN_EXCHANGE=peer
(default) or nccl.  Results: gpurun_out/nccl_check_P_<transport>.json.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2109_07893_b200 as pk  # noqa: E402
from paper_2109_07893_b200.synth import churn_graph  # noqa: E402

CASES = {"cd64": ("cd-gcn", 64, 64), "cd32x64": ("cd-gcn", 32, 64), "tm32": ("tm-gcn", 32, 32),
         "eg32": ("egcn-o", 32, 32)}


def problem(arch, hidden, embed):
    g = churn_graph(20_000, 8, 30_000, 0.10, seed=5)
    cfg = pk.ModelConfig(arch, hidden_features=hidden, embed_features=embed)
    data = pk.prepare_training_data(cfg, g)
    train, _ = pk.sample_link_prediction_sets(g, 0.1, 9)
    params = pk.init_params(cfg, 4)
    rng = np.random.default_rng(1)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    return cfg, data, train, params


def two_epochs(cfg, data, train, params, P):
    out = []
    st = pk.init_adam(params)
    p = {k: v.copy() for k, v in params.items()}
    for _ in range(2):
        comm, tr = pk.CommLedger(), pk.TransferLedger()
        loss, grads, comm, tr = pk.distributed_epoch(cfg, data, train, p, P, 2, comm=comm, transfer=tr)
        out.append((loss, grads, comm, tr))
        pk.adam_step(p, grads, st, 0.01)
    return out


def main():
    ref = "--ref" in sys.argv
    world = int(os.environ.get("WORLD_SIZE", "1"))
    P = int(sys.argv[sys.argv.index("--ref") + 1]) if ref else world
    transport = os.environ.get("DGNN_EXCHANGE", "peer")
    if not ref:
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    report = {"P": P, "transport": transport, "cases": {}}
    ok_all = True
    for case, (arch, hidden, embed) in CASES.items():
        cfg, data, train, params = problem(arch, hidden, embed)
        res = two_epochs(cfg, data, train, params, P)
        pk.api.clear_engines()
        path = ROOT / "gpurun_out" / f"nccl_ref_{P}_{case}.npz"
        keys = sorted(res[0][1])
        if ref:
            np.savez(path, **{f"e{e}_loss": r[0] for e, r in enumerate(res)},
                     **{f"e{e}_units": r[2].redistribution_units for e, r in enumerate(res)},
                     **{f"e{e}_g_{k}": r[1][k] for e, r in enumerate(res) for k in keys})
            print(f"ref P={P} {case}: losses {[r[0] for r in res]}", flush=True)
            continue
        rank = torch.distributed.get_rank()
        r = np.load(path)
        ent = {}
        for e, (loss, grads, comm, tr) in enumerate(res):
            worst = max(float(np.max(np.abs(grads[k] - r[f"e{e}_g_{k}"])))
                        / max(float(np.max(np.abs(r[f"e{e}_g_{k}"]))), 1e-30) for k in keys)
            units = torch.tensor([comm.redistribution_units], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(units)
            h2d = torch.tensor([tr.h2d_bytes, tr.full_built_bytes, tr.full_equiv_bytes], dtype=torch.float64,
                               device="cuda")
            torch.distributed.all_reduce(h2d)
            ok_loss = abs(loss - float(r[f"e{e}_loss"])) <= 1e-12 * max(1.0, abs(float(r[f"e{e}_loss"])))
            ok = ok_loss and worst <= 1e-12 and int(units.item()) in (int(r[f"e{e}_units"]),
                                                                        int(r[f"e{e}_units"]) * P)
            ok_all &= ok
            ent[f"epoch{e + 1}"] = {"loss": loss, "ref_loss": float(r[f"e{e}_loss"]), "worst_grad_rel_diff": worst,
                                    "units": int(units.item()), "ref_units": int(r[f"e{e}_units"]),
                                    "h2d_bytes": int(h2d[0].item()), "full_built_bytes": int(h2d[1].item()),
                                    "full_equiv_bytes": int(h2d[2].item()), "ok": ok}
            print(f"rank {rank} {case} epoch {e + 1}: loss {loss!r} (ref {float(r[f'e{e}_loss'])!r}) "
                  f"worst grad rel diff {worst:.3e} units {int(units.item())} ok={ok}", flush=True)
        report["cases"][case] = ent
    if ref:
        return
    rank = torch.distributed.get_rank()
    flags = torch.tensor([0.0 if ok_all else 1.0], device="cuda")
    torch.distributed.all_reduce(flags)
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()
    if rank == 0:
        report["all_ranks_ok"] = flags.item() == 0
        (ROOT / "gpurun_out" / f"nccl_check_{P}_{transport}.json").write_text(json.dumps(report, indent=1))
    if not ok_all:
        raise SystemExit(f"rank {rank}: the multi-process epoch differs from the emulated-rank epoch")
    if rank == 0:
        print(f"multi-process parity OK (P={P}, {transport})")


if __name__ == "__main__":
    main()

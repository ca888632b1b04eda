"""World-size-2 `gloo` tests (CPU) of the multi-rank host logic.

The engine's NCCL fabric (`engine.NcclFabric`) moves the snapshot-major
"owner layout" [dest q][owned step c][N/P][W] of every rank onto the
vertex-major [block step t][N/P][W] of every other rank with one equal-split
all_to_all_single and sums gradients with all_reduce (`dist.py:505-589`,
SnapshotPartition `dist.py:125-162`).  Here two real processes run the same
fabric calls over gloo on CPU tensors and the result is checked against the
single-process emulation (`LocalFabric`) and against the reference's
ownership semantics: on rank q, vertex-major step t = p * chunk + c holds
rank p's owned step c rows for q's vertex chunk.
"""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_07893_b200.engine import LocalFabric, NcclFabric, Plan

WORLD = 2


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _owner_buffer(plan: Plan, p: int, W: int) -> torch.Tensor:
    """Rank p's owner layout, every element encoding (p, q, c, row, col)."""
    P, C, NP = plan.P, plan.chunk, plan.NP
    q, c, v, k = np.meshgrid(np.arange(P), np.arange(C), np.arange(NP), np.arange(W), indexing="ij")
    code = (((p * 10 + q) * 10 + c) * 1000 + v) * 100 + k
    return torch.from_numpy(code.astype(np.float64).reshape(-1))


def _worker(rank, port, W, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        plan = Plan(T=8, P=WORLD, nblk=2, N=6)
        src = _owner_buffer(plan, rank, W)
        dst = torch.zeros_like(src)
        count = plan.chunk * plan.NP * W
        fab = NcclFabric()
        fab.exchange([rank], lambda r: src, lambda r: dst, count)
        g = torch.arange(5, dtype=torch.float64) * (rank + 1)
        red = fab.allreduce([g])
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), dst=dst.numpy(), red=red.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W", [4, 12])
def test_gloo_exchange_matches_emulation_and_ownership(W):
    plan = Plan(T=8, P=WORLD, nblk=2, N=6)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(_free_port(), W, d), nprocs=WORLD, join=True)
        got = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(WORLD)]
    # single-process emulation of the same exchange
    srcs = [_owner_buffer(plan, p, W) for p in range(WORLD)]
    dsts = [torch.zeros_like(s) for s in srcs]
    LocalFabric().exchange(list(range(WORLD)), lambda r: srcs[r], lambda r: dsts[r], plan.chunk * plan.NP * W)
    for q in range(WORLD):
        assert np.array_equal(got[q]["dst"], dsts[q].numpy())
        # ownership semantics: vertex-major step t = p*chunk + c comes from rank p's owned step c
        vm = got[q]["dst"].reshape(plan.bsize, plan.NP, W)
        for t in range(plan.bsize):
            p, c = plan.owner_of(t), t % plan.chunk
            assert p * plan.chunk + c == t
            want = _owner_buffer(plan, p, W).numpy().reshape(WORLD, plan.chunk, plan.NP, W)[q, c]
            assert np.array_equal(vm[t], want)
        # all-reduce: rank-order sum, identical on every rank
        assert np.array_equal(got[q]["red"], np.arange(5) * 3.0)


def test_plan_partition_matches_reference_rules():
    """SnapshotPartition (dist.py:125-162): contiguous ownership per block,
    every step owned once, divisibility errors as in the reference."""
    plan = Plan(T=32, P=4, nblk=4, N=1000)
    owned = sorted(t for p in range(4) for t in plan.owned(p))
    assert owned == list(range(32))
    for p in range(4):
        for t in plan.owned(p):
            assert plan.owner_of(t) == p
    from paper_2109_07893_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        Plan(T=32, P=3, nblk=4, N=999)
    with pytest.raises(ConfigError):
        Plan(T=30, P=2, nblk=4, N=1000)

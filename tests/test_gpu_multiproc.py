"""One process per GPU (torchrun, NCCL + symmetric memory) against the same
ranks emulated in one process: two epochs of cd-gcn (hidden = embed and
hidden < embed), tm-gcn and egcn-o, peer-push and NCCL transports
(scripts/nccl_check.py).  Needs >= 2 GPUs; skipped on a one-GPU box (the
committed results of the 2- and 4-GPU runs are in profiles/r02_parity/)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_two_processes_equal_emulated_ranks(transport):
    env = dict(os.environ, DGNN_EXCHANGE=transport, CUDA_VISIBLE_DEVICES="0,1")
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    subprocess.run([sys.executable, "scripts/nccl_check.py", "--ref", "2"], cwd=ROOT, env=env, check=True,
                   timeout=900)
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                    "--master-addr", "127.0.0.1", "--master-port", "29811", "scripts/nccl_check.py"],
                   cwd=ROOT, env=env, check=True, timeout=900)
    rep = json.loads((ROOT / "gpurun_out" / f"nccl_check_2_{transport}.json").read_text())
    assert rep["all_ranks_ok"]
    assert set(rep["cases"]) == {"cd64", "cd32x64", "tm32", "eg32"}

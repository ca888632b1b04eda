"""Time K3 (dgnn_gcn_forward, aggregation + transform + ReLU, skip cell) at
the configs[1] layer-1 shape: N = 750k, nnz = 1.22M (self loops + 468,750
random edges), F = H = 64, X larger than L2 (L2 flushed between launches).
DGNN_LIB_PATH selects a library variant (scripts/gcn_fwd_roles.sh)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2109_07893_b200 import _lib
from paper_2109_07893_b200._lib import call, ptr

dev = torch.device("cuda", 0)
C3 = "--c3" in sys.argv
n, m, F, H = (1_000_000, 2_000_000, 32, 32) if C3 else (750_000, 468_750, 64, 64)
rng = np.random.default_rng(1)
if C3:   # configs[2]: AMLSim-style heavy-tailed snapshot, plain cell
    from paper_2109_07893_b200.synth import aml_graph
    g0 = aml_graph(n, 1, m, 0.02, seed=1).snapshots[0]
    src, dst = np.asarray(g0.rows), np.asarray(g0.cols)
else:
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
rows = np.concatenate([np.arange(n), src])
cols = np.concatenate([np.arange(n), dst])
order = np.lexsort((cols, rows))
rows, cols = rows[order], cols[order]
rowptr = np.zeros(n + 1, np.int32)
np.add.at(rowptr, rows + 1, 1)
rowptr = np.cumsum(rowptr).astype(np.int32)
rp = torch.from_numpy(rowptr).to(dev)
col = torch.from_numpy(cols.astype(np.int32)).to(dev)
val = torch.rand(len(cols), device=dev) * 0.5
x = torch.randn(n, F, device=dev)
w = torch.randn(F, H, device=dev) * 0.2
SKIP = 0 if C3 else 1
s_out = torch.empty(n, F, device=dev)
r_out = torch.empty(n, F * SKIP + H, device=dev)
flush = torch.empty(1 << 28, device=dev)
st = _lib.stream_handle()
ts = []
for it in range(12):
    flush.fill_(it)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    call("dgnn_gcn_forward", n, ptr(rp), ptr(col), ptr(val), _lib.frame(x, F), F, ptr(w), H, SKIP,
         _lib.frame(s_out, F), _lib.frame(r_out, F * SKIP + H), st)
    b.record()
    torch.cuda.synchronize()
    if it >= 2:
        ts.append(a.elapsed_time(b) * 1e3)
nnz = len(cols)
byts = 4 * (n + 1) + 8 * nnz + 4 * F * nnz + 4 * n * (F + F * SKIP + H)
us = float(np.median(ts))
print(f"{'c3 ' if C3 else ''}{os.path.basename(os.environ.get('DGNN_LIB_PATH', 'libdgnn_b200.so'))}: {us:.1f} us  "
      f"{byts / us / 1e3:.0f} GB/s (gather-inclusive)")

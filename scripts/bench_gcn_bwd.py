"""Time the GCN backward pieces (tcgen05 vs SIMT) at the bench shapes."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2109_07893_b200 import _lib
from paper_2109_07893_b200._lib import call, ptr, query

dev = torch.device("cuda", 0)
n = 750_000
for fp, hp, skip in ((64, 64, True), (4, 64, True)):
    rw = fp + hp
    dr = torch.randn(n, rw, device=dev)
    r = torch.relu(torch.randn(n, rw, device=dev))
    s = torch.randn(n, fp, device=dev)
    w = torch.randn(fp, hp, device=dev) * 0.2
    ds = torch.empty(n, fp, device=dev)
    gw = torch.zeros(fp * hp, dtype=torch.float64, device=dev)
    ws = torch.empty(query("dgnn_gcn_weight_grad_workspace", fp, hp), dtype=torch.uint8, device=dev)
    st = _lib.stream_handle()
    for tc in (1, 0):
        call("dgnn_set_gcn_tensor_cores", tc)
        for what in ("dw", "rows"):
            if what == "rows" and fp < 16:
                continue
            def run():
                if what == "dw":
                    call("dgnn_gcn_weight_grad", n, _lib.frame(s, fp), _lib.frame(dr, rw), _lib.frame(r, rw), fp, hp,
                         int(skip), ptr(gw), ptr(ws), ws.numel(), st)
                else:
                    call("dgnn_gcn_backward_rows", n, _lib.frame(dr, rw), _lib.frame(r, rw), fp, ptr(w), hp,
                         int(skip), _lib.frame(ds, fp), st)
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                run()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            byts = 4 * n * ((fp + 2 * hp) if what == "dw" else (2 * rw + fp))
            print(f"fp={fp} hp={hp} tc={tc} {what}: {us:.1f} us  {byts / us / 1e3:.0f} GB/s", flush=True)
call("dgnn_set_gcn_tensor_cores", 1)

# SpMM: gather pipeline (tcgen05 flag on) vs SIMT, avg degree ~1.6 (bench shape)
rng = np.random.default_rng(0)
nnz = int(1.62 * n)
rows = np.sort(rng.integers(0, n, size=nnz))
cols = rng.integers(0, n, size=nnz).astype(np.int32)
rp = torch.from_numpy(np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))]).astype(np.int32)).to(dev)
cd = torch.from_numpy(cols).to(dev)
vd = torch.rand(nnz, device=dev)
for f in (64,):
    x = torch.randn(n, f, device=dev)
    out = torch.empty(n, f, device=dev)
    for tc in (1, 0):
        call("dgnn_set_gcn_tensor_cores", tc)
        run = lambda: call("dgnn_spmm_f32", n, ptr(rp), ptr(cd), ptr(vd), _lib.frame(x, f), f, _lib.frame(out, f), st)
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        byts = 4 * (n + 1) + 8 * nnz + 4 * f * nnz + 4 * n * f
        print(f"spmm f={f} tc={tc}: {us:.1f} us  {byts / us / 1e3:.0f} GB/s (gather-incl.)", flush=True)
call("dgnn_set_gcn_tensor_cores", 1)

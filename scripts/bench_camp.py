"""Does the relative offset of dr and r (same layout) change the GCN
backward kernels' bandwidth?  (channel conflicts between arrays walked in
lockstep)"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2109_07893_b200 import _lib
from paper_2109_07893_b200._lib import call, ptr, query

dev = torch.device("cuda", 0)
n, fp, hp = 750_000, 64, 64
rw = fp + hp
w = torch.randn(fp, hp, device=dev) * 0.2
ds = torch.empty(n, fp, device=dev)
gw = torch.zeros(fp * hp, dtype=torch.float64, device=dev)
ws = torch.empty(query("dgnn_gcn_weight_grad_workspace", fp, hp), dtype=torch.uint8, device=dev)
st = _lib.stream_handle()
for shift in (0, 64, 128, 256, 512, 1024, 4096, 65536 + 256, 1 << 20, (1 << 20) + 4096 + 256):
    big = torch.empty(2 * n * rw + shift // 4 + 1024, device=dev)
    dr = big[: n * rw].view(n, rw)
    r = big[n * rw + shift // 4: n * rw + shift // 4 + n * rw].view(n, rw)
    dr.normal_()
    r.normal_().relu_()
    sbig = torch.empty(n * fp + 8192 + shift // 4, device=dev)
    s = sbig[shift // 4 + 4096: shift // 4 + 4096 + n * fp].view(n, fp).normal_()
    res = []
    for what in ("dw", "rows"):
        def run():
            if what == "dw":
                call("dgnn_gcn_weight_grad", n, _lib.frame(s, fp), _lib.frame(dr, rw), _lib.frame(r, rw), fp, hp, 1,
                     ptr(gw), ptr(ws), ws.numel(), st)
            else:
                call("dgnn_gcn_backward_rows", n, _lib.frame(dr, rw), _lib.frame(r, rw), fp, ptr(w), hp, 1,
                     _lib.frame(ds, fp), st)
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 10 * 1e3)
    print(f"shift {shift:8d}: dw {res[0]:6.1f} us  rows {res[1]:6.1f} us", flush=True)
    del big, sbig, dr, r, s
# plain copy rate for reference
a = torch.empty(n * rw * 2, device=dev); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): b.copy_(a)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 10 * 1e3
print(f"copy {a.numel()*4/1e6:.0f} MB: {us:.1f} us  {2*a.numel()*4/us/1e3:.0f} GB/s")

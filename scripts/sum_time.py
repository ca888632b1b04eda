"""Time dgnn_sum_f64 (CUDA events) at the per-step pair counts of configs[1]/[2]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_07893_b200 import _lib
from paper_2109_07893_b200._lib import call, ptr
dev = torch.device("cuda", 0)
st = _lib.stream_handle()
out = torch.zeros(1, dtype=torch.float64, device=dev)
for n in (90_000, 400_000, 1_000_000, 4_000_000):
    x = torch.randn(n, dtype=torch.float64, device=dev)
    for _ in range(5):
        call("dgnn_sum_f64", n, ptr(x), out.data_ptr(), 0, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(100):
        call("dgnn_sum_f64", n, ptr(x), out.data_ptr(), 0, st)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n}: {e0.elapsed_time(e1) * 10:.1f} us per call (L2-warm)")

"""Time dgnn_head_loss_grad (CUDA events, isolated) at the configs[1] shape
(750k vertices, E = 64, 94k pairs per step) and the configs[2] shape (1M
vertices, E = 32, 400k pairs).  DGNN_LIB_PATH selects the library (A/B)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_07893_b200 import _lib
from paper_2109_07893_b200._lib import call, ptr, query
dev = torch.device("cuda", 0)
st = _lib.stream_handle()
g = torch.Generator(device=dev).manual_seed(1)
for n, ep, npairs in ((750_000, 64, 94_000), (1_000_000, 32, 400_000)):
    z = torch.randn(n * ep, device=dev, generator=g)
    u = torch.randint(0, n, (npairs,), device=dev, dtype=torch.int32, generator=g)
    v = torch.randint(0, n, (npairs,), device=dev, dtype=torch.int32, generator=g)
    y = torch.randint(0, 2, (npairs,), device=dev, dtype=torch.int32, generator=g)
    hw = torch.randn(2 * ep * 2, device=dev, generator=g) * 0.1
    hb = torch.zeros(2, device=dev)
    lpp = torch.empty(npairs, dtype=torch.float64, device=dev)
    dlg = torch.empty(2 * npairs, dtype=torch.float64, device=dev)
    ghw = torch.zeros(2 * ep * 2, dtype=torch.float64, device=dev)
    ghb = torch.zeros(2, dtype=torch.float64, device=dev)
    ws = torch.empty(query("dgnn_head_grad_workspace", ep, 2), dtype=torch.uint8, device=dev)
    fr = _lib.Frame(z.data_ptr(), ep, 0, 0)
    args = (npairs, ptr(u), ptr(v), ptr(y), fr, ep, 2, ptr(hw), ptr(hb), 1.0 / npairs, ptr(lpp), npairs, ptr(dlg),
            ptr(ghw), ptr(ghb), ptr(ws), ws.numel(), st)
    for _ in range(5):
        call("dgnn_head_loss_grad", *args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        call("dgnn_head_loss_grad", *args)
    e1.record()
    torch.cuda.synchronize()
    print(f"{os.path.basename(str(_lib.LIB_PATH))} n={n} ep={ep} pairs={npairs}: {e0.elapsed_time(e1) * 20:.1f} us per call"
          f"  loss[0..2]={lpp[:2].tolist()}")

"""Precision of the tcgen05 3xTF32 mainloop vs fp64 and vs plain fp32."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2109_07893_b200.ops import tc_gemm
rng = np.random.default_rng(0)
for k in (192, 1024, 4096):
    m, n = 2048, 256
    a = rng.standard_normal((m, k)).astype(np.float32)
    w = rng.standard_normal((n, k)).astype(np.float32)
    ref = a.astype(np.float64) @ w.astype(np.float64).T
    scale = np.abs(a).astype(np.float64) @ np.abs(w).astype(np.float64).T
    got = tc_gemm(a, w)
    f32 = (torch.from_numpy(a).cuda() @ torch.from_numpy(w).cuda().T)
    torch.backends.cuda.matmul.allow_tf32 = False
    f32 = (torch.from_numpy(a).cuda().double().float() @ torch.from_numpy(w).cuda().T).double().cpu().numpy()
    for name, x in (("tc3xtf32", got), ("fp32", f32)):
        e = (x - ref) / scale
        print(f"k={k:5d} {name:9s} max|e|={np.abs(e).max():.2e} mean(e)={e.mean():+.2e} rms={np.sqrt((e**2).mean()):.2e}")
    # positive-only data: bias shows up
    ap, wp = np.abs(a), np.abs(w)
    refp = ap.astype(np.float64) @ wp.astype(np.float64).T
    gp = tc_gemm(ap, wp)
    print(f"k={k:5d} positive  rel bias={(gp / refp - 1).mean():+.2e} max={np.abs(gp / refp - 1).max():.2e}")

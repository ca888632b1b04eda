import sys, os
import numpy as np
sys.path.insert(0, ".")
from paper_2109_07893_b200.ops import lstm_weight_grad_tc
hp, kx = 64, 128
rows = 16
for (r0, j0, k0) in ((0, 0, 0), (0, 5, 7), (3, 17, 33), (9, 130, 150), (15, 255, 191)):
    x = np.zeros((rows, kx), np.float32); h = np.zeros((rows, hp), np.float32)
    dz = np.zeros((rows, 4 * hp), np.float32)
    if k0 < kx: x[r0, k0] = 1.0
    else: h[r0, k0 - kx] = 1.0
    dz[r0, j0] = 1.0
    gw, gb = lstm_weight_grad_tc(x, h, h, dz, rows)
    nz = np.argwhere(gw != 0)
    print((r0, j0, k0), "nonzeros (k, j):", nz[:8].tolist(), "vals", gw[gw != 0][:8])

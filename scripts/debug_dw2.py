import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2109_07893_b200.ops import lstm_weight_grad_tc
hp, kx = 64, 128
for rows in (16, 32, 48, 64, 512, 528):
    x = np.ones((rows, kx), np.float32)
    h = np.ones((rows, hp), np.float32)
    h0 = np.ones((rows, hp), np.float32)
    dz = np.ones((rows, 4 * hp), np.float32)
    gw, gb = lstm_weight_grad_tc(x, h, h0, dz, rows)
    vals, counts = np.unique(gw, return_counts=True)
    print(rows, "unique values", list(zip(vals[:6], counts[:6])), "db", gb[:2])
# row-dependent data: dz row r = r+1 -> sum identifies which rows were counted
rows = 64
x = np.ones((rows, kx), np.float32); h = np.ones((rows, hp), np.float32)
dz = np.repeat(np.arange(1, rows + 1, dtype=np.float32)[:, None], 4 * hp, 1)
gw, gb = lstm_weight_grad_tc(x, h, h, dz, rows)
print("rowsum check: got", np.unique(gw)[:5], "expected", dz[:, 0].sum())
# column dependent: x column k = k+1, dz = 1 -> gw[k][j] = rows*(k+1)
x = np.repeat(np.arange(1, kx + 1, dtype=np.float32)[None, :], rows, 0)
gw, gb = lstm_weight_grad_tc(x, np.zeros((rows, hp), np.float32), np.zeros((rows, hp), np.float32),
                             np.ones((rows, 4 * hp), np.float32), rows)
print("k-dependence: got col j=0 for k=0..20:", gw[:20, 0] / rows)
print("j-dependence: got row k=5 for j=0..20:", gw[5, :20] / rows)

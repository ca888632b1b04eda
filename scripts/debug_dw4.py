import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2109_07893_b200.ops import lstm_weight_grad_tc
hp, kx, rows = 64, 128, 16
x = np.ones((rows, kx), np.float32); h = np.ones((rows, hp), np.float32); dz = np.ones((rows, 4 * hp), np.float32)
gw, gb = lstm_weight_grad_tc(x, h, h, dz, rows)
print("gw[0,0:4]", gw[0, :4], "gw[0:4,0]", gw[:4, 0], "unique", np.unique(gw)[:8])

"""Debug: per-epoch parameter trajectory of train_distributed vs the oracle."""
import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import dtgnn_oracle as O
import paper_2109_07893_b200 as pk
from conftest import load, jload, labels_from
from helpers import product_case

fx, cfg, data, train, test, _ = product_case("cdgcn_small")
n = int(fx["g_n"]); T = int(fx["g_T"])
snaps = [O.Coo(n, fx[f"g_rows{t}"], fx[f"g_cols{t}"], fx[f"g_vals{t}"]) for t in range(T)]
ocfg = O.Cfg("cd-gcn", 2, 8, 8)
P = O.prepare(ocfg, snaps)
params = O.init_params(ocfg, 3)
st = O.adam_state(params)
mine = {k: v.copy() for k, v in params.items()}
mst = pk.init_adam(mine)
for e in range(3):
    loss, g, _, _ = O.distributed_epoch(ocfg, P, train.by_time, params, 2, 2)
    l2, g2, _, _ = pk.distributed_epoch(cfg, data, train, mine, 2, 2)
    print("epoch", e + 1, "loss", loss, l2, (l2 - loss) / loss)
    for k in sorted(g):
        d = np.abs(g[k] - g2[k])
        print(f"  grad {k:12s} max|ref| {np.abs(g[k]).max():.3e} maxdiff {d.max():.3e} "
              f"min|ref| {np.abs(g[k]).min():.3e}")
    O.adam(params, g, st, 0.01)
    pk.adam_step(mine, g2, mst, 0.01)
    for k in sorted(params):
        print(f"  param {k:12s} maxdiff {np.abs(params[k] - mine[k]).max():.3e}")

"""Debug the tcgen05 weight-gradient kernel: error structure vs fp64."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2109_07893_b200.ops import lstm_weight_grad_tc
hp, kx = int(sys.argv[1]), int(sys.argv[2])
for np_rows, steps in ((16, 1), (8, 2), (1024, 1), (20000, 3)):
    rng = np.random.default_rng(1)
    rows = np_rows * steps
    x = rng.standard_normal((rows, kx)).astype(np.float32)
    h = rng.standard_normal((rows, hp)).astype(np.float32)
    h0 = rng.standard_normal((np_rows, hp)).astype(np.float32)
    dz = rng.standard_normal((rows, 4 * hp)).astype(np.float32)
    gw, gb = lstm_weight_grad_tc(x, h, h0, dz, np_rows)
    hprev = np.concatenate([h0, h[:-np_rows]]).astype(np.float64) if steps > 1 else h0.astype(np.float64)
    xcat = np.concatenate([x.astype(np.float64), hprev], axis=1)
    ref = xcat.T @ dz.astype(np.float64)
    err = np.abs(gw - ref) / (np.abs(xcat).T @ np.abs(dz.astype(np.float64)))
    print(f"hp={hp} kx={kx} rows={rows}: max rel err {err.max():.3e}; db err {np.abs(gb - dz.sum(0)).max():.2e}")
    if err.max() > 1e-4:
        K = kx + hp
        blk = err.reshape(K, 4 * hp)
        # per (16-col k atom, 16-col j atom)
        bad = [(i, j, float(blk[16*i:16*i+16, 16*j:16*j+16].max())) for i in range((K + 15)//16) for j in range(4*hp//16)]
        print("   worst blocks (katom, jatom, err):", sorted(bad, key=lambda t: -t[2])[:6])
        print("   good blocks:", sum(1 for b in bad if b[2] < 1e-4), "of", len(bad))
        # is the result a permutation of the reference? check correlation with transposed-ish variants
        print("   sample got/ref row0:", gw[0, :4], ref[0, :4])

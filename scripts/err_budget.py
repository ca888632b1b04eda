"""Measured error budget of the engine (GPU): for every gradient tensor, the
absolute floor (as a fraction of ||r||_inf) that the guarded 1e-4 relative
check needs, for the tcgen05 engine and the SIMT A/B engine.

    python scripts/err_budget.py [--out gpurun_out/err_budget.json]

needed_atol_frac = max_i max(0, |g_i - r_i| - 1e-4 max(|g_i|, |r_i|)) / ||r||_inf
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tests", ROOT / "oracle"):
    sys.path.insert(0, str(p))


def budget(got: dict, ref: dict, rtol=1e-4):
    out = {}
    for k in sorted(ref):
        g, r = np.asarray(got[k], np.float64), np.asarray(ref[k], np.float64)
        scale = float(np.abs(r).max()) if r.size else 0.0
        ex = np.maximum(0.0, np.abs(g - r) - rtol * np.maximum(np.abs(g), np.abs(r)))
        out[k] = {"needed_atol_frac": float(ex.max() / scale) if scale else 0.0,
                  "norm_rel": float(np.linalg.norm(g - r) / (np.linalg.norm(r) + 1e-300))}
    return out


def cases():
    import paper_2109_07893_b200 as pk
    import dtgnn_oracle as O
    from conftest import params_from
    from helpers import product_case
    from paper_2109_07893_b200.synth import churn_graph
    for name in ("cdgcn_small", "tmgcn_small"):
        fx, cfg, data, train, _, params = product_case(name)
        yield name, (lambda cfg=cfg, data=data, train=train, params=params:
                     pk.distributed_epoch(cfg, data, train, params, 2, 2)[:2]), \
            float(fx["dist2x2_loss"]), params_from(fx, "dist2x2_g_")
    g = churn_graph(20_000, 8, 30_000, 0.10, seed=5)
    for H in (32, 64):
        cfg = pk.ModelConfig("cd-gcn", hidden_features=H, embed_features=H)
        data = pk.prepare_training_data(cfg, g)
        train, _ = pk.sample_link_prediction_sets(g, 0.1, 9)
        params = pk.init_params(cfg, 4)
        rng = np.random.default_rng(1)
        params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
        ocfg = O.Cfg("cd-gcn", 2, H, H)
        Pp = O.prepare(ocfg, [O.Coo(s.dim, s.rows, s.cols, s.vals) for s in g.snapshots])
        lo, go = O.backward_checkpoint(ocfg, Pp, train.by_time, params, 2)
        yield f"mid20k_H{H}", (lambda cfg=cfg, data=data, train=train, params=params:
                               pk.backward_checkpoint(cfg, data, train, params, 2)), lo, go


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "err_budget.json"))
    args = ap.parse_args()
    import paper_2109_07893_b200 as pk
    res = {}
    for name, run, ref_loss, ref_g in cases():
        for tc in (True, False):
            pk.api.TENSOR_CORES = tc
            loss, grads = run()
            pk.api.clear_engines()
            b = budget(grads, ref_g)
            tag = f"{name}/{'tcgen05' if tc else 'simt'}"
            res[tag] = {"loss_rel": abs(loss - ref_loss) / abs(ref_loss),
                        "worst_needed_atol_frac": max(v["needed_atol_frac"] for v in b.values()),
                        "tensors": b}
            print(tag, f"loss_rel {res[tag]['loss_rel']:.2e}",
                  f"worst atol_frac {res[tag]['worst_needed_atol_frac']:.2e}",
                  " ".join(f"{k}:{v['needed_atol_frac']:.1e}" for k, v in b.items() if v["needed_atol_frac"] > 1e-6))
    pk.api.TENSOR_CORES = True
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

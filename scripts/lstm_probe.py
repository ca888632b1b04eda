"""Time the temporal-stage kernels alone at the bench shapes (GPU):
K5 forward step with / without the gate cache, K6 backward step, the block
weight gradient -- per layer of configs[1] (rows 750k, hidden 64) or any
(rows, kx, hp) -- with the 3xTF32 and HBM floors of each launch.

    python scripts/lstm_probe.py [--rows 750000] [--hp 64] [--kx 68,128] [--steps 8]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2109_07893_b200 import _lib  # noqa: E402
from paper_2109_07893_b200._lib import call, ptr, query  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=750_000)
    ap.add_argument("--hp", type=int, default=64)
    ap.add_argument("--kx", default="68,128")
    ap.add_argument("--steps", type=int, default=8, help="block steps for the weight gradient")
    args = ap.parse_args()
    pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(pk.get("hbm_gbs", 6650.0))
    tf = float(pk.get("bf16_tflops", 1590.0)) / 6
    dev = torch.device("cuda", 0)
    st = _lib.stream_handle()
    n, hp = args.rows, args.hp
    out = {}
    for kx in (int(k) for k in args.kx.split(",")):
        K = kx + hp
        N4 = 4 * hp
        x = torch.randn(n, kx, device=dev) * 0.5
        h = torch.randn(n, hp, device=dev) * 0.5
        c = torch.randn(n, hp, device=dev) * 0.5
        w = torch.randn(K, N4, device=dev) * 0.1
        wt = w.t().contiguous()
        img = torch.zeros(query("dgnn_tc_weight_image_bytes", N4, K) // 4, device=dev)
        call("dgnn_tc_weight_image", N4, K, ptr(wt), K, ptr(img), st)
        nb = (K + 15) // 16 * 16
        bimg = torch.zeros(query("dgnn_tc_weight_image_bytes", nb, N4) // 4, device=dev)
        call("dgnn_tc_weight_image_ex", nb, K, N4, ptr(w), N4, hp, ptr(bimg), st)
        b = torch.zeros(N4, device=dev)
        ho, co = torch.empty(n, hp, device=dev), torch.empty(n, hp, device=dev)
        g = torch.empty(n, N4, device=dev)
        flops = 2.0 * n * K * N4
        res = {}
        for fn, tag in (("dgnn_lstm_forward_step_ws", "fwd"), ("dgnn_lstm_forward_step_pair", "fwd_pair")):
            for keep in (False, True):
                us = timed(lambda: call(fn, n, kx, hp, ptr(x), kx, ptr(h), ptr(c), ptr(img),
                                        ptr(b), ptr(ho), ptr(co), ptr(g) if keep else None, st))
                byts = 4.0 * n * (kx + hp + hp + 2 * hp + (N4 if keep else 0))
                res[tag + ("_keep" if keep else "")] = dict(
                    us=us, floor_tf_us=flops / tf / 1e6, floor_hbm_us=byts / hbm / 1e3,
                    frac_tf=flops / tf / 1e6 / us, frac_hbm=byts / hbm / 1e3 / us)
        dy, dhi, dci = torch.randn(n, hp, device=dev), torch.randn(n, hp, device=dev), torch.randn(n, hp, device=dev)
        dx, dho, dco = torch.empty(n, kx, device=dev), torch.empty(n, hp, device=dev), torch.empty(n, hp, device=dev)
        gg = torch.rand(n, N4, device=dev)

        def bwd():
            call("dgnn_lstm_backward_step_ws", n, kx, hp, ptr(dy), ptr(dhi), ptr(dci), ptr(gg), ptr(c), ptr(co),
                 ptr(bimg), ptr(dx), kx, ptr(dho), ptr(dco), st)
        us = timed(bwd)
        byts = 4.0 * n * (hp + hp + hp + N4 + hp + hp + N4 + kx + hp + hp)
        res["bwd"] = dict(us=us, floor_tf_us=flops / tf / 1e6, floor_hbm_us=byts / hbm / 1e3,
                          frac_tf=flops / tf / 1e6 / us, frac_hbm=byts / hbm / 1e3 / us)
        B = args.steps
        X = torch.randn(B * n, kx, device=dev) * 0.5
        Y = torch.randn(B * n, hp, device=dev) * 0.5
        DZ = torch.randn(B * n, N4, device=dev) * 0.01
        gw = torch.zeros(K * N4, dtype=torch.float64, device=dev)
        gb = torch.zeros(N4, dtype=torch.float64, device=dev)
        ws = torch.empty(query("dgnn_lstm_weight_grad_tc_workspace", kx, hp), dtype=torch.uint8, device=dev)
        us = timed(lambda: call("dgnn_lstm_weight_grad_tc", B * n, n, kx, hp, ptr(X), kx, ptr(Y), ptr(h), ptr(DZ),
                                ptr(gw), ptr(gb), ptr(ws), ws.numel(), st), reps=3)
        fl = 2.0 * B * n * K * N4
        byts = 4.0 * B * n * (kx + hp + N4)
        res["dw"] = dict(us=us, floor_tf_us=fl / tf / 1e6, floor_hbm_us=byts / hbm / 1e3, frac_tf=fl / tf / 1e6 / us,
                         frac_hbm=byts / hbm / 1e3 / us)
        us = timed(lambda: call("dgnn_lstm_weight_grad_ts", B * n, n, kx, hp, ptr(X), kx, ptr(Y), ptr(h), ptr(DZ),
                                ptr(gw), ptr(gb), ptr(ws), ws.numel(), st), reps=3)
        res["dw_ts"] = dict(us=us, floor_tf_us=fl / tf / 1e6, floor_hbm_us=byts / hbm / 1e3,
                            frac_tf=fl / tf / 1e6 / us, frac_hbm=byts / hbm / 1e3 / us)
        out[f"kx{kx}_hp{hp}"] = res
        for k, v in res.items():
            print(f"kx={kx} hp={hp} {k:9s} {v['us']:8.1f} us  3xTF32 floor {v['floor_tf_us']:7.1f} "
                  f"({v['frac_tf']:.2f})  HBM floor {v['floor_hbm_us']:7.1f} ({v['frac_hbm']:.2f})", flush=True)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "lstm_probe.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

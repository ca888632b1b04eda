#!/usr/bin/env python
"""Training-epoch benchmark of the dynamic-GNN hot path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "Epinions-scale"): cd-gcn (skip-GCN +
LSTM, 2 layers, hidden = embed = 64) on a synthetic exact-churn dynamic
graph with N = 750k vertices, T = 32 snapshots, 468,750 edges per snapshot
(15M edges in total), 10% churn per step, link-prediction labels with
theta = 0.1, gradient checkpointing with nblk = 4 (bsize = 8).  Under
torchrun with N GPUs the graph grows with N (N x 750k vertices, N x 468,750
edges per snapshot: weak scaling, snapshot-partitioned as in the paper).

A step = one full training epoch (checkpointed forward sweep + rerun +
backward + gradient all-reduce + Adam).  `value` = edge*snapshots/s of the
whole job with the graph encoding resident in HBM (the per-pass CSR
rebuild still runs on device); `e2e` = the same metric through the public
drop-in API `distributed_epoch` with host parameters in, host gradients
out and every pass's graph deltas copied from pinned host memory.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# workloads: c2 = BASELINE configs[1] (the default, the headline line);
# c3 = configs[2] (TM-GCN, banded M-product, AMLSim-style graph); c4 =
# configs[3] (3M vertices, 300M edges); c5 = configs[4] (10M vertices, 1B
# edges, 1% churn) -- c4 / c5 are generated and encoded on the GPU
# (synth.device_churn_graph).  c3-c5 scale strongly: the whole graph is
# split over the GPUs.  nblk per GPU count: the checkpoint block count the
# HBM plan needs.
CONFIGS = {
    "c2": dict(arch="cd-gcn", n=750_000, m=468_750, T=32, hidden=64, churn=0.10, nblk={1: 1, 2: 1, 4: 1, 8: 1},
               gen="churn",
               scaling="weak", cpu_scale=64,
               workload="configs[1] Epinions-scale: cd-gcn (skip-GCN+LSTM, 2 layers) hidden=64, "
                        "N=750k/GPU, T=32, 468,750 edges/snapshot/GPU (15M/GPU total), 10% churn"),
    "c3": dict(arch="tm-gcn", n=1_000_000, m=2_000_000, T=64, hidden=32, churn=0.02, nblk=1, gen="aml",
               scaling="strong", cpu_scale=128,
               workload="configs[2] TM-GCN (plain GCN + banded M-product, window 2) hidden=32 on an "
                        "AMLSim-style transaction graph: N=1M, T=64, 2M edges/snapshot (128M total), "
                        "heavy-tailed degrees, 2% churn"),
    "c4": dict(arch="cd-gcn", n=3_000_000, m=4_687_500, T=64, hidden=32, churn=0.10,
               nblk={1: 4, 2: 2, 4: 1, 8: 1}, gen="device", scaling="strong", cpu_scale=256,
               workload="configs[3] Flickr/YouTube-scale: cd-gcn (skip-GCN+LSTM, 2 layers) hidden=32, "
                        "N=3M, T=64, 4,687,500 edges/snapshot (300M total), 10% churn, snapshot-partitioned"),
    "c5": dict(arch="cd-gcn", n=10_000_000, m=15_625_000, T=64, hidden=32, churn=0.01,
               nblk={1: 16, 2: 16, 4: 4, 8: 2}, gen="device", scaling="strong", cpu_scale=1024,
               workload="configs[4] billion-edge: cd-gcn (skip-GCN+LSTM, 2 layers) hidden=32, N=10M, T=64, "
                        "15,625,000 edges/snapshot (1B total), 1% churn, gradient checkpointing"),
}
CFG = CONFIGS["c2"]
N_PER_GPU = CFG["n"]
EDGES_PER_GPU = CFG["m"]
T = CFG["T"]
HIDDEN = CFG["hidden"]
CHURN = CFG["churn"]
THETA = 0.10
NBLK = CFG["nblk"]
CONFIG_KEY = "c2"


def select_config(name):
    global CFG, N_PER_GPU, EDGES_PER_GPU, T, HIDDEN, CHURN, NBLK, CONFIG_KEY
    CFG = CONFIGS[name]
    CONFIG_KEY = name
    N_PER_GPU, EDGES_PER_GPU, T, HIDDEN, CHURN, NBLK = (CFG[k] for k in ("n", "m", "T", "hidden", "churn", "nblk"))


NBLK_OVERRIDE = None


def nblk_for(P: int) -> int:
    if NBLK_OVERRIDE:
        return NBLK_OVERRIDE
    return NBLK[P] if isinstance(NBLK, dict) else NBLK


METRIC = "training epoch time and edges·snapshots/sec at 1/2/4/8 B200; SpMM HBM GB/s"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, out: Path | None):
        self.proc = None
        self.gpu = gpu
        self.out = out

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]
            if self.out is not None:
                self.out.write_text("\n".join(self.lines) + "\n")
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload


def scale_of(P: int) -> int:
    return P if CFG["scaling"] == "weak" else 1


def make_workload(P: int, seed: int = 1):
    """(cfg, graph, data, train labels, params).  c2 / c3: host generator and
    the reference's own pair sampler (vectorised, same pairs); c4 / c5: the
    device generator + encoder and its device pair sampler."""
    import paper_2109_07893_b200 as pk
    n = N_PER_GPU * scale_of(P)
    m = EDGES_PER_GPU * scale_of(P)
    cfg = pk.ModelConfig(CFG["arch"], in_features=2, hidden_features=HIDDEN, embed_features=HIDDEN)
    if CFG["gen"] == "device":
        import torch
        from paper_2109_07893_b200.synth import device_churn_graph
        g = device_churn_graph(n, T, m, CHURN, seed, torch.device("cuda", torch.cuda.current_device()))
        train, _ = g.sample_pairs(THETA, seed + 1000003)
        g.drop_keys()
        data = pk.TrainingData(graph=g, laps=None, feats=None, s1=None)
    else:
        from paper_2109_07893_b200.synth import aml_graph, churn_graph
        gen = churn_graph if CFG["gen"] == "churn" else aml_graph
        g = gen(n, T, m, CHURN, seed=seed)
        data = pk.prepare_training_data(cfg, g)
        train, _ = pk.sample_link_prediction_sets(g, THETA, seed + 1000003)
    params = pk.init_params(cfg, 0)
    rng = np.random.default_rng(77)          # non-zero head: every upstream gradient is live
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    params["head.b"] = rng.uniform(-0.1, 0.1, size=params["head.b"].shape)
    return cfg, g, data, train, params


def edge_snapshots(g) -> int:
    """Whole job: edge*snapshots per epoch (raw graph), the paper's metric."""
    if hasattr(g, "snapshots"):
        return int(sum(s.nnz for s in g.snapshots))
    return int(sum(g.nnz))


def pcie_h2d_peak(nbytes: int = 1 << 30, reps: int = 5):
    """Pinned host -> HBM copy rate on this box (GB/s): the PCIe roofline."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


# ---------------------------------------------------------------------------
# algorithmic work per kernel call (for the roofline)


TENSOR_KERNELS = ("dgnn_lstm_forward_step", "dgnn_lstm_backward_step", "dgnn_lstm_forward_step_tc",
                  "dgnn_lstm_forward_step_ws", "dgnn_lstm_backward_step_ws", "dgnn_lstm_backward_step_tc",
                  "dgnn_lstm_weight_grad_tc", "dgnn_gemm_tn")


def kernel_work(name, args, ctx):
    """(flops, bytes) of one C-ABI call from its arguments (DESIGN §4's
    algorithmic units); ctx: l2 bytes, real LSTM widths by padded kx, the
    mean nnz of Ahat per snapshot.  bytes None: not modelled."""
    l2, layers_real, nnz = ctx["l2"], ctx["layers_real"], ctx["nnz"]

    def agg(n, f):
        gather = 4 * f * nnz if 4 * n * f > l2 else 4 * n * f
        return 4 * (n + 1) + 8 * nnz + gather

    if name in ("dgnn_lstm_forward_step", "dgnn_lstm_forward_step_tc", "dgnn_lstm_forward_step_ws"):
        rows, kx, hp, gates = args[0], args[1], args[2], args[11]
        kin, h = layers_real.get(kx, (kx, hp))
        return 2 * rows * (kin + h) * 4 * h, 4 * rows * (kin + 4 * h + (4 * h if gates else 0))
    if name in ("dgnn_lstm_backward_step", "dgnn_lstm_backward_step_tc", "dgnn_lstm_backward_step_ws"):
        rows, kx, hp = args[0], args[1], args[2]
        kin, h = layers_real.get(kx, (kx, hp))
        return 2 * rows * 4 * h * (kin + h), 4 * rows * (h * 4 + 4 * h + 4 * h + kin + 2 * h)
    if name == "dgnn_lstm_weight_grad_tc":
        rows, kx, hp = args[0], args[2], args[3]
        kin, h = layers_real.get(kx, (kx, hp))
        return 2 * rows * (kin + h) * 4 * h, 4 * rows * (kin + h + 4 * h)
    if name == "dgnn_gemm_tn":
        rows, m, n = args[0], args[1], args[2]
        return 2 * rows * m * n, 4 * rows * (m + n)
    if name == "dgnn_gcn_forward":
        n, rp, fp, hg, skip, s_out = args[0], args[1], args[5], args[7], args[8], args[9]
        rw = fp + hg if skip else hg
        byts = 4 * n * rw + (4 * n * fp if s_out.ptr else 0)
        byts += agg(n, fp) if rp is not None else 4 * n * fp
        return 2 * n * fp * hg, byts
    if name == "dgnn_spmm_f32":
        n, f = args[0], args[5]
        return 2 * nnz * f, agg(n, f) + 4 * n * f
    if name == "dgnn_frames_combine":
        return 0, None      # bytes depend on the table: not modelled per call
    if name == "dgnn_axpy_frame":
        cnt, init = args[0], args[4]
        return 2 * cnt, (8 if init else 12) * cnt
    if name == "dgnn_gcn_weight_grad":
        n, fp, hg, skip = args[0], args[4], args[5], args[6]
        rw = fp + hg if skip else hg
        return 2 * n * fp * hg, 4 * n * (fp + 2 * rw)
    if name == "dgnn_gcn_backward_rows":
        n, fp, hg, skip = args[0], args[3], args[5], args[6]
        rw = fp + hg if skip else hg
        return 2 * n * fp * hg, 4 * n * (2 * rw + fp)
    return 0, None


# C-ABI entry -> kernel name prefix in the committed ncu launch list
NCU_KERNEL = {"dgnn_lstm_forward_step_ws": "lstm_fwd_ws_kernel", "dgnn_lstm_backward_step_ws": "lstm_bwd_ws_kernel",
              "dgnn_lstm_weight_grad_tc": "lstm_dw_tc_kernel", "dgnn_gcn_forward": "gcn_fwd_tc_kernel<64, 64, 1, 1",
              "dgnn_gcn_weight_grad": "gcn_dw_tc_kernel"}


def ncu_traffic(entry):
    """DRAM bytes per launch of the kernel behind a C-ABI entry, from the
    latest committed ncu launch list (profiles/*_traffic.json, written by
    scripts/ncu_summary.py from `dram__bytes_read.sum + dram__bytes_write.sum`)."""
    # the launch list of this config when one is committed (r*_<config>_traffic.json), else configs[1]'s
    files = sorted((ROOT / "profiles").glob(f"r*_{CONFIG_KEY}_traffic.json")) or \
        sorted(p for p in (ROOT / "profiles").glob("r*_traffic.json") if p.stem.count("_") == 1)
    pref = NCU_KERNEL.get(entry)
    if entry == "dgnn_gcn_forward":   # the aggregating instance at this config's width / cell
        pref = f"gcn_fwd_tc_kernel<{HIDDEN}, {HIDDEN}, {int(CFG['arch'] == 'cd-gcn')}, 1"
    elif pref is not None and pref.startswith("lstm_"):   # the instance at this config's hidden width
        pref = f"{pref}<{HIDDEN}>"
    if not files or pref is None:
        return None
    d = json.loads(files[-1].read_text())
    hits = {k: v for k, v in d.items() if k.startswith(pref)}
    if not hits:
        return None
    n = sum(v["launches"] for v in hits.values())
    b = sum(v["dram_bytes_per_launch"] * v["launches"] for v in hits.values())
    return {"dram_bytes_per_launch": b / n, "source": f"{files[-1].name}: " + ", ".join(sorted(hits))}


def spmm_bytes(n, nnz, f, write_width, l2):
    gather = 4 * f * nnz if 4 * n * f > l2 else 4 * n * f
    return 4 * (n + 1) + 8 * nnz + gather + 4 * n * write_width, 4 * n * f > l2


def spmm_isolated(eng, l2, hbm, reps=10):
    """The layer-1 fused SpMM (K3) of one snapshot timed alone (CUDA events,
    after the timed region): inputs exceed L2, s kept as in the rerun."""
    import torch
    from paper_2109_07893_b200 import _lib
    from paper_2109_07893_b200._lib import call, ptr
    r0 = eng.ranks[0]
    Ly = eng.layout.layers[1]
    sl = r0.slots[0]
    n = eng.plan.N
    t = sl.t
    w = eng.params.w("gcn1.w")
    st = _lib.stream_handle()
    args = (n, ptr(sl.rowptr), ptr(sl.col), ptr(sl.val), r0.own(r0.Y_own[0], Ly.fp, 0), Ly.fp, ptr(w), Ly.hg, 1,
            r0.plain(r0.S_own[1], Ly.fp, 0), r0.own(r0.R_own[1], Ly.rw, 0), st)
    for _ in range(3):
        call("dgnn_gcn_forward", *args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        call("dgnn_gcn_forward", *args)
    e1.record()
    torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) / reps / 1e3
    nnz = int(eng.enc.nnz_hat[t])
    byts, gath = spmm_bytes(n, nnz, Ly.fp, Ly.rw, l2)
    byts += 4 * n * Ly.fp          # the s cache
    return {"avg_launch_us": secs * 1e6, "achieved": byts / secs / 1e9, "frac": byts / secs / 1e9 / hbm,
            "bytes_per_launch": byts, "nnz": nnz}


# ---------------------------------------------------------------------------
# the GPU arm


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    P = world
    if args.gpus != P:
        if P == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    if P > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2109_07893_b200 as pk
    from paper_2109_07893_b200 import _lib
    from paper_2109_07893_b200.engine import Engine, LocalFabric, NcclFabric

    nblk = nblk_for(P)
    t0 = time.time()
    cfg, g, data, train, params = make_workload(P)
    prep_s = time.time() - t0
    fabric = NcclFabric() if P > 1 else LocalFabric()
    eng = Engine(cfg, data.graph, P, nblk, resident=True, fabric=fabric,
                 m_matrix=None if data.m_matrix is None else np.asarray(data.m_matrix.matrix),
                 feats_host=None if cfg.architecture == "cd-gcn"
                 else [np.asarray(f, np.float64) for f in data.feats.frames])
    eng.set_labels(train.by_time, None)
    eng.params.load(params)
    count = train.total_pairs()
    total_es = edge_snapshots(g)

    def step():
        loss_dev, grads = eng.epoch(None, None, None, count, "mean")
        eng.params.adam(0.01)
        return loss_dev

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    layers_real = {}
    for Ly in eng.layout.layers:
        layers_real[Ly.kx] = (Ly.fin + Ly.gout, Ly.out)
    ctx = {"l2": l2, "layers_real": layers_real, "nnz": float(np.mean(eng.enc.nnz_hat))}
    timed_names = list(TENSOR_KERNELS) + [
        "dgnn_gcn_forward", "dgnn_spmm_f32", "dgnn_gcn_weight_grad", "dgnn_gcn_backward_rows",
        "dgnn_axpy_frame", "dgnn_frames_combine", "dgnn_csr_apply_delta", "dgnn_laplacian", "dgnn_csr_transpose_staged",
        "dgnn_head_loss", "dgnn_head_grad", "dgnn_head_loss_grad", "dgnn_head_scatter", "dgnn_head_scatter_active"]
    if args.timeline:   # every C-ABI call, for the per-stream idle breakdown
        timed_names = list(_lib._SIGS.keys())
    timer = _lib.KernelTimer(timed_names)
    clocks = ClockSampler(local, ROOT / "gpurun_out" / f"clocks_rank{rank}.csv"
                          if (ROOT / "gpurun_out").exists() else None)

    def timed_region(instrumented):
        """K steps between events (barrier + synchronize on both sides); with
        `instrumented`, CUDA events around every timed C-ABI call too (their
        host-side cost inflates launch-heavy configs, so the headline comes
        from the plain region and the per-kernel roofline from this one)."""
        if P > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = _lib.launch_count()
        import paper_2109_07893_b200.engine as engine_mod
        overlap = engine_mod.DW_OVERLAP
        if instrumented:
            _lib.set_timer(timer)
            # per-call events must not span another stream's kernels: the
            # weight gradient runs in order here (the plain region overlaps it)
            engine_mod.DW_OVERLAP = False
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            out = step()
        b.record()
        torch.cuda.synchronize()
        _lib.set_timer(None)
        engine_mod.DW_OVERLAP = overlap
        nl = _lib.launch_count() - l0
        if P > 1:
            dist.barrier()
        m = a.elapsed_time(b) / args.steps
        if P > 1:
            t = torch.tensor([m], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            m = float(t.item())
        return m, nl, out, a

    # DGNN_PROFILE_REGION=1: ncu --profile-from-start off captures exactly the
    # uninstrumented timed region (scripts/profile_r02.sh)
    prof = os.environ.get("DGNN_PROFILE_REGION") == "1"
    if prof:
        torch.cuda.cudart().cudaProfilerStart()
    with clocks:
        ms, launches, loss_dev, e0 = timed_region(False)
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    if eng.peer is not None:
        eng.peer.log = []       # NVLink copy timing: the instrumented region
    ms_instr, _, _, e0i = timed_region(True)
    timeline = timer.gaps(e0i) if args.timeline else None
    if timeline is not None and (ROOT / "gpurun_out").exists():
        (ROOT / "gpurun_out" / f"timeline_{args.config}_n{P}_rank{rank}.json").write_text(
            json.dumps({"ms_per_step_instrumented": ms_instr, "streams": timeline}, indent=1))
    loss = float(loss_dev.item()) * eng.scale
    durs = timer.durations()

    # ---- roofline of the dominant kernel (time share over the timed region)
    hbm, bf16, bf16_s, peak_kind = peaks()
    tot = {k: sum(d for d, _ in v) for k, v in durs.items()}
    # dominant kernel of the compute stream (the graph-rebuild kernels run
    # concurrently on their own stream; their event spans include the time
    # they wait for SMs, so they are not candidates)
    graph_side = {"dgnn_laplacian", "dgnn_csr_transpose_staged", "dgnn_csr_apply_delta",
                  "dgnn_rowptr_from_sorted_rows"}
    cand = {k: v for k, v in tot.items() if k not in graph_side and kernel_work(k, durs[k][0][1], ctx)[1]}
    dom = max(cand, key=cand.get) if cand else None
    roof = None
    if dom is not None:
        fl = sum(kernel_work(dom, a, ctx)[0] for _, a in durs[dom])
        by = sum(kernel_work(dom, a, ctx)[1] for _, a in durs[dom])
        secs = tot[dom] / 1e3
        tr = ncu_traffic(dom)
        roof = {"kernel": dom, "share_of_step": tot[dom] / (ms_instr * args.steps),
                "measured_in": "the instrumented region (events around every call), ms_per_step_instrumented",
                "launches": len(durs[dom]), "avg_launch_us": tot[dom] / len(durs[dom]) * 1e3,
                "algorithmic_bytes_per_launch": by / len(durs[dom]),
                "traffic": tr and tr["dram_bytes_per_launch"], "traffic_source": tr and tr["source"],
                "hbm_achieved_gbs": by / secs / 1e9, "hbm_frac": by / secs / 1e9 / hbm}
        t_tensor, t_hbm = fl / (bf16_s / 6 * 1e12), by / (hbm * 1e9)
        if dom in TENSOR_KERNELS and t_tensor > t_hbm:
            roof.update({"bound": "tensor", "achieved": fl / secs / 1e12, "peak": bf16_s, "unit": "TFLOP/s",
                         "frac": fl / secs / 1e12 / bf16_s,
                         "peak_source": f"{peak_kind} bf16 dense sustained (MEASURED_PEAKS.json)",
                         "note": "tcgen05 kind::tf32 with the fp32-accurate 3xTF32 split: 3 MMAs per product at "
                                 "half the bf16 rate, so the useful-flop ceiling is bf16/6 (frac_3xtf32_ceiling); "
                                 "the binding roofline is the larger of the 3xTF32 and HBM times",
                         "frac_3xtf32_ceiling": fl / secs / 1e12 / (bf16_s / 6),
                         "frac_binding": max(t_tensor, t_hbm) / secs})
        elif dom in TENSOR_KERNELS:
            roof.update({"bound": "hbm", "achieved": by / secs / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": by / secs / 1e9 / hbm,
                         "peak_source": f"{peak_kind} HBM copy (MEASURED_PEAKS.json)",
                         "note": "a tcgen05 (3xTF32) kernel whose algorithmic bytes take longer at the HBM peak "
                                 "than its useful flops at the 3xTF32 ceiling (bf16/6): HBM binds",
                         "tflops_achieved": fl / secs / 1e12, "frac_3xtf32_ceiling": fl / secs / 1e12 / (bf16_s / 6),
                         "frac_binding": max(t_tensor, t_hbm) / secs})
        else:
            roof.update({"bound": "hbm", "achieved": by / secs / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": by / secs / 1e9 / hbm,
                         "peak_source": f"{peak_kind} HBM copy (MEASURED_PEAKS.json)"})
    # per-kernel algorithmic rates of everything timed
    kernel_table = {}
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        fl = sum(kernel_work(k, a, ctx)[0] for _, a in durs[k])
        byl = [kernel_work(k, a, ctx)[1] for _, a in durs[k]]
        ent = {"ms_total": v, "launches": len(durs[k]), "share": v / (ms_instr * args.steps)}
        if all(b is not None for b in byl) and v > 0:
            ent["hbm_frac"] = sum(byl) / (v / 1e3) / 1e9 / hbm
            if k in TENSOR_KERNELS:
                ent["frac_3xtf32_ceiling"] = fl / (v / 1e3) / 1e12 / (bf16_s / 6)
        kernel_table[k] = ent
    # SpMM (fused GCN forward with aggregation, last layer) HBM rate
    spmm = None
    sl = [(d, a) for d, a in durs.get("dgnn_gcn_forward", []) if a[1] is not None]
    if not sl:      # split GCN (P > 1) / tm-gcn: the aggregation runs as dgnn_spmm_f32
        sl = durs.get("dgnn_spmm_f32", [])
    if sl:
        nm = "dgnn_gcn_forward" if sl[0][1][1] is not None and len(sl[0][1]) == 12 else "dgnn_spmm_f32"
        byts = sum(kernel_work(nm, a, ctx)[1] for _, a in sl)
        secs = sum(d for d, _ in sl) / 1e3
        n = eng.plan.N
        Ly = eng.layout.layers[-1]
        ctx_c = dict(ctx, l2=1 << 62)
        cb = sum(kernel_work(nm, a, ctx_c)[1] for _, a in sl)
        spmm = {"kernel": f"{nm} (CSR SpMM over Ahat_t" + (" + W + ReLU" if nm == "dgnn_gcn_forward" else "") + ")",
                "bound": "hbm", "achieved": byts / secs / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": byts / secs / 1e9 / hbm,
                "bytes_model": "gather-inclusive" if 4 * n * Ly.fp > l2 else "compulsory",
                "compulsory_gbs": cb / secs / 1e9, "avg_launch_us": secs / len(sl) * 1e6,
                "nnz_per_snapshot": ctx["nnz"], "launches": len(sl),
                "note": "live in the epoch: launches share the GPU with the graph-rebuild stream"}
        tr = ncu_traffic("dgnn_gcn_forward")
        if tr and nm == "dgnn_gcn_forward":
            spmm["traffic"] = tr["dram_bytes_per_launch"]
            spmm["traffic_source"] = tr["source"]
        if P == 1 and cfg.architecture == "cd-gcn":
            spmm["isolated"] = spmm_isolated(eng, l2, hbm)
    nvlink = None
    if eng.peer is not None:
        nv = eng.peer.nvlink_summary()
        eng.peer.log = None
        if nv:
            nvlink = dict(nv, peak_gbs=900.0, frac=nv["achieved_gbs"] / 900.0 if nv["achieved_gbs"] else None,
                          bytes_per_epoch=nv["bytes"] / args.steps,
                          share_of_step_copying=nv["copy_ms"] / (ms_instr * args.steps),
                          note="copy-engine pushes into NVLink peer memory (rank 0), overlapping compute; "
                               "achieved = bytes / summed copy durations; peak 900 GB/s per direction")
    graph_kernels_ms = sum(tot.get(k, 0.0) for k in graph_side) / args.steps
    hbm_peak_gb = torch.cuda.max_memory_allocated() / 2**30
    keep_graphs = eng.keep_graphs
    del eng
    import gc
    gc.collect()               # Engine <-> Rank reference cycles hold the device buffers
    torch.cuda.empty_cache()

    # ---- e2e through the public drop-in API (host buffers, deltas streamed)
    e2e = None
    if not args.skip_e2e:
        # each rank alone on the bus (the uncontended pinned H2D rate is the roofline)
        pcie_peak = None
        for q in range(P):
            if P > 1:
                dist.barrier()
            if q == rank:
                pcie_peak = pcie_h2d_peak()
        if P > 1:
            dist.barrier()
        comm, transfer = pk.CommLedger(), pk.TransferLedger()
        hp = {k: v.copy() for k, v in params.items()}
        st = pk.init_adam(hp)
        pk.distributed_epoch(cfg, data, train, hp, P, nblk)        # build + warm the engine
        e2e_eng = pk.api.get_engine(cfg, data, P, nblk)
        for r in e2e_eng.ranks:
            r.mat.copy_log = []
        torch.cuda.synchronize()
        if P > 1:
            dist.barrier()
        ts = time.perf_counter()
        for _ in range(args.steps):
            loss_e, grads, _, _ = pk.distributed_epoch(cfg, data, train, hp, P, nblk, comm=comm,
                                                       transfer=transfer)
            pk.adam_step(hp, grads, st, 0.01)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - ts) / args.steps
        if P > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        # graph bytes of the whole job (every rank's copies), like the ratio's denominator
        tb = torch.tensor([transfer.h2d_bytes, transfer.full_built_bytes, transfer.full_equiv_bytes],
                          dtype=torch.float64, device="cuda")
        if P > 1:
            dist.all_reduce(tb)
        job_h2d, job_built, job_equiv = (float(x) for x in tb.tolist())
        log = [x for r in e2e_eng.ranks for x in (r.mat.copy_log or [])]
        copy_ms = sum(a.elapsed_time(b) for a, b, _ in log)
        copy_bytes = sum(b for _, _, b in log)
        for r in e2e_eng.ranks:
            r.mat.copy_log = None
        pbytes = 8 * e2e_eng.layout.count
        e2e = {"value": total_es / e2e_s, "unit": "edge*snapshots/s", "ms_per_step": e2e_s * 1e3,
               "h2d_bytes_per_step": int(transfer.h2d_bytes / args.steps) + pbytes,
               "d2h_bytes_per_step": pbytes + 8,
               "graph_h2d_bytes_per_step": int(transfer.h2d_bytes / args.steps),
               "graph_h2d_bytes_per_step_all_ranks": int(job_h2d / args.steps),
               "delta_vs_full_bytes": (job_built / job_h2d) if job_h2d else None,
               "delta_vs_full_bytes_reference_schedule": (job_equiv / job_h2d) if job_h2d else None,
               "delta_vs_full_bytes_rank0": (transfer.full_built_bytes / transfer.h2d_bytes)
               if transfer.h2d_bytes else None,
               "delta_note": "delta_vs_full_bytes (all ranks): full-snapshot bytes of the chunks streamed and "
                             "rebuilt / bytes copied (like for like: same u32-pair encoding, heads rebuilt "
                             "from 1-step deltas); _reference_schedule: every snapshot of every pass (forward + "
                             "checkpoint rerun) streamed in full, as dtgnn's stream_block does, / bytes copied",
               "pcie": {"peak_h2d_gbs": pcie_peak, "copy_ms_per_step": copy_ms / args.steps,
                        "achieved_gbs": copy_bytes / (copy_ms / 1e3) / 1e9 if copy_ms > 0 else None,
                        "frac": (copy_bytes / (copy_ms / 1e3) / 1e9 / pcie_peak) if copy_ms > 0 else None,
                        "share_of_step": copy_ms / (e2e_s * 1e3 * args.steps),
                        "note": "rank 0: pinned-host -> HBM graph copies on the copy stream (overlapping "
                                "compute); peak = 1 GiB pinned copy measured in this run"},
               "api": "paper_2109_07893_b200.distributed_epoch + adam_step"}
        pk.api.clear_engines()

    cpu = None
    if rank == 0 and P == 1 and not args.skip_cpu:
        cpu = cpu_baseline(sample_scale=args.cpu_scale, threads=True, linearity=True)

    if rank == 0:
        line = {
            "metric": METRIC, "value": total_es / (ms / 1e3), "unit": "edge*snapshots/s", "n_gpus": P,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "ms_per_step_instrumented": ms_instr,
            "scaling": CFG["scaling"], "vs_baseline": None, "dtype": "fp32 (fp64 graph values / master weights)",
            "data": "synthetic exact-churn dynamic graph, random-init weights",
            "config": {"workload": CFG["workload"], "config_key": args.config,
                       "model": CFG["arch"], "num_vertices": N_PER_GPU * scale_of(P), "num_timesteps": T,
                       "edges_per_snapshot": EDGES_PER_GPU * scale_of(P), "hidden": HIDDEN, "nblk": nblk,
                       "theta": THETA, "train_pairs": count, "parallelism": f"snapshot-partitioned x{P}",
                       "l2": "inputs larger than L2 (per-epoch working set ~tens of GB)",
                       "graph_in_timed_region": "delta-encoded graph resident in HBM, CSR/Laplacian "
                                                "rebuilt on device every epoch (forward sweep; the rerun "
                                                "reuses the kept snapshots)"},
            "loss": loss,
            "gpu_launches": launches,
            "roofline": roof,
            "spmm_roofline": spmm,
            "nvlink": nvlink,
            "graph_kernels_ms_per_step": graph_kernels_ms,
            "hbm_peak_gb": hbm_peak_gb, "keep_graphs": keep_graphs,
            "kernels": kernel_table,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "prep_seconds": prep_s,
            "timeline": timeline,
        }
        print(json.dumps(line))
    if P > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port of the reference algorithm


def cpu_sample(scale: int):
    n = N_PER_GPU // scale
    n -= n % 8
    m = EDGES_PER_GPU // scale
    return n, m


def cpu_epoch_rate(sample_scale: int, threads: bool, steps: int = 1, warmup: int = 0):
    """The oracle port (numpy fp64 restatement of dtgnn's distributed_epoch,
    threads scheduler) + Adam on the workload scaled 1/sample_scale."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import dtgnn_oracle as O
    from paper_2109_07893_b200.synth import aml_keys, churn_keys
    n, m = cpu_sample(sample_scale)
    keys = (aml_keys if CFG["gen"] == "aml" else churn_keys)(n, T, m, CHURN, seed=1)
    snaps = [O.Coo(n, k // n, k % n, np.ones(k.shape[0])) for k in keys]
    cfg = O.Cfg(CFG["arch"], 2, HIDDEN, HIDDEN)
    Pp = O.prepare(cfg, snaps)
    train, _ = O.sample_labels(snaps, THETA, 1 + 1000003)
    params = O.init_params(cfg, 0)
    rng = np.random.default_rng(77)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    cores = os.cpu_count() or 1
    nblk = nblk_for(1)
    bsize = T // nblk
    workers = max(p for p in range(1, min(cores, bsize) + 1) if bsize % p == 0 and n % p == 0) if threads else 1
    st = O.adam_state(params)

    def step():
        loss, grads, _, _ = O.distributed_epoch(cfg, Pp, train, params, workers, nblk, threads=threads)
        O.adam(params, grads, st, 0.01)

    for _ in range(warmup):
        step()
    c0 = time.process_time()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    util = (time.process_time() - c0) / (dt * steps)
    es = int(sum(k.shape[0] for k in keys))
    return {"value": es / dt, "seconds_per_epoch": dt, "cores": workers, "cpu_utilisation": util,
            "host_cpus": cores, "n": n, "edges_per_snapshot": m, "nblk": nblk}


def cpu_baseline(sample_scale: int | None = None, threads: bool = True, steps: int = 1, warmup: int = 0,
                 linearity: bool = False):
    scale = sample_scale or CFG["cpu_scale"]
    r = cpu_epoch_rate(scale, threads, steps, warmup)
    out = {"value": r["value"], "unit": "edge*snapshots/s", "cores": r["cores"], "kind": "port",
           "seconds_per_epoch": r["seconds_per_epoch"], "cpu_utilisation": r["cpu_utilisation"],
           "host_cpus": r["host_cpus"], "sample_scale": scale,
           "sample": f"oracle port (numpy fp64 restatement of dtgnn distributed_epoch, threads scheduler, "
                     f"P={r['cores']}) + Adam on the {CFG['workload'].split(':')[0]} shape scaled 1/{scale}: "
                     f"N={r['n']}, T={T}, {r['edges_per_snapshot']} edges/snapshot, {CHURN:.0%} churn, "
                     f"{CFG['arch']} H={HIDDEN}, nblk={r['nblk']}"}
    if linearity:
        # the sample's rate at 4x and 2x smaller scales (one epoch each): how
        # the per-edge rate moves with size (cache effects favour small samples)
        pts = [{"scale": sc, "value": cpu_epoch_rate(sc, threads)["value"]} for sc in (scale * 4, scale * 2)]
        out["linearity"] = pts + [{"scale": scale, "value": r["value"]}]
    return out


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_baseline(sample_scale=args.cpu_scale_ref, threads=True, steps=args.steps, warmup=args.warmup)
    line = {"metric": METRIC, "value": cb["value"], "unit": "edge*snapshots/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["seconds_per_epoch"] * 1e3,
            "higher_is_better": True, "scaling": CFG["scaling"], "vs_baseline": None, "dtype": "fp64",
            "data": "synthetic exact-churn dynamic graph, random-init weights",
            "config": {"workload": CFG["workload"] + " (CPU sample, see cpu_baseline)", "model": CFG["arch"],
                       "config_key": args.config},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "edge*snapshots/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--timeline", action="store_true", help="per-stream busy / idle breakdown (diagnostic)")
    ap.add_argument("--cpu-scale", type=int, default=None, help="CPU sample scale (default: per config)")
    ap.add_argument("--cpu-scale-ref", type=int, default=None)
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2",
                    help="workload (c2: the headline configs[1] line; c3: TM-GCN configs[2]; c4 / c5: "
                         "configs[3] / configs[4])")
    ap.add_argument("--nblk", type=int, default=None, help="checkpoint block count (default: per config / GPU count)")
    args = ap.parse_args()
    select_config(args.config)
    global NBLK_OVERRIDE
    NBLK_OVERRIDE = args.nblk
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

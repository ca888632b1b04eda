"""Generate golden fixtures by running the REFERENCE (`dtgnn` 0.1.0).

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \
        python tests/golden/make_golden.py

Writes small `.npz` / `.json` fixtures next to this script.  The fixtures pin
(1) the CPU oracle in `oracle/dtgnn_oracle.py` and (2) the GPU path, on the
same seeded inputs.  Graphs are stored inside the fixtures, so nothing here
needs to be re-run on the GPU box.
"""

from __future__ import annotations

import io
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

import dtgnn  # noqa: E402  (the reference)
from dtgnn import delta as rdelta  # noqa: E402
from dtgnn import dist as rdist  # noqa: E402
from dtgnn import training as rtrain  # noqa: E402
from dtgnn.core import SparseMatrix as RSparse  # noqa: E402
from dtgnn.dtdg import DynamicGraph as RGraph  # noqa: E402

from paper_2109_07893_b200.synth import churn_keys  # noqa: E402


def ref_graph_from_keys(n, keys_list, vals_list=None):
    snaps = []
    for i, k in enumerate(keys_list):
        v = None if vals_list is None else vals_list[i]
        snaps.append(RSparse.from_entries(n, k // n, k % n, v))
    return RGraph(n, snaps)


def pack_graph(prefix, g, out):
    out[f"{prefix}n"] = np.int64(g.num_vertices)
    out[f"{prefix}T"] = np.int64(g.num_timesteps)
    for t, s in enumerate(g.snapshots):
        out[f"{prefix}rows{t}"] = s.rows
        out[f"{prefix}cols{t}"] = s.cols
        out[f"{prefix}vals{t}"] = s.vals


def pack_sparse(prefix, s, out):
    out[f"{prefix}rows"] = s.rows
    out[f"{prefix}cols"] = s.cols
    out[f"{prefix}vals"] = s.vals


def randomize_head(params, seed=77):
    # the reference test-suite fixture (conftest.py:42-48)
    rng = np.random.default_rng(seed)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    params["head.b"] = rng.uniform(-0.1, 0.1, size=params["head.b"].shape)
    return params


def pack_params(prefix, p, out):
    for k, v in p.items():
        out[f"{prefix}{k}"] = v


def codec_fixture():
    out = {}
    n = 40
    keys = churn_keys(n, 6, 60, 0.2, seed=3)
    g = ref_graph_from_keys(n, keys)
    pack_graph("g_", g, out)
    for t, s in enumerate(g.snapshots):
        pack_sparse(f"lap{t}_", dtgnn.normalize_laplacian(s), out)
    feats = dtgnn.degree_features(g)
    laps = [dtgnn.normalize_laplacian(s) for s in g.snapshots]
    s1 = dtgnn.precompute_first_layer(laps, feats)
    for t in range(g.num_timesteps):
        out[f"feat{t}"] = feats.frames[t]
        out[f"s1_{t}"] = s1[t]
    for t in range(1, g.num_timesteps):
        d = rdelta.diff(g.snapshots[t - 1], g.snapshots[t])
        out[f"ext_prev{t}"] = d.ext_prev
        out[f"ext_next{t}"] = d.ext_next
    led = rdelta.TransferLedger()
    list(rdelta.stream_block(laps, led))
    out["stream_ledger"] = np.array(json.dumps(led.as_dict()))
    # weighted (edge-life smoothed) variant: value-carrying codec + Laplacian
    gw = dtgnn.apply_edge_life(g, 3)
    pack_graph("gw_", gw, out)
    for t, s in enumerate(gw.snapshots):
        pack_sparse(f"lapw{t}_", dtgnn.normalize_laplacian(s), out)
    # negative self-loop weights: exercises zero-elided diagonals
    rng = np.random.default_rng(9)
    rows = np.concatenate([np.arange(10), rng.integers(0, 12, 30)])
    cols = np.concatenate([np.arange(10), rng.integers(0, 12, 30)])
    vals = np.concatenate([-np.ones(10), rng.uniform(0.5, 2.0, 30)])
    sneg = RSparse.from_entries(12, rows, cols, vals)
    pack_sparse("neg_", sneg, out)
    pack_sparse("lapneg_", dtgnn.normalize_laplacian(sneg), out)
    np.savez_compressed(HERE / "codec.npz", **out)


def spmm_fixture():
    out = {}
    rng = np.random.default_rng(21)
    dim = 30
    keys = rng.choice(dim * dim, 140, replace=False)
    vals = rng.standard_normal(140)
    a = RSparse.from_entries(dim, keys // dim, keys % dim, vals)
    x = rng.standard_normal((dim, 5))
    pack_sparse("a_", a, out)
    out["x"] = x
    out["spmm"] = dtgnn.spmm(a, x)
    out["spmm_t"] = dtgnn.spmm_transpose(a, x)
    np.savez_compressed(HERE / "spmm.npz", **out)


def lstm_fixture():
    from dtgnn.models import LstmCellParams
    out = {}
    rng = np.random.default_rng(5)
    rows, fin, hid = 7, 5, 4
    cell = LstmCellParams(wx=rng.standard_normal((fin, 4 * hid)) * 0.5,
                          wh=rng.standard_normal((hid, 4 * hid)) * 0.5,
                          b=rng.standard_normal(4 * hid) * 0.1)
    h0, c0 = rng.standard_normal((rows, hid)) * 0.3, rng.standard_normal((rows, hid)) * 0.3
    ts = [3, 4, 5]
    xs = {t: rng.standard_normal((rows, fin)) for t in ts}
    ys, (h, c), cache = rtrain.lstm_block_forward(cell, (h0, c0), ts, xs)
    dys = {t: rng.standard_normal((rows, hid)) for t in ts}
    dh0, dc0 = rng.standard_normal((rows, hid)), rng.standard_normal((rows, hid))
    dxs, (dh, dc), dcell = rtrain.lstm_block_backward(cell, ts, cache, dys, (dh0, dc0))
    out.update(wx=cell.wx, wh=cell.wh, b=cell.b, h0=h0, c0=c0, h=h, c=c, dh0=dh0, dc0=dc0,
               dh=dh, dc=dc, dwx=dcell["wx"], dwh=dcell["wh"], db=dcell["b"])
    for t in ts:
        out[f"x{t}"], out[f"y{t}"], out[f"dy{t}"], out[f"dx{t}"] = xs[t], ys[t], dys[t], dxs[t]
    np.savez_compressed(HERE / "lstm.npz", **out)


def model_case(arch, n, t_count, m, churn, hidden, seed_graph, theta, label_seed, param_seed,
               window=2):
    keys = churn_keys(n, t_count, m, churn, seed=seed_graph)
    g = ref_graph_from_keys(n, keys)
    cfg = dtgnn.ModelConfig(architecture=arch, in_features=2, hidden_features=hidden,
                            embed_features=hidden, window=window)
    data = rtrain.prepare_training_data(cfg, g)
    train, test = rtrain.sample_link_prediction_sets(g, theta, label_seed)
    params = randomize_head(dtgnn.init_params(cfg, param_seed))
    return g, cfg, data, train, test, params


def pack_labels(prefix, ls, out):
    out[f"{prefix}frames"] = np.array(sorted(ls.by_time), dtype=np.int64)
    for t, (p, l) in ls.by_time.items():
        out[f"{prefix}pairs{t}"] = p
        out[f"{prefix}labels{t}"] = l


def model_fixture(name, arch, **kw):
    out = {}
    g, cfg, data, train, test, params = model_case(arch, **kw)
    pack_graph("g_", g, out)
    pack_labels("train_", train, out)
    pack_labels("test_", test, out)
    pack_params("p_", params, out)
    out["cfg"] = np.array(json.dumps({"architecture": arch, "hidden": kw["hidden"],
                                      "window": kw.get("window", 2)}))
    fresh = dtgnn.init_params(cfg, kw["param_seed"])
    pack_params("init_", fresh, out)
    loss, grads = rtrain.backward_full(cfg, data, train, params)
    out["full_loss"] = np.float64(loss)
    pack_params("full_g_", grads, out)
    for nblk in (1, 2, 4):
        if data.num_timesteps % nblk:
            continue
        loss, grads = rtrain.backward_checkpoint(cfg, data, train, params, nblk=nblk)
        out[f"ckpt{nblk}_loss"] = np.float64(loss)
        pack_params(f"ckpt{nblk}_g_", grads, out)
    for workers, nblk in ((2, 2), (4, 1), (2, 1)):
        comm = rdist.CommLedger()
        tr = rdelta.TransferLedger()
        loss, grads, comm, tr = rdist.distributed_epoch(cfg, data, train, params, workers, nblk,
                                                        comm=comm, transfer=tr)
        tag = f"dist{workers}x{nblk}"
        out[f"{tag}_loss"] = np.float64(loss)
        pack_params(f"{tag}_g_", grads, out)
        out[f"{tag}_comm"] = np.array(json.dumps(comm.as_dict()))
        out[f"{tag}_events"] = np.array(json.dumps(comm.events))
        out[f"{tag}_transfer"] = np.array(json.dumps(tr.as_dict()))
    # eval forward
    z = dtgnn.model_forward(cfg, data.laps, data.feats, params)
    for t, f in enumerate(z.frames):
        out[f"z{t}"] = f
    # 3 epochs of train_distributed (reference trainer incl. Adam + eval)
    trace, fparams, comm, tr, act = rdist.train_distributed(cfg, data, train, test, epochs=3,
                                                            seed=kw["param_seed"], workers=2,
                                                            nblk=2)
    out["train_trace"] = np.array(json.dumps(trace))
    pack_params("train_p_", fparams, out)
    out["train_comm"] = np.array(json.dumps(comm.as_dict()))
    out["train_transfer"] = np.array(json.dumps(tr.as_dict()))
    out["train_act_peak"] = np.float64(act.peak)
    np.savez_compressed(HERE / f"{name}.npz", **out)


def c1_pins():
    """Pins at the first BASELINE config (N=10k, T=8, 50k edges/snapshot,
    10% churn, cd-gcn H=32): the graph is regenerated deterministically from
    the in-repo generator, the reference's outputs are stored as scalars."""
    n, t_count, m = 10_000, 8, 50_000
    keys = churn_keys(n, t_count, m, 0.10, seed=1)
    g = ref_graph_from_keys(n, keys)
    cfg = dtgnn.ModelConfig(architecture="cd-gcn", in_features=2, hidden_features=32,
                            embed_features=32)
    data = rtrain.prepare_training_data(cfg, g)
    train, _ = rtrain.sample_link_prediction_sets(g, 0.1, 1 + 1000003)
    params = randomize_head(dtgnn.init_params(cfg, 0))
    loss, grads = rtrain.backward_checkpoint(cfg, data, train, params, nblk=2)
    out = {"loss": np.float64(loss)}
    for k, v in grads.items():
        out[f"g_{k}"] = v  # the grads are small (<= 2x(2H)x4H)
    out["lap_nnz"] = np.array([l.nnz for l in data.laps])
    out["lap_valsum"] = np.array([float(np.sum(l.vals)) for l in data.laps])
    out["s1_sum"] = np.array([float(np.sum(s)) for s in data.s1])
    out["train_pairs"] = np.array([train.by_time[t][0].shape[0] for t in sorted(train.by_time)])
    np.savez_compressed(HERE / "c1_pins.npz", **out)


def cli_report():
    """The reference's frozen CLI golden run (test_cli.py:124-137), produced
    here by the reference CLI, plus the graph it trained on."""
    from dtgnn.cli import main
    from dtgnn.dtdg import read_edge_list
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        gpath, rpath = os.path.join(d, "g.txt"), os.path.join(d, "r.json")
        main(["generate", "--timesteps", "4", "--vertices", "8", "--density", "2",
              "--seed", "1", "--out", gpath])
        main(["train", "--data", gpath, "--model", "tm-gcn", "--epochs", "2",
              "--workers", "2", "--blocks", "2", "--seed", "0", "--report", rpath])
        g = read_edge_list(gpath)
        rep = json.load(open(rpath))
    del rep["timing"]
    out = {"report": np.array(json.dumps(rep, sort_keys=True))}
    pack_graph("g_", g, out)
    np.savez_compressed(HERE / "cli_report.npz", **out)


def delta_bytes():
    a = RSparse.from_entries(2, [0], [1], [1.0])
    b = RSparse.from_entries(2, [1], [1], [2.5])
    buf = io.BytesIO()
    rdelta.write_delta_stream([a, b], buf)
    (HERE / "delta_record.bin").write_bytes(buf.getvalue())


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "egcn":
    # the EGCN-O fixture alone (added in round 2; the others are unchanged)
    model_fixture("egcn_small", "egcn-o", n=16, t_count=8, m=24, churn=0.25, hidden=8,
                  seed_graph=8, theta=0.5, label_seed=9, param_seed=4)
    sys.exit(0)

if __name__ == "__main__":
    codec_fixture()
    spmm_fixture()
    lstm_fixture()
    model_fixture("cdgcn_small", "cd-gcn", n=16, t_count=8, m=24, churn=0.25, hidden=8,
                  seed_graph=4, theta=0.5, label_seed=5, param_seed=3)
    model_fixture("tmgcn_small", "tm-gcn", n=16, t_count=8, m=24, churn=0.25, hidden=8,
                  seed_graph=6, theta=0.5, label_seed=7, param_seed=2)
    model_fixture("egcn_small", "egcn-o", n=16, t_count=8, m=24, churn=0.25, hidden=8,
                  seed_graph=8, theta=0.5, label_seed=9, param_seed=4)
    cli_report()
    delta_bytes()
    c1_pins()
    print("fixtures written to", HERE)

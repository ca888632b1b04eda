"""GPU parity of the training engine (drop-in API) against the reference's
golden runs and the CPU oracle.

Tolerance (north star): losses and gradients within 1e-4 relative in fp32,
guarded as |g - r| <= 1e-4 max(|g|, |r|) + 1e-6 ||r||_inf per tensor (the
reference's own guarded form, conftest.py:71-86).  Ledgers (communication
and transfer counters) must be exactly equal.  Test accuracy is an argmax,
compared with a small count tolerance.
"""

import json

import numpy as np
import pytest
import torch

import paper_2109_07893_b200 as pk

from conftest import ENGINE_ATOL, assert_grads_close, guarded_close, jload, labels_from, load, params_from
from helpers import product_case, product_graph

pytestmark = pytest.mark.gpu
RTOL = 1e-4


@pytest.fixture(autouse=True)
def _fresh_engines():
    yield
    pk.api.clear_engines()


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small", "egcn_small"])
@pytest.mark.parametrize("nblk", [1, 2, 4])
def test_backward_checkpoint_vs_reference(name, nblk):
    fx, cfg, data, train, _, params = product_case(name)
    loss, grads = pk.backward_checkpoint(cfg, data, train, params, nblk)
    assert loss == pytest.approx(float(fx[f"ckpt{nblk}_loss"]), rel=RTOL)
    assert_grads_close(grads, params_from(fx, f"ckpt{nblk}_g_"), RTOL, ENGINE_ATOL)


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small", "egcn_small"])
def test_backward_full_vs_reference(name):
    fx, cfg, data, train, _, params = product_case(name)
    loss, grads = pk.backward_full(cfg, data, train, params)
    assert loss == pytest.approx(float(fx["full_loss"]), rel=RTOL)
    assert_grads_close(grads, params_from(fx, "full_g_"), RTOL, ENGINE_ATOL)


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small", "egcn_small"])
@pytest.mark.parametrize("workers,nblk", [(2, 2), (4, 1), (2, 1)])
def test_distributed_epoch_vs_reference(name, workers, nblk):
    fx, cfg, data, train, _, params = product_case(name)
    tag = f"dist{workers}x{nblk}"
    for sched in ("round-robin", "threads"):
        loss, grads, comm, tr = pk.distributed_epoch(cfg, data, train, params, workers, nblk, scheduler=sched)
        assert loss == pytest.approx(float(fx[f"{tag}_loss"]), rel=RTOL)
        assert_grads_close(grads, params_from(fx, f"{tag}_g_"), RTOL, ENGINE_ATOL)
        assert comm.as_dict() == jload(fx[f"{tag}_comm"])
        assert comm.events == jload(fx[f"{tag}_events"])
        assert tr.as_dict() == jload(fx[f"{tag}_transfer"])


def test_results_are_bit_reproducible():
    fx, cfg, data, train, _, params = product_case("cdgcn_small")
    a = pk.distributed_epoch(cfg, data, train, params, 2, 2)
    pk.api.clear_engines()
    b = pk.distributed_epoch(cfg, data, train, params, 2, 2)
    assert a[0] == b[0]
    for k in a[1]:
        assert np.array_equal(a[1][k], b[1][k])


def test_multi_rank_matches_single_rank():
    fx, cfg, data, train, _, params = product_case("cdgcn_small")
    l1, g1 = pk.backward_checkpoint(cfg, data, train, params, 2)
    l4, g4, _, _ = pk.distributed_epoch(cfg, data, train, params, 4, 1)
    assert l4 == pytest.approx(l1, rel=RTOL)
    assert_grads_close(g4, g1, RTOL, ENGINE_ATOL)


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small", "egcn_small"])
def test_train_distributed_vs_reference(name):
    fx, cfg, data, train, test, _ = product_case(name)
    seed = {"cdgcn_small": 3, "tmgcn_small": 2, "egcn_small": 4}[name]
    trace, params, comm, tr, act = pk.train_distributed(cfg, data, train, test, epochs=3, seed=seed,
                                                        workers=2, nblk=2)
    ref = jload(fx["train_trace"])
    for a, b in zip(trace, ref):
        assert a["epoch"] == b["epoch"]
        assert a["loss"] == pytest.approx(b["loss"], rel=RTOL)
        npairs = sum(p.shape[0] for p, _ in test.by_time.values())
        assert abs(a["test_accuracy"] - b["test_accuracy"]) <= 1.0 / npairs + 1e-12
    ref_p = params_from(fx, "train_p_")
    for k in ref_p:
        ok, worst, _ = guarded_close(params[k], ref_p[k], 1e-4, 1e-5)
        assert ok, (k, worst)
    assert comm.as_dict() == jload(fx["train_comm"])
    assert tr.as_dict() == jload(fx["train_transfer"])
    assert act.peak == float(fx["train_act_peak"])


def test_cli_golden_report_through_engine():
    """The reference CLI's frozen golden run (tm-gcn, P=2, nblk=2, 2 epochs)."""
    fx = load("cli_report")
    rep = jload(fx["report"])
    c = rep["config"]
    g = product_graph(fx)
    cfg = pk.ModelConfig(c["model"], hidden_features=c["hidden"], embed_features=c["embed"], window=c["window"])
    data = pk.prepare_training_data(cfg, g)
    train, test = pk.sample_link_prediction_sets(g, c["theta"], c["seed"] + 1000003)
    trace, _, comm, tr, act = pk.train_distributed(cfg, data, train, test, c["epochs"], c["seed"],
                                                   c["workers"], c["blocks"], lr=c["lr"])
    assert comm.as_dict() == rep["comm"]
    assert tr.as_dict() == rep["transfer"]
    assert act.peak == rep["activation_peak"]
    for a, b in zip(trace, rep["epochs"]):
        assert a["loss"] == pytest.approx(b["loss"], rel=RTOL)


def test_c1_config_vs_reference():
    """BASELINE config 1 (N=10k, T=8, 50k edges/snapshot, 10% churn,
    cd-gcn H=32) against the reference's stored loss and gradients."""
    from paper_2109_07893_b200.synth import churn_graph
    fx = load("c1_pins")
    g = churn_graph(10_000, 8, 50_000, 0.10, seed=1)
    cfg = pk.ModelConfig("cd-gcn", hidden_features=32, embed_features=32)
    data = pk.prepare_training_data(cfg, g)
    train, _ = pk.sample_link_prediction_sets(g, 0.1, 1 + 1000003)
    params = pk.init_params(cfg, 0)
    rng = np.random.default_rng(77)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    params["head.b"] = rng.uniform(-0.1, 0.1, size=params["head.b"].shape)
    loss, grads = pk.backward_checkpoint(cfg, data, train, params, 2)
    assert loss == pytest.approx(float(fx["loss"]), rel=RTOL)
    assert_grads_close(grads, {k[2:]: fx[k] for k in fx if k.startswith("g_")}, RTOL, ENGINE_ATOL)


def test_midsize_multi_rank_parity_vs_oracle(oracle):
    """N=20k, T=8, H=64: emulated P=4 vs P=1 vs the oracle."""
    from paper_2109_07893_b200.synth import churn_graph
    g = churn_graph(20_000, 8, 30_000, 0.10, seed=5)
    cfg = pk.ModelConfig("cd-gcn", hidden_features=64, embed_features=64)
    data = pk.prepare_training_data(cfg, g)
    train, _ = pk.sample_link_prediction_sets(g, 0.1, 9)
    params = pk.init_params(cfg, 4)
    rng = np.random.default_rng(1)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    l1, g1 = pk.backward_checkpoint(cfg, data, train, params, 2)
    l4, g4, comm, tr = pk.distributed_epoch(cfg, data, train, params, 4, 2)
    ocfg = oracle.Cfg("cd-gcn", 2, 64, 64)
    P = oracle.prepare(ocfg, [oracle.Coo(s.dim, s.rows, s.cols, s.vals) for s in g.snapshots])
    lo, go = oracle.backward_checkpoint(ocfg, P, train.by_time, params, 2)
    assert l1 == pytest.approx(lo, rel=RTOL)
    assert l4 == pytest.approx(lo, rel=RTOL)
    assert_grads_close(g1, go, RTOL, ENGINE_ATOL)
    assert_grads_close(g4, go, RTOL, ENGINE_ATOL)
    assert comm.redistribution_units == 6 * 2 * 8 * 20_000 * 3 // 4


def test_reference_objects_are_accepted():
    """Duck typing: a reference-shaped TrainingData/ModelConfig works."""
    fx, cfg, data, train, _, params = product_case("cdgcn_small")

    class RefCfg:
        architecture, in_features, hidden_features, embed_features = "cd-gcn", 2, 8, 8
        layers, window, edge_life, classes = 2, 2, 2, 2

    loss, grads = pk.backward_checkpoint(RefCfg, data, train, params, 1)
    assert loss == pytest.approx(float(fx["ckpt1_loss"]), rel=RTOL)


def test_errors_match_reference_types():
    fx, cfg, data, train, _, params = product_case("cdgcn_small")
    with pytest.raises(pk.ConfigError):
        pk.distributed_epoch(cfg, data, train, params, 3, 1)
    with pytest.raises(pk.ConfigError):
        pk.distributed_epoch(cfg, data, train, params, 2, 3)
    with pytest.raises(pk.ConfigError):
        pk.distributed_epoch(cfg, data, train, params, 1, 1, scheduler="fibers")
    with pytest.raises(pk.ConfigError):
        pk.backward_checkpoint(cfg, data, train, params, 3)


def test_simt_engine_meets_the_strict_floor():
    """A/B: with the SIMT fp32 temporal kernels the engine meets the strict
    1e-6 x ||r||_inf floor on the reference fixtures."""
    old = pk.api.TENSOR_CORES
    pk.api.TENSOR_CORES = False
    try:
        for name in ("cdgcn_small", "tmgcn_small"):
            fx, cfg, data, train, _, params = product_case(name)
            loss, grads, _, _ = pk.distributed_epoch(cfg, data, train, params, 2, 2)
            assert loss == pytest.approx(float(fx["dist2x2_loss"]), rel=RTOL)
            assert_grads_close(grads, params_from(fx, "dist2x2_g_"), RTOL, 1e-6)
    finally:
        pk.api.TENSOR_CORES = old


@pytest.mark.parametrize("keep", ["0", "1"])
@pytest.mark.parametrize("workers,nblk", [(1, 4), (2, 2), (4, 1)])
def test_graph_residency_modes_match_reference(keep, workers, nblk, monkeypatch):
    """Kept snapshots (the rerun and evaluation reuse the forward sweep's
    rebuild) and the two-set rebuild-every-pass mode give the reference's
    results and exact ledgers; kept mode copies each chunk once per epoch."""
    import paper_2109_07893_b200.engine as E
    monkeypatch.setattr(E, "KEEP_GRAPHS", keep)
    fx, cfg, data, train, _, params = product_case("cdgcn_small")
    tag = f"dist{workers}x{nblk}" if workers > 1 else f"ckpt{nblk}"
    for epoch in range(2):
        tr = pk.TransferLedger()
        loss, grads, comm, tr = pk.distributed_epoch(cfg, data, train, params, workers, nblk, transfer=tr)
        assert loss == pytest.approx(float(fx[f"{tag}_loss"]), rel=RTOL)
        assert_grads_close(grads, params_from(fx, f"{tag}_g_"), RTOL, ENGINE_ATOL)
        if workers > 1:
            assert tr.as_dict() == jload(fx[f"{tag}_transfer"])
        if keep == "1" and epoch == 1:     # steady state: one rebuild per epoch
            assert tr.full_equiv_bytes == 2 * tr.full_built_bytes
        if keep == "1" or workers == 1:    # every head after t = 0 rebuilt from a delta
            assert tr.h2d_bytes < tr.full_built_bytes


def test_train_report_matches_reference_cli_golden():
    """§8f.3: the dtgnn.report/1 document of the reference CLI's frozen
    golden run, produced by this package on the GPU (timing excluded)."""
    from paper_2109_07893_b200 import wire
    fx = load("cli_report")
    ref = jload(fx["report"])
    g = product_graph(fx)
    rep, _ = wire.train_report(g, dict(ref["config"]))
    assert rep["schema"] == ref["schema"] == "dtgnn.report/1"
    assert set(rep) == set(ref) | {"timing"}
    assert rep["config"] == ref["config"]
    assert rep["comm"] == ref["comm"] and rep["transfer"] == ref["transfer"]
    assert rep["activation_peak"] == ref["activation_peak"]
    for a, b in zip(rep["epochs"], ref["epochs"]):
        assert a["epoch"] == b["epoch"] and a["loss"] == pytest.approx(b["loss"], rel=RTOL)


def test_egcn_midsize_vs_oracle(oracle):
    """§8f.4 EGCN-O at N = 20k, T = 8, hidden 32: P = 1 and emulated P = 4
    against the oracle's checkpointed backward (pinned to the reference by
    tests/test_oracle_golden.py::test_egcn_oracle_pinned)."""
    from paper_2109_07893_b200.synth import churn_graph
    g = churn_graph(20_000, 8, 30_000, 0.10, seed=6)
    cfg = pk.ModelConfig("egcn-o", hidden_features=32, embed_features=32)
    data = pk.prepare_training_data(cfg, g)
    train, _ = pk.sample_link_prediction_sets(g, 0.1, 10)
    params = pk.init_params(cfg, 5)
    rng = np.random.default_rng(2)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    l1, g1 = pk.backward_checkpoint(cfg, data, train, params, 2)
    l4, g4, comm, tr = pk.distributed_epoch(cfg, data, train, params, 4, 2)
    ocfg = oracle.Cfg("egcn-o", 2, 32, 32)
    P = oracle.prepare(ocfg, [oracle.Coo(s.dim, s.rows, s.cols, s.vals) for s in g.snapshots])
    lo, go = oracle.backward_checkpoint(ocfg, P, train.by_time, params, 2)
    assert l1 == pytest.approx(lo, rel=RTOL)
    assert l4 == pytest.approx(lo, rel=RTOL)
    assert_grads_close(g1, go, RTOL, ENGINE_ATOL)
    assert_grads_close(g4, go, RTOL, ENGINE_ATOL)
    assert comm.redistribution_units == 0 and comm.alltoall_events() == []


@pytest.mark.parametrize("arch", ["cd-gcn", "tm-gcn", "egcn-o"])
def test_first_layer_products_bit_exact(oracle, arch):
    """H5 (`models.py:326-332`, `training.py:212`): the device's s1[t] =
    Ahat_t X_t -- degree features (of the raw graph, M-smoothed for tm-gcn,
    of the edge-life graph for egcn-o) and the fp64 SpMM in canonical order
    -- equals the oracle's fp64 s1 rounded once to fp32, for every t."""
    from paper_2109_07893_b200.synth import aml_graph
    g = aml_graph(5000, 6, 20_000, 0.1, seed=3)
    cfg = pk.ModelConfig(arch, hidden_features=16, embed_features=16)
    data = pk.prepare_training_data(cfg, g)
    eng = pk.api.get_engine(cfg, data, 1, 2)
    eng.set_labels({}, None)
    ocfg = oracle.Cfg(arch, 2, 16, 16)
    P = oracle.prepare(ocfg, [oracle.Coo(s.dim, s.rows, s.cols, s.vals) for s in g.snapshots])
    r = eng.ranks[0]
    for t in range(g.num_timesteps):
        got = r.s1[t].view(g.num_vertices, -1).cpu().numpy()
        assert np.array_equal(got[:, :2], P.s1[t].astype(np.float32)), t
        assert not got[:, 2:].any()


@pytest.mark.parametrize("workers,nblk,window", [(2, 2, 2), (4, 2, 2), (4, 1, 2), (2, 2, 3), (2, 1, 3)])
def test_tm_halo_matches_redistribution_bitwise(workers, nblk, window, monkeypatch):
    """tm-gcn at P > 1: the M-product on each rank's own snapshots with a
    (w - 1)-frame halo (previous rank's operator inputs, next rank's output
    gradients, cross-block trailing / owed frames) against the reference's
    snapshot <-> vertex redistribution: identical loss, gradients (bit for
    bit) and ledgers."""
    import paper_2109_07893_b200.engine as engine_mod
    fx = load("tmgcn_small")
    meta = jload(fx["cfg"])
    cfg = pk.ModelConfig(architecture="tm-gcn", in_features=2, hidden_features=meta["hidden"],
                         embed_features=meta["hidden"], window=window)
    data = pk.prepare_training_data(cfg, product_graph(fx))
    train = pk.LabelSet(2, labels_from(fx, "train_"))
    params = params_from(fx, "p_")
    out = {}
    for halo in ("1", "0"):
        monkeypatch.setattr(engine_mod, "TM_HALO", halo)
        pk.api.clear_engines()
        out[halo] = pk.distributed_epoch(cfg, data, train, params, workers, nblk)
    (la, ga, ca, ta), (lb, gb, cb, tb) = out["1"], out["0"]
    assert la == lb
    for k in ga:
        assert np.array_equal(ga[k], gb[k]), k
    assert ca.as_dict() == cb.as_dict() and ca.events == cb.events
    assert ta.as_dict() == tb.as_dict()


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small"])
def test_block0_slot_sets_do_not_change_results(name, monkeypatch):
    """keep_graphs with two or three block-0 slot sets (the next epochs'
    rebuilds overlap one or two epochs of compute): identical trajectories
    over three epochs (every epoch rebuilds its graphs into a rotated set)."""
    import paper_2109_07893_b200.engine as engine_mod
    fx, cfg, data, train, test, _ = product_case(name)
    out = {}
    for sets in ("2", "3"):
        monkeypatch.setattr(engine_mod, "BLOCK0_SETS", sets)
        monkeypatch.setattr(engine_mod, "KEEP_GRAPHS", "auto")
        pk.api.clear_engines()
        out[sets] = pk.train_distributed(cfg, data, train, test, epochs=3, seed=3, workers=2, nblk=1)
    (ta, pa, *_), (tb, pb, *_) = out["2"], out["3"]
    assert [a["loss"] for a in ta] == [b["loss"] for b in tb]
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k

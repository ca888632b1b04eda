"""Pin the CPU oracle (oracle/dtgnn_oracle.py) against golden vectors that the
reference itself produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import graph_keys, jload, labels_from, load, params_from


def coo_list(O, fx, prefix="g_"):
    n, snaps = graph_keys(fx, prefix)
    return n, [O.Coo(n, r, c, v) for r, c, v in snaps]


def test_canonical_from_entries(oracle):
    a = oracle.coo_from_entries(3, [2, 0, 2], [1, 2, 1], [1.0, 2.0, 3.0])
    assert list(zip(a.rows, a.cols, a.vals)) == [(0, 2, 2.0), (2, 1, 4.0)]
    assert oracle.coo_from_entries(3, [1, 1], [1, 1], [2.0, -2.0]).nnz == 0


@pytest.mark.parametrize("graph,lap", [("g_", "lap"), ("gw_", "lapw")])
def test_laplacian_bit_exact(oracle, graph, lap):
    fx = load("codec")
    n, snaps = coo_list(oracle, fx, graph)
    for t, s in enumerate(snaps):
        got = oracle.laplacian(s)
        assert np.array_equal(got.rows, fx[f"{lap}{t}_rows"])
        assert np.array_equal(got.cols, fx[f"{lap}{t}_cols"])
        assert np.array_equal(got.vals, fx[f"{lap}{t}_vals"])  # bitwise


def test_laplacian_zero_elided_diagonal(oracle):
    fx = load("codec")
    s = oracle.Coo(12, fx["neg_rows"], fx["neg_cols"], fx["neg_vals"])
    got = oracle.laplacian(s)
    assert np.array_equal(got.rows, fx["lapneg_rows"])
    assert np.array_equal(got.cols, fx["lapneg_cols"])
    assert np.array_equal(got.vals, fx["lapneg_vals"])


def test_degree_features_and_s1_bit_exact(oracle):
    fx = load("codec")
    n, snaps = coo_list(oracle, fx)
    feats = oracle.degree_feats(snaps)
    for t, s in enumerate(snaps):
        assert np.array_equal(feats[t], fx[f"feat{t}"])
        s1 = oracle.spmm(oracle.laplacian(s), feats[t])
        assert np.array_equal(s1, fx[f"s1_{t}"])


def test_delta_encode_apply_and_ledger(oracle):
    fx = load("codec")
    n, snaps = coo_list(oracle, fx)
    for t in range(1, len(snaps)):
        ep, en, vals = oracle.delta_encode(snaps[t - 1], snaps[t])
        assert np.array_equal(ep, fx[f"ext_prev{t}"])
        assert np.array_equal(en, fx[f"ext_next{t}"])
        assert oracle.delta_apply(snaps[t - 1], ep, en, vals).same(snaps[t])
    led = oracle.Transfer()
    laps = [oracle.laplacian(s) for s in snaps]
    rebuilt = oracle.stream(laps, led)
    assert all(a.same(b) for a, b in zip(rebuilt, laps))
    assert led.as_dict() == jload(fx["stream_ledger"])


def test_delta_corruption_detected(oracle):
    a = oracle.coo_from_entries(4, [0], [1], [1.0])
    with pytest.raises(oracle.OracleCorruptDelta):
        oracle.delta_apply(a, np.array([[2, 2]]), np.zeros((0, 2), np.int64), np.array([1.0]))
    with pytest.raises(oracle.OracleCorruptDelta):
        oracle.delta_apply(a, np.zeros((0, 2), np.int64), np.array([[0, 1]]), np.array([1.0]))
    with pytest.raises(oracle.OracleCorruptDelta):
        oracle.delta_apply(a, np.zeros((0, 2), np.int64), np.zeros((0, 2), np.int64),
                           np.array([1.0, 2.0]))


def test_spmm_bit_exact(oracle):
    fx = load("spmm")
    a = oracle.Coo(30, fx["a_rows"], fx["a_cols"], fx["a_vals"])
    assert np.array_equal(oracle.spmm(a, fx["x"]), fx["spmm"])
    assert np.array_equal(oracle.spmm_t(a, fx["x"]), fx["spmm_t"])


def test_lstm_block(oracle):
    fx = load("lstm")
    ts = [3, 4, 5]
    xs = {t: fx[f"x{t}"] for t in ts}
    ys, (h, c), cache = oracle.lstm_fwd(fx["wx"], fx["wh"], fx["b"], (fx["h0"], fx["c0"]), ts, xs)
    for t in ts:
        np.testing.assert_allclose(ys[t], fx[f"y{t}"], rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(c, fx["c"], rtol=1e-13, atol=1e-14)
    dys = {t: fx[f"dy{t}"] for t in ts}
    dxs, (dh, dc), (dwx, dwh, db) = oracle.lstm_bwd(fx["wx"], fx["wh"], ts, cache, dys,
                                                    (fx["dh0"], fx["dc0"]))
    for got, key in ((dh, "dh"), (dc, "dc"), (dwx, "dwx"), (dwh, "dwh"), (db, "db")):
        np.testing.assert_allclose(got, fx[key], rtol=1e-12, atol=1e-13)
    for t in ts:
        np.testing.assert_allclose(dxs[t], fx[f"dx{t}"], rtol=1e-12, atol=1e-13)


def _case(oracle, name):
    fx = load(name)
    meta = jload(fx["cfg"])
    cfg = oracle.Cfg(meta["architecture"], 2, meta["hidden"], meta["hidden"], 2, meta["window"])
    n, snaps = coo_list(oracle, fx)
    P = oracle.prepare(cfg, snaps)
    return fx, cfg, P


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small"])
def test_init_params_bit_exact(oracle, name):
    fx = load(name)
    meta = jload(fx["cfg"])
    cfg = oracle.Cfg(meta["architecture"], 2, meta["hidden"], meta["hidden"], 2, meta["window"])
    seed = 3 if name.startswith("cd") else 2
    got = oracle.init_params(cfg, seed)
    ref = params_from(fx, "init_")
    assert sorted(got) == sorted(ref)
    for k in ref:
        assert np.array_equal(got[k], ref[k]), k


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small"])
def test_label_sampler_bit_exact(oracle, name):
    fx, cfg, P = _case(oracle, name)
    seed = 5 if name.startswith("cd") else 7
    train, test = oracle.sample_labels(P.graph if cfg.architecture == "cd-gcn" else
                                       coo_list(oracle, fx)[1], 0.5, seed)
    ref_train, ref_test = labels_from(fx, "train_"), labels_from(fx, "test_")
    for got, ref in ((train, ref_train), (test, ref_test)):
        assert sorted(got) == sorted(ref)
        for t in ref:
            assert np.array_equal(got[t][0], ref[t][0])
            assert np.array_equal(got[t][1], ref[t][1])


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small"])
def test_checkpoint_engine(oracle, name):
    fx, cfg, P = _case(oracle, name)
    params = params_from(fx, "p_")
    train = labels_from(fx, "train_")
    for nblk in (1, 2, 4):
        loss, grads = oracle.backward_checkpoint(cfg, P, train, params, nblk)
        assert loss == pytest.approx(float(fx[f"ckpt{nblk}_loss"]), rel=1e-12)
        ref = params_from(fx, f"ckpt{nblk}_g_")
        for k in ref:
            np.testing.assert_allclose(grads[k], ref[k], rtol=1e-9, atol=1e-12, err_msg=k)


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small"])
@pytest.mark.parametrize("workers,nblk", [(2, 2), (4, 1), (2, 1)])
def test_distributed_epoch_and_ledgers(oracle, name, workers, nblk):
    fx, cfg, P = _case(oracle, name)
    params = params_from(fx, "p_")
    train = labels_from(fx, "train_")
    tag = f"dist{workers}x{nblk}"
    for threads in (False, True):
        loss, grads, comm, tr = oracle.distributed_epoch(cfg, P, train, params, workers, nblk,
                                                         threads=threads)
        assert loss == pytest.approx(float(fx[f"{tag}_loss"]), rel=1e-12)
        ref = params_from(fx, f"{tag}_g_")
        for k in ref:
            np.testing.assert_allclose(grads[k], ref[k], rtol=1e-9, atol=1e-12, err_msg=k)
        assert comm.as_dict() == jload(fx[f"{tag}_comm"])
        assert comm.events == jload(fx[f"{tag}_events"])
        assert tr.as_dict() == jload(fx[f"{tag}_transfer"])


@pytest.mark.parametrize("name", ["cdgcn_small", "tmgcn_small"])
def test_model_forward_and_training(oracle, name):
    fx, cfg, P = _case(oracle, name)
    params = params_from(fx, "p_")
    z = oracle.model_forward(cfg, P, params)
    for t, f in enumerate(z):
        np.testing.assert_allclose(f, fx[f"z{t}"], rtol=1e-11, atol=1e-13)
    seed = 3 if name.startswith("cd") else 2
    trace, fparams, comm, tr = oracle.train_distributed(
        cfg, P, labels_from(fx, "train_"), labels_from(fx, "test_"), 3, seed, 2, 2)
    ref_trace = jload(fx["train_trace"])
    for a, b in zip(trace, ref_trace):
        assert a["epoch"] == b["epoch"]
        assert a["loss"] == pytest.approx(b["loss"], rel=1e-10)
        assert a["test_accuracy"] == b["test_accuracy"]
    ref_p = params_from(fx, "train_p_")
    for k in ref_p:
        np.testing.assert_allclose(fparams[k], ref_p[k], rtol=1e-8, atol=1e-11, err_msg=k)
    assert comm.as_dict() == jload(fx["train_comm"])
    assert tr.as_dict() == jload(fx["train_transfer"])


def test_cli_golden_report_counters(oracle):
    """The reference's frozen CLI report (tm-gcn, P=2, nblk=2, 2 epochs)."""
    fx = load("cli_report")
    rep = jload(fx["report"])
    n, snaps = coo_list(oracle, fx)
    c = rep["config"]
    cfg = oracle.Cfg(c["model"], 2, c["hidden"], c["embed"], c["layers"], c["window"])
    P = oracle.prepare(cfg, snaps)
    train, test = oracle.sample_labels(snaps, c["theta"], c["seed"] + 1000003)
    trace, _, comm, tr = oracle.train_distributed(cfg, P, train, test, c["epochs"], c["seed"],
                                                  c["workers"], c["blocks"], lr=c["lr"])
    assert comm.as_dict() == rep["comm"]
    assert tr.as_dict() == rep["transfer"]
    for a, b in zip(trace, rep["epochs"]):
        assert a["loss"] == pytest.approx(b["loss"], rel=1e-12)
        assert a["test_accuracy"] == b["test_accuracy"]


def test_delta_record_golden_bytes():
    """Reference binary record layout (delta.py:181-197, test_delta.py:200-215)."""
    from pathlib import Path
    blob = (Path(__file__).parent / "golden" / "delta_record.bin").read_bytes()
    assert blob == (b"\x01\x00\x00\x00" b"\x00\x00\x00\x00\x01\x00\x00\x00"
                    b"\x01\x00\x00\x00" b"\x01\x00\x00\x00\x01\x00\x00\x00"
                    b"\x01\x00\x00\x00" b"\x00\x00\x00\x00\x00\x00\x04\x40")


def test_c1_pins(oracle):
    """BASELINE config 1 (N=10k, T=8, 50k edges, 10% churn, cd-gcn H=32):
    the oracle's checkpointed epoch vs the reference's stored result."""
    from paper_2109_07893_b200.synth import churn_keys
    fx = load("c1_pins")
    n = 10_000
    snaps = [oracle.Coo(n, k // n, k % n, np.ones(k.shape[0]))
             for k in churn_keys(n, 8, 50_000, 0.10, seed=1)]
    cfg = oracle.Cfg("cd-gcn", 2, 32, 32)
    P = oracle.prepare(cfg, snaps)
    assert [l.nnz for l in P.laps] == fx["lap_nnz"].tolist()
    assert np.array_equal(np.array([float(np.sum(l.vals)) for l in P.laps]), fx["lap_valsum"])
    train, _ = oracle.sample_labels(snaps, 0.1, 1 + 1000003)
    assert [train[t][0].shape[0] for t in sorted(train)] == fx["train_pairs"].tolist()
    params = oracle.init_params(cfg, 0)
    rng = np.random.default_rng(77)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    params["head.b"] = rng.uniform(-0.1, 0.1, size=params["head.b"].shape)
    loss, grads = oracle.backward_checkpoint(cfg, P, train, params, 2)
    assert loss == pytest.approx(float(fx["loss"]), rel=1e-12)
    for k in grads:
        np.testing.assert_allclose(grads[k], fx[f"g_{k}"], rtol=1e-8, atol=1e-12, err_msg=k)


@pytest.mark.parametrize("arch", ["cd-gcn", "tm-gcn"])
def test_cone_forward_equals_full_forward(oracle, arch):
    """The dependency-cone forward used by the large-config parity tests is
    bit-identical to the full forward on the sampled rows."""
    from paper_2109_07893_b200.synth import aml_keys, churn_keys
    n = 400
    keys = (churn_keys if arch == "cd-gcn" else aml_keys)(n, 6, 900, 0.1, seed=3)
    snaps = [oracle.Coo(n, k // n, k % n, np.ones(k.shape[0])) for k in keys]
    cfg = oracle.Cfg(arch, 2, 8, 8)
    P = oracle.prepare(cfg, snaps)
    params = oracle.init_params(cfg, 1)
    full = oracle.model_forward(cfg, P, params)
    rows = np.array([3, 50, 51, 399, 200])
    part = oracle.model_forward_rows(cfg, lambda t: P.laps[t], lambda t: P.feats[t], P.T, params, rows, P.m,
                                     P.window)
    for t in range(P.T):
        assert np.array_equal(full[t][np.unique(rows)], part[t])


def test_egcn_oracle_pinned(oracle):
    """§8f.4 EGCN-O: the oracle's restatement (edge life, weight-evolution
    chain forward / backward, initial-weight gradient) against the
    reference's own outputs: init params, full backward, checkpointed
    backward at nblk 1 / 2 / 4, forward frames."""
    fx, cfg, P = _case(oracle, "egcn_small")
    init = oracle.init_params(cfg, 4)
    ref_init = params_from(fx, "init_")
    assert sorted(init) == sorted(ref_init)
    for k in ref_init:
        assert np.array_equal(init[k], ref_init[k]), k
    params = params_from(fx, "p_")
    train = labels_from(fx, "train_")
    for nblk, tag in ((1, "full"), (1, "ckpt1"), (2, "ckpt2"), (4, "ckpt4")):
        loss, grads = oracle.backward_checkpoint(cfg, P, train, params, nblk)
        assert loss == pytest.approx(float(fx[f"{tag}_loss"]), rel=1e-12)
        ref = params_from(fx, f"{tag}_g_")
        assert sorted(grads) == sorted(ref)
        for k in ref:
            np.testing.assert_allclose(grads[k], ref[k], rtol=1e-9, atol=1e-12, err_msg=(tag, k))
    z = oracle.model_forward(cfg, P, params)
    for t, f in enumerate(z):
        np.testing.assert_allclose(f, fx[f"z{t}"], rtol=1e-11, atol=1e-13)

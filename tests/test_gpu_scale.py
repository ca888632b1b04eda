"""Parity at the benchmarked shapes (SURVEY §8c large-config protocol).

Full-graph oracle epochs are infeasible at configs[1] / configs[2] (the
reference needs > 62 GB and ~45 min per c2 epoch), so these shapes are
checked the way §8c prescribes:

* per-kernel oracle checks on real snapshots of the config: the device
  rebuild (K1 + transpose + K2) bit-exact against the oracle Laplacian of
  the same snapshot (structure, fp64 and fp32 values, both operands), the
  fused GCN (K3: SpMM + W + ReLU) and the transpose SpMM (K4) on sampled
  rows against fp64;
* a vertex-sampled forward check of the full-shape model: the rows of the
  SpMM and the per-vertex LSTM / M-product timelines are independent
  (`test_models.py:267-285`), so the oracle runs the forward on the
  dependency cone of a vertex sample (`dtgnn_oracle.model_forward_rows`)
  and every output frame's sampled rows are compared;
* emulated P = 4 against P = 1 over a full training epoch (loss and every
  gradient).

Tolerance: the north star's 1e-4 relative, guarded by the measured tcgen05
floor (conftest.ENGINE_ATOL = 1e-5 x ||r||_inf; measured worst ~2e-6 for
forward activations, ~7e-6 for layer-0 gradients at hidden 64 -- DESIGN §5);
kernel-level checks at 1e-6 x ||r||_inf; graph work bit-exact.
"""

import numpy as np
import pytest
import torch

import paper_2109_07893_b200 as pk

from conftest import ENGINE_ATOL, assert_grads_close, guarded_close

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _head(params, seed=77):
    rng = np.random.default_rng(seed)
    params["head.w"] = rng.uniform(-0.5, 0.5, size=params["head.w"].shape)
    params["head.b"] = rng.uniform(-0.1, 0.1, size=params["head.b"].shape)
    return params


@pytest.fixture(scope="module")
def c2(oracle):
    """configs[1]: N = 750k, T = 32, 468,750 edges per snapshot, 10% churn,
    cd-gcn hidden 64, nblk 4 -- exactly the bench workload."""
    from paper_2109_07893_b200.synth import churn_graph
    g = churn_graph(750_000, 32, 468_750, 0.10, seed=1)
    cfg = pk.ModelConfig("cd-gcn", hidden_features=64, embed_features=64)
    data = pk.prepare_training_data(cfg, g)
    train, _ = pk.sample_link_prediction_sets(g, 0.1, 1 + 1000003)
    params = _head(pk.init_params(cfg, 0))
    coos = [oracle.Coo(g.num_vertices, np.asarray(s.rows), np.asarray(s.cols), np.asarray(s.vals))
            for s in g.snapshots]
    yield dict(g=g, cfg=cfg, data=data, train=train, params=params, coos=coos, laps={})
    pk.api.clear_engines()


def _lap(oracle, case, t):
    if t not in case["laps"]:
        case["laps"][t] = oracle.laplacian(case["coos"][t])
    return case["laps"][t]


def _check_slot(s, ref, n):
    rp = s.rowptr.cpu().numpy()
    m = int(rp[-1])
    assert m == ref.nnz
    assert np.array_equal(np.repeat(np.arange(n), np.diff(rp)), ref.rows)
    assert np.array_equal(s.col[:m].cpu().numpy(), ref.cols)
    assert np.array_equal(s.val[:m].cpu().numpy(), ref.vals.astype(np.float32))
    order = np.lexsort((ref.rows, ref.cols))
    trp = s.t_rowptr.cpu().numpy()
    assert np.array_equal(np.repeat(np.arange(n), np.diff(trp)), ref.cols[order])
    assert np.array_equal(s.t_col[:m].cpu().numpy(), ref.rows[order])
    assert np.array_equal(s.t_val[:m].cpu().numpy(), ref.vals[order].astype(np.float32))


def test_c2_snapshots_rebuilt_bit_exact(oracle, c2):
    """The engine's rebuild of real configs[1] snapshots (chunks of the
    nblk = 4 schedule: heads from the previous chunk's last snapshot, then
    1-step deltas) against the oracle Laplacians, bit for bit."""
    from paper_2109_07893_b200.materialize import Materializer, SnapshotEncoding
    g = c2["g"]
    n = g.num_vertices
    enc = SnapshotEncoding(g)
    mat = Materializer(enc, "cuda", slots=8, resident=False, with_f64=True)
    for ts in (list(range(0, 8)), list(range(8, 16)), list(range(24, 32))):
        slots = mat.materialize(ts)
        mat.wait()
        torch.cuda.synchronize()
        for s, t in zip(slots, ts):
            if t in (0, 7, 8, 15, 24, 31):
                ref = _lap(oracle, c2, t)
                _check_slot(s, ref, n)
                assert np.array_equal(s.val64[:ref.nnz].cpu().numpy(), ref.vals)
    mat.check()
    # the third chunk's head (t = 24) followed nothing: shipped in full
    assert [b[2] for b in mat.builds] == [False, True, False]


def test_c2_fused_gcn_and_transpose_spmm_sampled_rows(oracle, c2):
    """K3 (SpMM + W + ReLU, tcgen05) and K4 (Ahat^T SpMM) on a real
    configs[1] snapshot at the layer-1 width (64), 4096 sampled rows vs fp64."""
    from paper_2109_07893_b200.ops import gcn_forward, spmm_f32
    g = c2["g"]
    n = g.num_vertices
    ref = _lap(oracle, c2, 9)
    rng = np.random.default_rng(9)
    x = rng.standard_normal((n, 64)).astype(np.float32)
    w = (rng.standard_normal((64, 64)) * 0.2).astype(np.float32)
    rowptr = np.concatenate([[0], np.cumsum(np.bincount(ref.rows, minlength=n))]).astype(np.int32)
    s, r = gcn_forward(n, rowptr, ref.cols.astype(np.int32), ref.vals.astype(np.float32), x, w, True)
    rows = np.sort(rng.choice(n, 4096, replace=False))
    idx = oracle._rows_of(ref, rows)
    want = np.zeros((rows.size, 64))
    np.add.at(want, np.searchsorted(rows, ref.rows[idx]), ref.vals[idx][:, None] * x.astype(np.float64)[ref.cols[idx]])
    ok, worst, nbad = guarded_close(s[rows], want, RTOL, 1e-6)
    assert ok, (worst, nbad)
    q = np.maximum(want @ w.astype(np.float64), 0.0)
    ok, worst, nbad = guarded_close(r[rows, 64:], q, RTOL, 1e-6)
    assert ok, (worst, nbad)
    assert np.array_equal(r[rows, :64], np.maximum(s[rows], 0))
    # K4: Ahat^T g over the transposed operand (CSR of Ahat^T)
    order = np.lexsort((ref.rows, ref.cols))
    trp = np.concatenate([[0], np.cumsum(np.bincount(ref.cols, minlength=n))]).astype(np.int32)
    gy = rng.standard_normal((n, 64)).astype(np.float32)
    dt = spmm_f32(trp, ref.rows[order].astype(np.int32), ref.vals[order].astype(np.float32), gy)
    tcols = ref.cols[order]
    lo, hi = np.searchsorted(tcols, rows, "left"), np.searchsorted(tcols, rows, "right")
    tidx = np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)])
    want_t = np.zeros((rows.size, 64))
    np.add.at(want_t, np.searchsorted(rows, tcols[tidx]),
              ref.vals[order][tidx][:, None] * gy.astype(np.float64)[ref.rows[order][tidx]])
    ok, worst, nbad = guarded_close(dt[rows], want_t, RTOL, 1e-6)
    assert ok, (worst, nbad)


def test_c2_forward_sampled_vertices_vs_oracle(oracle, c2):
    """The full configs[1] forward (T = 32, nblk = 4, 750k vertices) on the
    device; 512 sampled vertices' rows of all 32 output frames against the
    oracle forward on their dependency cone."""
    g, cfg, params = c2["g"], c2["cfg"], c2["params"]
    n = g.num_vertices
    rng = np.random.default_rng(3)
    rows = np.sort(rng.choice(n, 512, replace=False))
    got = pk.model_forward_frames(cfg, c2["data"], params, nblk=4, rows=rows)
    feats = oracle.degree_feats(c2["coos"])
    want = oracle.model_forward_rows(oracle.Cfg("cd-gcn", 2, 64, 64), lambda t: _lap(oracle, c2, t),
                                     lambda t: feats[t], g.num_timesteps, params, rows)
    need = 0.0
    for t in range(g.num_timesteps):
        ok, worst, nbad = guarded_close(got[t], want[t], RTOL, ENGINE_ATOL)
        assert ok, (t, worst, nbad)
        ex = np.maximum(0.0, np.abs(got[t] - want[t]) - RTOL * np.maximum(np.abs(got[t]), np.abs(want[t])))
        need = max(need, float(ex.max() / np.abs(want[t]).max()))
    # measured error budget: the tcgen05 temporal GEMMs
    # (3xTF32, truncating fp32 accumulation) leave ~2e-6 x ||r||_inf on
    # near-zero embeddings after 32 recurrent steps
    print(f"c2 forward: needed atol fraction {need:.2e}")
    assert need <= 5e-6


def test_c2_emulated_four_ranks_equal_one_rank(c2):
    """A full configs[1] training epoch: emulated P = 4 (split GCN, owner /
    vertex-major layouts, head chain) against P = 1: loss and every
    gradient, plus the reference's communication volume law."""
    cfg, data, train, params = c2["cfg"], c2["data"], c2["train"], c2["params"]
    l1, g1 = pk.backward_checkpoint(cfg, data, train, params, 4)
    pk.api.clear_engines()
    l4, g4, comm, tr = pk.distributed_epoch(cfg, data, train, params, 4, 4)
    pk.api.clear_engines()
    assert l4 == pytest.approx(l1, rel=1e-6)
    assert_grads_close(g4, g1, RTOL, ENGINE_ATOL)
    n, T = data.num_vertices, data.num_timesteps
    assert comm.redistribution_units == 6 * 2 * T * n * 3 // 4
    # the whole job streamed every snapshot after t = 0 as a 1-step delta
    assert tr.full_built_bytes / tr.h2d_bytes > 4.0


@pytest.fixture(scope="module")
def c3(oracle):
    """configs[2]: TM-GCN (window 2) hidden 32 on the AMLSim-style graph,
    N = 1M, T = 64, 2M edges per snapshot, heavy-tailed degrees, 2% churn,
    nblk 8 -- the bench workload (smoothed on the device)."""
    from paper_2109_07893_b200.synth import aml_graph
    g = aml_graph(1_000_000, 64, 2_000_000, 0.02, seed=1)
    cfg = pk.ModelConfig("tm-gcn", hidden_features=32, embed_features=32)
    data = pk.prepare_training_data(cfg, g)
    params = _head(pk.init_params(cfg, 0))
    coos = [oracle.Coo(g.num_vertices, np.asarray(s.rows), np.asarray(s.cols), np.asarray(s.vals))
            for s in g.snapshots]
    m = data.m_matrix.matrix
    yield dict(g=g, cfg=cfg, data=data, params=params, coos=coos, m=m, laps={})
    pk.api.clear_engines()


def _slap(oracle, case, t):
    """Oracle Laplacian of the M-smoothed snapshot t (dtdg.py:239-252, 178-191)."""
    if t not in case["laps"]:
        m = case["m"]
        terms = [(m[t, k], case["coos"][k]) for k in range(max(0, t - 1), t + 1)]
        case["laps"][t] = oracle.laplacian(oracle.weighted_sum(terms))
    return case["laps"][t]


def test_c3_smoothed_snapshots_rebuilt_bit_exact(oracle, c3):
    """configs[2] smoothed snapshots rebuilt on the device (raw graph
    differences -> weighted merge -> transpose -> Laplacian) against the
    oracle's host smoothing + Laplacian, bit for bit, hub rows included."""
    from paper_2109_07893_b200.materialize import Materializer
    enc = c3["data"].graph.encoding
    n = c3["g"].num_vertices
    mat = Materializer(enc, "cuda", slots=8, resident=False, with_f64=True)
    for ts in (list(range(0, 8)), list(range(8, 16)), list(range(56, 64))):
        slots = mat.materialize(ts)
        mat.wait()
        torch.cuda.synchronize()
        for s, t in zip(slots, ts):
            if t in (0, 1, 8, 56, 63):
                ref = _slap(oracle, c3, t)
                _check_slot(s, ref, n)
                assert np.array_equal(s.val64[:ref.nnz].cpu().numpy(), ref.vals)
    mat.check()


def test_c3_forward_sampled_vertices_vs_oracle(oracle, c3):
    """The full configs[2] tm-gcn forward (T = 64, nblk = 8, 1M vertices,
    device smoothing) against the oracle's forward on the dependency cone of
    256 sampled vertices (GCN rows + per-vertex M-product timelines)."""
    g, cfg, params = c3["g"], c3["cfg"], c3["params"]
    n, T = g.num_vertices, g.num_timesteps
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(n, 256, replace=False))
    got = pk.model_forward_frames(cfg, c3["data"], params, nblk=8, rows=rows)
    feats = oracle.m_transform_frames(oracle.degree_feats(c3["coos"]), c3["m"], 2)
    want = oracle.model_forward_rows(oracle.Cfg("tm-gcn", 2, 32, 32), lambda t: _slap(oracle, c3, t),
                                     lambda t: feats[t], T, params, rows, c3["m"], 2)
    need = 0.0
    for t in range(T):
        ok, worst, nbad = guarded_close(got[t], want[t], RTOL, 1e-6)
        assert ok, (t, worst, nbad)
        ex = np.maximum(0.0, np.abs(got[t] - want[t]) - RTOL * np.maximum(np.abs(got[t]), np.abs(want[t])))
        need = max(need, float(ex.max() / max(np.abs(want[t]).max(), 1e-300)))
    print(f"c3 forward: needed atol fraction {need:.2e}")


def test_c3_emulated_four_ranks_equal_one_rank(c3):
    """A full configs[2] training epoch (device smoothing, value-carrying
    smoothed Laplacians rebuilt every epoch, M-product trailing frames):
    emulated P = 4 against P = 1."""
    cfg, data, params = c3["cfg"], c3["data"], c3["params"]
    train, _ = pk.sample_link_prediction_sets(c3["g"], 0.1, 1 + 1000003)
    l1, g1 = pk.backward_checkpoint(cfg, data, train, params, 8)
    pk.api.clear_engines()
    l4, g4, comm, tr = pk.distributed_epoch(cfg, data, train, params, 4, 8)
    pk.api.clear_engines()
    assert l4 == pytest.approx(l1, rel=1e-6)
    assert_grads_close(g4, g1, RTOL, ENGINE_ATOL)
    assert tr.full_built_bytes / tr.h2d_bytes > 3.0


def test_c5_shape_device_generated_snapshots_rebuilt_exactly():
    """configs[4] shape (N = 10M, 15,625,000 edges per snapshot, 1% churn):
    the device generator's encoding, streamed as the engine does (full head,
    then 1-step deltas; the next chunk's head from the previous chunk's last
    snapshot), rebuilds every snapshot's CSR exactly (size-independent
    property: structure == the generator's sorted keys; the Laplacian keeps
    A plus the diagonal)."""
    from paper_2109_07893_b200.materialize import Materializer
    from paper_2109_07893_b200.synth import device_churn_graph
    n, T, m = 10_000_000, 4, 15_625_000
    g = device_churn_graph(n, T, m, 0.01, 1, torch.device("cuda"))
    mat = Materializer(g.encoding, "cuda", slots=2, sets=2)
    diag = torch.arange(n, dtype=torch.int64, device="cuda") * (n + 1)
    for i, ts in enumerate(([0, 1], [2, 3])):
        slots = mat.materialize(ts, set_idx=i)
        mat.wait()
        for s, t in zip(slots, ts):
            rp = s.rowptr.long()
            nnz = int(rp[-1])
            rows = torch.repeat_interleave(torch.arange(n, device="cuda"), rp[1:] - rp[:-1])
            got = rows * n + s.col[:nnz].long()
            want = torch.unique(torch.cat([g._keys[t], diag]))
            assert torch.equal(got, want), t
    assert [b[2] for b in mat.builds] == [False, True]
    mat.check()
    g.drop_keys()

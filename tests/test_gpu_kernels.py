"""GPU parity of the individual kernels against golden fixtures produced by
the reference and against the CPU oracle.  Integer / graph work must be
bit-exact; fp64 kernels bit-exact; fp32 training kernels within 1e-4
relative (guarded: |g - r| <= 1e-4 max(|g|,|r|) + 1e-6 ||r||_inf)."""

import numpy as np
import pytest
import torch

import paper_2109_07893_b200 as pk

from conftest import guarded_close, load
from helpers import product_graph

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def sm(fx, prefix, n):
    return pk.SparseMatrix.from_canonical(n, fx[f"{prefix}rows"], fx[f"{prefix}cols"], fx[f"{prefix}vals"])


def test_spmm_and_transpose_bit_exact():
    fx = load("spmm")
    a = sm(fx, "a_", 30)
    assert np.array_equal(pk.spmm(a, fx["x"]), fx["spmm"])
    assert np.array_equal(pk.spmm_transpose(a, fx["x"]), fx["spmm_t"])


def test_spmm_empty_and_identity():
    x = np.arange(6, dtype=np.float64).reshape(3, 2)
    assert np.array_equal(pk.spmm(pk.SparseMatrix.identity(3), x), x)
    assert np.array_equal(pk.spmm(pk.SparseMatrix.empty(3), x), np.zeros((3, 2)))
    with pytest.raises(pk.InputError):
        pk.spmm(pk.SparseMatrix.identity(3), np.ones((2, 2)))


@pytest.mark.parametrize("graph,lap", [("g_", "lap"), ("gw_", "lapw")])
def test_laplacian_bit_exact(graph, lap):
    fx = load("codec")
    g = product_graph(fx, graph)
    for t, s in enumerate(g.snapshots):
        got = pk.normalize_laplacian(s)
        assert np.array_equal(got.rows, fx[f"{lap}{t}_rows"])
        assert np.array_equal(got.cols, fx[f"{lap}{t}_cols"])
        assert np.array_equal(got.vals, fx[f"{lap}{t}_vals"])


def test_laplacian_zero_elision_and_transpose_form():
    from paper_2109_07893_b200.ops import normalize_laplacian_transpose
    fx = load("codec")
    s = sm(fx, "neg_", 12)
    got = pk.normalize_laplacian(s)
    assert np.array_equal(got.rows, fx["lapneg_rows"])
    assert np.array_equal(got.vals, fx["lapneg_vals"])
    g = product_graph(fx, "gw_")
    for t, snap in enumerate(g.snapshots):
        tr = normalize_laplacian_transpose(snap)
        ref = pk.SparseMatrix.from_entries(snap.dim, fx[f"lapw{t}_cols"], fx[f"lapw{t}_rows"],
                                           fx[f"lapw{t}_vals"])
        assert tr == ref


def test_apply_round_trip_and_reference_deltas():
    fx = load("codec")
    g = product_graph(fx)
    for t in range(1, g.num_timesteps):
        d = pk.diff(g.snapshots[t - 1], g.snapshots[t])
        assert np.array_equal(d.ext_prev, fx[f"ext_prev{t}"])
        assert pk.apply(g.snapshots[t - 1], d) == g.snapshots[t]
    gw = product_graph(fx, "gw_")
    for a, b in zip(gw.snapshots, gw.snapshots[1:]):
        assert pk.apply(a, pk.diff(a, b)) == b


def test_apply_corruption_errors():
    a = pk.SparseMatrix.from_entries(4, [0], [1], [1.0])
    bad = pk.SnapshotDelta(4, np.array([[2, 2]]), np.zeros((0, 2), np.int64), np.array([1.0]))
    with pytest.raises(pk.CorruptDeltaError):
        pk.apply(a, bad)
    bad = pk.SnapshotDelta(4, np.zeros((0, 2), np.int64), np.array([[0, 1]]), np.array([1.0]))
    with pytest.raises(pk.CorruptDeltaError):
        pk.apply(a, bad)
    bad = pk.SnapshotDelta(4, np.zeros((0, 2), np.int64), np.zeros((0, 2), np.int64), np.array([1.0, 2.0]))
    with pytest.raises(pk.CorruptDeltaError):
        pk.apply(a, bad)


def test_apply_randomized_round_trips(oracle):
    rng = np.random.default_rng(0)
    for _ in range(40):
        n = int(rng.integers(1, 12))
        def rnd():
            k = int(rng.integers(0, 20))
            return pk.SparseMatrix.from_entries(n, rng.integers(0, n, k), rng.integers(0, n, k),
                                                rng.choice([-2.0, 1.0, 0.5, 3.0], k))
        a, b = rnd(), rnd()
        got = pk.apply(a, pk.diff(a, b))
        assert got == b


def test_stream_block_ledger():
    import json
    fx = load("codec")
    g = product_graph(fx)
    laps = [pk.SparseMatrix.from_canonical(g.num_vertices, fx[f"lap{t}_rows"], fx[f"lap{t}_cols"],
                                           fx[f"lap{t}_vals"]) for t in range(g.num_timesteps)]
    led = pk.TransferLedger()
    out = list(pk.stream_block(laps, led))
    assert all(a == b for a, b in zip(out, laps))
    assert led.as_dict() == json.loads(str(fx["stream_ledger"]))


def test_materializer_rebuild_bit_exact(oracle):
    """K1 + transpose + K2 through the engine's materialiser, chunked like a
    P=2 partition (first snapshot full, rest deltas), both input modes."""
    from paper_2109_07893_b200.materialize import Materializer, SnapshotEncoding
    fx = load("codec")
    for prefix in ("g_", "gw_"):
        g = product_graph(fx, prefix)
        enc = SnapshotEncoding(g)
        for resident in (False, True):
            mat = Materializer(enc, "cuda", slots=3, resident=resident, with_f64=True)
            for ts in ([0, 1, 2], [3, 4, 5]):
                slots = mat.materialize(ts)
                mat.wait()
                torch.cuda.synchronize()
                for s, t in zip(slots, ts):
                    ref = oracle.laplacian(oracle.Coo(g.num_vertices, np.asarray(g.snapshots[t].rows),
                                                      np.asarray(g.snapshots[t].cols),
                                                      np.asarray(g.snapshots[t].vals)))
                    rp = s.rowptr.cpu().numpy()
                    m = int(rp[-1])
                    assert m == ref.nnz
                    rows = np.repeat(np.arange(g.num_vertices), np.diff(rp))
                    assert np.array_equal(rows, ref.rows)
                    assert np.array_equal(s.col[:m].cpu().numpy(), ref.cols)
                    assert np.array_equal(s.val64[:m].cpu().numpy(), ref.vals)
                    assert np.array_equal(s.val[:m].cpu().numpy(), ref.vals.astype(np.float32))
                    # transposed operand: CSR of Ahat^T
                    trp = s.t_rowptr.cpu().numpy()
                    trow = np.repeat(np.arange(g.num_vertices), np.diff(trp))
                    order = np.lexsort((ref.rows, ref.cols))
                    assert np.array_equal(trow, ref.cols[order])
                    assert np.array_equal(s.t_col[:m].cpu().numpy(), ref.rows[order])
                    assert np.array_equal(s.t_val64[:m].cpu().numpy(), ref.vals[order])
            mat.check()


def test_materializer_large_random_round_trip():
    """Size-independent property at scale: rebuilt structure equals the host
    snapshots (checksum of every snapshot) for a 200k-vertex churn graph."""
    from paper_2109_07893_b200.materialize import Materializer, SnapshotEncoding
    from paper_2109_07893_b200.synth import churn_keys
    n, T = 200_000, 6
    keys = churn_keys(n, T, 150_000, 0.1, seed=11)
    g = pk.DynamicGraph(n, [pk.SparseMatrix.from_canonical(n, k // n, k % n) for k in keys])
    enc = SnapshotEncoding(g)
    mat = Materializer(enc, "cuda", slots=T)
    slots = mat.materialize(list(range(T)))
    mat.wait()
    for s, k in zip(slots, keys):
        rp = s.rowptr.cpu().numpy().astype(np.int64)
        m = int(rp[-1])
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
        got = rows * n + s.col[:m].cpu().numpy()
        want = np.union1d(k, np.arange(n, dtype=np.int64) * (n + 1))
        assert np.array_equal(got, want)
    mat.check()


def test_lstm_block_fp32_vs_reference():
    from paper_2109_07893_b200.params import ModelConfig  # noqa: F401
    fx = load("lstm")

    class Cell:
        wx, wh, b = fx["wx"], fx["wh"], fx["b"]

    ts = [3, 4, 5]
    xs = {t: fx[f"x{t}"] for t in ts}
    ys, (h, c), cache = pk.lstm_block_forward(Cell, (fx["h0"], fx["c0"]), ts, xs)
    for t in ts:
        ok, worst, _ = guarded_close(ys[t], fx[f"y{t}"], RTOL)
        assert ok, worst
    assert guarded_close(c, fx["c"], RTOL)[0]
    dys = {t: fx[f"dy{t}"] for t in ts}
    dxs, (dh, dc), dcell = pk.lstm_block_backward(Cell, ts, cache, dys, (fx["dh0"], fx["dc0"]))
    for got, key in ((dh, "dh"), (dc, "dc"), (dcell["wx"], "dwx"), (dcell["wh"], "dwh"), (dcell["b"], "db")):
        ok, worst, _ = guarded_close(got, fx[key], RTOL)
        assert ok, (key, worst)
    for t in ts:
        assert guarded_close(dxs[t], fx[f"dx{t}"], RTOL)[0]


@pytest.mark.parametrize("H", [16, 32, 64, 128])
def test_lstm_kernels_wide_vs_oracle(oracle, H):
    rng = np.random.default_rng(H)
    rows, fin = 1000, 2 * H

    class Cell:
        wx = rng.uniform(-0.2, 0.2, (fin, 4 * H))
        wh = rng.uniform(-0.2, 0.2, (H, 4 * H))
        b = rng.uniform(-0.1, 0.1, 4 * H)

    ts = [0, 1, 2, 3]
    xs = {t: np.maximum(rng.standard_normal((rows, fin)), 0) for t in ts}
    st = (rng.standard_normal((rows, H)) * 0.1, rng.standard_normal((rows, H)) * 0.1)
    ys, (h, c), cache = pk.lstm_block_forward(Cell, st, ts, xs, tensor_cores=False)
    rys, (rh, rc), rcache = oracle.lstm_fwd(Cell.wx, Cell.wh, Cell.b, st, ts, xs)
    for t in ts:
        assert guarded_close(ys[t], rys[t], RTOL)[0]
    dys = {t: rng.standard_normal((rows, H)) for t in ts}
    dst = (rng.standard_normal((rows, H)), rng.standard_normal((rows, H)))
    dxs, dstate, dcell = pk.lstm_block_backward(Cell, ts, cache, dys, dst, tensor_cores=False)
    rdxs, rdstate, (rdwx, rdwh, rdb) = oracle.lstm_bwd(Cell.wx, Cell.wh, ts, rcache, dys, dst)
    for got, ref in ((dcell["wx"], rdwx), (dcell["wh"], rdwh), (dcell["b"], rdb), (dstate[0], rdstate[0]),
                     (dstate[1], rdstate[1])):
        ok, worst, nbad = guarded_close(got, ref, RTOL)
        assert ok, (worst, nbad)
    for t in ts:
        assert guarded_close(dxs[t], rdxs[t], RTOL)[0]


@pytest.mark.parametrize("n", [64, 128, 256])
@pytest.mark.parametrize("m,k", [(128, 16), (300, 132), (1000, 192)])
def test_tcgen05_3xtf32_gemm_is_fp32_accurate(n, m, k):
    """tcgen05 kind::tf32 mainloop with the 3xTF32 split: descriptor /
    swizzle / TMEM plumbing check against an fp64 product."""
    from paper_2109_07893_b200.ops import tc_gemm
    rng = np.random.default_rng(n + m + k)
    a = rng.standard_normal((m, k)).astype(np.float32)
    w = rng.standard_normal((n, k)).astype(np.float32)
    got = tc_gemm(a, w)
    ref = a.astype(np.float64) @ w.astype(np.float64).T
    err = np.abs(got - ref) / (np.abs(a).astype(np.float64) @ np.abs(w).astype(np.float64).T)
    assert err.max() < 2e-6, err.max()


@pytest.mark.parametrize("H", [16, 32, 64, 128])
def test_lstm_forward_tensor_cores_vs_oracle(oracle, H):
    rng = np.random.default_rng(10 + H)
    rows, fin = 777, 2 * H + 2

    class Cell:
        wx = rng.uniform(-0.3, 0.3, (fin, 4 * H))
        wh = rng.uniform(-0.3, 0.3, (H, 4 * H))
        b = rng.uniform(-0.1, 0.1, 4 * H)

    ts = [0, 1, 2]
    xs = {t: np.maximum(rng.standard_normal((rows, fin)), 0) for t in ts}
    st = (rng.standard_normal((rows, H)) * 0.2, rng.standard_normal((rows, H)) * 0.2)
    ys, (h, c), _ = pk.lstm_block_forward(Cell, st, ts, xs, tensor_cores=True)
    ys2, _, _ = pk.lstm_block_forward(Cell, st, ts, xs, tensor_cores=False)
    rys, (rh, rc), _ = oracle.lstm_fwd(Cell.wx, Cell.wh, Cell.b, st, ts, xs)
    for t in ts:
        assert np.abs(ys[t] - rys[t]).max() < 2e-5
        assert np.abs(ys[t] - ys2[t]).max() < 2e-5
    assert np.abs(c - rc).max() < 2e-5


def test_transpose_with_hub_columns_bit_exact(oracle):
    """Columns with > 32 entries take the block-per-segment sort path."""
    rng = np.random.default_rng(3)
    n = 600
    rows = np.concatenate([rng.permutation(n)[:500], rng.permutation(n)[:100], rng.integers(0, n, 800)])
    cols = np.concatenate([np.full(500, 3), np.full(100, 7), rng.integers(0, n, 800)])
    vals = rng.standard_normal(rows.shape[0])
    a = pk.SparseMatrix.from_entries(n, rows, cols, vals)
    g = rng.standard_normal((n, 3))
    oa = oracle.Coo(n, a.rows, a.cols, a.vals)
    assert np.array_equal(pk.spmm_transpose(a, g), oracle.spmm_t(oa, g))
    from paper_2109_07893_b200.ops import normalize_laplacian_transpose
    lt = normalize_laplacian_transpose(a)
    ref = oracle.laplacian(oa)
    assert lt == pk.SparseMatrix.from_entries(n, ref.cols, ref.rows, ref.vals)


@pytest.mark.parametrize("H", [16, 32, 64])
def test_lstm_backward_tensor_cores_vs_oracle(oracle, H):
    rng = np.random.default_rng(20 + H)
    rows, fin = 555, 2 * H

    class Cell:
        wx = rng.uniform(-0.3, 0.3, (fin, 4 * H))
        wh = rng.uniform(-0.3, 0.3, (H, 4 * H))
        b = rng.uniform(-0.1, 0.1, 4 * H)

    ts = [0, 1, 2]
    xs = {t: np.maximum(rng.standard_normal((rows, fin)), 0) for t in ts}
    st = (rng.standard_normal((rows, H)) * 0.2, rng.standard_normal((rows, H)) * 0.2)
    ys, _, cache = pk.lstm_block_forward(Cell, st, ts, xs, tensor_cores=True)
    rys, _, rcache = oracle.lstm_fwd(Cell.wx, Cell.wh, Cell.b, st, ts, xs)
    dys = {t: rng.standard_normal((rows, H)) for t in ts}
    dst = (rng.standard_normal((rows, H)), rng.standard_normal((rows, H)))
    dxs, dstate, dcell = pk.lstm_block_backward(Cell, ts, cache, dys, dst, tensor_cores=True)
    rdxs, rdstate, (rdwx, rdwh, rdb) = oracle.lstm_bwd(Cell.wx, Cell.wh, ts, rcache, dys, dst)
    for got, ref in ((dstate[0], rdstate[0]), (dstate[1], rdstate[1]), (dcell["wx"], rdwx),
                     (dcell["wh"], rdwh), (dcell["b"], rdb)):
        ok, worst, nbad = guarded_close(got, ref, RTOL, 1e-5)
        assert ok, (worst, nbad)
    for t in ts:
        assert guarded_close(dxs[t], rdxs[t], RTOL, 1e-5)[0]


@pytest.mark.parametrize("variant", ["tc", "ts"])
@pytest.mark.parametrize("hp,kx", [(64, 128), (64, 68), (32, 36), (32, 96)])
def test_lstm_weight_grad_tc_long_reduction(hp, kx, variant):
    """Block weight gradient over 120k (step, vertex) rows: many CTAs, many
    TMEM promotion periods; fp64 reference.  Both kernels: dz from shared
    memory ("tc") and dz from TMEM ("ts")."""
    from paper_2109_07893_b200.ops import lstm_weight_grad_tc
    rng = np.random.default_rng(hp + kx)
    np_rows, steps = 20_000, 6
    rows = np_rows * steps
    x = np.maximum(rng.standard_normal((rows, kx)), 0).astype(np.float32)
    h = np.tanh(rng.standard_normal((rows, hp))).astype(np.float32)
    h0 = np.tanh(rng.standard_normal((np_rows, hp))).astype(np.float32)
    dz = (rng.standard_normal((rows, 4 * hp)) * 1e-3).astype(np.float32)
    gw, gb = lstm_weight_grad_tc(x, h, h0, dz, np_rows, variant)
    hprev = np.concatenate([h0, h[:-np_rows]]).astype(np.float64)
    xcat = np.concatenate([x.astype(np.float64), hprev], axis=1)
    ref = xcat.T @ dz.astype(np.float64)
    scale = np.abs(xcat).T @ np.abs(dz.astype(np.float64))
    assert np.abs(gw - ref).max() / scale.max() < 2e-5
    assert (np.abs(gw - ref) / scale).max() < 5e-5
    assert np.allclose(gb, dz.astype(np.float64).sum(0), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("H", [16, 32, 64])
def test_warp_specialized_lstm_steps_match_tc_bitwise(H):
    """Persistent warp-specialised kernels (several tiles per CTA, both TMEM
    buffers in use) issue the same MMAs in the same order as the one-tile
    kernels: outputs must be bit-identical."""
    rng = np.random.default_rng(30 + H)
    rows, fin = 128 * 148 * 2 + 77, 2 * H

    class Cell:
        wx = rng.uniform(-0.3, 0.3, (fin, 4 * H))
        wh = rng.uniform(-0.3, 0.3, (H, 4 * H))
        b = rng.uniform(-0.1, 0.1, 4 * H)

    ts = [0, 1]
    xs = {t: np.maximum(rng.standard_normal((rows, fin)), 0) for t in ts}
    st = (rng.standard_normal((rows, H)) * 0.2, rng.standard_normal((rows, H)) * 0.2)
    ys_w, (hw, cw), cache_w = pk.lstm_block_forward(Cell, st, ts, xs, warp_specialized=True)
    ys_t, (ht, ct), cache_t = pk.lstm_block_forward(Cell, st, ts, xs, warp_specialized=False)
    for t in ts:
        assert np.array_equal(ys_w[t], ys_t[t])
    assert np.array_equal(cw, ct)
    dys = {t: rng.standard_normal((rows, H)) for t in ts}
    dst = (rng.standard_normal((rows, H)), rng.standard_normal((rows, H)))
    dxw, dsw, dcw = pk.lstm_block_backward(Cell, ts, cache_w, dys, dst, warp_specialized=True)
    dxt, dst_t, dct = pk.lstm_block_backward(Cell, ts, cache_t, dys, dst, warp_specialized=False)
    for t in ts:
        assert np.array_equal(dxw[t], dxt[t])
    assert np.array_equal(dsw[0], dst_t[0]) and np.array_equal(dsw[1], dst_t[1])
    for k in dcw:
        assert np.array_equal(dcw[k], dct[k])


@pytest.mark.gpu
@pytest.mark.parametrize("fp,hp,skip,agg", [(64, 64, True, True), (32, 16, False, True), (16, 64, True, True),
                                            (64, 32, False, True), (64, 64, True, False), (4, 64, True, False),
                                            (4, 32, False, False)])
def test_gcn_forward_tensor_cores(fp, hp, skip, agg):
    """K3 tcgen05 instance (gather warps + 3xTF32 transform) against fp64:
    ragged last tile, empty rows, and a hub row whose tile overflows the
    staged-index capacity (global-index path).  The aggregation s is the
    same fp32 FMA sequence as the SIMT kernel: bitwise equal."""
    from paper_2109_07893_b200.ops import gcn_forward
    rng = np.random.default_rng(fp * 7 + hp + skip)
    n = 5000 + 37
    deg = rng.integers(0, 4, size=n)
    deg[1234] = 3000
    deg[777] = 100                  # a hub row just past kHubRow (64)
    deg[2000:2140] = 60             # a tile of rows just below it
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, size=rows.size).astype(np.int32)
    val = rng.uniform(-1, 1, size=rows.size).astype(np.float32)
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    x = rng.standard_normal((n, fp)).astype(np.float32)
    w = (rng.standard_normal((fp, hp)) * 0.2).astype(np.float32)
    args = (rowptr, cols, val) if agg else (None, None, None)
    s, r = gcn_forward(n, *args, x, w, skip)
    s2, r2 = gcn_forward(n, *args, x, w, skip, tensor_cores=False)
    assert np.array_equal(s, s2)
    if agg:
        ref_s = np.zeros((n, fp))
        np.add.at(ref_s, rows, val.astype(np.float64)[:, None] * x.astype(np.float64)[cols])
    else:
        ref_s = x.astype(np.float64)
    sc = np.abs(ref_s).max()
    assert np.abs(s - ref_s).max() <= 1e-5 * sc
    q = s.astype(np.float64) @ w.astype(np.float64)
    qs = (np.abs(s).astype(np.float64) @ np.abs(w).astype(np.float64)).max()
    got_q = r[:, fp:] if skip else r
    assert np.abs(got_q - np.maximum(q, 0)).max() <= 2e-6 * qs
    if skip:
        assert np.array_equal(r[:, :fp], np.maximum(s, 0))
    assert np.abs((r2[:, fp:] if skip else r2) - got_q).max() <= 2e-6 * qs


@pytest.mark.gpu
@pytest.mark.parametrize("fp,hp,skip,slabs,n", [(64, 64, True, 0, 70001), (4, 64, True, 0, 20011),
                                                (32, 16, False, 0, 9000), (64, 64, True, 2, 30002),
                                                (16, 32, True, 4, 5003), (64, 128, False, 0, 3000)])
def test_gcn_backward_tensor_cores(fp, hp, skip, slabs, n):
    """K4 rows (tcgen05 BWD instance of K3) and the tcgen05 GCN weight
    gradient against fp64: masked dq, skip term, ragged tails, split
    owner-layout frames, long reductions (period promotion), and the SIMT
    kernels on the same inputs."""
    from paper_2109_07893_b200.ops import gcn_backward
    rng = np.random.default_rng(fp + 3 * hp + n)
    rw = fp + hp if skip else hp
    dr = rng.standard_normal((n, rw)).astype(np.float32)
    r = np.maximum(rng.standard_normal((n, rw)), 0).astype(np.float32)
    s = rng.standard_normal((n, fp)).astype(np.float32)
    w = (rng.standard_normal((fp, hp)) * 0.2).astype(np.float32)
    rows_ds = fp >= 16
    ds, gw = gcn_backward(dr, r, s, w, skip, slabs=slabs, rows_ds=rows_ds)
    ds2, gw2 = gcn_backward(dr, r, s, w, skip, tensor_cores=False, rows_ds=rows_ds)
    dpre = dr.astype(np.float64) * (r > 0)
    dq = dpre[:, fp:] if skip else dpre
    ref_gw = s.astype(np.float64).T @ dq
    scale = np.abs(s).astype(np.float64).T @ np.abs(dq)
    assert np.all(np.abs(gw - ref_gw) <= 2e-6 * scale + 1e-9), np.abs(gw - ref_gw).max()
    assert np.all(np.abs(gw2 - ref_gw) <= 2e-6 * scale + 1e-9)
    if rows_ds:
        ref_ds = dq @ w.astype(np.float64).T + (dpre[:, :fp] if skip else 0.0)
        sc = (np.abs(dq) @ np.abs(w.astype(np.float64)).T).max() + 1.0
        assert np.abs(ds - ref_ds).max() <= 2e-6 * sc
        assert np.abs(ds2 - ref_ds).max() <= 2e-6 * sc
    # deterministic: the same inputs give bitwise the same results
    ds3, gw3 = gcn_backward(dr, r, s, w, skip, slabs=slabs, rows_ds=rows_ds)
    assert np.array_equal(gw, gw3)
    if rows_ds:
        assert np.array_equal(ds, ds3)


@pytest.mark.gpu
@pytest.mark.parametrize("f", [16, 32, 64])
def test_spmm_f32_large(f):
    """dgnn_spmm_f32 (K4 aggregation) at several rows per warp: run-to-run
    bitwise reproducible and within fp32 rounding of the fp64 sum; empty
    rows, a hub row, ragged tail."""
    from paper_2109_07893_b200.ops import spmm_f32
    rng = np.random.default_rng(f)
    n = 148 * 128 * 5 + 13          # several tiles per persistent CTA
    deg = rng.integers(0, 5, size=n)
    deg[4321] = 2500
    deg[999] = 65
    deg[3000:3200] = 64
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, size=rows.size).astype(np.int32)
    val = rng.uniform(-1, 1, size=rows.size).astype(np.float32)
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    x = rng.standard_normal((n, f)).astype(np.float32)
    a = spmm_f32(rowptr, cols, val, x)
    b = spmm_f32(rowptr, cols, val, x, tensor_cores=False)
    assert np.array_equal(a, b)
    ref = np.zeros((n, f))
    np.add.at(ref, rows, val.astype(np.float64)[:, None] * x.astype(np.float64)[cols])
    assert np.abs(a - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.gpu
def test_laplacian_and_transpose_heavy_tailed_bit_exact(oracle):
    """Hub rows (> 16 entries: CTA-per-row count / write / scatter, with and
    without a stored diagonal, entries on both sides of it, one chunk or
    many, the last row among them, zero products
    elided) and hub columns (past 1024 entries: chunk rank sorts merged by
    binary-search ranks, 5 and 17 chunks) against the oracle, bit-exact."""
    rng = np.random.default_rng(11)
    n = 20000
    parts_r, parts_c = [rng.integers(0, n, 30000)], [rng.integers(0, n, 30000)]
    for h in (5, 77, 12345):                       # hub rows
        parts_r.append(np.full(3000, h))
        parts_c.append(rng.permutation(n)[:3000])
    for h, d in ((n - 1, 300), (600, 40)):         # a ragged second chunk; a single chunk
        parts_r.append(np.full(d, h))
        parts_c.append(rng.permutation(n)[:d])
    parts_r.append(np.array([77]))                  # row 77 stores its diagonal
    parts_c.append(np.array([77]))
    parts_r.append(rng.permutation(n)[:17000])      # a 17-chunk column
    parts_c.append(np.full(17000, 9))
    parts_r.append(rng.permutation(n)[:5000])       # a 5-chunk column
    parts_c.append(np.full(5000, 4242))
    rows, cols = np.concatenate(parts_r), np.concatenate(parts_c)
    vals = rng.standard_normal(rows.shape[0])
    vals[rng.random(rows.shape[0]) < 0.01] = 0.0    # explicit zeros vanish
    a = pk.SparseMatrix.from_entries(n, rows, cols, vals)
    oa = oracle.Coo(n, a.rows, a.cols, a.vals)
    ref = oracle.laplacian(oa)
    got = pk.normalize_laplacian(a)
    assert np.array_equal(got.rows, ref.rows) and np.array_equal(got.cols, ref.cols)
    assert np.array_equal(got.vals, ref.vals)
    from paper_2109_07893_b200.ops import normalize_laplacian_transpose
    lt = normalize_laplacian_transpose(a)
    assert lt == pk.SparseMatrix.from_entries(n, ref.cols, ref.rows, ref.vals)
    g = rng.standard_normal((n, 3))
    assert np.array_equal(pk.spmm_transpose(a, g), oracle.spmm_t(oa, g))


@pytest.mark.gpu
def test_apply_hub_rows_round_trip_and_corruption():
    """Rows longer than 16 entries go through the CTA-per-row merge: round
    trips through diff / apply on hub rows, and the corrupt-delta checks
    (delete absent, insert present) still fire on them."""
    rng = np.random.default_rng(5)
    n = 3000

    def hubby():
        r = np.concatenate([rng.integers(0, n, 4000), np.full(900, 17), np.full(300, 2999)])
        c = np.concatenate([rng.integers(0, n, 4000), rng.permutation(n)[:900], rng.permutation(n)[:300]])
        return pk.SparseMatrix.from_entries(n, r, c, rng.choice([1.0, 0.5, -2.0], r.shape[0]))

    for _ in range(3):
        a, b = hubby(), hubby()
        assert pk.apply(a, pk.diff(a, b)) == b
    a = hubby()
    hub_cols = a.cols[a.rows == 17]
    absent = np.setdiff1d(np.arange(n), hub_cols)[:1]
    bad = pk.SnapshotDelta(n, np.array([[17, absent[0]]]), np.zeros((0, 2), np.int64), a.vals)
    with pytest.raises(pk.CorruptDeltaError):
        pk.apply(a, bad)
    bad = pk.SnapshotDelta(n, np.zeros((0, 2), np.int64), np.array([[17, hub_cols[5]]]),
                           np.concatenate([a.vals, [1.0]]))
    with pytest.raises(pk.CorruptDeltaError):
        pk.apply(a, bad)


@pytest.mark.gpu
def test_materializer_chunk_heads_rebuilt_from_deltas():
    """SURVEY §7 hard part 3, fixes 2/3: a chunk whose head follows the
    materialiser's own last snapshot, or a neighbour's (read in place on a
    shared graph stream), is rebuilt from the 1-step delta -- bit-exact, and
    only t = 0 crosses PCIe in full."""
    from paper_2109_07893_b200.materialize import Materializer, SnapshotEncoding
    from paper_2109_07893_b200.synth import churn_keys
    n, T = 30_000, 8
    keys = churn_keys(n, T, 60_000, 0.1, seed=21)
    g = pk.DynamicGraph(n, [pk.SparseMatrix.from_canonical(n, k // n, k % n) for k in keys])
    enc = SnapshotEncoding(g)

    def check(slots, ts):
        for s, t in zip(slots, ts):
            rp = s.rowptr.cpu().numpy().astype(np.int64)
            m = int(rp[-1])
            got = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp)) * n + s.col[:m].cpu().numpy()
            assert np.array_equal(got, np.union1d(keys[t], np.arange(n, dtype=np.int64) * (n + 1))), t

    # own chain: consecutive chunks, one materialiser
    mat = Materializer(enc, "cuda", slots=2, sets=2)
    for i, ts in enumerate(([0, 1], [2, 3], [4, 5], [6, 7])):
        slots = mat.materialize(ts, set_idx=i % 2)
        mat.wait()
        check(slots, ts)
    assert mat.bytes_h2d == 4 * (int(enc.full_off[1]) + int(enc.delta_off[T] - enc.delta_off[1]))
    assert [b[2] for b in mat.builds] == [False, True, True, True]
    # neighbour chain: two materialisers on one graph stream (emulated ranks)
    gs = torch.cuda.Stream()
    a = Materializer(enc, "cuda", slots=2, graph_stream=gs)
    b = Materializer(enc, "cuda", slots=2, graph_stream=gs)
    sa = a.materialize([0, 1])
    sb = b.materialize([2, 3], head_prev=a.raw())
    b.wait()
    check(sa, [0, 1])
    check(sb, [2, 3])
    assert b.builds[0][2] and b.bytes_h2d == 4 * int(enc.delta_off[4] - enc.delta_off[2])
    # not following anything: the head travels in full
    c = Materializer(enc, "cuda", slots=2)
    sc = c.materialize([5, 6])
    c.wait()
    check(sc, [5, 6])
    assert not c.builds[0][2]
    for m in (mat, a, b, c):
        m.check()


@pytest.mark.gpu
def test_device_smoothing_bit_exact(oracle):
    """§8f.1: tm-gcn's M-smoothed snapshots rebuilt on the device from the raw
    graph differences (weighted merge of A_{t-1}, A_t, then transpose and
    Laplacian) equal the oracle's m_transform_snaps + laplacian bit for bit:
    heads after the own last snapshot, after nothing (A_{t0-1} shipped in
    full) and after a neighbour's snapshot; heavy-tailed (hub) rows."""
    from paper_2109_07893_b200.graph import SmoothedGraph
    from paper_2109_07893_b200.materialize import Materializer
    from paper_2109_07893_b200.synth import aml_graph
    n, T = 20_000, 8
    g = aml_graph(n, T, 60_000, 0.05, seed=8)
    m = pk.build_m_matrix(T, 2)
    enc = SmoothedGraph(g, m).encoding
    coos = [oracle.Coo(n, np.asarray(s.rows), np.asarray(s.cols), np.asarray(s.vals)) for s in g.snapshots]
    sm = oracle.m_transform_snaps(coos, m.matrix, 2)

    def check(slots, ts):
        for s, t in zip(slots, ts):
            ref = oracle.laplacian(sm[t])
            rp = s.rowptr.cpu().numpy()
            mm = int(rp[-1])
            assert mm == ref.nnz, t
            assert np.array_equal(np.repeat(np.arange(n), np.diff(rp)), ref.rows)
            assert np.array_equal(s.col[:mm].cpu().numpy(), ref.cols)
            assert np.array_equal(s.val64[:mm].cpu().numpy(), ref.vals), t
            order = np.lexsort((ref.rows, ref.cols))
            assert np.array_equal(s.t_col[:mm].cpu().numpy(), ref.rows[order])
            assert np.array_equal(s.t_val64[:mm].cpu().numpy(), ref.vals[order])

    mat = Materializer(enc, "cuda", slots=3, with_f64=True, sets=2)
    for i, ts in enumerate(([0, 1, 2], [3, 4, 5], [6, 7])):      # own-chain heads
        check(mat.materialize(ts, set_idx=i % 2), ts)
    other = Materializer(enc, "cuda", slots=3, with_f64=True)
    check(other.materialize([4, 5, 6]), [4, 5, 6])                # head after nothing: A_3 in full
    gs = torch.cuda.Stream()
    a = Materializer(enc, "cuda", slots=3, with_f64=True, graph_stream=gs)
    b = Materializer(enc, "cuda", slots=3, with_f64=True, graph_stream=gs)
    sa = a.materialize([1, 2, 3])
    sb = b.materialize([4, 5, 6], head_prev=a.raw())               # neighbour's A_3
    b.wait()
    check(sb, [4, 5, 6])
    check(sa, [1, 2, 3])
    assert [x[2] for x in mat.builds] == [False, True, True] and other.builds[0][2]
    for x in (mat, other, a, b):
        x.check()


@pytest.mark.gpu
@pytest.mark.parametrize("hp,kx", [(64, 128), (64, 68), (32, 64), (32, 36)])
@pytest.mark.parametrize("rows", [1, 200, 256 * 74 * 2 + 77, 300_001])
def test_pair_lstm_forward_matches_single_cta_bitwise(hp, kx, rows):
    """K5 on CTA pairs (cta_group::2, M = 256, each CTA half of the weight
    chunk) against the one-CTA warp-specialised kernel: h, c and the gate
    cache bitwise equal, with and without the cache, ragged pair tiles
    (a lone 128-row half, rows < 128) and more pair tiles than pairs."""
    from paper_2109_07893_b200 import _lib
    from paper_2109_07893_b200._lib import call, ptr, query
    g = torch.Generator(device="cuda").manual_seed(rows + hp + kx)
    dev = torch.device("cuda")
    K, N4 = kx + hp, 4 * hp
    x = torch.randn(rows, kx, device=dev, generator=g)
    h = torch.randn(rows, hp, device=dev, generator=g) * 0.5
    c = torch.randn(rows, hp, device=dev, generator=g) * 0.5
    wt = (torch.randn(N4, K, device=dev, generator=g) * 0.1).contiguous()
    img = torch.zeros(query("dgnn_tc_weight_image_bytes", N4, K) // 4, device=dev)
    st = _lib.stream_handle()
    call("dgnn_tc_weight_image", N4, K, ptr(wt), K, ptr(img), st)
    b = torch.randn(N4, device=dev, generator=g) * 0.1
    outs = {}
    for fn in ("dgnn_lstm_forward_step_ws", "dgnn_lstm_forward_step_pair"):
        for keep in (False, True):
            ho, co = torch.full((rows, hp), 7.0, device=dev), torch.full((rows, hp), 7.0, device=dev)
            gg = torch.full((rows, N4), 7.0, device=dev)
            call(fn, rows, kx, hp, ptr(x), kx, ptr(h), ptr(c), ptr(img), ptr(b), ptr(ho), ptr(co),
                 ptr(gg) if keep else None, st)
            torch.cuda.synchronize()
            outs[fn, keep] = (ho, co, gg if keep else None)
    for keep in (False, True):
        a, p = outs["dgnn_lstm_forward_step_ws", keep], outs["dgnn_lstm_forward_step_pair", keep]
        assert torch.equal(a[0], p[0]) and torch.equal(a[1], p[1])
        if keep:
            assert torch.equal(a[2], p[2])


@pytest.mark.parametrize("ep,classes,slabs", [(64, 2, 1), (32, 2, 4), (16, 3, 1)])
def test_head_scatter_active_matches_full_pass(ep, classes, slabs):
    """dz seeds over the active-vertex list (zero-fill pass + gathers of the
    vertices with incident pairs) equal the all-vertex pass bit for bit,
    hub vertices and owner-layout (slabbed) frames included, and both match
    the per-vertex sums computed in numpy."""
    from paper_2109_07893_b200 import _lib
    from paper_2109_07893_b200._lib import call, ptr
    from paper_2109_07893_b200.labels import frame_labels_device
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(ep + classes)
    n, npairs = 50_000, 20_000
    pairs = rng.integers(0, n, (npairs, 2))
    pairs[:3000, 0] = 7                         # hubs (summed by a whole warp)
    pairs[3000:3200, 1] = 11
    pairs[3200:3265, 0] = 13                    # just above the warp threshold
    lab = rng.integers(0, classes, npairs)
    d = frame_labels_device(pairs, lab, n, classes, dev)
    assert d["nact"] == len(np.unique(pairs))
    dl = torch.from_numpy(rng.standard_normal((npairs, classes))).to(dev)
    hw = torch.from_numpy(rng.standard_normal((2 * ep, classes)).astype(np.float32)).to(dev)
    rps = n // slabs
    outs = []
    for active in (False, True):
        buf = torch.full((slabs * rps * ep + 4 * ep,), float("nan"), device=dev)
        fr = _lib.Frame(buf.data_ptr(), ep, rps if slabs > 1 else 0, rps * ep if slabs > 1 else 0)
        if active:
            call("dgnn_head_scatter_active", n, ptr(d["ptr"]), ptr(d["slot"]), d["nact"], ptr(d["act"]), ptr(dl),
                 ptr(hw), ep, classes, fr, _lib.stream_handle())
        else:
            call("dgnn_head_scatter", n, ptr(d["ptr"]), ptr(d["slot"]), ptr(dl), ptr(hw), ep, classes, fr,
                 _lib.stream_handle())
        outs.append(buf[:n * ep].cpu().numpy())
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    # against the per-vertex sums in numpy (fp64): dz[x] = S_u[x] W_u^T + S_v[x] W_v^T
    dln, hwn = dl.cpu().numpy(), hw.cpu().numpy().astype(np.float64)
    su, sv = np.zeros((n, classes)), np.zeros((n, classes))
    np.add.at(su, pairs[:, 0], dln)
    np.add.at(sv, pairs[:, 1], dln)
    ref = su @ hwn[:ep].T + sv @ hwn[ep:].T
    got = outs[1].reshape(n, ep).astype(np.float64)
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref) + 1e-9 * np.abs(ref).max())


@pytest.mark.parametrize("n", [0, 1, 7, 8191, 8192 * 8 + 3, 1_000_003])
def test_sum_f64_deterministic(n):
    """dgnn_sum_f64 (one 8-CTA cluster, fixed order): within fp64 rounding of
    an exact (math.fsum) sum, accumulate adds onto *out, and repeated calls
    agree bit for bit."""
    import math
    from paper_2109_07893_b200 import _lib
    from paper_2109_07893_b200._lib import call, ptr
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) * np.exp(rng.uniform(-5, 5, n))
    xd = torch.from_numpy(x).to(dev)
    out = torch.zeros(3, dtype=torch.float64, device=dev)
    out[2] = 0.25
    st = _lib.stream_handle()
    call("dgnn_sum_f64", n, ptr(xd), out.data_ptr(), 0, st)
    call("dgnn_sum_f64", n, ptr(xd), out.data_ptr() + 8, 0, st)
    call("dgnn_sum_f64", n, ptr(xd), out.data_ptr() + 16, 1, st)
    got = out.cpu().numpy()
    exact = math.fsum(x)
    assert got[0] == got[1]
    assert abs(got[0] - exact) <= 1e-15 * max(1.0, float(np.abs(x).sum()))
    assert got[2] == 0.25 + got[0]

"""CPU tests: C-ABI library exports, host-side logic of the boundary (no
kernel launches)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2109_07893_b200 as pk
from paper_2109_07893_b200 import _lib
from paper_2109_07893_b200.params import ParamLayout, padded_layers

from conftest import ROOT, load, params_from
from helpers import product_graph


def header_symbols():
    text = (ROOT / "include" / "dgnn_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|void|size_t|long long|const char\*)\s+(dgnn_\w+)\(", text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.lib()
    declared = header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.dgnn_abi_version() == 1


def test_binding_covers_the_header():
    assert set(_lib.exported_symbols()) == set(header_symbols())


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_init_params_matches_reference_fixture():
    for name, seed in (("cdgcn_small", 3), ("tmgcn_small", 2)):
        fx = load(name)
        arch = "cd-gcn" if name.startswith("cd") else "tm-gcn"
        cfg = pk.ModelConfig(arch, hidden_features=8, embed_features=8)
        got = pk.init_params(cfg, seed)
        ref = params_from(fx, "init_")
        assert sorted(got) == sorted(ref)
        for k in ref:
            assert np.array_equal(got[k], ref[k])


def test_param_layout_round_trip_and_disjoint_positions():
    for arch, h in (("cd-gcn", 8), ("cd-gcn", 64), ("tm-gcn", 6)):
        cfg = pk.ModelConfig(arch, hidden_features=h, embed_features=h)
        lay = ParamLayout(cfg)
        p = pk.init_params(cfg, 1)
        flat = lay.flatten(p)
        back = lay.unflatten(flat)
        for k in p:
            assert np.array_equal(back[k], p[k])
        assert np.unique(lay.pos0).shape[0] == lay.count
        assert lay.pos0.max() < lay.size
        sec = lay.pos1[lay.pos1 >= 0]
        assert np.intersect1d(sec, lay.pos0).size == 0


def test_padding_rules():
    cfg = pk.ModelConfig("cd-gcn", hidden_features=64, embed_features=64)
    l0, l1 = padded_layers(cfg)
    assert (l0.fp, l0.hg, l0.ho, l0.rw) == (4, 64, 64, 68)
    assert (l1.fp, l1.hg, l1.ho, l1.rw) == (64, 64, 64, 128)
    with pytest.raises(pk.ConfigError):
        padded_layers(pk.ModelConfig("cd-gcn", hidden_features=200, embed_features=200))


def test_encoding_matches_reference_deltas_and_ledger():
    from paper_2109_07893_b200.materialize import SnapshotEncoding
    fx = load("codec")
    g = product_graph(fx)
    enc = SnapshotEncoding(g, pin=False)
    for t in range(1, g.num_timesteps):
        o = int(enc.delta_off[t])
        nd, ni = int(enc.n_del[t]), int(enc.n_ins[t])
        d = enc.delta[o:o + 2 * (nd + ni)].numpy()
        assert np.array_equal(np.stack([d[:nd], d[nd:2 * nd]], 1), fx[f"ext_prev{t}"])
        assert np.array_equal(np.stack([d[2 * nd:2 * nd + ni], d[2 * nd + ni:]], 1), fx[f"ext_next{t}"])
    led = pk.TransferLedger()
    enc.charge(led, list(range(g.num_timesteps)))
    import json
    assert led.as_dict() == json.loads(str(fx["stream_ledger"]))
    # weighted graph: value-carrying mode, Laplacian structure counts exact
    gw = product_graph(fx, "gw_")
    encw = SnapshotEncoding(gw, pin=False)
    assert not encw.unit
    for t in range(gw.num_timesteps):
        assert encw.nnz_hat[t] == fx[f"lapw{t}_vals"].shape[0]


def test_delta_bytes_ratio_formula():
    """Like-for-like per-pass ratio L / (1 + (L-1) 2 churn)."""
    from paper_2109_07893_b200.materialize import SnapshotEncoding
    from paper_2109_07893_b200.synth import churn_graph
    g = churn_graph(2000, 8, 4000, 0.10, seed=3)
    enc = SnapshotEncoding(g, pin=False)
    ts = list(range(8))
    ratio = enc.full_bytes(ts) / enc.chunk_bytes(ts)
    assert ratio == pytest.approx(8 / (1 + 7 * 0.2), rel=1e-9)


def test_plan_and_partition_errors():
    from paper_2109_07893_b200.engine import Plan
    p = Plan(12, 3, 2, 9)
    assert p.steps_of(1, 1) == [8, 9]
    assert [p.owner_of(t) for t in range(6)] == [0, 0, 1, 1, 2, 2]
    with pytest.raises(pk.ConfigError):
        Plan(6, 4, 1, 8)
    with pytest.raises(pk.ConfigError):
        Plan(8, 2, 3, 8)
    with pytest.raises(pk.ConfigError):
        Plan(8, 4, 1, 6)
    sp = pk.plan_snapshot_partition(12, 3, 2)
    assert sp.steps_of(2, 1) == [10, 11]


def test_label_incidence_order():
    from paper_2109_07893_b200.labels import frame_labels
    pairs = np.array([[1, 2], [2, 1], [1, 1], [0, 2]])
    fl = frame_labels(pairs, np.array([1, 0, 1, 0]), 3, 2)
    # vertex 1: side-0 slots of pairs 0, 2 then side-1 slots of pairs 1, 2
    s = fl.inc_slot[fl.inc_ptr[1]:fl.inc_ptr[2]].tolist()
    assert s == [0, 4, 3, 5]


def test_engines_refuse_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    fx = load("cdgcn_small")
    g = product_graph(fx)
    cfg = pk.ModelConfig("cd-gcn", hidden_features=8, embed_features=8)
    data = pk.prepare_training_data(cfg, g)
    with pytest.raises(pk.ConfigError):
        pk.backward_checkpoint(cfg, data, pk.LabelSet(2, {}), pk.init_params(cfg, 0), 1)


def test_synthetic_generator_exact_churn():
    from paper_2109_07893_b200.synth import churn_keys
    ks = churn_keys(500, 5, 1000, 0.1, seed=2)
    for a, b in zip(ks, ks[1:]):
        assert a.shape[0] == b.shape[0] == 1000
        assert np.setdiff1d(a, b).shape[0] == 100
    assert all(np.all(k[1:] > k[:-1]) for k in ks)
    ks2 = churn_keys(500, 5, 1000, 0.1, seed=2)
    assert all(np.array_equal(a, b) for a, b in zip(ks, ks2))


@pytest.mark.parametrize("name", ["cdgcn_small"])
def test_vectorised_sampler_equals_reference_pairs(name):
    """§8f.2: the vectorised sampler returns the reference's pairs (golden
    fixtures made by the reference's own sampler)."""
    from helpers import product_graph
    from conftest import labels_from
    fx = load(name)
    g = product_graph(fx)
    seed = 5 if name.startswith("cd") else 7
    train, test = pk.sample_link_prediction_sets(g, 0.5, seed)
    if name.startswith("cd"):
        for got, ref in ((train.by_time, labels_from(fx, "train_")), (test.by_time, labels_from(fx, "test_"))):
            assert sorted(got) == sorted(ref)
            for t in ref:
                assert np.array_equal(got[t][0], ref[t][0]) and np.array_equal(got[t][1], ref[t][1])


@pytest.mark.parametrize("n,m,theta", [(12, 60, 0.9), (40, 300, 0.5), (2000, 20000, 0.1), (300, 80000, 1.0)])
def test_vectorised_sampler_equals_key_loop(n, m, theta):
    """Dense graphs (heavy rejection, duplicate draws within and across
    batches) and sparse ones: identical pairs to the literal key loop."""
    from paper_2109_07893_b200.labels import sample_link_prediction_sets_loop
    from paper_2109_07893_b200.synth import churn_graph
    g = churn_graph(n, 4, min(m, n * n - 1), 0.1, seed=n)
    a_tr, a_te = pk.sample_link_prediction_sets(g, theta, 17)
    b_tr, b_te = sample_link_prediction_sets_loop(g, theta, 17)
    for a, b in ((a_tr.by_time, b_tr.by_time), (a_te.by_time, b_te.by_time)):
        assert sorted(a) == sorted(b)
        for t in a:
            assert np.array_equal(a[t][0], b[t][0]) and np.array_equal(a[t][1], b[t][1])


def test_device_generator_encoding_equals_host_encoding():
    """The device-built encoding (configs[3]/[4] generator) equals the host
    encoding of the same snapshots; exact churn; pair-sampler invariants."""
    import torch
    from paper_2109_07893_b200.materialize import SnapshotEncoding
    from paper_2109_07893_b200.synth import device_churn_graph
    n, T, m = 5000, 6, 20000
    g = device_churn_graph(n, T, m, 0.1, 3, "cpu", pin=False)
    keys = [k.numpy() for k in g._keys]
    host = pk.DynamicGraph(n, [pk.SparseMatrix.from_canonical(n, k // n, k % n) for k in keys])
    ref = SnapshotEncoding(host, pin=False)
    for a in ("nnz", "n_del", "n_ins", "nnz_hat", "dhat", "full_off", "delta_off"):
        assert np.array_equal(getattr(g.encoding, a), getattr(ref, a)), a
    assert torch.equal(g.encoding.full, ref.full) and torch.equal(g.encoding.delta, ref.delta)
    for t in range(1, T):
        assert np.intersect1d(keys[t - 1], keys[t]).shape[0] == m - 2000
    train, test = g.sample_pairs(0.1, 5)
    assert sorted(train.by_time) == list(range(T - 1)) and list(test.by_time) == [T - 2]
    for t, (p, lab) in train.by_time.items():
        k = p[:, 0] * n + p[:, 1]
        assert p.shape[0] == 2 * 2000 and np.unique(k).shape[0] == k.shape[0]
        assert np.all(np.isin(k[lab == 1], keys[t])) and not np.any(np.isin(k[lab == 0], keys[t]))


def test_smoothed_encoding_counts_equal_host_smoothing():
    """§8f.1: the raw-graph encoding with device smoothing charges exactly the
    reference ledger counts of the smoothed Laplacians (`delta.py:75-84` over
    `m_transform_graph` snapshots), AMLSim-style graph with hubs."""
    from paper_2109_07893_b200.graph import SmoothedGraph
    from paper_2109_07893_b200.materialize import SnapshotEncoding
    from paper_2109_07893_b200.synth import aml_graph
    g = aml_graph(3000, 7, 9000, 0.05, seed=4)
    m = pk.build_m_matrix(7, 2)
    sg = SmoothedGraph(g, m)
    assert sg.device_smoothing
    dev = sg.encoding
    host = SnapshotEncoding(pk.DynamicGraph(g.num_vertices, pk.m_transform_graph(g, m).snapshots), pin=False)
    assert np.array_equal(dev.nnz_hat, host.nnz_hat)
    assert np.array_equal(dev.dhat, host.dhat)
    assert np.array_equal(dev.nnz_sm, host.nnz)
    assert dev.unit and not host.unit


def test_delta_stream_wire_format():
    """§8f.3: the reference's record layout -- golden bytes
    (`test_delta.py:200-215`), round trip, truncation, and a record file
    loaded straight into the engine's encoding."""
    import io
    from pathlib import Path
    from helpers import product_graph
    from paper_2109_07893_b200 import wire
    from paper_2109_07893_b200.materialize import SnapshotEncoding
    a = pk.SparseMatrix.from_entries(2, [0], [1], [1.0])
    b = pk.SparseMatrix.from_entries(2, [1], [1], [2.5])
    buf = io.BytesIO()
    wire.write_delta_stream([a, b], buf)
    assert buf.getvalue() == (Path(__file__).parent / "golden" / "delta_record.bin").read_bytes()
    for prefix in ("g_", "gw_"):
        g = product_graph(load("codec"), prefix)
        buf = io.BytesIO()
        wire.write_delta_stream(g.snapshots, buf)
        raw = buf.getvalue()
        buf.seek(0)
        back = wire.graph_from_delta_stream(g.snapshots[0], buf)
        assert all(x == y for x, y in zip(back.snapshots, g.snapshots))
        enc = wire.encoding_from_delta_stream(g.snapshots[0], io.BytesIO(raw), pin=False)
        ref = SnapshotEncoding(g, pin=False)
        assert enc.unit == ref.unit and torch_equal(enc.delta, ref.delta) and torch_equal(enc.full, ref.full)
        assert np.array_equal(enc.nnz_hat, ref.nnz_hat) and np.array_equal(enc.dhat, ref.dhat)
        with pytest.raises(pk.CorruptDeltaError):
            wire.read_delta_stream(io.BytesIO(raw[:-3]), g.num_vertices)


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))

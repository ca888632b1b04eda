"""Wire formats of the reference around the hot path.

* The delta-stream record layout (`delta.py:181-227`): per snapshot
  transition, little-endian [u32 n_ext_prev][u32 row, u32 col pairs]
  [u32 n_ext_next][pairs][u32 n_values][f64 values].  `write_delta_stream`
  / `read_delta_stream` keep the reference's API and bytes (golden:
  `test_delta.py:200-215`); `encoding_from_delta_stream` loads such a file
  straight into the engine's pinned-host graph encoding (full first
  snapshot + structure deltas, values kept only when not all 1.0), so a
  record file written by the reference feeds the device rebuild directly.
* The run report `dtgnn.report/1` (`cli.py:194-204`): `train_report`
  runs the reference CLI's `train` pipeline (sampling, preprocessing,
  `train_distributed`) through this package and returns the same JSON
  document.
"""

from __future__ import annotations

import struct
import time

import numpy as np

from .errors import CorruptDeltaError, InputError
from .graph import DynamicGraph, SparseMatrix
from .ops import SnapshotDelta, diff

REPORT_SCHEMA = "dtgnn.report/1"
_REPORT_CONFIG_KEYS = ("model", "hidden", "embed", "layers", "window", "edge_life", "epochs", "lr", "theta",
                       "workers", "blocks", "scheduler", "seed")


def write_delta_stream(snapshots, fh) -> None:
    """`delta.py:181-195`: the delta records of a snapshot run (everything
    after the full first snapshot)."""
    snapshots = list(snapshots)
    for prev, nxt in zip(snapshots, snapshots[1:]):
        d = diff(prev, nxt)
        for pairs in (d.ext_prev, d.ext_next):
            fh.write(struct.pack("<I", pairs.shape[0]))
            fh.write(np.ascontiguousarray(pairs, dtype="<u4").tobytes())
        fh.write(struct.pack("<I", d.values_next.shape[0]))
        fh.write(np.ascontiguousarray(d.values_next, dtype="<f8").tobytes())


def read_delta_stream(fh, dim: int) -> list:
    """`delta.py:198-227`: decode the records; truncation raises
    CorruptDeltaError."""
    def _read(size):
        buf = fh.read(size)
        if len(buf) != size:
            raise CorruptDeltaError("truncated delta stream")
        return buf

    out = []
    while True:
        head = fh.read(4)
        if not head:
            break
        if len(head) != 4:
            raise CorruptDeltaError("truncated delta stream")
        n_prev = struct.unpack("<I", head)[0]
        ext_prev = np.frombuffer(_read(8 * n_prev), dtype="<u4").reshape(-1, 2)
        n_next = struct.unpack("<I", _read(4))[0]
        ext_next = np.frombuffer(_read(8 * n_next), dtype="<u4").reshape(-1, 2)
        n_vals = struct.unpack("<I", _read(4))[0]
        vals = np.frombuffer(_read(8 * n_vals), dtype="<f8")
        out.append(SnapshotDelta(dim, ext_prev.astype(np.int64), ext_next.astype(np.int64),
                                 vals.astype(np.float64)))
    return out


def _apply_keys(keys: np.ndarray, d: SnapshotDelta, n: int) -> np.ndarray:
    """Sorted keys of A_next from A_i's sorted keys and a delta, with the
    reference's consistency checks (`delta.py:126-146`)."""
    gone = d.ext_prev[:, 0] * np.int64(n) + d.ext_prev[:, 1]
    new = d.ext_next[:, 0] * np.int64(n) + d.ext_next[:, 1]
    if gone.size:
        pos = np.minimum(np.searchsorted(keys, gone), max(keys.size - 1, 0))
        if keys.size == 0 or not np.all(keys[pos] == gone):
            raise CorruptDeltaError("ext_prev names an entry absent from the previous snapshot")
    keep = np.ones(keys.size, bool)
    if gone.size:
        keep[np.searchsorted(keys, gone)] = False
    common = keys[keep]
    if new.size and common.size:
        pos = np.minimum(np.searchsorted(common, new), common.size - 1)
        if np.any(common[pos] == new):
            raise CorruptDeltaError("ext_next names an entry already in the common structure")
    return np.union1d(common, new)


def graph_from_delta_stream(first: SparseMatrix, fh) -> DynamicGraph:
    """The snapshot run a record file describes, given its full first
    snapshot (the stream carries only the transitions)."""
    n = first.dim
    snaps = [first]
    keys = np.asarray(first.rows, np.int64) * np.int64(n) + np.asarray(first.cols, np.int64)
    for d in read_delta_stream(fh, n):
        keys = _apply_keys(keys, d, n)
        if d.values_next.shape[0] != keys.shape[0]:
            raise CorruptDeltaError("value count does not match the rebuilt structure")
        snaps.append(SparseMatrix.from_canonical(n, keys // n, keys % n, d.values_next))
    return DynamicGraph(n, snaps)


def encoding_from_delta_stream(first: SparseMatrix, fh, pin: bool = True):
    """The engine's pinned-host graph encoding of a record file (first
    snapshot + records): structure deltas for every transition, values only
    if some value is not 1.0 (the device recomputes unit-valued Laplacians
    bit-exactly).  Pass the result to the engine as `encoding=`."""
    from .materialize import SnapshotEncoding
    return SnapshotEncoding(graph_from_delta_stream(first, fh), pin=pin)


# ---------------------------------------------------------------------------
# run report


def train_report(graph, opts: dict) -> tuple:
    """The reference CLI's `train` pipeline on this package (`cli.py:168-210`):
    label sampling with seed + 1000003, preprocessing, `train_distributed`;
    returns (report dict in the dtgnn.report/1 schema, trained params).
    `opts` holds the CLI's config keys (model, hidden, embed, layers,
    window, edge_life, epochs, lr, theta, workers, blocks, scheduler, seed)."""
    from . import __version__
    from .api import plan_snapshot_partition, prepare_training_data, train_distributed
    from .labels import sample_link_prediction_sets
    from .params import ModelConfig
    missing = [k for k in _REPORT_CONFIG_KEYS if k not in opts]
    if missing:
        raise InputError(f"report options missing: {missing}")
    if graph.num_timesteps < 2:
        from .errors import ConfigError
        raise ConfigError("training needs at least two snapshots (final one is held out)")
    cfg = ModelConfig(architecture=opts["model"], in_features=2, hidden_features=int(opts["hidden"]),
                      embed_features=int(opts["embed"]), layers=int(opts["layers"]), window=int(opts["window"]),
                      edge_life=int(opts["edge_life"]))
    plan_snapshot_partition(graph.num_timesteps, int(opts["workers"]), int(opts["blocks"]))
    t0 = time.perf_counter()
    train, test = sample_link_prediction_sets(graph, float(opts["theta"]), int(opts["seed"]) + 1000003)
    data = prepare_training_data(cfg, graph)
    t_prep = time.perf_counter() - t0
    t0 = time.perf_counter()
    trace, params, comm, transfer, act = train_distributed(
        cfg, data, train, test, epochs=int(opts["epochs"]), seed=int(opts["seed"]), workers=int(opts["workers"]),
        nblk=int(opts["blocks"]), scheduler=opts["scheduler"], lr=float(opts["lr"]))
    t_train = time.perf_counter() - t0
    config = {k: opts[k] for k in _REPORT_CONFIG_KEYS}
    config["num_vertices"] = graph.num_vertices
    config["num_timesteps"] = graph.num_timesteps
    report = {"schema": REPORT_SCHEMA, "version": __version__, "command": "train", "config": config,
              "epochs": trace, "comm": comm.as_dict(), "transfer": transfer.as_dict(),
              "activation_peak": act.peak,
              "timing": {"preprocess_seconds": t_prep, "train_seconds": t_train}}
    return report, params

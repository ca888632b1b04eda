"""Drop-in training API (the reference's model/trainer boundary).

Same names, signatures, return values and error types as the reference
engines:

* `distributed_epoch(cfg, data, labels, params, workers, nblk, scheduler,
  comm, transfer, act_ledger)` -> (loss, grads, comm, transfer)   dist.py:505
* `train_distributed(cfg, data, train, test, epochs, seed, workers, nblk,
  scheduler, lr)` -> (trace, params, comm, transfer, act)          dist.py:592
* `backward_checkpoint(cfg, data, labels, params, nblk, reduction,
  act_ledger)` -> (loss, grads)                                    training.py:798
* `backward_full`, `train_epochs`                                  training.py:772, 903

Inputs may be this package's objects or the reference's own (duck typed).
Parameters and gradients cross the boundary as float64 numpy dicts; inside,
everything is device resident (fp32 compute, fp64 master weights / Adam /
gradient accumulation).  With `workers > 1` in a single process the P ranks
are emulated on the current GPU; under `torchrun` with a process group of P
ranks each process drives one GPU and the exchanges are NCCL all-to-alls.
"""

from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import Engine, LocalFabric, NcclFabric, Plan
from .errors import ConfigError, InputError, ProtocolError
from .graph import (DynamicGraph, FeatureSequence, LazyDegreeFeatures, MMatrix, SmoothedGraph, build_m_matrix,
                    degree_features, edge_life_matrix, m_transform_features, m_transform_graph)
from .params import ModelConfig, as_config, init_params, parameter_count

SCHEDULERS = ("round-robin", "threads")


# ---------------------------------------------------------------------------
# ledgers (reference-equivalent counters, dist.py:82-122, delta.py:57-100,
# training.py:292-335) plus measured device quantities


@dataclass
class CommLedger:
    redistribution_units: int = 0
    all_reduce_scalars: int = 0
    messages: int = 0
    events: list = field(default_factory=list)

    def record_alltoall(self, units: int, messages: int, phase: str, block: int, layer: int):
        self.redistribution_units += units
        self.messages += messages
        self.events.append({"kind": "alltoall", "phase": phase, "block": block, "layer": layer,
                            "units": units})

    def record_allreduce(self, scalars: int, workers: int):
        self.all_reduce_scalars += scalars
        if workers > 1:
            self.messages += workers - 1
        self.events.append({"kind": "allreduce", "scalars": scalars})

    def alltoall_events(self, phase=None):
        evs = [e for e in self.events if e["kind"] == "alltoall"]
        return evs if phase is None else [e for e in evs if e["phase"] == phase]

    def as_dict(self) -> dict:
        return {"redistribution_units": self.redistribution_units,
                "all_reduce_scalars": self.all_reduce_scalars,
                "messages": self.messages,
                "alltoall_count": len(self.alltoall_events())}


INDEX_ENTRY_BYTES = 8
VALUE_ENTRY_BYTES = 8


@dataclass
class TransferLedger:
    """Reference counters for the Laplacian stream (`delta.py:57-100`);
    `h2d_bytes` is what this package actually copied over PCIe,
    `full_equiv_bytes` what the reference schedule (every snapshot of every
    pass streamed) would cost with full snapshots in the same encoding, and
    `full_built_bytes` the full-snapshot bytes of the passes that were
    actually streamed and rebuilt (like for like)."""
    index_entries_sent: int = 0
    value_entries_sent: int = 0
    snapshots_full: int = 0
    snapshots_delta: int = 0
    h2d_bytes: int = 0
    full_equiv_bytes: int = 0
    full_built_bytes: int = 0

    def charge_full(self, snapshot) -> None:
        self.index_entries_sent += snapshot.nnz
        self.value_entries_sent += snapshot.nnz
        self.snapshots_full += 1

    def charge_delta(self, delta) -> None:
        self.index_entries_sent += delta.index_entries
        self.value_entries_sent += int(np.asarray(delta.values_next).shape[0])
        self.snapshots_delta += 1

    def merge(self, other: "TransferLedger") -> None:
        for k in ("index_entries_sent", "value_entries_sent", "snapshots_full", "snapshots_delta",
                  "h2d_bytes", "full_equiv_bytes", "full_built_bytes"):
            setattr(self, k, getattr(self, k) + getattr(other, k))

    def delta_fraction(self) -> float:
        tot = self.snapshots_full + self.snapshots_delta
        return self.snapshots_delta / tot if tot else 0.0

    def bytes_sent(self) -> int:
        return self.index_entries_sent * INDEX_ENTRY_BYTES + self.value_entries_sent * VALUE_ENTRY_BYTES

    def as_dict(self) -> dict:
        return {"index_entries_sent": self.index_entries_sent,
                "value_entries_sent": self.value_entries_sent,
                "snapshots_full": self.snapshots_full,
                "snapshots_delta": self.snapshots_delta,
                "delta_fraction": self.delta_fraction(),
                "bytes_sent": self.bytes_sent()}


class ActivationLedger:
    """Logical retained-activation accounting (`training.py:292-335`)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.live_activations = 0.0
        self.live_checkpoints = 0.0
        self.peak = 0.0
        self.peak_activations = 0.0
        self.peak_checkpoints = 0.0

    def _bump(self):
        total = self.live_activations + self.live_checkpoints
        self.peak = max(self.peak, total)
        self.peak_activations = max(self.peak_activations, self.live_activations)
        self.peak_checkpoints = max(self.peak_checkpoints, self.live_checkpoints)

    def alloc_activations(self, amount: float):
        with self._lock:
            self.live_activations += amount
            self._bump()

    def free_activations(self, amount: float):
        with self._lock:
            self.live_activations -= amount

    def alloc_checkpoint(self, amount: float = 1.0):
        with self._lock:
            self.live_checkpoints += amount
            self._bump()

    def free_checkpoint(self, amount: float = 1.0):
        with self._lock:
            self.live_checkpoints -= amount


@dataclass(frozen=True)
class SnapshotPartition:
    """`dist.py:125-162`."""
    num_timesteps: int
    workers: int
    nblk: int

    def __post_init__(self):
        if self.workers < 1:
            raise ConfigError("worker count must be >= 1")
        if self.nblk < 1 or self.num_timesteps % self.nblk != 0:
            raise ConfigError(f"block count {self.nblk} must divide the timeline length {self.num_timesteps}")
        if self.bsize % self.workers != 0:
            raise ConfigError(f"worker count {self.workers} must divide the block size {self.bsize}")

    @property
    def bsize(self) -> int:
        return self.num_timesteps // self.nblk

    @property
    def chunk(self) -> int:
        return self.bsize // self.workers

    def owner_of(self, t: int) -> int:
        return (t % self.bsize) // self.chunk

    def block_steps(self, b: int) -> list:
        return list(range(b * self.bsize, (b + 1) * self.bsize))

    def steps_of(self, p: int, b: int) -> list:
        start = b * self.bsize + p * self.chunk
        return list(range(start, start + self.chunk))


def plan_snapshot_partition(num_timesteps: int, workers: int, nblk: int) -> SnapshotPartition:
    return SnapshotPartition(num_timesteps, workers, nblk)


@dataclass(frozen=True)
class BlockPlan:
    """`training.py:253-277`."""
    num_timesteps: int
    nblk: int

    def __post_init__(self):
        if self.nblk < 1:
            raise ConfigError("block count must be >= 1")
        if self.num_timesteps % self.nblk != 0:
            raise ConfigError(f"block count {self.nblk} must divide the timeline length {self.num_timesteps}")

    @property
    def bsize(self) -> int:
        return self.num_timesteps // self.nblk

    def block_steps(self, b: int) -> list:
        return list(range(b * self.bsize, (b + 1) * self.bsize))

    def blocks(self):
        return [(b, self.block_steps(b)) for b in range(self.nblk)]


# ---------------------------------------------------------------------------
# training data


@dataclass(frozen=True, eq=False)
class TrainingData:
    """`training.py:204-221`.  `laps` and `s1` are produced on device by the
    engine (from `graph`), so they may be None here; a reference
    `TrainingData` (with host Laplacians) is accepted as well."""
    graph: DynamicGraph
    laps: list | None
    feats: FeatureSequence
    s1: list | None
    m_matrix: MMatrix | None = None

    @property
    def num_timesteps(self) -> int:
        return self.graph.num_timesteps

    @property
    def num_vertices(self) -> int:
        return self.graph.num_vertices


def prepare_training_data(cfg, graph) -> TrainingData:
    """Host preprocessing (`training.py:224-250`): tm-gcn smooths the graph
    and the degree features with the M-transform; cd-gcn uses raw snapshots.
    Laplacians and first-layer products are left to the device."""
    cfg = as_config(cfg)
    m = None
    if cfg.architecture == "tm-gcn":
        m = build_m_matrix(graph.num_timesteps, cfg.window)
        # smoothed on the device by the engine (graph.SmoothedGraph); the
        # host smoothing runs only if something reads .snapshots
        smoothed = SmoothedGraph(graph, m)
        feats = m_transform_features(degree_features(graph), m)
    elif cfg.architecture == "cd-gcn":
        smoothed, feats = graph, degree_features(graph)
    else:
        # egcn-o (training.py:238-240): edge life (dtdg.py:194-208) applied on
        # the device like the tm-gcn smoothing; the degree features of the
        # smoothed graph are computed on the device too (host copy on demand)
        smoothed = SmoothedGraph(graph, edge_life_matrix(graph.num_timesteps, cfg.edge_life))
        feats = LazyDegreeFeatures(smoothed)
    if feats.width != cfg.in_features:
        raise ConfigError(f"configured in_features={cfg.in_features} but input frames have width {feats.width}")
    return TrainingData(graph=smoothed, laps=None, feats=feats, s1=None, m_matrix=m)


# ---------------------------------------------------------------------------
# engine cache: one device engine per (data, config, workers, nblk)

_ENGINES: dict = {}
# temporal-stage GEMMs on tcgen05 (default) or on the SIMT fp32 kernels (A/B, strict-parity tests)
TENSOR_CORES = True
_LOCK = threading.Lock()


def _fabric():
    if torch.distributed.is_available() and torch.distributed.is_initialized() \
            and torch.distributed.get_world_size() > 1:
        return NcclFabric()
    return LocalFabric()


def get_engine(cfg, data, workers: int, nblk: int, resident: bool = False) -> Engine:
    cfg = as_config(cfg)
    if not torch.cuda.is_available():
        raise ConfigError("no CUDA device: this package has no CPU execution path")
    graph = data.graph
    key = (id(data), cfg, int(workers), int(nblk), bool(resident), bool(TENSOR_CORES))
    with _LOCK:
        eng = _ENGINES.get(key)
        if eng is None:
            # share the host encoding between engines built on the same data
            enc = next((e.enc for k, e in _ENGINES.items() if k[0] == id(data)), None)
            feats = None
            if cfg.architecture == "tm-gcn":
                feats = [np.asarray(f, np.float64) for f in data.feats.frames]
            m = None if data.m_matrix is None else np.asarray(data.m_matrix.matrix)
            eng = Engine(cfg, graph, workers, nblk, feats_host=feats, m_matrix=m, resident=resident,
                         fabric=_fabric(), encoding=enc, tensor_cores=TENSOR_CORES)
            _ENGINES[key] = eng
            try:
                weakref.finalize(data, _drop, id(data))
            except TypeError:
                pass
    return eng


def _drop(data_id):
    with _LOCK:
        for k in [k for k in _ENGINES if k[0] == data_id]:
            del _ENGINES[k]


def clear_engines():
    import gc
    with _LOCK:
        _ENGINES.clear()
    gc.collect()               # Engine <-> Rank reference cycles hold the device buffers
    torch.cuda.empty_cache()


def _check(cfg, data, workers, nblk, scheduler):
    if scheduler not in SCHEDULERS:
        raise ConfigError(f"unknown scheduler {scheduler!r}; expected one of {SCHEDULERS}")
    Plan(data.num_timesteps if hasattr(data, "num_timesteps") else data.graph.num_timesteps, workers,
         nblk, data.graph.num_vertices)


def _by_time(labels):
    if labels is None:
        return {}
    return labels if isinstance(labels, dict) else labels.by_time


_FINGERPRINTS: dict = {}


def _labels_key(*labelsets):
    """Content fingerprint of label sets (the engine caches device labels
    under it): per frame the pair count, coordinate and label sums and a
    label-weighted coordinate sum.  Unlike an object id it cannot be reused
    by a different label set; it is computed once per live label-set object
    (a weak reference identifies the object, so a new object is always
    fingerprinted; arrays mutated in place are not re-read)."""
    key = []
    for ls in labelsets:
        ent = _FINGERPRINTS.get(id(ls))
        if ent is not None and ent[0]() is ls and ls is not None:
            key.append(ent[1])
            continue
        fp = _fingerprint(ls)
        try:
            _FINGERPRINTS[id(ls)] = (weakref.ref(ls), fp)
        except TypeError:           # dicts / None: not weak-referenceable, fingerprinted each call
            pass
        key.append(fp)
    return tuple(key)


def _fingerprint(ls):
    bt = _by_time(ls)
    ent = []
    for t in sorted(bt):
        p, lab = bt[t]
        p = np.asarray(p, dtype=np.int64).reshape(-1, 2)
        lab = np.asarray(lab, dtype=np.int64)
        ent.append((int(t), p.shape[0], int(p.sum()), int(lab.sum()),
                    int(np.dot(p[:, 0] + 3 * p[:, 1], lab)) if p.shape[0] else 0))
    return tuple(ent)


def _bytes(eng):
    return tuple(sum(getattr(r.mat, k) for r in eng.ranks)
                 for k in ("bytes_h2d", "bytes_full_equiv", "bytes_full_built"))


def _charge_bytes(transfer, eng, before):
    now = _bytes(eng)
    transfer.h2d_bytes += now[0] - before[0]
    transfer.full_equiv_bytes += now[1] - before[1]
    transfer.full_built_bytes += now[2] - before[2]


def _count(labels):
    return sum(np.asarray(p).shape[0] for p, _ in _by_time(labels).values())


# ---------------------------------------------------------------------------
# engines


def distributed_epoch(cfg, data, labels, params: dict, workers: int, nblk: int,
                      scheduler: str = "round-robin", comm: CommLedger | None = None,
                      transfer: TransferLedger | None = None, act_ledger: ActivationLedger | None = None,
                      reduction: str = "mean"):
    """One training epoch under snapshot partitioning (`dist.py:505-589`).
    Returns (loss, grads, comm, transfer)."""
    cfg = as_config(cfg)
    _check(cfg, data, workers, nblk, scheduler)
    comm = comm if comm is not None else CommLedger()
    transfer = transfer if transfer is not None else TransferLedger()
    act = act_ledger if act_ledger is not None else ActivationLedger()
    eng = get_engine(cfg, data, workers, nblk)
    eng.set_labels(_by_time(labels), None, key=_labels_key(labels, None))
    eng.params.load(params)
    before = _bytes(eng)
    loss_dev, grads = eng.epoch(comm, transfer, act, _count(labels), reduction)
    loss = eng.finish(loss_dev, grads)
    _charge_bytes(transfer, eng, before)
    g = eng.layout.unflatten(grads.cpu().numpy())
    if not _count(labels):
        loss = 0.0
    return loss, g, comm, transfer


def backward_checkpoint(cfg, data, labels, params: dict, nblk: int, reduction: str = "mean",
                        act_ledger: ActivationLedger | None = None):
    """`training.py:798-865` -> (loss, grads); one rank, gradient checkpointing
    over nblk time blocks."""
    if reduction not in ("mean", "sum"):
        raise InputError(f"unknown reduction {reduction!r}")
    BlockPlan(data.graph.num_timesteps, nblk)
    loss, grads, _, _ = distributed_epoch(cfg, data, labels, params, 1, nblk, act_ledger=act_ledger,
                                          reduction=reduction)
    return loss, grads


def backward_full(cfg, data, labels, params: dict, reduction: str = "mean"):
    """`training.py:772-795`; identical to the checkpointed path at nblk = 1."""
    return backward_checkpoint(cfg, data, labels, params, 1, reduction)


def train_distributed(cfg, data, train_labels, test_labels, epochs: int, seed: int, workers: int, nblk: int,
                      scheduler: str = "round-robin", lr: float = 0.01):
    """`dist.py:592-614` -> (trace, params, comm, transfer, act_ledger)."""
    cfg = as_config(cfg)
    _check(cfg, data, workers, nblk, scheduler)
    params = init_params(cfg, seed)
    comm, transfer, act = CommLedger(), TransferLedger(), ActivationLedger()
    trace = []
    if epochs <= 0:
        return trace, params, comm, transfer, act
    eng = get_engine(cfg, data, workers, nblk)
    eng.set_labels(_by_time(train_labels), _by_time(test_labels),
                   key=_labels_key(train_labels, test_labels))
    eng.params.load(params)
    eng.params.step = 0
    eng.params.m.zero_()
    eng.params.v.zero_()
    count = _count(train_labels)
    for epoch in range(1, epochs + 1):
        before = _bytes(eng)
        loss_dev, grads = eng.epoch(comm, transfer, act, count, "mean")
        if count:
            loss = eng.finish(loss_dev, grads)
        else:
            loss = 0.0
            eng.check()
        _charge_bytes(transfer, eng, before)
        eng.params.adam(lr)
        acc = eng.evaluate()
        trace.append({"epoch": epoch, "loss": loss, "test_accuracy": acc})
    return trace, eng.params.to_host(), comm, transfer, act


def train_epochs(cfg, data, train_labels, test_labels, epochs: int, seed: int, nblk: int = 1, lr: float = 0.01):
    """`training.py:903-921` -> (trace, params)."""
    trace, params, _, _, _ = train_distributed(cfg, data, train_labels, test_labels, epochs, seed, 1, nblk,
                                               lr=lr)
    return trace, params


def model_forward_frames(cfg, data, params: dict, nblk: int = 1, rows=None, workers: int = 1) -> list:
    """Embedding frames of the straight-line forward (`models.py:275-323`);
    `rows`: only those vertex rows of every frame."""
    eng = get_engine(cfg, data, workers, nblk)
    eng.set_labels({}, None, key=("forward",)) if eng.prepared_labels is None else None
    eng.params.load(params)
    return eng.forward_frames(rows)


# ---------------------------------------------------------------------------
# host optimiser for callers that keep parameters on the host (training.py:872-900)


@dataclass
class AdamState:
    m: dict
    v: dict
    step: int = 0


def init_adam(params: dict) -> AdamState:
    return AdamState(m={k: np.zeros_like(v) for k, v in params.items()},
                     v={k: np.zeros_like(v) for k, v in params.items()})


def adam_step(params: dict, grads: dict, state: AdamState, lr: float = 0.01, beta1: float = 0.9,
              beta2: float = 0.999, eps: float = 1e-8) -> AdamState:
    """Reference Adam on host dicts (sorted key order, in place); the device
    engines use the fp64 kernel `dgnn_adam` with the same arithmetic."""
    state.step += 1
    t = state.step
    for k in sorted(params):
        g = grads[k]
        if g.shape != params[k].shape:
            raise InputError(f"gradient shape mismatch for {k}")
        state.m[k] = beta1 * state.m[k] + (1.0 - beta1) * g
        state.v[k] = beta2 * state.v[k] + (1.0 - beta2) * (g * g)
        m_hat = state.m[k] / (1.0 - beta1 ** t)
        v_hat = state.v[k] / (1.0 - beta2 ** t)
        params[k] -= lr * m_hat / (np.sqrt(v_hat) + eps)
    return state

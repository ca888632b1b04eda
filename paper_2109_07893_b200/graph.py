"""Host-side snapshot data model (the input format of the hot path).

`SparseMatrix` keeps the reference's canonical COO contract
(`core.py:39-129`): entries strictly sorted by (row, col), no duplicates,
no stored zeros, read-only arrays.  It is the format callers hand to the
engine; the engine turns it into device CSR/CSC once (full snapshot) or via
graph-difference deltas (`delta.py`).  Objects of the reference's own
classes are accepted anywhere a `SparseMatrix`/`DynamicGraph` is (duck
typing on `dim/rows/cols/vals` and `num_vertices/snapshots`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InputError


def _ro(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    a.flags.writeable = False
    return a


@dataclass(frozen=True, eq=False)
class SparseMatrix:
    """Square sparse matrix, canonical COO (`core.py:39-52`)."""

    dim: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    @staticmethod
    def from_entries(dim, rows, cols, vals=None) -> "SparseMatrix":
        """Canonicalise arbitrary entries (`core.py:54-87`): duplicates sum in
        input order, exact zeros are dropped."""
        if dim < 0:
            raise InputError(f"dimension must be non-negative, got {dim}")
        r = np.asarray(rows, dtype=np.int64).ravel()
        c = np.asarray(cols, dtype=np.int64).ravel()
        v = np.ones(r.shape[0]) if vals is None else np.asarray(vals, dtype=np.float64).ravel()
        if not (r.shape == c.shape == v.shape):
            raise InputError("rows, cols and vals must have equal lengths")
        if r.size and (r.min() < 0 or r.max() >= dim):
            raise InputError(f"row index out of range for dim {dim}")
        if c.size and (c.min() < 0 or c.max() >= dim):
            raise InputError(f"col index out of range for dim {dim}")
        if not np.all(np.isfinite(v)):
            raise InputError("entry values must be finite")
        keys = r * np.int64(dim) + c
        uk, inv = np.unique(keys, return_inverse=True)
        acc = np.zeros(uk.shape[0])
        np.add.at(acc, inv, v)
        nz = acc != 0.0
        uk = uk[nz]
        return SparseMatrix(int(dim), _ro(uk // dim), _ro(uk % dim), _ro(acc[nz]))

    @staticmethod
    def from_canonical(dim, rows, cols, vals=None) -> "SparseMatrix":
        """Trusted constructor for already-canonical arrays (generator, device
        read-back); `vals=None` means unit values."""
        r = np.asarray(rows, dtype=np.int64)
        v = np.ones(r.shape[0]) if vals is None else np.asarray(vals, dtype=np.float64)
        return SparseMatrix(int(dim), _ro(r), _ro(np.asarray(cols, dtype=np.int64)), _ro(v))

    @staticmethod
    def empty(dim: int) -> "SparseMatrix":
        return SparseMatrix.from_entries(dim, [], [], [])

    @staticmethod
    def identity(dim: int) -> "SparseMatrix":
        i = np.arange(dim, dtype=np.int64)
        return SparseMatrix.from_entries(dim, i, i, np.ones(dim))

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    def index_keys(self) -> np.ndarray:
        return self.rows * np.int64(self.dim) + self.cols

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.dim, self.dim))
        out[self.rows, self.cols] = self.vals
        return out

    def row_counts(self) -> np.ndarray:
        return np.bincount(self.rows, minlength=self.dim).astype(np.int64)

    def col_counts(self) -> np.ndarray:
        return np.bincount(self.cols, minlength=self.dim).astype(np.int64)

    def unit_valued(self) -> bool:
        return bool(np.all(self.vals == 1.0))

    def __eq__(self, other) -> bool:
        if not hasattr(other, "rows"):
            return NotImplemented
        return (self.dim == other.dim and np.array_equal(self.rows, other.rows)
                and np.array_equal(self.cols, other.cols)
                and np.array_equal(self.vals, other.vals))

    def __repr__(self) -> str:
        return f"SparseMatrix(dim={self.dim}, nnz={self.nnz})"


@dataclass(frozen=True)
class DynamicGraph:
    """Sequence of snapshots over a fixed vertex set (`dtdg.py:36-57`)."""

    num_vertices: int
    snapshots: list

    def __post_init__(self):
        if len(self.snapshots) < 1:
            raise InputError("a dynamic graph needs at least one snapshot")
        for i, s in enumerate(self.snapshots):
            if s.dim != self.num_vertices:
                raise InputError(f"snapshot {i} has dim {s.dim}, expected {self.num_vertices}")

    @property
    def num_timesteps(self) -> int:
        return len(self.snapshots)

    def total_nnz(self) -> int:
        return sum(s.nnz for s in self.snapshots)


@dataclass(frozen=True)
class FeatureSequence:
    """Dense N x F frames, one per timestep (`dtdg.py:60-84`)."""

    frames: list

    def __post_init__(self):
        if len(self.frames) < 1:
            raise InputError("a feature sequence needs at least one frame")
        shape = self.frames[0].shape
        for i, f in enumerate(self.frames):
            if f.shape != shape:
                raise InputError(f"frame {i} has shape {f.shape}, expected {shape}")

    @property
    def num_timesteps(self) -> int:
        return len(self.frames)

    @property
    def num_vertices(self) -> int:
        return self.frames[0].shape[0]

    @property
    def width(self) -> int:
        return self.frames[0].shape[1]


@dataclass(frozen=True)
class MMatrix:
    """Banded lower-triangular averaging matrix (`dtdg.py:87-98`)."""

    size: int
    window: int
    matrix: np.ndarray


def build_m_matrix(num_timesteps: int, window: int) -> MMatrix:
    """Row t (1-based) holds 1/min(w, t) on columns max(1, t-w+1)..t
    (`dtdg.py:211-221`)."""
    if num_timesteps < 1:
        raise InputError(f"timestep count must be >= 1, got {num_timesteps}")
    if window < 1:
        raise InputError(f"window must be >= 1, got {window}")
    m = np.zeros((num_timesteps, num_timesteps))
    for t0 in range(num_timesteps):
        lo = max(0, t0 - window + 1)
        m[t0, lo:t0 + 1] = 1.0 / min(window, t0 + 1)
    return MMatrix(num_timesteps, window, m)


def degree_features(g) -> FeatureSequence:
    """Host degree frames (`dtdg.py:255-266`): out-degree, in-degree."""
    frames = []
    for s in g.snapshots:
        f = np.zeros((g.num_vertices, 2))
        f[:, 0] = np.bincount(np.asarray(s.rows), minlength=g.num_vertices)
        f[:, 1] = np.bincount(np.asarray(s.cols), minlength=g.num_vertices)
        frames.append(f)
    return FeatureSequence(frames)


def m_transform_features(x: FeatureSequence, m: MMatrix) -> FeatureSequence:
    """First-mode product of the feature tensor (`dtdg.py:224-236`); host
    preprocessing for tm-gcn."""
    if x.num_timesteps != m.size:
        raise InputError(f"feature sequence has {x.num_timesteps} frames, M expects {m.size}")
    out = []
    for t in range(m.size):
        acc = np.zeros_like(x.frames[0])
        for k in range(max(0, t - m.window + 1), t + 1):
            acc += m.matrix[t, k] * x.frames[k]
        out.append(acc)
    return FeatureSequence(out)


def m_transform_graph(g, m: MMatrix) -> DynamicGraph:
    """First-mode product on the adjacency tensor (`dtdg.py:239-252`); host
    preprocessing for tm-gcn."""
    if g.num_timesteps != m.size:
        raise InputError(f"graph has {g.num_timesteps} snapshots, M expects {m.size}")
    out = []
    for t in range(m.size):
        terms = [(m.matrix[t, k], g.snapshots[k]) for k in range(max(0, t - m.window + 1), t + 1)]
        r = np.concatenate([np.asarray(s.rows) for _, s in terms])
        c = np.concatenate([np.asarray(s.cols) for _, s in terms])
        v = np.concatenate([float(w) * np.asarray(s.vals) for w, s in terms])
        out.append(SparseMatrix.from_entries(g.num_vertices, r, c, v))
    return DynamicGraph(g.num_vertices, out)


class SmoothedGraph:
    """The M-smoothed graph of tm-gcn (`training.py:234-237`: data.graph =
    m_transform_graph(raw, M)), smoothed on the device by the engine.

    The engine streams the *raw* snapshots' graph differences (structure
    only) and rebuilds A~_t = M[t,t-1] A_{t-1} + M[t,t] A_t per step with the
    bit-exact weighted merge (`dgnn_csr_weighted_merge`).  Host code that
    reads `snapshots` gets the reference's host smoothing, computed on first
    access.  Device smoothing applies to unit-valued raw graphs with window
    <= 2; otherwise the engine streams the host-smoothed snapshots with
    values (the reference's own path)."""

    def __init__(self, raw, m: MMatrix):
        if raw.num_timesteps != m.size:
            raise InputError(f"graph has {raw.num_timesteps} snapshots, M expects {m.size}")
        self.raw, self.m = raw, m
        self.num_vertices = raw.num_vertices
        self._host = None
        self._encoding = None

    @property
    def num_timesteps(self) -> int:
        return self.raw.num_timesteps

    @property
    def device_smoothing(self) -> bool:
        return (self.m.window <= 2 and bool(np.all(self.m.matrix >= 0.0))
                and all(bool(np.all(np.asarray(s.vals) == 1.0)) for s in self.raw.snapshots))

    @property
    def snapshots(self) -> list:
        if self._host is None:
            self._host = m_transform_graph(self.raw, self.m).snapshots
        return self._host

    def total_nnz(self) -> int:
        return sum(s.nnz for s in self.snapshots)

    @property
    def encoding(self):
        """The encoding the engine streams: raw graph differences with the
        smoothing plan attached, or (no device smoothing) the smoothed
        snapshots with values."""
        if self._encoding is None:
            from .materialize import SnapshotEncoding
            if self.device_smoothing:
                self._encoding = SnapshotEncoding(self.raw, smooth=(self.m.matrix, self.m.window))
            else:
                self._encoding = SnapshotEncoding(DynamicGraph(self.num_vertices, self.snapshots))
        return self._encoding


def edge_life_matrix(num_timesteps: int, life: int) -> MMatrix:
    """`apply_edge_life` (dtdg.py:194-208) as a weighting: snapshot t becomes
    sum_{k = max(0, t-life+1)}^{t} 1.0 * A_k (ascending k), i.e. the M-product
    with a banded matrix of ones -- smoothed by the same device merge."""
    if life < 1:
        raise InputError(f"edge life must be >= 1, got {life}")
    m = np.zeros((num_timesteps, num_timesteps))
    for t in range(num_timesteps):
        m[t, max(0, t - life + 1):t + 1] = 1.0
    return MMatrix(num_timesteps, life, m)


class LazyDegreeFeatures:
    """Degree features of a smoothed graph (`degree_features`,
    dtdg.py:255-266), built on the host only if read: the engine computes
    them on the device from the rebuilt snapshots."""

    def __init__(self, graph):
        self.graph = graph
        self._fs = None

    @property
    def width(self) -> int:
        return 2

    @property
    def num_timesteps(self) -> int:
        return self.graph.num_timesteps

    @property
    def num_vertices(self) -> int:
        return self.graph.num_vertices

    @property
    def frames(self) -> list:
        if self._fs is None:
            self._fs = degree_features(self.graph)
        return self._fs.frames

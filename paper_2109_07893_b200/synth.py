"""Seeded synthetic dynamic graphs with exact per-step churn (host prep).

The reference generator (`dtdg.py:288-310`) draws every snapshot
independently, which makes consecutive snapshots almost disjoint and the
graph-difference codec pointless.  The paper's datasets (and the north-star
configs) are evolving graphs, so this generator keeps an edge set and, per
step, deletes `k = round(churn * m)` uniformly chosen existing edges and
inserts `k` uniformly chosen absent pairs (self-loops allowed, as in the
reference).  Output snapshots are canonical (sorted, unit-valued), so both
this package and the reference consume the very same `DynamicGraph`.

Also: a vectorised link-prediction pair sampler for large configs (the
reference's `sample_link_prediction_sets`, `training.py:129-186`, loops in
Python over negatives; `labels.sample_link_prediction_sets` restates that
one exactly for parity runs).
"""

from __future__ import annotations

import math

import numpy as np

from .graph import DynamicGraph, SparseMatrix


def _draw_absent(rng, space: int, count: int, taken_sorted: np.ndarray, sampler=None) -> np.ndarray:
    """`count` distinct keys from [0, space) not in `taken_sorted`, in draw
    order; `sampler(rng, size)` draws candidate keys (default: uniform)."""
    got = np.zeros(0, dtype=np.int64)
    while got.shape[0] < count:
        need = count - got.shape[0]
        size = max(64, 2 * need + 16)
        cand = sampler(rng, size) if sampler is not None else rng.integers(0, space, size=size, dtype=np.int64)
        _, first = np.unique(cand, return_index=True)
        cand = cand[np.sort(first)]                      # distinct, draw order kept
        if taken_sorted.size:
            pos = np.searchsorted(taken_sorted, cand)
            pos = np.minimum(pos, taken_sorted.size - 1)
            cand = cand[taken_sorted[pos] != cand]
        if got.size:
            cand = cand[~np.isin(cand, got)]
        got = np.concatenate([got, cand[:need]])
    return got


def churn_keys(num_vertices: int, num_timesteps: int, edges_per_snapshot: int,
               churn: float, seed: int) -> list:
    """Sorted int64 key arrays (row * N + col), one per timestep."""
    n, m = int(num_vertices), int(edges_per_snapshot)
    space = n * n
    if m > space:
        raise ValueError("more edges than vertex pairs")
    rng = np.random.default_rng(seed)
    cur = np.sort(_draw_absent(rng, space, m, np.zeros(0, np.int64)))
    out = [cur]
    k = int(round(churn * m))
    for _ in range(1, num_timesteps):
        drop = rng.choice(cur.shape[0], size=k, replace=False)
        keep = np.ones(cur.shape[0], dtype=bool)
        keep[drop] = False
        ins = _draw_absent(rng, space, k, cur)
        cur = np.sort(np.concatenate([cur[keep], ins]))
        out.append(cur)
    return out


def aml_keys(num_vertices: int, num_timesteps: int, edges_per_snapshot: int, churn: float, seed: int,
             gamma: float = 2.5) -> list:
    """AMLSim-style transaction graph (BASELINE configs[2]): account degrees
    are heavy-tailed -- both endpoints are drawn by rank r = floor(n u^gamma)
    (u uniform; gamma = 2.5 gives the top 1% of accounts ~16% of the edges
    and hubs ~1000x the mean degree) through a seeded random relabelling -- and transactions
    persist: each step replaces `churn` of the edges with new draws from the
    same distribution.  Sorted int64 key arrays, one per timestep."""
    n, m = int(num_vertices), int(edges_per_snapshot)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n).astype(np.int64)

    def sampler(rng, size):
        ru = np.minimum((n * rng.random(size) ** gamma).astype(np.int64), n - 1)
        rv = np.minimum((n * rng.random(size) ** gamma).astype(np.int64), n - 1)
        return perm[ru] * n + perm[rv]

    cur = np.sort(_draw_absent(rng, n * n, m, np.zeros(0, np.int64), sampler))
    out = [cur]
    k = int(round(churn * m))
    for _ in range(1, num_timesteps):
        drop = rng.choice(cur.shape[0], size=k, replace=False)
        keep = np.ones(cur.shape[0], dtype=bool)
        keep[drop] = False
        ins = _draw_absent(rng, n * n, k, cur, sampler)
        cur = np.sort(np.concatenate([cur[keep], ins]))
        out.append(cur)
    return out


def aml_graph(num_vertices: int, num_timesteps: int, edges_per_snapshot: int, churn: float, seed: int,
              gamma: float = 2.5) -> DynamicGraph:
    n = int(num_vertices)
    return DynamicGraph(n, [SparseMatrix.from_canonical(n, k // n, k % n, None)
                            for k in aml_keys(n, num_timesteps, edges_per_snapshot, churn, seed, gamma)])


def churn_graph(num_vertices: int, num_timesteps: int, edges_per_snapshot: int,
                churn: float, seed: int) -> DynamicGraph:
    n = int(num_vertices)
    snaps = []
    for keys in churn_keys(n, num_timesteps, edges_per_snapshot, churn, seed):
        snaps.append(SparseMatrix.from_canonical(n, keys // n, keys % n, None))
    return DynamicGraph(n, snaps)


def sample_pairs_fast(graph: DynamicGraph, theta: float, seed: int):
    """Vectorised per-step positives/negatives with the reference's counts
    (ceil(theta * nnz) each, `training.py:150-156`) and keying (train frames
    0..T-2, test pairs of the last snapshot under frame T-2); the draws differ
    from the reference's Python-loop sampler."""
    from .labels import LabelSet

    rng = np.random.default_rng(seed)
    n = graph.num_vertices
    space = n * n

    def one(s: SparseMatrix):
        if s.nnz == 0:
            return np.zeros((0, 2), np.int64), np.zeros(0, np.int64)
        npos = math.ceil(theta * s.nnz)
        pick = rng.permutation(s.nnz)[:npos]
        pos = np.stack([s.rows[pick], s.cols[pick]], axis=1)
        nneg = min(npos, space - s.nnz)
        neg = _draw_absent(rng, space, nneg, s.index_keys())
        pairs = np.concatenate([pos, np.stack([neg // n, neg % n], axis=1)])
        lab = np.concatenate([np.ones(npos, np.int64), np.zeros(nneg, np.int64)])
        return pairs, lab

    train = {}
    for t in range(graph.num_timesteps - 1):
        p, l = one(graph.snapshots[t])
        if p.shape[0]:
            train[t] = (p, l)
    p, l = one(graph.snapshots[-1])
    test = {graph.num_timesteps - 2: (p, l)} if p.shape[0] else {}
    return LabelSet(2, train), LabelSet(2, test)

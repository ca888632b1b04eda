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


# ---------------------------------------------------------------------------
# device-side generation (configs[3] / configs[4]: 300M - 1B edges)
#
# The host generator above sorts and set-differences every snapshot in
# numpy (minutes and tens of GB of int64 at 1B edges).  The same exact-churn
# process runs here on the GPU with torch's generator: per step, k uniformly
# chosen edges are dropped (a random permutation prefix) and k absent
# uniform pairs inserted; the dropped / inserted keys are the graph
# difference itself, so the encoding needs no set operations.  Deterministic
# for a given seed on a given device type (every rank of a run regenerates
# the same graph); not the numpy generator's draws.


def _draw_absent_device(gen, space: int, count: int, taken_sorted, device, sampler=None):
    import torch
    got = torch.zeros(0, dtype=torch.int64, device=device)
    while got.numel() < count:
        need = count - got.numel()
        size = 2 * need + 1024
        cand = sampler(gen, size) if sampler is not None else \
            torch.randint(0, space, (size,), generator=gen, device=device, dtype=torch.int64)
        cand = torch.unique(cand)                                    # sorted, distinct
        if taken_sorted is not None and taken_sorted.numel():
            pos = torch.searchsorted(taken_sorted, cand).clamp_(max=taken_sorted.numel() - 1)
            cand = cand[taken_sorted[pos] != cand]
        if got.numel():
            gs = torch.sort(got).values
            pos = torch.searchsorted(gs, cand).clamp_(max=gs.numel() - 1)
            cand = cand[gs[pos] != cand]
        # a uniform subset of the surviving candidates (unique() sorted them)
        cand = cand[torch.randperm(cand.numel(), generator=gen, device=device)[:need]]
        got = torch.cat([got, cand])
    return got


def churn_keys_device(num_vertices: int, num_timesteps: int, edges_per_snapshot: int, churn: float,
                      seed: int, device, gamma: float | None = None):
    """Yields (t, keys, dropped, inserted) per timestep: sorted int64 device
    keys row * N + col of A_t, and the sorted keys removed from / added to
    A_{t-1} (None at t = 0).  `gamma`: AMLSim-style heavy-tailed endpoints
    (as `aml_keys`), else uniform pairs."""
    import torch
    n, m = int(num_vertices), int(edges_per_snapshot)
    space = n * n
    if m > space:
        raise ValueError("more edges than vertex pairs")
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    sampler = None
    if gamma is not None:
        perm = torch.randperm(n, generator=gen, device=device)

        def sampler(g, size):
            ru = (n * torch.rand(size, generator=g, device=device, dtype=torch.float64) ** gamma).long().clamp_(max=n - 1)
            rv = (n * torch.rand(size, generator=g, device=device, dtype=torch.float64) ** gamma).long().clamp_(max=n - 1)
            return perm[ru] * n + perm[rv]

    cur = torch.sort(_draw_absent_device(gen, space, m, None, device, sampler)).values
    yield 0, cur, None, None
    k = int(round(churn * m))
    for t in range(1, int(num_timesteps)):
        drop = torch.randperm(cur.numel(), generator=gen, device=device)[:k]
        keep = torch.ones(cur.numel(), dtype=torch.bool, device=device)
        keep[drop] = False
        ins = torch.sort(_draw_absent_device(gen, space, k, cur, device, sampler)).values
        dropped = cur[~keep]
        cur = torch.sort(torch.cat([cur[keep], ins])).values
        yield t, cur, dropped, ins


class EncodedGraph:
    """A dynamic graph held only as its encoding (no host COO snapshots):
    what `Engine` needs -- vertex / timestep counts, nnz per step and
    `encoding` -- plus the device keys of every snapshot for the pair
    sampler (freed by `drop_keys`).  Built by `device_churn_graph`."""

    def __init__(self, n: int, T: int, encoding, keys):
        self.num_vertices, self.num_timesteps = int(n), int(T)
        self.encoding = encoding
        self.nnz = [int(x) for x in encoding.nnz]
        self._keys = keys

    def sample_pairs(self, theta: float, seed: int):
        """Link-prediction sets with the reference's counts and keying
        (`training.py:129-186`: ceil(theta nnz) positives without replacement
        and as many distinct uniform non-edges per snapshot; train frames
        0..T-2, the last snapshot's pairs under frame T-2), drawn on device."""
        import torch
        from .labels import LabelSet
        n, T = self.num_vertices, self.num_timesteps
        dev = self._keys[0].device
        gen = torch.Generator(device=dev)
        gen.manual_seed(int(seed))
        out = []
        for keys in self._keys:
            nnz = keys.numel()
            npos = math.ceil(theta * nnz)
            pos = keys[torch.randperm(nnz, generator=gen, device=dev)[:npos]]
            nneg = min(npos, n * n - nnz)
            neg = _draw_absent_device(gen, n * n, nneg, keys, dev)
            k = torch.cat([pos, neg])
            out.append((torch.stack([k // n, k % n], dim=1).cpu().numpy(),
                        np.concatenate([np.ones(npos, np.int64), np.zeros(nneg, np.int64)])))
        train = {t: out[t] for t in range(T - 1) if out[t][0].shape[0]}
        test = {T - 2: out[T - 1]} if out[T - 1][0].shape[0] else {}
        return LabelSet(2, train), LabelSet(2, test)

    def drop_keys(self):
        import torch
        self._keys = []
        torch.cuda.empty_cache()


def device_churn_graph(num_vertices: int, num_timesteps: int, edges_per_snapshot: int, churn: float,
                       seed: int, device, gamma: float | None = None, pin: bool = True) -> EncodedGraph:
    """Exact-churn dynamic graph generated on `device` and encoded directly
    (full snapshots + graph differences in pinned host memory)."""
    from .materialize import SnapshotEncoding
    n, T = int(num_vertices), int(num_timesteps)
    enc = SnapshotEncoding.empty(n, T)
    keys = []
    for t, k, dropped, ins in churn_keys_device(n, T, edges_per_snapshot, churn, seed, device, gamma):
        enc.add_step(t, k, dropped, ins)
        keys.append(k)
    enc.finish(pin=pin)
    return EncodedGraph(n, T, enc, keys)

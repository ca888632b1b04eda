"""Supervised link-prediction pairs (host prep) and their device layout.

`LabelSet` and `sample_link_prediction_sets` keep the reference contract
(`training.py:78-99`, `training.py:129-186`; the sampler makes the same
generator calls in the same order, so it returns the reference's pairs for a
given seed).  `DeviceLabels` is the device-side form built once per label
set: int32 pair endpoints and labels per frame, plus an incidence CSR
(vertex -> pair endpoint slots, ascending pair order) so that the loss
gradient scatter `np.add.at(dz, pairs[:, s], ...)` (`training.py:733-734`)
becomes an atomic-free, deterministic gather.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import InputError


@dataclass(frozen=True)
class LabelSet:
    num_classes: int
    by_time: dict

    def __post_init__(self):
        for t, (pairs, labels) in self.by_time.items():
            if pairs.shape[0] != labels.shape[0]:
                raise InputError(f"pair/label count mismatch at step {t}")
            if labels.size and (labels.min() < 0 or labels.max() >= self.num_classes):
                raise InputError(f"label out of range [0, {self.num_classes}) at step {t}")

    def total_pairs(self) -> int:
        return sum(p.shape[0] for p, _ in self.by_time.values())


def sample_link_prediction_sets(g, theta: float, seed: int):
    """Reference sampler (`training.py:129-186`), vectorised but exact: the
    same generator calls in the same order, so it returns the reference's
    pairs for a given seed.

    The reference filters each negative batch key by key in Python (skip
    edges and keys already chosen, stop at nneg).  Here a batch is filtered
    as arrays -- membership in the snapshot's sorted edge keys by binary
    search, first occurrences within the batch, keys not chosen by earlier
    batches -- and its first (nneg - chosen) survivors are taken, which is
    the loop's result; the next batch size depends only on the chosen
    count, so the generator stream is consumed identically.  At configs[4]
    (15.6M edges per snapshot) a step takes ~1 s instead of minutes."""
    if not (0.0 < theta <= 1.0):
        raise InputError(f"theta must lie in (0, 1], got {theta}")
    if g.num_timesteps < 2:
        raise InputError("link prediction needs at least two snapshots")
    rng = np.random.default_rng(seed)
    n = g.num_vertices
    space = n * n

    def step(s):
        nnz = int(np.asarray(s.vals).shape[0]) if s.vals is not None else int(s.nnz)
        if nnz == 0:
            return np.zeros((0, 2), np.int64), np.zeros(0, np.int64)
        rows, cols = np.asarray(s.rows, np.int64), np.asarray(s.cols, np.int64)
        npos = math.ceil(theta * nnz)
        pick = rng.permutation(nnz)[:npos]
        pos = np.stack([rows[pick], cols[pick]], axis=1)
        edges = rows * np.int64(n) + cols            # canonical: sorted, distinct
        nneg = min(npos, space - nnz)
        neg = draw_absent_exact(rng, space, nneg, edges)
        pairs = np.concatenate([pos, np.stack([neg // n, neg % n], axis=1)])
        labels = np.concatenate([np.ones(npos, np.int64), np.zeros(nneg, np.int64)])
        return pairs, labels

    train = {}
    for t in range(g.num_timesteps - 1):
        p, l = step(g.snapshots[t])
        if p.shape[0]:
            train[t] = (p, l)
    p, l = step(g.snapshots[g.num_timesteps - 1])
    test = {g.num_timesteps - 2: (p, l)} if p.shape[0] else {}
    return LabelSet(2, train), LabelSet(2, test)


def _in_sorted(keys: np.ndarray, sorted_keys: np.ndarray) -> np.ndarray:
    if sorted_keys.size == 0:
        return np.zeros(keys.shape, bool)
    pos = np.minimum(np.searchsorted(sorted_keys, keys), sorted_keys.size - 1)
    return sorted_keys[pos] == keys


def draw_absent_exact(rng, space: int, count: int, taken_sorted: np.ndarray) -> np.ndarray:
    """`count` distinct keys in [0, space) not in `taken_sorted`, exactly as
    the reference's rejection loop draws them (`training.py:160-172`):
    batches of max(64, 2 * missing) uniform int64 keys, scanned in order."""
    chosen = np.zeros(0, np.int64)
    chosen_sorted = chosen
    while chosen.shape[0] < count:
        batch = rng.integers(0, space, size=max(64, 2 * (count - chosen.shape[0])))
        cand = batch[~_in_sorted(batch, taken_sorted)]
        _, first = np.unique(cand, return_index=True)
        cand = cand[np.sort(first)]                   # first occurrences, draw order
        cand = cand[~_in_sorted(cand, chosen_sorted)]
        chosen = np.concatenate([chosen, cand[:count - chosen.shape[0]]])
        chosen_sorted = np.sort(chosen)
    return chosen


def sample_link_prediction_sets_loop(g, theta: float, seed: int):
    """The reference's key-by-key loop, restated literally (test
    infrastructure for `sample_link_prediction_sets`)."""
    rng = np.random.default_rng(seed)
    n = g.num_vertices
    space = n * n

    def step(s):
        nnz = int(np.asarray(s.vals).shape[0])
        if nnz == 0:
            return np.zeros((0, 2), np.int64), np.zeros(0, np.int64)
        rows, cols = np.asarray(s.rows, np.int64), np.asarray(s.cols, np.int64)
        npos = math.ceil(theta * nnz)
        pick = rng.permutation(nnz)[:npos]
        pos = np.stack([rows[pick], cols[pick]], axis=1)
        edges = set((rows * np.int64(n) + cols).tolist())
        nneg = min(npos, space - nnz)
        chosen, seen = [], set()
        while len(chosen) < nneg:
            batch = rng.integers(0, space, size=max(64, 2 * (nneg - len(chosen))))
            for key in batch.tolist():
                if key in edges or key in seen:
                    continue
                seen.add(key)
                chosen.append(key)
                if len(chosen) == nneg:
                    break
        neg = np.asarray(chosen, dtype=np.int64)
        pairs = np.concatenate([pos, np.stack([neg // n, neg % n], axis=1)], axis=0)
        labels = np.concatenate([np.ones(npos, np.int64), np.zeros(nneg, np.int64)])
        return pairs, labels

    train = {}
    for t in range(g.num_timesteps - 1):
        p, l = step(g.snapshots[t])
        if p.shape[0]:
            train[t] = (p, l)
    p, l = step(g.snapshots[g.num_timesteps - 1])
    test = {g.num_timesteps - 2: (p, l)} if p.shape[0] else {}
    return LabelSet(2, train), LabelSet(2, test)


@dataclass
class FrameLabels:
    """One frame's pairs in device-ready host arrays."""
    count: int
    u: np.ndarray          # int32 [R]
    v: np.ndarray          # int32 [R]
    y: np.ndarray          # int32 [R]
    inc_ptr: np.ndarray    # int32 [N+1] over the vertex space
    inc_slot: np.ndarray   # int32 [2R]: pair * 2 + side, ascending per vertex


def frame_labels(pairs: np.ndarray, labels: np.ndarray, n: int, num_classes: int) -> FrameLabels:
    pairs = np.asarray(pairs, dtype=np.int64)
    labels = np.asarray(labels, dtype=np.int64)
    if pairs.ndim != 2 or pairs.shape[1] != 2:
        raise InputError("pairs must be an (R, 2) array")
    if pairs.size and (pairs.min() < 0 or pairs.max() >= n):
        raise InputError(f"vertex id out of range [0, {n})")
    if labels.size and (labels.min() < 0 or labels.max() >= num_classes):
        raise InputError(f"label out of range [0, {num_classes})")
    r = pairs.shape[0]
    # np.add.at(dz, pairs[:,0], .) runs before np.add.at(dz, pairs[:,1], .)
    # (training.py:733-734): order slots side-major, then pair index.
    verts = np.concatenate([pairs[:, 0], pairs[:, 1]])
    slots = np.concatenate([np.arange(r) * 2, np.arange(r) * 2 + 1])
    order = np.argsort(verts, kind="stable")
    counts = np.bincount(verts, minlength=n)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    return FrameLabels(r, pairs[:, 0].astype(np.int32), pairs[:, 1].astype(np.int32),
                       labels.astype(np.int32), ptr.astype(np.int32),
                       slots[order].astype(np.int32))


def frame_labels_device(pairs, labels, n: int, num_classes: int, device) -> dict:
    """`frame_labels` built on the device (prep of configs[3]/[4]: 3.1M
    pairs per frame): int32 endpoints / labels and the incidence CSR
    vertex -> pair * 2 + side, side-major then pair order per vertex (a
    stable sort, the order of `np.add.at` over pairs[:, 0] then pairs[:, 1],
    `training.py:733-734`)."""
    import torch
    p = torch.as_tensor(np.asarray(pairs, dtype=np.int64)).reshape(-1, 2).to(device)
    y = torch.as_tensor(np.asarray(labels, dtype=np.int64)).to(device)
    if p.shape[0] != y.shape[0]:
        raise InputError("pair/label count mismatch")
    if p.numel() and (int(p.min()) < 0 or int(p.max()) >= n):
        raise InputError(f"vertex id out of range [0, {n})")
    if y.numel() and (int(y.min()) < 0 or int(y.max()) >= num_classes):
        raise InputError(f"label out of range [0, {num_classes})")
    r = p.shape[0]
    verts = torch.cat([p[:, 0], p[:, 1]])
    ar = torch.arange(r, device=p.device, dtype=torch.int64) * 2
    slots = torch.cat([ar, ar + 1])
    order = torch.sort(verts, stable=True).indices
    ptr = torch.zeros(n + 1, dtype=torch.int64, device=p.device)
    ptr[1:] = torch.cumsum(torch.bincount(verts, minlength=n), 0)
    # vertices with incident pairs (ascending): dgnn_head_scatter_active gathers only these
    act = torch.nonzero(ptr[1:] != ptr[:-1]).reshape(-1).to(torch.int32)
    return dict(n=r, u=p[:, 0].to(torch.int32).contiguous(), v=p[:, 1].to(torch.int32).contiguous(),
                y=y.to(torch.int32), ptr=ptr.to(torch.int32), slot=slots[order].to(torch.int32), act=act,
                nact=int(act.numel()))

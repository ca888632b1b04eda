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
    """Reference sampler semantics (`training.py:129-186`)."""
    if not (0.0 < theta <= 1.0):
        raise InputError(f"theta must lie in (0, 1], got {theta}")
    if g.num_timesteps < 2:
        raise InputError("link prediction needs at least two snapshots")
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

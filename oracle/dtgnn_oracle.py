"""CPU ORACLE — test infrastructure only, never the product path.

A numpy (float64) restatement of the reference algorithm on the hot path of
arXiv 2109.07893 as implemented by the reference package `dtgnn` 0.1.0
(`/root/reference/pkg/src/dtgnn`).  Every function cites the reference
file:line it restates.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
module, and only as the checker (or the timed CPU baseline), never as the
thing measured for the GPU path.

Parity of this restatement is PINNED against golden vectors produced by
running the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`), see
`tests/test_oracle_golden.py`.

Numerics: float64 throughout, fixed accumulation orders, so the
restatement reproduces the reference bit-for-bit where the reference is
order-defined (canonical COO, Laplacian values, `np.add.at` SpMM) and to
~1e-12 where BLAS blocking decides the order.
"""

from __future__ import annotations

import math
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# errors (errors.py:4-29) -- the oracle raises plain ValueError / RuntimeError
# subclasses with the reference's names so tests can match by name.


class OracleConfigError(ValueError):
    pass


class OracleCorruptDelta(ValueError):
    pass


class OracleProtocolError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# canonical COO (core.py:39-129)


@dataclass(frozen=True, eq=False)
class Coo:
    dim: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    def keys(self) -> np.ndarray:
        # core.py:102-104
        return self.rows * np.int64(self.dim) + self.cols

    def same(self, other: "Coo") -> bool:
        return (self.dim == other.dim and np.array_equal(self.rows, other.rows)
                and np.array_equal(self.cols, other.cols)
                and np.array_equal(self.vals, other.vals))


def coo_from_entries(dim, rows, cols, vals=None) -> Coo:
    """core.py:54-87: sort by (row, col), sum duplicates in input order
    (np.add.at is sequential), drop exact zeros."""
    r = np.asarray(rows, dtype=np.int64).ravel()
    c = np.asarray(cols, dtype=np.int64).ravel()
    v = (np.ones(r.shape[0]) if vals is None
         else np.asarray(vals, dtype=np.float64).ravel())
    k = r * np.int64(dim) + c
    uk, inv = np.unique(k, return_inverse=True)
    acc = np.zeros(uk.shape[0])
    np.add.at(acc, inv, v)
    nz = acc != 0.0
    uk = uk[nz]
    return Coo(int(dim), uk // dim, uk % dim, acc[nz])


def coo_from_sparse(sm) -> Coo:
    """Adopt any object with dim/rows/cols/vals (the reference SparseMatrix
    or the product's) without re-canonicalising."""
    return Coo(int(sm.dim), np.asarray(sm.rows, np.int64), np.asarray(sm.cols, np.int64),
               np.asarray(sm.vals, np.float64))


# ---------------------------------------------------------------------------
# kernels (core.py:142-161)


def spmm(a: Coo, x: np.ndarray) -> np.ndarray:
    """core.py:142-152: out[i] += v * x[j] in canonical entry order."""
    out = np.zeros((a.dim, x.shape[1]))
    np.add.at(out, a.rows, a.vals[:, None] * x[a.cols])
    return out


def spmm_t(a: Coo, g: np.ndarray) -> np.ndarray:
    """core.py:155-161: out[j] += v * g[i] in canonical entry order."""
    out = np.zeros((a.dim, g.shape[1]))
    np.add.at(out, a.cols, a.vals[:, None] * g[a.rows])
    return out


# ---------------------------------------------------------------------------
# data model (dtdg.py)


def laplacian(a: Coo) -> Coo:
    """dtdg.py:178-191: D^-1/2 (A + I) D^-1/2 with D = 1 + structural
    out-degree; value (a*is_r)*is_c, A entries first then the identity."""
    deg = np.bincount(a.rows, minlength=a.dim).astype(np.float64)
    isq = 1.0 / np.sqrt(1.0 + deg)
    diag = np.arange(a.dim, dtype=np.int64)
    r = np.concatenate([a.rows, diag])
    c = np.concatenate([a.cols, diag])
    v = np.concatenate([a.vals, np.ones(a.dim)])
    return coo_from_entries(a.dim, r, c, (v * isq[r]) * isq[c])


def degree_feats(snaps) -> list:
    """dtdg.py:255-266: column 0 structural out-degree, column 1 in-degree."""
    out = []
    for s in snaps:
        f = np.zeros((s.dim, 2))
        f[:, 0] = np.bincount(s.rows, minlength=s.dim)
        f[:, 1] = np.bincount(s.cols, minlength=s.dim)
        out.append(f)
    return out


def m_matrix(t_count: int, w: int) -> np.ndarray:
    """dtdg.py:211-221: row t (1-based) averages columns max(1,t-w+1)..t."""
    m = np.zeros((t_count, t_count))
    for t0 in range(t_count):
        lo = max(0, t0 - w + 1)
        m[t0, lo:t0 + 1] = 1.0 / min(w, t0 + 1)
    return m


def m_transform_frames(frames, m: np.ndarray, w: int) -> list:
    """dtdg.py:224-236 (accumulation from zeros, ascending k)."""
    out = []
    for t in range(m.shape[0]):
        acc = np.zeros_like(frames[0])
        for k in range(max(0, t - w + 1), t + 1):
            acc += m[t, k] * frames[k]
        out.append(acc)
    return out


def weighted_sum(terms) -> Coo:
    """core.py:173-192."""
    dim = terms[0][1].dim
    r = np.concatenate([s.rows for _, s in terms])
    c = np.concatenate([s.cols for _, s in terms])
    v = np.concatenate([float(wt) * s.vals for wt, s in terms])
    return coo_from_entries(dim, r, c, v)


def m_transform_snaps(snaps, m: np.ndarray, w: int) -> list:
    """dtdg.py:239-252."""
    return [weighted_sum([(m[t, k], snaps[k]) for k in range(max(0, t - w + 1), t + 1)])
            for t in range(m.shape[0])]


# ---------------------------------------------------------------------------
# graph-difference codec (delta.py:37-178)


@dataclass
class Transfer:
    """delta.py:57-100 counters (index entry 8 B, value entry 8 B)."""
    index_entries_sent: int = 0
    value_entries_sent: int = 0
    snapshots_full: int = 0
    snapshots_delta: int = 0

    def as_dict(self) -> dict:
        tot = self.snapshots_full + self.snapshots_delta
        return {
            "index_entries_sent": self.index_entries_sent,
            "value_entries_sent": self.value_entries_sent,
            "snapshots_full": self.snapshots_full,
            "snapshots_delta": self.snapshots_delta,
            "delta_fraction": (self.snapshots_delta / tot) if tot else 0.0,
            "bytes_sent": 8 * (self.index_entries_sent + self.value_entries_sent),
        }

    def add(self, o: "Transfer"):
        self.index_entries_sent += o.index_entries_sent
        self.value_entries_sent += o.value_entries_sent
        self.snapshots_full += o.snapshots_full
        self.snapshots_delta += o.snapshots_delta


def delta_encode(prev: Coo, nxt: Coo):
    """delta.py:110-123: (ext_prev pairs, ext_next pairs, all values of nxt)."""
    kp, kn = prev.keys(), nxt.keys()
    gone = np.setdiff1d(kp, kn, assume_unique=True)
    new = np.setdiff1d(kn, kp, assume_unique=True)
    d = prev.dim
    return (np.stack([gone // d, gone % d], 1), np.stack([new // d, new % d], 1),
            nxt.vals.copy())


def delta_apply(prev: Coo, ext_prev, ext_next, values) -> Coo:
    """delta.py:126-146 with the same CorruptDelta checks."""
    d = np.int64(prev.dim)
    kp = prev.keys()
    gone = ext_prev[:, 0].astype(np.int64) * d + ext_prev[:, 1]
    new = ext_next[:, 0].astype(np.int64) * d + ext_next[:, 1]
    if not np.all(np.isin(gone, kp)):
        raise OracleCorruptDelta("ext_prev not in base")
    common = np.setdiff1d(kp, gone, assume_unique=True)
    if np.intersect1d(new, common).size:
        raise OracleCorruptDelta("ext_next overlaps common")
    keys = np.union1d(common, new)
    if keys.shape[0] != values.shape[0]:
        raise OracleCorruptDelta("value count mismatch")
    return coo_from_entries(prev.dim, keys // d, keys % d, values)


def stream(snaps, ledger: Transfer) -> list:
    """delta.py:149-170: first full, the rest rebuilt from deltas."""
    out = [snaps[0]]
    ledger.index_entries_sent += snaps[0].nnz
    ledger.value_entries_sent += snaps[0].nnz
    ledger.snapshots_full += 1
    cur = snaps[0]
    for nxt in snaps[1:]:
        ep, en, vals = delta_encode(cur, nxt)
        ledger.index_entries_sent += ep.shape[0] + en.shape[0]
        ledger.value_entries_sent += vals.shape[0]
        ledger.snapshots_delta += 1
        cur = delta_apply(cur, ep, en, vals)
        out.append(cur)
    return out


# ---------------------------------------------------------------------------
# model (models.py)


@dataclass(frozen=True)
class Cfg:
    """models.py:49-93 (only the fields the hot path reads)."""
    architecture: str
    in_features: int = 2
    hidden_features: int = 6
    embed_features: int = 6
    layers: int = 2
    window: int = 2
    edge_life: int = 2
    classes: int = 2

    def dims(self):
        """models.py:80-93 -> list of (fin, gcn_out, out)."""
        res, fin = [], self.in_features
        for l in range(self.layers):
            last = l == self.layers - 1
            if self.architecture == "cd-gcn":
                g, o = self.hidden_features, (self.embed_features if last else self.hidden_features)
            else:
                g = self.embed_features if last else self.hidden_features
                o = g
            res.append((fin, g, o))
            fin = o
        return res


def as_cfg(cfg) -> Cfg:
    return Cfg(cfg.architecture, cfg.in_features, cfg.hidden_features, cfg.embed_features,
               cfg.layers, cfg.window, cfg.edge_life, cfg.classes)


def init_params(cfg: Cfg, seed: int) -> dict:
    """models.py:138-177: Glorot-uniform draws in fixed key order, forget
    bias 1, zero head."""
    rng = np.random.default_rng(seed)

    def glorot(fi, fo):
        lim = np.sqrt(6.0 / (fi + fo))
        return rng.uniform(-lim, lim, size=(fi, fo))

    p = {}
    for l, (fin, g, o) in enumerate(cfg.dims()):
        if cfg.architecture == "egcn-o":
            # models.py:157-163: w0, then the four gate matrices; forget bias 1
            p[f"evolve{l}.w0"] = glorot(fin, g)
            p[f"evolve{l}.gates"] = np.stack([glorot(fin, g) for _ in range(4)])
            bias = np.zeros((4, fin, g))
            bias[1] = 1.0
            p[f"evolve{l}.bias"] = bias
            continue
        p[f"gcn{l}.w"] = glorot(fin, g)
        if cfg.architecture == "cd-gcn":
            k = fin + g
            p[f"lstm{l}.wx"] = np.concatenate([glorot(k, o) for _ in range(4)], axis=1)
            p[f"lstm{l}.wh"] = np.concatenate([glorot(o, o) for _ in range(4)], axis=1)
            b = np.zeros(4 * o)
            b[o:2 * o] = 1.0
            p[f"lstm{l}.b"] = b
    p["head.w"] = np.zeros((2 * cfg.embed_features, cfg.classes))
    p["head.b"] = np.zeros(cfg.classes)
    return p


def sig(x):
    return 1.0 / (1.0 + np.exp(-x))


# per-timestep cells (training.py:342-367)


def gcn_fwd(s, w, skip):
    q = s @ w
    if skip:
        r = np.maximum(np.concatenate([s, q], 1), 0.0)
        return r, (s, q, r)
    y = np.maximum(q, 0.0)
    return y, (s, y)


def gcn_bwd(cache, dr, w, skip):
    if skip:
        s, q, r = cache
        dpre = dr * (r > 0.0)
        f = s.shape[1]
        ds = dpre[:, :f].copy()
        dq = dpre[:, f:]
        dw = s.T @ dq
        ds += dq @ w.T
        return dw, ds
    s, y = cache
    dpre = dr * (y > 0.0)
    return s.T @ dpre, dpre @ w.T


# LSTM block (training.py:370-427)


def lstm_fwd(wx, wh, b, state, ts, xs):
    H = wh.shape[0]
    h, c = state
    ys, cache = {}, []
    for t in ts:
        x = xs[t]
        z = x @ wx + h @ wh + b
        i, f, o = sig(z[:, :H]), sig(z[:, H:2 * H]), sig(z[:, 2 * H:3 * H])
        g = np.tanh(z[:, 3 * H:])
        c2 = f * c + i * g
        tc = np.tanh(c2)
        h2 = o * tc
        cache.append((x, h, c, i, f, o, g, c2, tc))
        h, c = h2, c2
        ys[t] = h2
    return ys, (h, c), cache


def lstm_bwd(wx, wh, ts, cache, dys, dstate):
    dh_c, dc_c = dstate[0].copy(), dstate[1].copy()
    dwx, dwh, db = np.zeros_like(wx), np.zeros_like(wh), np.zeros(wx.shape[1])
    dxs = {}
    for t, (x, hp, cp, i, f, o, g, c2, tc) in zip(reversed(ts), reversed(cache)):
        dh = dys[t] + dh_c
        do = dh * tc
        dc = dh * o * (1.0 - tc * tc) + dc_c
        df, di, dg = dc * cp, dc * g, dc * i
        dc_c = dc * f
        dz = np.concatenate([di * i * (1.0 - i), df * f * (1.0 - f),
                             do * o * (1.0 - o), dg * (1.0 - g * g)], 1)
        dwx += x.T @ dz
        dwh += hp.T @ dz
        db += dz.sum(0)
        dxs[t] = dz @ wx.T
        dh_c = dz @ wh.T
    return dxs, (dh_c, dc_c), (dwx, dwh, db)


# M-product block (training.py:430-460)


def mprod_fwd(m, w, ts, frames):
    out = {}
    for t in ts:
        lo = max(0, t - w + 1)
        acc = m[t, lo] * frames[lo]
        for k in range(lo + 1, t + 1):
            acc = acc + m[t, k] * frames[k]
        out[t] = acc
    return out


def mprod_bwd(m, w, ts, dz, start, like):
    dy = {t: np.zeros_like(like) for t in ts}
    before = {}
    for t in ts:
        for k in range(max(0, t - w + 1), t + 1):
            g = m[t, k] * dz[t]
            if k >= start:
                dy[k] += g
            elif k in before:
                before[k] += g
            else:
                before[k] = g
    return dy, before


# ---------------------------------------------------------------------------
# loss and labels (training.py:102-197, 698-735; models.py:335-348)


def ce(logits, labels, mean=True):
    """training.py:102-126."""
    n = logits.shape[0]
    if n == 0:
        return 0.0, np.zeros_like(logits)
    sh = logits - logits.max(axis=1, keepdims=True)
    lp = sh - np.log(np.exp(sh).sum(axis=1, keepdims=True))
    loss = -lp[np.arange(n), labels]
    g = np.exp(lp)
    g[np.arange(n), labels] -= 1.0
    if mean:
        return float(loss.mean()), g / n
    return float(loss.sum()), g


def head_logits(z, pairs, hw, hb):
    """models.py:335-348."""
    return np.concatenate([z[pairs[:, 0]], z[pairs[:, 1]]], 1) @ hw + hb


def sample_labels(snaps, theta: float, seed: int):
    """training.py:129-186 with the same generator call sequence; returns
    (train_by_time, test_by_time) dicts of (pairs, labels)."""
    rng = np.random.default_rng(seed)
    n = snaps[0].dim
    space = n * n

    def one(s: Coo):
        if s.nnz == 0:
            return np.zeros((0, 2), np.int64), np.zeros(0, np.int64)
        npos = math.ceil(theta * s.nnz)
        pick = rng.permutation(s.nnz)[:npos]
        pos = np.stack([s.rows[pick], s.cols[pick]], 1)
        edges = set(int(k) for k in s.keys())
        nneg = min(npos, space - s.nnz)
        negs, seen = [], set()
        while len(negs) < nneg:
            batch = rng.integers(0, space, size=max(64, 2 * (nneg - len(negs))))
            for kk in batch:
                k = int(kk)
                if k in edges or k in seen:
                    continue
                seen.add(k)
                negs.append(k)
                if len(negs) == nneg:
                    break
        negs = np.asarray(negs, np.int64)
        pairs = np.concatenate([pos, np.stack([negs // n, negs % n], 1)], 0)
        lab = np.concatenate([np.ones(npos, np.int64), np.zeros(nneg, np.int64)])
        return pairs, lab

    train = {}
    for t in range(len(snaps) - 1):
        p, l = one(snaps[t])
        if p.shape[0]:
            train[t] = (p, l)
    p, l = one(snaps[-1])
    test = {len(snaps) - 2: (p, l)} if p.shape[0] else {}
    return train, test


def total_pairs(by_time) -> int:
    return sum(p.shape[0] for p, _ in by_time.values())


def loss_sum(params, zf, by_time, ts):
    """training.py:698-710."""
    tot, cnt = 0.0, 0
    for t in ts:
        if t in by_time:
            p, l = by_time[t]
            piece, _ = ce(head_logits(zf[t], p, params["head.w"], params["head.b"]), l, False)
            tot += piece
            cnt += l.shape[0]
    return tot, cnt


def loss_grads(E, params, zf, by_time, ts, scale):
    """training.py:713-735."""
    hw = params["head.w"]
    dz, dhw, dhb = {}, np.zeros_like(hw), np.zeros_like(params["head.b"])
    for t in ts:
        dz[t] = np.zeros_like(zf[t])
        if t not in by_time:
            continue
        p, l = by_time[t]
        cat = np.concatenate([zf[t][p[:, 0]], zf[t][p[:, 1]]], 1)
        _, dl = ce(cat @ hw + params["head.b"], l, False)
        dl = dl * scale
        dhw += cat.T @ dl
        dhb += dl.sum(0)
        dc = dl @ hw.T
        np.add.at(dz[t], p[:, 0], dc[:, :E])
        np.add.at(dz[t], p[:, 1], dc[:, E:])
    return dz, dhw, dhb


# ---------------------------------------------------------------------------
# prepared inputs (training.py:204-250)


@dataclass
class Prepared:
    graph: list          # (smoothed) raw snapshots, Coo
    laps: list           # normalised Laplacians, Coo
    feats: list          # N x in_features frames
    s1: list             # laps[t] @ feats[t]
    m: np.ndarray | None
    window: int

    @property
    def T(self):
        return len(self.laps)

    @property
    def N(self):
        return self.feats[0].shape[0]


def prepare(cfg: Cfg, snaps) -> Prepared:
    """training.py:224-250."""
    T = len(snaps)
    m = None
    if cfg.architecture == "tm-gcn":
        m = m_matrix(T, cfg.window)
        g = m_transform_snaps(snaps, m, cfg.window)
        feats = m_transform_frames(degree_feats(snaps), m, cfg.window)
    elif cfg.architecture == "cd-gcn":
        g, feats = list(snaps), degree_feats(snaps)
    else:
        # training.py:238-240: edge life (dtdg.py:194-208), degrees of the smoothed graph
        life = cfg.edge_life
        g = [weighted_sum([(1.0, snaps[k]) for k in range(max(0, t - life + 1), t + 1)]) for t in range(T)]
        feats = degree_feats(g)
    laps = [laplacian(s) for s in g]
    s1 = [spmm(a, x) for a, x in zip(laps, feats)]
    return Prepared(g, laps, feats, s1, m, cfg.window)


def from_reference_data(data, window: int) -> Prepared:
    return Prepared([coo_from_sparse(s) for s in data.graph.snapshots],
                    [coo_from_sparse(s) for s in data.laps],
                    [np.asarray(f) for f in data.feats.frames],
                    [np.asarray(s) for s in data.s1],
                    None if data.m_matrix is None else np.asarray(data.m_matrix.matrix),
                    window)


# ---------------------------------------------------------------------------
# sequential block engine (training.py:516-865)


def _state0(cfg, n, params=None, grads=False):
    """training.py:516-539: LSTM state, or the evolving weight (w0; zero for
    its gradient carry) for egcn-o."""
    out = []
    for l, (_, _, o) in enumerate(cfg.dims()):
        if cfg.architecture == "cd-gcn":
            out.append((np.zeros((n, o)), np.zeros((n, o))))
        elif cfg.architecture == "egcn-o":
            w0 = params[f"evolve{l}.w0"]
            out.append(np.zeros_like(w0) if grads else w0)
        else:
            out.append(None)
    return out


def evolve_fwd(gates, bias, w_in, ts):
    """training.py:466-484 (egcn_evolve, models.py:247-268): elementwise
    matrix-LSTM chain; returns ({t: W_t}, W_last, cache)."""
    w, w_by_t, cache = w_in, {}, []
    for t in ts:
        z = gates * w + bias
        i, f, o = sig(z[0]), sig(z[1]), sig(z[2])
        g = np.tanh(z[3])
        c = f * w + i * g
        tc = np.tanh(c)
        w_new = o * tc
        cache.append((w, i, f, o, g, tc))
        w_by_t[t] = w_new
        w = w_new
    return w_by_t, w, cache


def evolve_bwd(gates, ts, cache, seeds, dw_out):
    """training.py:487-509 -> (dgates, dbias, dw_in)."""
    dgates, dbias = np.zeros_like(gates), np.zeros_like(gates)
    carry = dw_out.copy()
    for t, (wp, i, f, o, g, tc) in zip(reversed(ts), reversed(cache)):
        dwn = carry + seeds[t] if t in seeds else carry
        do = dwn * tc
        dc = dwn * o * (1.0 - tc * tc)
        df, di, dg = dc * wp, dc * g, dc * i
        dwp = dc * f
        dzs = (di * i * (1.0 - i), df * f * (1.0 - f), do * o * (1.0 - o), dg * (1.0 - g * g))
        for k, dz in enumerate(dzs):
            dgates[k] += dz * wp
            dbias[k] += dz
            dwp = dwp + dz * gates[k]
        carry = dwp
    return dgates, dbias, carry


def block_forward(cfg, P: Prepared, params, ts, state_in, trailing, keep):
    """training.py:549-618 -> (z frames, state_out, trailing_out, caches)."""
    skip = cfg.architecture == "cd-gcn"
    cur, st_out, tr_out, caches = None, [], [], ([] if keep else None)
    for l, (fin, g, o) in enumerate(cfg.dims()):
        if cfg.architecture == "egcn-o":
            w_by_t, w_last, ev = evolve_fwd(params[f"evolve{l}.gates"], params[f"evolve{l}.bias"], state_in[l], ts)
            st_out.append(w_last)
            tr_out.append({})
            gout, gc = {}, {}
            for t in ts:
                s = P.s1[t] if l == 0 else spmm(P.laps[t], cur[t])
                gout[t], gc[t] = gcn_fwd(s, w_by_t[t], False)
            if keep:
                caches.append({"gcn": gc, "evolve": ev, "w_by_t": w_by_t})
            cur = gout
            continue
        w = params[f"gcn{l}.w"]
        gout, gc = {}, {}
        for t in ts:
            s = P.s1[t] if l == 0 else spmm(P.laps[t], cur[t])
            gout[t], gc[t] = gcn_fwd(s, w, skip)
        lc = {"gcn": gc}
        if skip:
            ys, st, lcache = lstm_fwd(params[f"lstm{l}.wx"], params[f"lstm{l}.wh"],
                                      params[f"lstm{l}.b"], state_in[l], ts, gout)
            lc["lstm"] = lcache
            out = ys
            st_out.append(st)
            tr_out.append({ts[-1]: ys[ts[-1]]})
        else:
            fr = dict(trailing[l])
            fr.update(gout)
            out = mprod_fwd(P.m, P.window, ts, fr)
            keepn = min(P.window, len(ts))
            tr_out.append({t: gout[t] for t in ts[-keepn:]})
            st_out.append(None)
        if keep:
            caches.append(lc)
        cur = out
    return cur, st_out, tr_out, caches


def block_backward(cfg, P: Prepared, params, ts, caches, dz, dstate, dtr_in):
    """training.py:621-691 -> (dparams, dstate_in, dtrailing_out)."""
    skip = cfg.architecture == "cd-gcn"
    dp, dst_in, dtr_out = {}, [None] * cfg.layers, [dict() for _ in range(cfg.layers)]
    dcur = dz
    for l in reversed(range(cfg.layers)):
        lc = caches[l]
        if cfg.architecture == "egcn-o":
            seeds, prev = {}, {}
            for t in ts:
                seeds[t], ds = gcn_bwd(lc["gcn"][t], dcur[t], lc["w_by_t"][t], False)
                if l > 0:
                    prev[t] = spmm_t(P.laps[t], ds)
            dg, dbias, dst_in[l] = evolve_bwd(params[f"evolve{l}.gates"], ts, lc["evolve"], seeds, dstate[l])
            dp[f"evolve{l}.gates"], dp[f"evolve{l}.bias"] = dg, dbias
            dcur = prev
            continue
        if skip:
            dy, dst, (dwx, dwh, db) = lstm_bwd(params[f"lstm{l}.wx"], params[f"lstm{l}.wh"],
                                               ts, lc["lstm"], dcur, dstate[l])
            dst_in[l] = dst
            dp[f"lstm{l}.wx"], dp[f"lstm{l}.wh"], dp[f"lstm{l}.b"] = dwx, dwh, db
        else:
            like = next(iter(dcur.values()))
            dy, before = mprod_bwd(P.m, P.window, ts, dcur, ts[0], like)
            for t, g in dtr_in[l].items():
                dy[t] += g
            dtr_out[l] = before
        w = params[f"gcn{l}.w"]
        dw = np.zeros_like(w)
        prev = {}
        for t in ts:
            dwt, ds = gcn_bwd(lc["gcn"][t], dy[t], w, skip)
            dw += dwt
            if l > 0:
                prev[t] = spmm_t(P.laps[t], ds)
        dp[f"gcn{l}.w"] = dw
        dcur = prev
    return dp, dst_in, dtr_out


def backward_checkpoint(cfg: Cfg, P: Prepared, by_time, params, nblk: int, mean=True):
    """training.py:798-865 (loss, grads)."""
    T = P.T
    if nblk < 1 or T % nblk:
        raise OracleConfigError("nblk must divide T")
    bs = T // nblk
    blocks = [list(range(b * bs, (b + 1) * bs)) for b in range(nblk)]
    state = _state0(cfg, P.N, params)
    trail = [dict() for _ in range(cfg.layers)]
    pis, tot, cnt = {}, 0.0, 0
    for b, ts in enumerate(blocks):
        zf, st, tr, _ = block_forward(cfg, P, params, ts, state, trail, False)
        piece, c = loss_sum(params, zf, by_time, ts)
        tot += piece
        cnt += c
        state = st
        pis[b] = st
        for l in range(cfg.layers):
            trail[l].update(tr[l])
    scale = (1.0 / cnt) if (mean and cnt) else 1.0
    loss = tot * scale
    grads = {k: np.zeros_like(v) for k, v in params.items()}
    dstate = _state0(cfg, P.N, params, grads=True)
    dtr = [dict() for _ in range(cfg.layers)]
    init = _state0(cfg, P.N, params)
    for b in reversed(range(nblk)):
        ts = blocks[b]
        zf, _, _, caches = block_forward(cfg, P, params, ts, pis[b - 1] if b else init, trail, True)
        dz, dhw, dhb = loss_grads(cfg.embed_features, params, zf, by_time, ts, scale)
        grads["head.w"] += dhw
        grads["head.b"] += dhb
        dtr_in = []
        for l in range(cfg.layers):
            own = [t for t in dtr[l] if t in set(ts)]
            dtr_in.append({t: dtr[l].pop(t) for t in own})
        dp, dstate, dtr_out = block_backward(cfg, P, params, ts, caches, dz, dstate, dtr_in)
        for k, v in dp.items():
            grads[k] += v
        for l in range(cfg.layers):
            for t, g in dtr_out[l].items():
                dtr[l][t] = dtr[l][t] + g if t in dtr[l] else g
    if cfg.architecture == "egcn-o":      # training.py:750-754: the initial weights' gradient
        for l in range(cfg.layers):
            grads[f"evolve{l}.w0"] += dstate[l]
    return loss, grads


def model_forward(cfg: Cfg, P: Prepared, params) -> list:
    """models.py:275-323 (cd-gcn / tm-gcn), straight-line over all T."""
    frames = list(P.feats)
    T, n = P.T, P.N
    skip = cfg.architecture == "cd-gcn"
    for l, (fin, g, o) in enumerate(cfg.dims()):
        if cfg.architecture == "egcn-o":       # models.py:315-321
            w_by_t, _, _ = evolve_fwd(params[f"evolve{l}.gates"], params[f"evolve{l}.bias"],
                                      params[f"evolve{l}.w0"], list(range(T)))
            frames = [np.maximum(spmm(P.laps[t], frames[t]) @ w_by_t[t], 0.0) for t in range(T)]
            continue
        w = params[f"gcn{l}.w"]
        if skip:
            h, c = np.zeros((n, o)), np.zeros((n, o))
            wx, wh, b = params[f"lstm{l}.wx"], params[f"lstm{l}.wh"], params[f"lstm{l}.b"]
            out = []
            for t in range(T):
                s = spmm(P.laps[t], frames[t])
                r = np.maximum(np.concatenate([s, s @ w], 1), 0.0)
                ys, (h, c), _ = lstm_fwd(wx, wh, b, (h, c), [t], {t: r})
                out.append(ys[t])
            frames = out
        else:
            out = [np.maximum(spmm(P.laps[t], frames[t]) @ w, 0.0) for t in range(T)]
            frames = m_transform_frames(out, P.m, P.window)
    return frames


def _rows_of(a: Coo, rows: np.ndarray):
    """Entries of canonical `a` whose row is in sorted `rows` (canonical order)."""
    lo = np.searchsorted(a.rows, rows, side="left")
    cnt = np.searchsorted(a.rows, rows, side="right") - lo
    if cnt.sum() == 0:
        return np.zeros(0, np.int64)
    start = np.repeat(lo - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
    return (start + np.arange(cnt.sum())).astype(np.int64)


def model_forward_rows(cfg: Cfg, laps_at, feats_at, T: int, params, rows, m=None, window: int = 2):
    """`model_forward` (models.py:275-323) restricted to output rows `rows`
    (test infrastructure for the large-config parity protocol, SURVEY §8c:
    rows of the SpMM and per-vertex LSTM / M-product timelines are
    independent, `test_models.py:267-285`).  Layer l needs its inputs only at
    the union over t of the Laplacian neighbourhoods of the rows it outputs,
    so the forward runs on that dependency cone -- identical arithmetic per
    row (spmm in canonical entry order, `core.py:142-152`).  `laps_at(t)` /
    `feats_at(t)` return the full Laplacian / input frame of step t.
    Returns {t: frame rows} for the requested rows (sorted)."""
    rows = np.unique(np.asarray(rows, np.int64))
    dims = cfg.dims()
    L = len(dims)
    need = [None] * L
    need[L - 1] = rows
    for l in range(L - 1, 0, -1):
        acc = [need[l]]
        for t in range(T):
            a = laps_at(t)
            acc.append(a.cols[_rows_of(a, need[l])])
        need[l - 1] = np.unique(np.concatenate(acc))
    skip = cfg.architecture == "cd-gcn"
    prev_rows, frames = None, None
    for l, (fin, g, o) in enumerate(dims):
        R = need[l]
        w = params[f"gcn{l}.w"]
        out = []
        if skip:
            h, c = np.zeros((R.size, o)), np.zeros((R.size, o))
            wx, wh, b = params[f"lstm{l}.wx"], params[f"lstm{l}.wh"], params[f"lstm{l}.b"]
        for t in range(T):
            a = laps_at(t)
            idx = _rows_of(a, R)
            x = feats_at(t) if l == 0 else frames[t]
            cols = a.cols[idx] if l == 0 else np.searchsorted(prev_rows, a.cols[idx])
            s = np.zeros((R.size, x.shape[1]))
            np.add.at(s, np.searchsorted(R, a.rows[idx]), a.vals[idx][:, None] * x[cols])
            if skip:
                r = np.maximum(np.concatenate([s, s @ w], 1), 0.0)
                ys, (h, c), _ = lstm_fwd(wx, wh, b, (h, c), [t], {t: r})
                out.append(ys[t])
            else:
                out.append(np.maximum(s @ w, 0.0))
        if not skip:
            out = m_transform_frames(out, m, window)
        prev_rows, frames = R, out
    return {t: frames[t] for t in range(T)}


def accuracy(z_frames, test_by_time, params):
    """training.py:189-197 (first-index argmax)."""
    ok = tot = 0
    for t, (p, l) in sorted(test_by_time.items()):
        lg = head_logits(z_frames[t], p, params["head.w"], params["head.b"])
        ok += int((lg.argmax(1) == l).sum())
        tot += l.shape[0]
    return ok / tot if tot else None


def adam(params, grads, st, lr=0.01, b1=0.9, b2=0.999, eps=1e-8):
    """training.py:886-900 (sorted key order, in place)."""
    st["step"] += 1
    t = st["step"]
    for k in sorted(params):
        g = grads[k]
        st["m"][k] = b1 * st["m"][k] + (1.0 - b1) * g
        st["v"][k] = b2 * st["v"][k] + (1.0 - b2) * (g * g)
        params[k] -= lr * (st["m"][k] / (1.0 - b1 ** t)) / (np.sqrt(st["v"][k] / (1.0 - b2 ** t)) + eps)


def adam_state(params):
    return {"step": 0, "m": {k: np.zeros_like(v) for k, v in params.items()},
            "v": {k: np.zeros_like(v) for k, v in params.items()}}


# ---------------------------------------------------------------------------
# snapshot-partitioned simulated workers (dist.py:82-589)


@dataclass
class Comm:
    """dist.py:82-122."""
    redistribution_units: int = 0
    all_reduce_scalars: int = 0
    messages: int = 0
    events: list = field(default_factory=list)

    def as_dict(self):
        return {"redistribution_units": self.redistribution_units,
                "all_reduce_scalars": self.all_reduce_scalars,
                "messages": self.messages,
                "alltoall_count": sum(1 for e in self.events if e["kind"] == "alltoall")}


class _Plan:
    """dist.py:125-173."""

    def __init__(self, T, P, nblk, N):
        if P < 1:
            raise OracleConfigError("P >= 1")
        if nblk < 1 or T % nblk:
            raise OracleConfigError("nblk must divide T")
        self.T, self.P, self.nblk, self.bs = T, P, nblk, T // nblk
        if self.bs % P:
            raise OracleConfigError("P must divide bsize")
        if N % P:
            raise OracleConfigError("P must divide N")
        self.ch, self.N, self.NP = self.bs // P, N, N // P

    def owner(self, t):
        return (t % self.bs) // self.ch

    def steps(self, p, b):
        s = b * self.bs + p * self.ch
        return list(range(s, s + self.ch))

    def block(self, b):
        return list(range(b * self.bs, (b + 1) * self.bs))


def _a2a_vertex(frames, plan: _Plan, comm: Comm, phase, b, l):
    """dist.py:176-199."""
    out = {q: {} for q in range(plan.P)}
    units, pairs = 0, set()
    for t in sorted(frames):
        p = plan.owner(t)
        for q in range(plan.P):
            out[q][t] = frames[t][q * plan.NP:(q + 1) * plan.NP]
            if q != p:
                units += plan.NP
                pairs.add((p, q))
    comm.redistribution_units += units
    comm.messages += len(pairs)
    comm.events.append({"kind": "alltoall", "phase": phase, "block": b, "layer": l, "units": units})
    return out


def _a2a_snapshot(rows, plan: _Plan, comm: Comm, phase, b, l):
    """dist.py:202-228."""
    ts = sorted(rows[0])
    for q in range(plan.P):
        if sorted(rows[q]) != ts:
            raise OracleProtocolError("missing chunk")
    frames, units, pairs = {}, 0, set()
    for t in ts:
        p = plan.owner(t)
        for q in range(plan.P):
            if q != p:
                units += rows[q][t].shape[0]
                pairs.add((q, p))
        frames[t] = np.vstack([rows[q][t] for q in range(plan.P)])
    comm.redistribution_units += units
    comm.messages += len(pairs)
    comm.events.append({"kind": "alltoall", "phase": phase, "block": b, "layer": l, "units": units})
    return frames


class _Rank:
    """dist.py:235-458 for cd-gcn / tm-gcn."""

    def __init__(self, q, cfg: Cfg, P: Prepared, params, plan: _Plan, by_time, scale):
        self.q, self.cfg, self.Pd, self.params, self.plan = q, cfg, P, params, plan
        self.by_time, self.scale = by_time, scale
        self.lo, self.hi = q * plan.NP, (q + 1) * plan.NP
        self.skip = cfg.architecture == "cd-gcn"
        self.L = cfg.layers
        self.transfer = Transfer()
        self.grads = {k: np.zeros_like(v) for k, v in params.items()}
        self.state = self._zero()
        self.dstate = self._zero()
        self.trail = [dict() for _ in range(self.L)]
        self.dtrail = [dict() for _ in range(self.L)]
        self.pi = {}

    def _zero(self):
        nr = self.hi - self.lo
        return [(np.zeros((nr, o)), np.zeros((nr, o))) if self.skip else None
                for (_, _, o) in self.cfg.dims()]

    def begin(self, b, keep):
        self.ts = self.plan.steps(self.q, b)
        self.keep = keep
        self.laps = dict(zip(self.ts, stream([self.Pd.laps[t] for t in self.ts], self.transfer)))
        self.x = {}
        self.caches = [dict() for _ in range(self.L)] if keep else None
        self.act = (list(self.pi[b - 1]) if b > 0 else self._zero()) if keep else list(self.state)

    def gcn_forward(self, b, l):
        w = self.params[f"gcn{l}.w"]
        out, gc = {}, {}
        for t in self.ts:
            s = self.Pd.s1[t] if l == 0 else spmm(self.laps[t], self.x[t])
            out[t], gc[t] = gcn_fwd(s, w, self.skip)
        if self.keep:
            self.caches[l]["gcn"] = gc
        return out

    def rnn_forward(self, b, l, rows):
        ts = self.plan.block(b)
        if not self.skip:
            fr = dict(self.trail[l])
            fr.update(rows)
            zs = mprod_fwd(self.Pd.m, self.Pd.window, ts, fr)
            for t in ts[-min(self.Pd.window, len(ts)):]:
                self.trail[l][t] = rows[t]
            return zs
        p = self.params
        ys, st, cache = lstm_fwd(p[f"lstm{l}.wx"], p[f"lstm{l}.wh"], p[f"lstm{l}.b"],
                                 self.act[l], ts, rows)
        self.act[l] = st
        if self.keep:
            self.caches[l]["lstm"] = cache
        return ys

    def set_input(self, b, l, frames):
        self.x = frames
        if l == self.L - 1:
            self.zf = frames

    def block_loss(self, b):
        return loss_sum(self.params, self.zf, self.by_time, self.ts)

    def store_pi(self, b):
        self.state = list(self.act)
        self.pi[b] = list(self.act)

    def loss_grads(self, b):
        dz, dhw, dhb = loss_grads(self.cfg.embed_features, self.params, self.zf, self.by_time,
                                  self.ts, self.scale)
        self.grads["head.w"] += dhw
        self.grads["head.b"] += dhb
        self.dcur = dz

    def rnn_backward(self, b, l, drows):
        ts = self.plan.block(b)
        if not self.skip:
            like = next(iter(drows.values()))
            dy, before = mprod_bwd(self.Pd.m, self.Pd.window, ts, drows, ts[0], like)
            for t in ts:
                if t in self.dtrail[l]:
                    dy[t] += self.dtrail[l].pop(t)
            for t, g in before.items():
                self.dtrail[l][t] = self.dtrail[l][t] + g if t in self.dtrail[l] else g
            return dy
        p = self.params
        dy, dst, (dwx, dwh, db) = lstm_bwd(p[f"lstm{l}.wx"], p[f"lstm{l}.wh"], ts,
                                           self.caches[l]["lstm"], drows, self.dstate[l])
        self.dstate[l] = dst
        self.grads[f"lstm{l}.wx"] += dwx
        self.grads[f"lstm{l}.wh"] += dwh
        self.grads[f"lstm{l}.b"] += db
        return dy

    def gcn_backward(self, b, l, dy):
        w = self.params[f"gcn{l}.w"]
        dw = np.zeros_like(w)
        prev = {}
        for t in self.ts:
            dwt, ds = gcn_bwd(self.caches[l]["gcn"][t], dy[t], w, self.skip)
            dw += dwt
            if l > 0:
                prev[t] = spmm_t(self.laps[t], ds)
        self.grads[f"gcn{l}.w"] += dw
        self.dcur = prev


def distributed_epoch(cfg: Cfg, P: Prepared, by_time, params, workers: int, nblk: int,
                      threads: bool = False, comm: Comm | None = None,
                      transfer: Transfer | None = None):
    """dist.py:505-589 -> (loss, grads, comm, transfer)."""
    plan = _Plan(P.T, workers, nblk, P.N)
    comm = comm if comm is not None else Comm()
    transfer = transfer if transfer is not None else Transfer()
    cnt = total_pairs(by_time)
    scale = (1.0 / cnt) if cnt else 1.0
    ranks = [_Rank(q, cfg, P, params, plan, by_time, scale) for q in range(workers)]
    pool = ThreadPoolExecutor(max_workers=workers) if threads else None

    def run(fn, *args, per=None):
        calls = [(getattr(r, fn), args + ((per[r.q],) if per is not None else ())) for r in ranks]
        if pool is None:
            return [f(*a) for f, a in calls]
        futs = [pool.submit(f, *a) for f, a in calls]
        return [x.result() for x in futs]

    def merge(pieces):
        out = {}
        for d in pieces:
            out.update(d)
        return out

    def own(frames, b):
        return {q: {t: frames[t] for t in plan.steps(q, b)} for q in range(workers)}

    def layers_forward(b, phase):
        for l in range(cfg.layers):
            fr = merge(run("gcn_forward", b, l))
            rows = _a2a_vertex(fr, plan, comm, phase, b, l)
            z = run("rnn_forward", b, l, per=rows)
            fr = _a2a_snapshot({q: z[q] for q in range(workers)}, plan, comm, phase, b, l)
            run("set_input", b, l, per=own(fr, b))

    try:
        from threadpoolctl import threadpool_limits  # BLAS pinned to 1 thread (core.py:195-209)
        blas = threadpool_limits(limits=1)
    except ImportError:  # pragma: no cover
        blas = None
    try:
        tot = 0.0
        for b in range(plan.nblk):
            run("begin", b, False)
            layers_forward(b, "forward")
            for piece, _ in run("block_loss", b):
                tot += piece
            run("store_pi", b)
        loss = tot * scale if cnt else 0.0
        for b in reversed(range(plan.nblk)):
            run("begin", b, True)
            layers_forward(b, "rerun")
            run("loss_grads", b)
            for l in reversed(range(cfg.layers)):
                dz = merge([r.dcur for r in ranks])
                drows = _a2a_vertex(dz, plan, comm, "backward", b, l)
                dy = run("rnn_backward", b, l, per=drows)
                dyf = _a2a_snapshot({q: dy[q] for q in range(workers)}, plan, comm, "backward", b, l)
                run("gcn_backward", b, l, per=own(dyf, b))
        grads = {k: np.sum(np.stack([r.grads[k] for r in ranks]), axis=0) for k in sorted(params)}
        n_scalars = sum(int(np.prod(v.shape)) for v in params.values())
        comm.all_reduce_scalars += n_scalars
        if workers > 1:
            comm.messages += workers - 1
        comm.events.append({"kind": "allreduce", "scalars": n_scalars})
        for r in ranks:
            transfer.add(r.transfer)
    finally:
        if pool is not None:
            pool.shutdown(wait=True)
        if blas is not None:
            blas.unregister()
    return loss, grads, comm, transfer


def train_distributed(cfg: Cfg, P: Prepared, train_bt, test_bt, epochs, seed, workers, nblk,
                      threads=False, lr=0.01):
    """dist.py:592-614 -> (trace, params, comm, transfer)."""
    params = init_params(cfg, seed)
    st = adam_state(params)
    comm, transfer, trace = Comm(), Transfer(), []
    for e in range(1, epochs + 1):
        loss, grads, _, _ = distributed_epoch(cfg, P, train_bt, params, workers, nblk, threads,
                                              comm, transfer)
        adam(params, grads, st, lr)
        acc = accuracy(model_forward(cfg, P, params), test_bt, params)
        trace.append({"epoch": e, "loss": loss, "test_accuracy": acc})
    return trace, params, comm, transfer


_lock = threading.Lock()  # reserved for callers that share an oracle across threads

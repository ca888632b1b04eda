"""Kernel-level drop-ins with the reference's host signatures.

Each function takes/returns numpy (float64) like the reference function it
replaces and runs the corresponding sm_100a kernel on the current device:

* `spmm`, `spmm_transpose` (core.py:142-161): fp64, bit-identical to the
  reference's `np.add.at` accumulation order;
* `normalize_laplacian` (dtdg.py:178-191): fp64 values, bit-identical;
* `diff` (host encode) / `apply` (device rebuild) / `stream_block`
  (delta.py:110-170) with the reference's CorruptDeltaError checks;
* `lstm_block_forward` / `lstm_block_backward` (training.py:370-427) and
  `skip_gcn_fwd_t` / `skip_gcn_bwd_t` (training.py:353-367): the fp32
  training kernels on padded device layouts.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, frame, ptr, query
from .errors import ConfigError, CorruptDeltaError, InputError
from .graph import SparseMatrix
from .params import pad_hidden, pad_input


def _dev():
    if not torch.cuda.is_available():
        raise ConfigError("no CUDA device: this package has no CPU execution path")
    return torch.device("cuda", torch.cuda.current_device())


def _i32(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)


def _f64(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


class _DevCsr:
    def __init__(self, a, dev, with_vals=True):
        n, m = int(a.dim), int(np.asarray(a.vals).shape[0])
        self.n, self.m = n, m
        self.rows = _i32(a.rows, dev) if m else torch.zeros(1, dtype=torch.int32, device=dev)
        self.col = _i32(a.cols, dev) if m else torch.zeros(1, dtype=torch.int32, device=dev)
        self.val = (_f64(a.vals, dev) if m else torch.zeros(1, dtype=torch.float64, device=dev)) \
            if with_vals else None
        self.rowptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
        call("dgnn_rowptr_from_sorted_rows", n, m, ptr(self.rows), ptr(self.rowptr), _lib.stream_handle())

    def transpose(self, dev):
        n, m = self.n, max(self.m, 1)
        t_rowptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
        t_col = torch.empty(m, dtype=torch.int32, device=dev)
        t_val = torch.empty(m, dtype=torch.float64, device=dev) if self.val is not None else None
        st_col = torch.empty(m, dtype=torch.int32, device=dev)
        st_val = torch.empty(m, dtype=torch.float64, device=dev) if self.val is not None else None
        ws = torch.empty(query("dgnn_csr_transpose_workspace", n), dtype=torch.uint8, device=dev)
        call("dgnn_csr_transpose_staged", n, self.m, ptr(self.rowptr), ptr(self.col), ptr(self.val),
             ptr(t_rowptr), ptr(t_col), ptr(t_val), ptr(st_col), ptr(st_val), ptr(ws), ws.numel(),
             _lib.stream_handle())
        return t_rowptr, t_col, t_val


def spmm(a, x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if a.dim != x.shape[0]:
        raise InputError(f"spmm dimension mismatch: {a.dim} vs {x.shape[0]}")
    dev = _dev()
    A = _DevCsr(a, dev)
    f = x.shape[1]
    xd = _f64(x, dev)
    out = torch.zeros(a.dim * max(f, 1), dtype=torch.float64, device=dev)
    call("dgnn_spmm_f64", a.dim, ptr(A.rowptr), ptr(A.col), ptr(A.val), ptr(xd), f, f, ptr(out), f,
         _lib.stream_handle())
    return out[:a.dim * f].view(a.dim, f).cpu().numpy()


def spmm_transpose(a, g: np.ndarray) -> np.ndarray:
    g = np.asarray(g, dtype=np.float64)
    if a.dim != g.shape[0]:
        raise InputError(f"spmm_transpose dimension mismatch: {a.dim} vs {g.shape[0]}")
    dev = _dev()
    A = _DevCsr(a, dev)
    t_rowptr, t_col, t_val = A.transpose(dev)
    f = g.shape[1]
    gd = _f64(g, dev)
    out = torch.zeros(a.dim * max(f, 1), dtype=torch.float64, device=dev)
    call("dgnn_spmm_f64", a.dim, ptr(t_rowptr), ptr(t_col), ptr(t_val), ptr(gd), f, f, ptr(out), f,
         _lib.stream_handle())
    return out[:a.dim * f].view(a.dim, f).cpu().numpy()


def _laplacian_dev(A: _DevCsr, dev, transposed_input=None, a_rowptr=None):
    n = A.n
    cap = A.m + n
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    col = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    v32 = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
    v64 = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
    ws = torch.empty(query("dgnn_laplacian_workspace", n), dtype=torch.uint8, device=dev)
    if transposed_input is None:
        m_rowptr, m_col, m_val, tr = A.rowptr, A.col, A.val, 0
    else:
        (m_rowptr, m_col, m_val), tr = transposed_input, 1
    call("dgnn_laplacian", n, ptr(a_rowptr if a_rowptr is not None else A.rowptr), ptr(m_rowptr), ptr(m_col),
         ptr(m_val), tr, ptr(rp), ptr(col), ptr(v32), ptr(v64), cap, ptr(ws), ws.numel(), _lib.stream_handle())
    return rp, col, v32, v64


def _csr_to_sparse(n, rp, col, val) -> SparseMatrix:
    rp = rp.cpu().numpy().astype(np.int64)
    m = int(rp[-1])
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    return SparseMatrix.from_canonical(n, rows, col[:m].cpu().numpy().astype(np.int64),
                                       val[:m].cpu().numpy())


def normalize_laplacian(a) -> SparseMatrix:
    dev = _dev()
    A = _DevCsr(a, dev)
    rp, col, _, v64 = _laplacian_dev(A, dev)
    return _csr_to_sparse(a.dim, rp, col, v64)


def normalize_laplacian_transpose(a) -> SparseMatrix:
    """normalize_laplacian(a) transposed, built from the CSC of a (the
    operand of the backward SpMM)."""
    dev = _dev()
    A = _DevCsr(a, dev)
    t = A.transpose(dev)
    rp, col, _, v64 = _laplacian_dev(A, dev, transposed_input=t)
    return _csr_to_sparse(a.dim, rp, col, v64)


@dataclass(frozen=True)
class SnapshotDelta:
    """`delta.py:37-54`."""
    dim: int
    ext_prev: np.ndarray
    ext_next: np.ndarray
    values_next: np.ndarray

    @property
    def index_entries(self) -> int:
        return int(self.ext_prev.shape[0] + self.ext_next.shape[0])


def diff(a_i, a_next) -> SnapshotDelta:
    """Three-way split (`delta.py:110-123`) -- host encode, done once at prep
    by the engine."""
    if a_i.dim != a_next.dim:
        raise InputError(f"diff dimension mismatch: {a_i.dim} vs {a_next.dim}")
    d = np.int64(a_i.dim)
    ki = np.asarray(a_i.rows, np.int64) * d + np.asarray(a_i.cols, np.int64)
    kn = np.asarray(a_next.rows, np.int64) * d + np.asarray(a_next.cols, np.int64)
    gone = np.setdiff1d(ki, kn, assume_unique=True)
    new = np.setdiff1d(kn, ki, assume_unique=True)
    return SnapshotDelta(a_i.dim, np.stack([gone // d, gone % d], 1), np.stack([new // d, new % d], 1),
                         np.array(a_next.vals, dtype=np.float64))


def apply(a_i, d: SnapshotDelta) -> SparseMatrix:
    """Device rebuild of the next snapshot (`delta.py:126-146`)."""
    if a_i.dim != d.dim:
        raise InputError(f"apply dimension mismatch: {a_i.dim} vs {d.dim}")
    dev = _dev()
    n = a_i.dim
    A = _DevCsr(a_i, dev, with_vals=False)

    def pairs(p):
        p = np.asarray(p, dtype=np.int64).reshape(-1, 2)
        if p.size and (p.min() < 0 or p.max() >= n):
            raise CorruptDeltaError("delta pair outside the matrix")
        o = np.lexsort((p[:, 1], p[:, 0]))
        p = p[o]
        return _i32(p[:, 0], dev) if p.shape[0] else torch.zeros(1, dtype=torch.int32, device=dev), \
            _i32(p[:, 1], dev) if p.shape[0] else torch.zeros(1, dtype=torch.int32, device=dev), p.shape[0]

    dr, dc, nd = pairs(d.ext_prev)
    ir, ic, ni = pairs(d.ext_next)
    cap = A.m + ni
    nrp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    ncol = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    ws = torch.empty(query("dgnn_csr_apply_delta_workspace", n), dtype=torch.uint8, device=dev)
    status = torch.zeros(4, dtype=torch.int32, device=dev)
    call("dgnn_csr_apply_delta", n, ptr(A.rowptr), ptr(A.col), nd, ptr(dr), ptr(dc), ni, ptr(ir), ptr(ic),
         ptr(nrp), ptr(ncol), cap, ptr(ws), ws.numel(), ptr(status), _lib.stream_handle())
    if int(status[0].item()):
        raise CorruptDeltaError("delta inconsistent with the base snapshot (ext_prev absent or ext_next "
                                "overlapping the common set)")
    vals = np.asarray(d.values_next, dtype=np.float64)
    m = int(nrp[-1].item())
    if m != vals.shape[0]:
        raise CorruptDeltaError(f"value count {vals.shape[0]} does not match reconstructed index count {m}")
    rp = nrp.cpu().numpy().astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    cols = ncol[:m].cpu().numpy().astype(np.int64)
    keep = vals != 0.0                     # from_entries drops exact zeros (core.py:80)
    return SparseMatrix.from_canonical(n, rows[keep], cols[keep], vals[keep])


def stream_block(snapshots, ledger):
    """`delta.py:149-170`: first snapshot forwarded, the rest rebuilt on
    device from their deltas, charging the ledger as the reference does."""
    snapshots = list(snapshots)
    if not snapshots:
        raise InputError("stream_block needs a non-empty snapshot run")

    def gen():
        prev = snapshots[0]
        ledger.charge_full(prev)
        yield prev
        for nxt in snapshots[1:]:
            d = diff(prev, nxt)
            ledger.charge_delta(d)
            prev = apply(prev, d)
            yield prev

    return gen()


def naive_cost(snapshots):
    from .api import TransferLedger
    led = TransferLedger()
    for s in snapshots:
        led.charge_full(s)
    return led


# ---------------------------------------------------------------------------
# temporal / graph-convolution cells on padded device layouts


def _pad_rows(a: np.ndarray, width: int, dev) -> torch.Tensor:
    out = np.zeros((a.shape[0], width), dtype=np.float32)
    out[:, :a.shape[1]] = a
    return torch.from_numpy(out).to(dev)


def _lstm_weights(wx, wh, b, dev):
    fin, four_h = wx.shape
    H = four_h // 4
    hp = pad_hidden(H)
    kx = (fin + 3) // 4 * 4
    K = kx + hp
    wc = np.zeros((K, 4 * hp), dtype=np.float32)
    bb = np.zeros(4 * hp, dtype=np.float32)
    for g in range(4):
        wc[:fin, g * hp:g * hp + H] = wx[:, g * H:(g + 1) * H]
        wc[kx:kx + H, g * hp:g * hp + H] = wh[:, g * H:(g + 1) * H]
        bb[g * hp:g * hp + H] = b[g * H:(g + 1) * H]
    wct = np.ascontiguousarray(wc.T)
    return H, hp, kx, torch.from_numpy(wc).to(dev), torch.from_numpy(wct).to(dev), torch.from_numpy(bb).to(dev)


def _tile(t: torch.Tensor, w: int, to_blocked: bool) -> torch.Tensor:
    """rows x w row-major <-> tile-blocked (the LSTM cache layout, see
    include/dgnn_b200.h)."""
    out = torch.empty_like(t)
    call("dgnn_tile_block" if to_blocked else "dgnn_tile_unblock", 1, t.shape[0], w, ptr(t), ptr(out),
         _lib.stream_handle())
    return out


def tc_gemm(a: np.ndarray, w: np.ndarray) -> np.ndarray:
    """a @ w.T on the tcgen05 3xTF32 mainloop (self-test of the tensor-core
    path); a: m x k, w: n x k with n in {64, 128, 256}, k % 4 == 0."""
    dev = _dev()
    m, k = a.shape
    n = w.shape[0]
    ad = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)
    wd = torch.from_numpy(np.ascontiguousarray(w, np.float32)).to(dev)
    img = torch.zeros(query("dgnn_tc_weight_image_bytes", n, k) // 4, dtype=torch.float32, device=dev)
    st = _lib.stream_handle()
    call("dgnn_tc_weight_image", n, k, ptr(wd), k, ptr(img), st)
    out = torch.zeros(m, n, dtype=torch.float32, device=dev)
    call("dgnn_tc_gemm_test", m, n, k, ptr(ad), k, ptr(img), ptr(out), n, st)
    return out.double().cpu().numpy()


def gcn_forward(n: int, rowptr: np.ndarray | None, col: np.ndarray | None, val: np.ndarray | None,
                x: np.ndarray, w: np.ndarray, skip: bool, tensor_cores: bool = True):
    """Test hook of K3 `dgnn_gcn_forward`: s = (A x if rowptr is given else x),
    r = relu([s, s w]) (skip) | relu(s w); fp32.  Returns (s, r)."""
    dev = _dev()
    fp, hp = w.shape
    xd = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dev)
    wd = torch.from_numpy(np.ascontiguousarray(w, np.float32)).to(dev)
    rw = fp + hp if skip else hp
    s_out = torch.full((n, fp), np.nan, dtype=torch.float32, device=dev)
    r_out = torch.full((n, rw), np.nan, dtype=torch.float32, device=dev)
    st = _lib.stream_handle()
    agg = rowptr is not None
    rp = _i32(rowptr, dev) if agg else None
    cd = _i32(col if len(col) else np.zeros(1), dev) if agg else None
    vd = torch.from_numpy(np.ascontiguousarray(val if len(val) else np.zeros(1), np.float32)).to(dev) if agg else None
    call("dgnn_set_gcn_tensor_cores", int(tensor_cores))
    try:
        call("dgnn_gcn_forward", n, ptr(rp), ptr(cd), ptr(vd), _lib.frame(xd, fp), fp, ptr(wd), hp, int(skip),
             _lib.frame(s_out, fp), _lib.frame(r_out, rw), st)
    finally:
        call("dgnn_set_gcn_tensor_cores", 1)
    return s_out.cpu().numpy(), r_out.cpu().numpy()


def spmm_f32(rowptr: np.ndarray, col: np.ndarray, val: np.ndarray, x: np.ndarray, tensor_cores: bool = True):
    """Test hook of `dgnn_spmm_f32` (fp32 CSR SpMM, core.py:142-152 order):
    the K3 gather pipeline (default) or the SIMT kernel."""
    dev = _dev()
    n, f = rowptr.shape[0] - 1, x.shape[1]
    xd = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dev)
    out = torch.full((n, f), np.nan, dtype=torch.float32, device=dev)
    rp = _i32(rowptr, dev)
    cd = _i32(col if len(col) else np.zeros(1), dev)
    vd = torch.from_numpy(np.ascontiguousarray(val if len(val) else np.zeros(1), np.float32)).to(dev)
    call("dgnn_set_gcn_tensor_cores", int(tensor_cores))
    try:
        call("dgnn_spmm_f32", n, ptr(rp), ptr(cd), ptr(vd), _lib.frame(xd, f), f, _lib.frame(out, f),
             _lib.stream_handle())
    finally:
        call("dgnn_set_gcn_tensor_cores", 1)
    return out.cpu().numpy()


def gcn_backward(dr: np.ndarray, r: np.ndarray, s: np.ndarray, w: np.ndarray, skip: bool,
                 tensor_cores: bool = True, slabs: int = 0, rows_ds: bool = True):
    """Test hook of K4's row part and weight gradient (`dgnn_gcn_backward_rows`,
    `dgnn_gcn_weight_grad`, training.py:347-350, 359-367): with dpre =
    dr (.) [r > 0] and dq = dpre[:, F:] (skip) | dpre, returns (ds, gw) =
    (dpre[:, :F] + dq w^T (skip) | dq w^T, s^T dq) -- ds None when rows_ds is
    False.  `slabs` > 0 passes the inputs as split (owner-layout) frames."""
    dev = _dev()
    n = dr.shape[0]
    fp, hp = w.shape
    rw = dr.shape[1]

    def dev_frame(a, wdt):
        t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)
        if slabs <= 0:
            return t, _lib.frame(t, wdt)
        rps = -(-n // slabs)
        buf = torch.full((slabs, rps + 3, wdt), np.nan, dtype=torch.float32, device=dev)
        for q in range(slabs):
            part = t[q * rps:(q + 1) * rps]
            buf[q, :part.shape[0]] = part
        return buf, _lib.frame(buf, wdt, rps, (rps + 3) * wdt)

    keep = []
    drd, fdr = dev_frame(dr, rw)
    rd, fr = dev_frame(r, rw)
    sd, fs = dev_frame(s, fp)
    keep += [drd, rd, sd]
    wd = torch.from_numpy(np.ascontiguousarray(w, np.float32)).to(dev)
    ds = torch.full((n, fp), np.nan, dtype=torch.float32, device=dev)
    gw = torch.zeros(fp * hp, dtype=torch.float64, device=dev)
    ws = torch.empty(query("dgnn_gcn_weight_grad_workspace", fp, hp), dtype=torch.uint8, device=dev)
    st = _lib.stream_handle()
    call("dgnn_set_gcn_tensor_cores", int(tensor_cores))
    try:
        call("dgnn_gcn_weight_grad", n, fs, fdr, fr, fp, hp, int(skip), ptr(gw), ptr(ws), ws.numel(), st)
        if rows_ds:
            call("dgnn_gcn_backward_rows", n, fdr, fr, fp, ptr(wd), hp, int(skip), _lib.frame(ds, fp), st)
    finally:
        call("dgnn_set_gcn_tensor_cores", 1)
    return (ds.cpu().numpy() if rows_ds else None), gw.view(fp, hp).cpu().numpy()


def lstm_weight_grad_tc(x: np.ndarray, h_out: np.ndarray, h0: np.ndarray, dz: np.ndarray, np_rows: int,
                        variant: str = "tc"):
    """Tensor-core block weight gradient (test hook of dgnn_lstm_weight_grad_tc,
    variant "ts": dgnn_lstm_weight_grad_ts): returns (sum_r xcat[r]^T dz[r]
    as (kx+hp) x 4hp, sum_r dz[r]) in fp64."""
    dev = _dev()
    rows, kx = x.shape
    hp = h0.shape[1]
    t = [torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev) for a in (x, h_out, h0, dz)]
    blk = torch.empty_like(t[3])     # dz is tile-blocked per step of np_rows rows
    call("dgnn_tile_block", rows // np_rows, np_rows, 4 * hp, ptr(t[3]), ptr(blk), _lib.stream_handle())
    t[3] = blk
    gw = torch.zeros((kx + hp) * 4 * hp, dtype=torch.float64, device=dev)
    gb = torch.zeros(4 * hp, dtype=torch.float64, device=dev)
    ws = torch.empty(query("dgnn_lstm_weight_grad_tc_workspace", kx, hp), dtype=torch.uint8, device=dev)
    call(f"dgnn_lstm_weight_grad_{variant}", rows, np_rows, kx, hp, ptr(t[0]), kx, ptr(t[1]), ptr(t[2]),
         ptr(t[3]), ptr(gw), ptr(gb), ptr(ws), ws.numel(), _lib.stream_handle())
    return gw.view(kx + hp, 4 * hp).cpu().numpy(), gb.cpu().numpy()


def lstm_block_forward(cell, state_in, ts, xs: dict, tensor_cores: bool = True, warp_specialized: bool = True):
    """fp32 device LSTM over a block (training.py:370-391).  Returns
    (ys, (h, c), cache) with a device cache for lstm_block_backward."""
    dev = _dev()
    wx, wh, b = (np.asarray(cell.wx), np.asarray(cell.wh), np.asarray(cell.b))
    H, hp, kx, wc, wct, bb = _lstm_weights(wx, wh, b, dev)
    img = None
    if tensor_cores:
        img = torch.zeros(query("dgnn_tc_weight_image_bytes", 4 * hp, kx + hp) // 4, dtype=torch.float32,
                          device=dev)
        call("dgnn_tc_weight_image", 4 * hp, kx + hp, ptr(wct), kx + hp, ptr(img), _lib.stream_handle())
    h0, c0 = state_in
    rows = h0.shape[0]
    st = _lib.stream_handle()
    h = _pad_rows(np.asarray(h0), hp, dev)
    c = _tile(_pad_rows(np.asarray(c0), hp, dev), hp, True)
    cache = {"h0": h, "c0": c, "x": [], "h": [], "c": [], "g": [], "H": H, "hp": hp, "kx": kx,
             "wc": wc, "wct": wct, "rows": rows}
    ys = {}
    for t in ts:
        x = _pad_rows(np.asarray(xs[t]), kx, dev)
        hn = torch.zeros(rows, hp, device=dev)
        cn = torch.zeros(rows, hp, device=dev)
        g = torch.zeros(rows, 4 * hp, device=dev)
        if img is not None:
            call("dgnn_lstm_forward_step_ws" if (warp_specialized and hp <= 64) else "dgnn_lstm_forward_step_tc", rows, kx, hp, ptr(x), kx, ptr(h), ptr(c), ptr(img), ptr(bb),
                 ptr(hn), ptr(cn), ptr(g), st)
        else:
            call("dgnn_lstm_forward_step", rows, kx, hp, ptr(x), kx, ptr(h), ptr(c), ptr(wc), ptr(bb), ptr(hn),
                 ptr(cn), ptr(g), st)
        cache["x"].append(x)
        cache["h"].append(hn)
        cache["c"].append(cn)
        cache["g"].append(g)
        h, c = hn, cn
        ys[t] = hn[:, :H].double().cpu().numpy()
    c = _tile(c, hp, False)
    return ys, (h[:, :H].double().cpu().numpy(), c[:, :H].double().cpu().numpy()), cache


def lstm_block_backward(cell, ts, cache, dys: dict, dstate_out, tensor_cores: bool = True,
                        warp_specialized: bool = True):
    """fp32 device BPTT over a block (training.py:394-427)."""
    dev = _dev()
    H, hp, kx, rows = cache["H"], cache["hp"], cache["kx"], cache["rows"]
    st = _lib.stream_handle()
    bimg = None
    if tensor_cores and hp <= 64 and kx + hp <= 256:
        nb = (kx + hp + 15) // 16 * 16
        bimg = torch.zeros(query("dgnn_tc_weight_image_bytes", nb, 4 * hp) // 4, dtype=torch.float32, device=dev)
        call("dgnn_tc_weight_image_ex", nb, kx + hp, 4 * hp, ptr(cache["wc"]), 4 * hp, hp, ptr(bimg), st)
    dh = _pad_rows(np.asarray(dstate_out[0]), hp, dev)
    dc = _tile(_pad_rows(np.asarray(dstate_out[1]), hp, dev), hp, True)
    K4 = 4 * hp
    gwc = torch.zeros((kx + hp) * K4, dtype=torch.float64, device=dev)
    gb = torch.zeros(K4, dtype=torch.float64, device=dev)
    ws = torch.empty(query("dgnn_gemm_tn_workspace", max(kx, hp), K4), dtype=torch.uint8, device=dev)
    dxs = {}
    B = len(ts)
    dzs = [None] * B
    for i in reversed(range(B)):
        t = ts[i]
        dy = _pad_rows(np.asarray(dys[t]), hp, dev)
        c_prev = cache["c"][i - 1] if i > 0 else cache["c0"]
        dz = torch.zeros(rows, K4, device=dev)
        dx = torch.zeros(rows, kx, device=dev)
        dh2 = torch.zeros(rows, hp, device=dev)
        dc2 = torch.zeros(rows, hp, device=dev)
        if bimg is not None:
            dz.copy_(cache["g"][i])      # the tensor-core step writes dz over the gate cache
            call("dgnn_lstm_backward_step_ws" if warp_specialized else "dgnn_lstm_backward_step_tc", rows, kx, hp,
                 ptr(dy), ptr(dh), ptr(dc), ptr(dz), ptr(c_prev),
                 ptr(cache["c"][i]), ptr(bimg), ptr(dx), kx, ptr(dh2), ptr(dc2), st)
        else:
            call("dgnn_lstm_backward_step", rows, kx, hp, ptr(dy), ptr(dh), ptr(dc), ptr(cache["g"][i]),
                 ptr(c_prev), ptr(cache["c"][i]), ptr(cache["wct"]), ptr(dz), ptr(dx), kx, ptr(dh2), ptr(dc2), st)
        h_prev = cache["h"][i - 1] if i > 0 else cache["h0"]
        if bimg is not None and hp >= 32:
            dzs[i] = dz
        else:
            dzr = _tile(dz, K4, False)
            call("dgnn_gemm_tn", rows, kx, K4, ptr(cache["x"][i]), kx, ptr(dzr), K4, ptr(gwc), K4, ptr(gb),
                 ptr(ws), ws.numel(), st)
            call("dgnn_gemm_tn", rows, hp, K4, ptr(h_prev), hp, ptr(dzr), K4, ptr(gwc[kx * K4:]), K4, None,
                 ptr(ws), ws.numel(), st)
        fin = np.asarray(cell.wx).shape[0]
        dxs[t] = dx[:, :fin].double().cpu().numpy()
        dh, dc = dh2, dc2
    if bimg is not None and hp >= 32:
        # one tensor-core pass over all (step, row) pairs of the block
        xs_all = torch.cat(cache["x"][:B]).contiguous()
        hs_all = torch.cat(cache["h"][:B]).contiguous()
        dz_all = torch.cat(dzs).contiguous()
        wsd = torch.empty(query("dgnn_lstm_weight_grad_tc_workspace", kx, hp), dtype=torch.uint8, device=dev)
        call("dgnn_lstm_weight_grad_tc", B * rows, rows, kx, hp, ptr(xs_all), kx, ptr(hs_all), ptr(cache["h0"]),
             ptr(dz_all), ptr(gwc), ptr(gb), ptr(wsd), wsd.numel(), st)
    g = gwc.view(kx + hp, K4).cpu().numpy()
    gbv = gb.cpu().numpy()
    fin = np.asarray(cell.wx).shape[0]
    dwx = np.zeros((fin, 4 * H))
    dwh = np.zeros((H, 4 * H))
    db = np.zeros(4 * H)
    for gi in range(4):
        dwx[:, gi * H:(gi + 1) * H] = g[:fin, gi * hp:gi * hp + H]
        dwh[:, gi * H:(gi + 1) * H] = g[kx:kx + H, gi * hp:gi * hp + H]
        db[gi * H:(gi + 1) * H] = gbv[gi * hp:gi * hp + H]
    dc = _tile(dc, hp, False)
    return dxs, (dh[:, :H].double().cpu().numpy(), dc[:, :H].double().cpu().numpy()), \
        {"wx": dwx, "wh": dwh, "b": db}

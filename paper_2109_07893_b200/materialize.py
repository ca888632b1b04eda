"""Graph-difference snapshot materialisation.

Host side (`SnapshotEncoding`, built once per graph -- the encoding is
input-static, so the reference's per-pass `diff` (`delta.py:110-123`,
recomputed inside `stream_block` every pass) becomes a one-time prep):

* full snapshot t: sorted (row, col) int32 pairs of the raw adjacency A_t;
* delta t (t >= 1): ext_prev / ext_next of A_{t-1} -> A_t as sorted pairs;
* values (fp64) only when A is not unit-valued (value-carrying mode, like
  the reference which always ships `values_next`); unit-valued graphs ship
  structure only and the device recomputes the Laplacian values bit-exactly.

The reference streams the normalised Laplacians (`dist.py:308-312`); the
ledger counters it would charge for them (index / value entries of Ahat) are
computed exactly here at prep so `TransferLedger` stays reference-equivalent,
next to the real bytes this package moves.

Device side (`Materializer`): per pass and per owned chunk of a checkpoint
block, the first snapshot arrives in full and the rest as deltas (pinned
host -> HBM `cudaMemcpyAsync` on a copy stream), and kernels on a graph
stream rebuild CSR(A_t) (K1), transpose it, and build CSR(Ahat_t) and
CSR(Ahat_t^T) with fp64 values (K2) -- overlapped with the layer-0 compute,
which does not need the graph (its aggregation is precomputed).
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, query
from .errors import CorruptDeltaError, InputError

# priority of the graph-rebuild stream (-1: ahead of the compute stream's
# kernels when both have work queued)
GRAPH_PRIORITY = int(os.environ.get("DGNN_GRAPH_PRIORITY", "-1"))


def _lap_keys(n: int, rows: np.ndarray, cols: np.ndarray, vals: np.ndarray | None) -> np.ndarray:
    """Sorted int64 keys of normalize_laplacian(A) (dtdg.py:178-191), i.e. the
    structure of A plus the diagonal, minus entries whose value is exactly 0."""
    keys = rows * np.int64(n) + cols
    diag = np.arange(n, dtype=np.int64) * (n + 1)
    if vals is None:                                   # unit values: nothing can vanish
        return np.union1d(keys, diag)
    deg = np.bincount(rows, minlength=n).astype(np.float64)
    isq = 1.0 / np.sqrt(1.0 + deg)
    v = (vals * isq[rows]) * isq[cols]
    on_diag = rows == cols
    dvals = isq * isq                                  # identity term
    dsum = dvals.copy()
    dsum[rows[on_diag]] = v[on_diag] + dvals[rows[on_diag]]
    off = keys[(~on_diag) & (v != 0.0)]
    dk = diag[dsum != 0.0]
    return np.union1d(off, dk)


@dataclass
class ChunkPlan:
    ts: list
    full_range: tuple      # (offset, count) int32 elements in the full region
    delta_range: tuple     # (offset, count) int32 elements in the delta region
    val_range: tuple       # (offset, count) fp64 elements (value-carrying only)


class SnapshotEncoding:
    """Pinned host encoding of a dynamic graph (see module docstring)."""

    def __init__(self, graph, pin: bool = True, smooth=None):
        """`smooth` = (M matrix, window <= 2): `graph` is the raw, unit-valued
        graph of a tm-gcn run whose M-smoothed snapshots are rebuilt on the
        device; the ledger counts are those of the smoothed Laplacians."""
        n = int(graph.num_vertices)
        T = int(graph.num_timesteps)
        if n >= 2 ** 31 - 1:
            raise InputError("vertex ids must fit int32")
        self.n, self.T = n, T
        snaps = graph.snapshots
        rows = [np.asarray(s.rows, np.int64) for s in snaps]
        cols = [np.asarray(s.cols, np.int64) for s in snaps]
        vals = [np.asarray(s.vals, np.float64) for s in snaps]
        self.unit = all(bool(np.all(v == 1.0)) for v in vals)
        keys = [r * np.int64(n) + c for r, c in zip(rows, cols)]
        for t, k in enumerate(keys):
            if k.size > 1 and not np.all(k[1:] > k[:-1]):
                raise InputError(f"snapshot {t} is not canonical (sorted, duplicate-free)")
        self.nnz = np.array([k.shape[0] for k in keys], dtype=np.int64)

        # full region: [rows_t | cols_t] per t
        full_off = np.zeros(T + 1, dtype=np.int64)
        full_off[1:] = np.cumsum(2 * self.nnz)
        # delta region: [del_r | del_c | ins_r | ins_c] per t >= 1
        self.n_del = np.zeros(T, dtype=np.int64)
        self.n_ins = np.zeros(T, dtype=np.int64)
        deltas = [None]
        for t in range(1, T):
            gone = np.setdiff1d(keys[t - 1], keys[t], assume_unique=True)
            new = np.setdiff1d(keys[t], keys[t - 1], assume_unique=True)
            self.n_del[t], self.n_ins[t] = gone.shape[0], new.shape[0]
            deltas.append((gone, new))
        delta_off = np.zeros(T + 1, dtype=np.int64)
        delta_off[1:] = np.cumsum(2 * (self.n_del + self.n_ins))
        self.full_off, self.delta_off = full_off, delta_off
        val_off = np.zeros(T + 1, dtype=np.int64)
        val_off[1:] = np.cumsum(self.nnz)
        self.val_off = val_off

        full = np.empty(int(full_off[-1]), dtype=np.int32)
        for t in range(T):
            o, m = int(full_off[t]), int(self.nnz[t])
            full[o:o + m] = rows[t]
            full[o + m:o + 2 * m] = cols[t]
        dl = np.empty(int(delta_off[-1]), dtype=np.int32)
        for t in range(1, T):
            gone, new = deltas[t]
            o = int(delta_off[t])
            a, b = gone.shape[0], new.shape[0]
            dl[o:o + a] = gone // n
            dl[o + a:o + 2 * a] = gone % n
            dl[o + 2 * a:o + 2 * a + b] = new // n
            dl[o + 2 * a + b:o + 2 * a + 2 * b] = new % n
        self.full = torch.from_numpy(full)
        self.delta = torch.from_numpy(dl)
        self.vals = None if self.unit else torch.from_numpy(np.concatenate(vals) if vals else np.zeros(0))
        if pin and torch.cuda.is_available():
            self.full = self.full.pin_memory()
            self.delta = self.delta.pin_memory()
            if self.vals is not None:
                self.vals = self.vals.pin_memory()

        # reference-equivalent ledger counts for the Laplacians (delta.py:75-84)
        self.nnz_hat = np.zeros(T, dtype=np.int64)
        self.dhat = np.zeros(T, dtype=np.int64)
        self.smooth = None
        if smooth is not None:
            if not self.unit or smooth[1] > 2:
                raise InputError("device smoothing needs a unit-valued raw graph and window <= 2")
            self.smooth = (np.asarray(smooth[0], np.float64), int(smooth[1]))
            self._smoothed_counts(keys)
        elif self.unit:
            # Ahat = A + I structurally and nothing can cancel: the diagonal is
            # always present, so diagonal entries of the A-delta do not change Ahat
            for t in range(T):
                self.nnz_hat[t] = self.nnz[t] + n - int(np.count_nonzero(rows[t] == cols[t]))
            for t in range(1, T):
                gone, new = deltas[t]
                off = int(np.count_nonzero(gone // n != gone % n) + np.count_nonzero(new // n != new % n))
                self.dhat[t] = off
        else:
            hat = [_lap_keys(n, rows[t], cols[t], vals[t]) for t in range(T)]
            self.nnz_hat = np.array([h.shape[0] for h in hat], dtype=np.int64)
            for t in range(1, T):
                self.dhat[t] = (np.setdiff1d(hat[t - 1], hat[t], assume_unique=True).shape[0]
                                + np.setdiff1d(hat[t], hat[t - 1], assume_unique=True).shape[0])
        self.cap_a = int(max(1, self.nnz.max()))
        self.cap_hat = int(max(1, self.nnz_hat.max()))

    def _smoothed_counts(self, keys) -> None:
        """nnz of A~_t (union of the window's structures: positive weights,
        unit values -- nothing cancels), and the ledger counts of its
        Laplacian L_t = A~_t + I: nnz_hat = |L_t|, dhat = |L_{t-1} xor L_t|.
        Sorted-key set algebra in torch (on the GPU when there is one)."""
        n, T = self.n, self.T
        dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
        diag = torch.arange(n, dtype=torch.int64, device=dev) * (n + 1)
        w = self.smooth[1]
        self.nnz_sm = np.zeros(T, dtype=np.int64)
        prev_k, prev_l = None, None
        for t in range(T):
            k = torch.from_numpy(np.ascontiguousarray(keys[t])).to(dev)
            sm = torch.unique(torch.cat([prev_k, k])) if (prev_k is not None and w == 2) else k
            lap = torch.unique(torch.cat([sm, diag]))
            self.nnz_sm[t] = sm.numel()
            self.nnz_hat[t] = lap.numel()
            if prev_l is not None:
                pos = torch.searchsorted(prev_l, lap).clamp_(max=prev_l.numel() - 1)
                common = int((prev_l[pos] == lap).sum().item())
                self.dhat[t] = prev_l.numel() + lap.numel() - 2 * common
            prev_k, prev_l = k, lap

    # -- incremental construction from device keys (synth.device_churn_graph)
    @classmethod
    def empty(cls, n: int, T: int) -> "SnapshotEncoding":
        """An encoding filled step by step with `add_step` (unit-valued
        graphs given as sorted device keys row * n + col and their graph
        differences), then `finish`."""
        self = cls.__new__(cls)
        self.n, self.T, self.unit = int(n), int(T), True
        self.nnz = np.zeros(T, dtype=np.int64)
        self.n_del = np.zeros(T, dtype=np.int64)
        self.n_ins = np.zeros(T, dtype=np.int64)
        self.nnz_hat = np.zeros(T, dtype=np.int64)
        self.dhat = np.zeros(T, dtype=np.int64)
        self._full_parts, self._delta_parts = [], []
        self.vals = None
        return self

    def add_step(self, t: int, keys, dropped=None, inserted=None) -> None:
        import torch as _t
        n = self.n
        r, c = keys // n, keys % n
        self.nnz[t] = keys.numel()
        self.nnz_hat[t] = keys.numel() + n - int((r == c).sum().item())
        self._full_parts.append(_t.cat([r, c]).to(_t.int32).cpu())
        if t > 0:
            self.n_del[t], self.n_ins[t] = dropped.numel(), inserted.numel()
            self.dhat[t] = int(((dropped // n) != (dropped % n)).sum().item()
                               + ((inserted // n) != (inserted % n)).sum().item())
            self._delta_parts.append(_t.cat([dropped // n, dropped % n, inserted // n, inserted % n])
                                     .to(_t.int32).cpu())

    def finish(self, pin: bool = True) -> "SnapshotEncoding":
        T = self.T
        self.full_off = np.zeros(T + 1, dtype=np.int64)
        self.full_off[1:] = np.cumsum(2 * self.nnz)
        self.delta_off = np.zeros(T + 1, dtype=np.int64)
        self.delta_off[1:] = np.cumsum(2 * (self.n_del + self.n_ins))
        self.val_off = np.zeros(T + 1, dtype=np.int64)
        self.val_off[1:] = np.cumsum(self.nnz)
        self.full = torch.cat(self._full_parts) if self._full_parts else torch.zeros(0, dtype=torch.int32)
        self.delta = torch.cat(self._delta_parts) if self._delta_parts else torch.zeros(0, dtype=torch.int32)
        del self._full_parts, self._delta_parts
        if pin and torch.cuda.is_available():
            self.full = self.full.pin_memory()
            self.delta = self.delta.pin_memory()
        self.cap_a = int(max(1, self.nnz.max()))
        self.cap_hat = int(max(1, self.nnz_hat.max()))
        return self

    # -- accounting ---------------------------------------------------------
    def chunk(self, ts) -> ChunkPlan:
        t0, t1 = ts[0], ts[-1]
        if list(ts) != list(range(t0, t1 + 1)):
            raise InputError("a streamed chunk must be a contiguous run of timesteps")
        fr = (int(self.full_off[t0]), int(2 * self.nnz[t0]))
        dr = (int(self.delta_off[t0 + 1]), int(self.delta_off[t1 + 1] - self.delta_off[t0 + 1]))
        vr = (int(self.val_off[t0]), int(self.val_off[t1 + 1] - self.val_off[t0]))
        return ChunkPlan(list(ts), fr, dr, vr)

    def chunk_bytes(self, ts) -> int:
        c = self.chunk(ts)
        b = 4 * (c.full_range[1] + c.delta_range[1])
        if not self.unit:
            b += 8 * c.val_range[1]
        return b

    def full_bytes(self, ts) -> int:
        """Bytes if every snapshot of the chunk travelled in full (same encoding)."""
        b = sum(8 * int(self.nnz[t]) for t in ts)
        if not self.unit:
            b += sum(8 * int(self.nnz[t]) for t in ts)
        return b

    def charge(self, ledger, ts) -> None:
        """Reference TransferLedger charges of stream_block over the
        chunk's Laplacians (delta.py:75-84, 161-167)."""
        t0 = ts[0]
        ledger.index_entries_sent += int(self.nnz_hat[t0])
        ledger.value_entries_sent += int(self.nnz_hat[t0])
        ledger.snapshots_full += 1
        for t in ts[1:]:
            ledger.index_entries_sent += int(self.dhat[t])
            ledger.value_entries_sent += int(self.nnz_hat[t])
            ledger.snapshots_delta += 1


@dataclass
class LapSlot:
    """CSR of Ahat_t and of Ahat_t^T for one materialised timestep."""
    rowptr: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor
    t_rowptr: torch.Tensor
    t_col: torch.Tensor
    t_val: torch.Tensor
    val64: torch.Tensor | None = None
    t_val64: torch.Tensor | None = None
    a_rowptr: torch.Tensor | None = None   # raw CSR of A_t (valid until the next rebuild)
    a_t_rowptr: torch.Tensor | None = None
    t: int = -1


class Materializer:
    """Device-side rebuild of the snapshots a rank owns, chunk by chunk."""

    def __init__(self, enc: SnapshotEncoding, device, slots: int, resident: bool = False,
                 with_f64: bool = False, sets: int = 1, graph_stream=None):
        self.enc = enc
        self.device = torch.device(device)
        n = enc.n
        i32 = dict(dtype=torch.int32, device=self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        f32 = dict(dtype=torch.float32, device=self.device)
        self.resident = resident
        self.copy_stream = torch.cuda.Stream(device=self.device)
        # high priority: the rebuild kernels take SMs as soon as they free up, so
        # a graph-bound pass (large value-carrying graphs) is not starved by
        # the compute stream's persistent kernels
        self.graph_stream = graph_stream if graph_stream is not None else \
            torch.cuda.Stream(device=self.device, priority=GRAPH_PRIORITY)
        # encoded input on device: everything (resident) or a chunk-sized staging area
        if resident:
            self.full_dev = enc.full.to(self.device)
            self.delta_dev = enc.delta.to(self.device)
            self.vals_dev = None if enc.unit else enc.vals.to(self.device)
        else:
            self.full_dev = torch.empty(int(2 * enc.nnz.max()) + 1, **i32)
            self.delta_dev = torch.empty(int(enc.delta_off[-1]) + 1, **i32)
            self.vals_dev = None if enc.unit else torch.empty(int(enc.val_off[-1]) + 1, **f64)
        cap_a, cap_h = enc.cap_a, enc.cap_hat
        # M-smoothing on the device (tm-gcn, window <= 2, unit raw graph): the
        # rebuilt raw A_{t-1}, A_t are merged into A~_t, which then goes
        # through the transpose and the Laplacian like a value-carrying graph
        self.smooth = getattr(enc, "smooth", None)
        cap_g = 2 * cap_a if self.smooth is not None else cap_a      # the graph the Laplacian reads
        valued = (not enc.unit) or self.smooth is not None
        self.a_rowptr = [torch.empty(n + 1, **i32) for _ in range(2)]
        self.a_col = [torch.empty(cap_a, **i32) for _ in range(2)]
        self.at_rowptr = torch.empty(n + 1, **i32)
        self.at_col = torch.empty(cap_g, **i32)
        self.stage_col = torch.empty(cap_g, **i32)
        self.at_val = torch.empty(cap_g, **f64) if valued else None
        self.stage_val = torch.empty(cap_g, **f64) if valued else None
        if self.smooth is not None:
            self.sm_rowptr = torch.empty(n + 1, **i32)
            self.sm_col = torch.empty(cap_g, **i32)
            self.sm_val = torch.empty(cap_g, **f64)
            self.zero_rowptr = torch.zeros(n + 1, **i32)
            self.ws_merge = torch.empty(query("dgnn_csr_weighted_merge_workspace", n, cap_a), dtype=torch.uint8,
                                        device=self.device)
        self.ws_apply = torch.empty(query("dgnn_csr_apply_delta_workspace", n), dtype=torch.uint8,
                                    device=self.device)
        self.ws_tr = torch.empty(query("dgnn_csr_transpose_workspace", n), dtype=torch.uint8,
                                 device=self.device)
        self.ws_lap = torch.empty(query("dgnn_laplacian_workspace", n), dtype=torch.uint8,
                                  device=self.device)
        self.status = torch.zeros(4, **i32)
        # `sets` independent slot sets: with two, the next block's graph is
        # rebuilt on the graph stream while the current block computes
        self.sets = []
        self.ready_sets = []
        self.nslots, self.with_f64 = slots, with_f64
        self.add_sets(sets)
        self.slots = self.sets[0]
        self.bytes_h2d = 0            # bytes this materialiser copied host -> device
        self.bytes_full_equiv = 0     # full-snapshot bytes of every pass consumed (reference schedule)
        self.bytes_full_built = 0     # full-snapshot bytes of every chunk actually built (like for like)
        self.builds = []              # (ts, bytes copied, head rebuilt from a delta) per counted build
        self.ready = torch.cuda.Event()
        self.raw_t = -1               # timestep whose raw CSR sits in a_rowptr[cur] / a_col[cur]
        self.cur = 0
        # when a list: (start event, end event, bytes) of every chunk's H2D copies (PCIe timing)
        self.copy_log = None

    def materialize(self, ts, ledger=None, count_bytes: bool = True, set_idx: int = 0, after=None,
                    head_prev=None, consume: bool = True, handoff=None):
        """Rebuild Ahat_t for the contiguous run `ts` into slots 0..len(ts)-1
        of slot set `set_idx`.  Returns the slots; the set's ready event (and
        `self.ready`) is recorded on the graph stream.  `after`: an event
        marking the end of the set's previous consumers (default: everything
        already enqueued on the current stream).

        Chunk head (graph difference across chunks, SURVEY §7 hard part 3):
        the reference ships the first snapshot of every chunk in full
        (`delta.py:161-163`).  Here the head A_{t0} is rebuilt from the
        1-step delta of t0 whenever A_{t0-1} is on the device at this point
        of the graph stream: this materialiser's own last snapshot (chunks
        built in time order, e.g. consecutive blocks at P = 1), or
        `head_prev` = (rowptr, col) of A_{t0-1} from the rank that owns t0-1
        (a neighbouring rank's raw CSR, same device or received over NVLink;
        `head_prev[2]`, if given, is an event or callable the graph stream
        waits on first; `head_prev[3]`, if given, is called once A_{t0-1}
        has been read).  Only t = 0 then travels in full.  With device
        smoothing a head that follows nothing ships A_{t0-1} in full (the
        smoothed A~_{t0} needs it) and A_{t0} as its delta.

        `count_bytes` charges the real H2D bytes of this build; `consume`
        also charges the pass that consumes it (`account`) -- the engine
        builds ahead of the consuming pass and charges that pass itself.

        `handoff(rowptr, col, nnz)`: the chunk's last raw snapshot is wanted
        by another rank as its head.  It is then rebuilt first, by the raw
        delta chain alone (`_raw_chain`, private buffers, before waiting for
        the slots' consumers), and handed over (enqueued on the graph
        stream) before the chunk's smoothing / transposes / Laplacians:
        rank q's head no longer waits for rank q-1's whole chunk build,
        only for its chain of 1-step deltas."""
        enc = self.enc
        self.slots = self.sets[set_idx]
        self.ready = self.ready_sets[set_idx]
        if len(ts) > len(self.slots):
            raise InputError("chunk longer than the materialiser's slot count")
        plan = enc.chunk(ts)
        n = enc.n
        gs = self.graph_stream
        gsh = gs.cuda_stream
        t0 = ts[0]
        sm = self.smooth
        if t0 > 0 and self.raw_t == t0 - 1:
            head = "own"
        elif t0 > 0 and head_prev is not None:
            head = "neighbor"
        elif t0 > 0 and sm is not None:
            head = "full_prev"
        else:
            head = "full"
        # H2D ranges of this build: deltas of t0+1..t1 (and of t0 itself when
        # the head is rebuilt from A_{t0-1}), the full head (or A_{t0-1}) otherwise
        fo, fc = plan.full_range
        do, dc = plan.delta_range
        if head != "full":
            do = int(enc.delta_off[t0])
            dc = int(enc.delta_off[ts[-1] + 1] - enc.delta_off[t0])
            if head == "full_prev":
                fo, fc = int(enc.full_off[t0 - 1]), int(2 * enc.nnz[t0 - 1])
            else:
                fc = 0
        vo, vc = plan.val_range
        if self.resident:
            fbase, dbase, vbase = fo, do, vo
        else:
            fbase = dbase = vbase = 0
            cs = self.copy_stream
            cs.wait_stream(gs)                 # staging is free once the previous chunk's rebuild ran
            with torch.cuda.stream(cs):
                if self.copy_log is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(cs)
                if fc:
                    self.full_dev[:fc].copy_(enc.full[fo:fo + fc], non_blocking=True)
                if dc:
                    self.delta_dev[:dc].copy_(enc.delta[do:do + dc], non_blocking=True)
                if not enc.unit:
                    self.vals_dev[:vc].copy_(enc.vals[vo:vo + vc], non_blocking=True)
                if self.copy_log is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(cs)
                    self.copy_log.append((e0, e1, 4 * (fc + dc) + (0 if enc.unit else 8 * vc)))
            gs.wait_stream(cs)
        built_bytes = 4 * (fc + dc) + (0 if enc.unit else 8 * vc)
        if count_bytes:
            self.bytes_h2d += built_bytes
            self.bytes_full_built += enc.full_bytes(ts)
            self.builds.append((list(ts), built_bytes, head != "full"))
        if consume:
            self.account(ts, ledger, count_bytes)
        voff = vbase
        if head == "neighbor" and len(head_prev) > 2 and head_prev[2] is not None:
            with torch.cuda.stream(gs):
                w = head_prev[2]
                w() if callable(w) else gs.wait_event(w)
        if handoff is not None:
            with torch.cuda.stream(gs):
                rp, col = self._raw_chain(ts, head, head_prev, fbase, dbase)
                handoff(rp, col, int(enc.nnz[ts[-1]]))
        # slots are overwritten: wait for their consumers on the compute stream
        if after is not None:
            gs.wait_event(after)
        else:
            gs.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(gs):
            cur = self.cur
            dpos = dbase
            release = None
            prev_rp = prev_col = None
            if head == "neighbor":
                prev_rp, prev_col = head_prev[0], head_prev[1]
                release = head_prev[3] if len(head_prev) > 3 else None
            elif head == "own":
                prev_rp, prev_col = self.a_rowptr[cur], self.a_col[cur]
            elif head == "full_prev":
                mp = int(enc.nnz[t0 - 1])
                call("dgnn_rowptr_from_sorted_rows", n, mp, ptr(self.full_dev[fbase:fbase + mp]),
                     ptr(self.a_rowptr[cur]), gsh)
                self.a_col[cur][:mp].copy_(self.full_dev[fbase + mp:fbase + 2 * mp])
                prev_rp, prev_col = self.a_rowptr[cur], self.a_col[cur]
            for i, t in enumerate(ts):
                m = int(enc.nnz[t])
                if i == 0 and head == "full":
                    rows = self.full_dev[fbase:fbase + m]
                    call("dgnn_rowptr_from_sorted_rows", n, m, ptr(rows), ptr(self.a_rowptr[cur]), gsh)
                    a_rowptr = self.a_rowptr[cur]
                    # the raw CSR lives in a_rowptr / a_col (the staging area is reused)
                    a_col = self.a_col[cur]
                    a_col[:m].copy_(self.full_dev[fbase + m:fbase + 2 * m])
                else:
                    if i > 0:
                        prev_rp, prev_col = a_rowptr, a_col
                    nd, ni = int(enc.n_del[t]), int(enc.n_ins[t])
                    d = self.delta_dev[dpos:dpos + 2 * (nd + ni)]
                    dpos += 2 * (nd + ni)
                    nxt = 1 - cur
                    call("dgnn_csr_apply_delta", n, ptr(prev_rp), ptr(prev_col), nd, ptr(d[:nd]),
                         ptr(d[nd:2 * nd]), ni, ptr(d[2 * nd:2 * nd + ni]), ptr(d[2 * nd + ni:]),
                         ptr(self.a_rowptr[nxt]), ptr(self.a_col[nxt]), enc.cap_a, ptr(self.ws_apply),
                         self.ws_apply.numel(), ptr(self.status), gsh)
                    cur = nxt
                    a_rowptr, a_col = self.a_rowptr[cur], self.a_col[cur]
                if sm is not None:
                    # A~_t = M[t,t-1] A_{t-1} + M[t,t] A_t (dtdg.py:239-252), window <= 2
                    mm, w = sm
                    if t == 0 or w == 1:
                        pa, ca, na, wa = self.zero_rowptr, self.a_col[1 - cur], 0, 0.0
                    else:
                        pa, ca, na, wa = prev_rp, prev_col, int(enc.nnz[t - 1]), float(mm[t, t - 1])
                    call("dgnn_csr_weighted_merge", n, ptr(pa), ptr(ca), None, na, wa, ptr(a_rowptr), ptr(a_col),
                         None, m, float(mm[t, t]), ptr(self.sm_rowptr), ptr(self.sm_col), ptr(self.sm_val),
                         self.sm_col.numel(), ptr(self.ws_merge), self.ws_merge.numel(), gsh)
                    g_rowptr, g_col, g_val, g_m = self.sm_rowptr, self.sm_col, self.sm_val, int(enc.nnz_sm[t])
                else:
                    g_val = None if enc.unit else self.vals_dev[voff:voff + m]
                    g_rowptr, g_col, g_m = a_rowptr, a_col, m
                voff += m
                if i == 0 and release is not None:
                    release()           # A_{t0-1} (the neighbour's hand-off) has been read
                    release = None
                call("dgnn_csr_transpose_staged", n, g_m, ptr(g_rowptr), ptr(g_col), ptr(g_val),
                     ptr(self.at_rowptr), ptr(self.at_col), ptr(self.at_val), ptr(self.stage_col),
                     ptr(self.stage_val), ptr(self.ws_tr), self.ws_tr.numel(), gsh)
                s = self.slots[i]
                call("dgnn_laplacian", n, ptr(g_rowptr), ptr(g_rowptr), ptr(g_col), ptr(g_val), 0,
                     ptr(s.rowptr), ptr(s.col), ptr(s.val), ptr(s.val64), enc.cap_hat,
                     ptr(self.ws_lap), self.ws_lap.numel(), gsh)
                call("dgnn_laplacian", n, ptr(g_rowptr), ptr(self.at_rowptr), ptr(self.at_col),
                     ptr(self.at_val), 1, ptr(s.t_rowptr), ptr(s.t_col), ptr(s.t_val), ptr(s.t_val64),
                     enc.cap_hat, ptr(self.ws_lap), self.ws_lap.numel(), gsh)
                s.a_rowptr, s.a_t_rowptr, s.t = g_rowptr, self.at_rowptr, t
            if release is not None:
                release()
            self.cur = cur
            self.raw_t = ts[-1]
            self.ready.record(gs)
        return self.slots[:len(ts)]

    def _raw_chain(self, ts, head, head_prev, fbase, dbase):
        """Raw CSR of A_{ts[-1]} from the chunk's head source and the 1-step
        deltas of ts alone, in private ping-pong buffers (graph stream
        current).  Same kernels and inputs as materialize's chain, hence
        the same bits."""
        enc, n = self.enc, self.enc.n
        gsh = self.graph_stream.cuda_stream
        if getattr(self, "ch_rowptr", None) is None:
            i32 = dict(dtype=torch.int32, device=self.device)
            self.ch_rowptr = [torch.empty(n + 1, **i32) for _ in range(2)]
            self.ch_col = [torch.empty(enc.cap_a, **i32) for _ in range(2)]
        t0 = ts[0]
        cur, dpos, first = 0, dbase, 0
        if head == "full":
            m = int(enc.nnz[t0])
            call("dgnn_rowptr_from_sorted_rows", n, m, ptr(self.full_dev[fbase:fbase + m]), ptr(self.ch_rowptr[0]),
                 gsh)
            self.ch_col[0][:m].copy_(self.full_dev[fbase + m:fbase + 2 * m])
            prev_rp, prev_col, first = self.ch_rowptr[0], self.ch_col[0], 1
        elif head == "neighbor":
            prev_rp, prev_col = head_prev[0], head_prev[1]
        elif head == "own":
            prev_rp, prev_col = self.a_rowptr[self.cur], self.a_col[self.cur]
        else:   # full_prev: A_{t0-1} in full
            mp = int(enc.nnz[t0 - 1])
            call("dgnn_rowptr_from_sorted_rows", n, mp, ptr(self.full_dev[fbase:fbase + mp]), ptr(self.ch_rowptr[0]),
                 gsh)
            self.ch_col[0][:mp].copy_(self.full_dev[fbase + mp:fbase + 2 * mp])
            prev_rp, prev_col = self.ch_rowptr[0], self.ch_col[0]
        for t in ts[first:]:
            nd, ni = int(enc.n_del[t]), int(enc.n_ins[t])
            d = self.delta_dev[dpos:dpos + 2 * (nd + ni)]
            dpos += 2 * (nd + ni)
            nxt = 1 - cur
            call("dgnn_csr_apply_delta", n, ptr(prev_rp), ptr(prev_col), nd, ptr(d[:nd]), ptr(d[nd:2 * nd]), ni,
                 ptr(d[2 * nd:2 * nd + ni]), ptr(d[2 * nd + ni:]), ptr(self.ch_rowptr[nxt]), ptr(self.ch_col[nxt]),
                 enc.cap_a, ptr(self.ws_apply), self.ws_apply.numel(), ptr(self.status), gsh)
            cur = nxt
            prev_rp, prev_col = self.ch_rowptr[cur], self.ch_col[cur]
        return prev_rp, prev_col

    def add_sets(self, k: int) -> None:
        """k more slot sets of `slots` slots each."""
        n, cap_h = self.enc.n, self.enc.cap_hat
        i32 = dict(dtype=torch.int32, device=self.device)
        f32 = dict(dtype=torch.float32, device=self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        for _ in range(k):
            self.sets.append([LapSlot(
                torch.empty(n + 1, **i32), torch.empty(cap_h, **i32), torch.empty(cap_h, **f32),
                torch.empty(n + 1, **i32), torch.empty(cap_h, **i32), torch.empty(cap_h, **f32),
                torch.empty(cap_h, **f64) if self.with_f64 else None,
                torch.empty(cap_h, **f64) if self.with_f64 else None) for _ in range(self.nslots)])
            self.ready_sets.append(torch.cuda.Event())

    @staticmethod
    def slot_bytes(enc, with_f64: bool = False) -> int:
        return 2 * 4 * (enc.n + 1) + 2 * enc.cap_hat * (4 + 4 + (8 if with_f64 else 0))

    def raw(self):
        """(rowptr, col) of the last rebuilt raw snapshot A_{raw_t} (valid at
        the current end of the graph stream, until the next rebuild)."""
        return self.a_rowptr[self.cur], self.a_col[self.cur]

    def account(self, ts, ledger=None, count_bytes: bool = True):
        """Charge one streaming pass of `ts` as the reference schedule sees it
        (`stream_block` at every pass, `dist.py:301-312`): the reference
        ledger counters, and `bytes_full_equiv` = the bytes of this pass's
        snapshots sent in full.  The real H2D bytes are charged when a chunk
        is built (`materialize`); a pass that reuses kept snapshots (the
        checkpoint rerun) copies nothing."""
        if count_bytes:
            self.bytes_full_equiv += self.enc.full_bytes(ts)
        if ledger is not None:
            self.enc.charge(ledger, ts)

    def wait(self, stream=None):
        (stream or torch.cuda.current_stream(self.device)).wait_event(self.ready)

    def check(self):
        """Raise CorruptDeltaError if any rebuild saw an inconsistent delta."""
        bad = int(self.status[0].item())
        if bad:
            self.status.zero_()
            raise CorruptDeltaError(f"{bad} inconsistent delta entries during CSR rebuild")

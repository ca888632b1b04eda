"""ctypes binding of libdgnn_b200.so (the C ABI in include/dgnn_b200.h).

This is the only place the package touches native code.  The library is
loaded lazily on first use and the product path fails loudly when it is
missing -- there is no CPU fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes
from ctypes import c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_void_p
import os
from pathlib import Path

from .errors import CorruptDeltaError, DeviceError, InputError

LIB_PATH = Path(__file__).resolve().parent / "libdgnn_b200.so"
# bottleneck-probe builds (scripts/*probe*) substitute a variant library
if os.environ.get("DGNN_LIB_PATH"):
    LIB_PATH = Path(os.environ["DGNN_LIB_PATH"])


class Frame(ctypes.Structure):
    """`dgnn_frame`: row i at ptr + (i / rows_per_slab) * slab_stride + (i % rows_per_slab) * ld."""
    _fields_ = [("ptr", c_void_p), ("ld", c_int64), ("rows_per_slab", c_int64), ("slab_stride", c_int64)]


P = c_void_p
_SIGS = {
    "dgnn_last_error": (ctypes.c_char_p, []),
    "dgnn_abi_version": (c_int, []),
    "dgnn_launch_count": (ctypes.c_longlong, []),
    "dgnn_device_check": (c_int, [c_int]),
    "dgnn_set_sm_reserve": (None, [c_int]),
    "dgnn_rowptr_from_sorted_rows": (c_int, [c_int32, c_int64, P, P, P]),
    "dgnn_csr_apply_delta_workspace": (c_size_t, [c_int32]),
    "dgnn_csr_apply_delta": (c_int, [c_int32, P, P, c_int64, P, P, c_int64, P, P, P, P, c_int64, P,
                                     c_size_t, P, P]),
    "dgnn_csr_transpose_workspace": (c_size_t, [c_int32]),
    "dgnn_csr_transpose_staged": (c_int, [c_int32, c_int64, P, P, P, P, P, P, P, P, P, c_size_t, P]),
    "dgnn_laplacian_workspace": (c_size_t, [c_int32]),
    "dgnn_laplacian": (c_int, [c_int32, P, P, P, P, c_int, P, P, P, P, c_int64, P, c_size_t, P]),
    "dgnn_degree_features": (c_int, [c_int32, P, P, P, c_int64, P]),
    "dgnn_csr_weighted_merge_workspace": (c_size_t, [c_int32, c_int64]),
    "dgnn_scatter_f64": (c_int, [c_int64, P, P, P, P]),
    "dgnn_evolve_forward": (c_int, [c_int64, c_int32, P, P, P, P, P, P, P]),
    "dgnn_evolve_backward": (c_int, [c_int64, c_int32, P, P, P, P, P, P, P]),
    "dgnn_csr_weighted_merge": (c_int, [c_int32, P, P, P, c_int64, c_double, P, P, P, c_int64, c_double, P, P, P,
                                        c_int64, P, c_size_t, P]),
    "dgnn_spmm_f64": (c_int, [c_int32, P, P, P, P, c_int64, c_int32, P, c_int64, P]),
    "dgnn_spmm_f32": (c_int, [c_int32, P, P, P, Frame, c_int32, Frame, P]),
    "dgnn_gcn_forward": (c_int, [c_int32, P, P, P, Frame, c_int32, P, c_int32, c_int, Frame, Frame, P]),
    "dgnn_set_gcn_tensor_cores": (None, [c_int]),
    "dgnn_gcn_backward_rows": (c_int, [c_int32, Frame, Frame, c_int32, P, c_int32, c_int, Frame, P]),
    "dgnn_gcn_weight_grad_workspace": (c_size_t, [c_int32, c_int32]),
    "dgnn_gcn_weight_grad": (c_int, [c_int32, Frame, Frame, Frame, c_int32, c_int32, c_int, P, P,
                                     c_size_t, P]),
    "dgnn_tile_block": (c_int, [c_int64, c_int64, c_int32, P, P, P]),
    "dgnn_tile_unblock": (c_int, [c_int64, c_int64, c_int32, P, P, P]),
    "dgnn_lstm_forward_step": (c_int, [c_int64, c_int32, c_int32, P, c_int64, P, P, P, P, P, P, P, P]),
    "dgnn_tc_weight_image_bytes": (c_size_t, [c_int32, c_int32]),
    "dgnn_tc_weight_image": (c_int, [c_int32, c_int32, P, c_int64, P, P]),
    "dgnn_tc_weight_image_ex": (c_int, [c_int32, c_int32, c_int32, P, c_int64, c_int32, P, P]),
    "dgnn_lstm_weight_grad_tc_workspace": (c_size_t, [c_int32, c_int32]),
    "dgnn_lstm_weight_grad_tc": (c_int, [c_int64, c_int64, c_int32, c_int32, P, c_int64, P, P, P, P, P, P,
                                         c_size_t, P]),
    "dgnn_lstm_weight_grad_ts": (c_int, [c_int64, c_int64, c_int32, c_int32, P, c_int64, P, P, P, P, P, P,
                                         c_size_t, P]),
    "dgnn_lstm_backward_step_tc": (c_int, [c_int64, c_int32, c_int32, P, P, P, P, P, P, P, P, c_int64, P, P,
                                           P]),
    "dgnn_tc_gemm_test": (c_int, [c_int32, c_int32, c_int32, P, c_int64, P, P, c_int64, P]),
    "dgnn_lstm_forward_step_tc": (c_int, [c_int64, c_int32, c_int32, P, c_int64, P, P, P, P, P, P, P, P]),
    "dgnn_lstm_forward_step_ws": (c_int, [c_int64, c_int32, c_int32, P, c_int64, P, P, P, P, P, P, P, P]),
    "dgnn_lstm_forward_step_pair": (c_int, [c_int64, c_int32, c_int32, P, c_int64, P, P, P, P, P, P, P, P]),
    "dgnn_lstm_backward_step_ws": (c_int, [c_int64, c_int32, c_int32, P, P, P, P, P, P, P, P, c_int64, P, P,
                                           P]),
    "dgnn_lstm_backward_step": (c_int, [c_int64, c_int32, c_int32, P, P, P, P, P, P, P, P, P, c_int64,
                                        P, P, P]),
    "dgnn_gemm_tn_workspace": (c_size_t, [c_int32, c_int32]),
    "dgnn_gemm_tn": (c_int, [c_int64, c_int32, c_int32, P, c_int64, P, c_int64, P, c_int64, P, P,
                             c_size_t, P]),
    "dgnn_axpy_frame": (c_int, [c_int64, c_float, P, P, c_int, P]),
    "dgnn_frames_combine": (c_int, [c_int64, c_int32, P, P, P, P, P, P]),
    "dgnn_head_loss": (c_int, [c_int64, P, P, P, Frame, c_int32, c_int32, P, P, c_double, P, c_int32,
                               P, P]),
    "dgnn_head_grad_workspace": (c_size_t, [c_int32, c_int32]),
    "dgnn_head_grad": (c_int, [c_int64, P, P, Frame, c_int32, c_int32, P, P, P, P, c_size_t, P]),
    "dgnn_head_loss_grad": (c_int, [c_int64, P, P, P, Frame, c_int32, c_int32, P, P, c_double, P, c_int32, P, P, P,
                                    P, c_size_t, P]),
    "dgnn_head_scatter": (c_int, [c_int32, P, P, P, P, c_int32, c_int32, Frame, P]),
    "dgnn_head_scatter_active": (c_int, [c_int32, P, P, c_int32, P, P, P, c_int32, c_int32, Frame, P]),
    "dgnn_head_predict": (c_int, [c_int64, P, P, P, Frame, c_int32, c_int32, P, P, P, P]),
    "dgnn_sum_f64": (c_int, [c_int64, P, P, c_int, P]),
    "dgnn_adam": (c_int, [c_int64, P, P, P, P, c_double, c_double, c_double, c_double, c_double,
                          c_double, c_double, c_double, P]),
    "dgnn_params_to_device": (c_int, [c_int64, P, P, P, P, P]),
    "dgnn_grads_gather": (c_int, [c_int64, P, P, P, P]),
    "dgnn_fill_f32": (c_int, [c_int64, c_float, P, P]),
    "dgnn_cast_f64_to_f32_frame": (c_int, [c_int32, c_int32, P, c_int64, Frame, P]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(f"{LIB_PATH.name} is missing; build it with "
                              "`python -m paper_2109_07893_b200.build` (nvcc, sm_100a)")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list:
    return sorted(_SIGS)


class KernelTimer:
    """Records CUDA events around every C-ABI call whose name is in `names`,
    on the stream the call was enqueued on (its last argument).  Used by
    bench.py for per-kernel durations inside the timed region."""

    def __init__(self, names):
        self.names = set(names)
        self.records = {}      # name -> list of (start, end, args)
        self._streams = {}
        self.order = []        # (stream handle, name, start, end) in issue order

    def stream(self, handle):
        import torch
        if handle not in self._streams:
            self._streams[handle] = torch.cuda.ExternalStream(handle)
        return self._streams[handle]

    def gaps(self, t0, top: int = 8):
        """Per stream: busy ms inside the recorded calls, idle ms between
        consecutive calls (waits on other streams / the fabric / the host),
        and the calls preceded by the largest total idle time.  `t0` is an
        event recorded at the start of the timed region."""
        import torch
        torch.cuda.synchronize()
        out = {}
        last = {}
        for st, name, e0, e1 in self.order:
            d = out.setdefault(str(st), {"busy_ms": 0.0, "idle_ms": 0.0, "idle_before": {}, "busy_by_call": {}})
            dt = e0.elapsed_time(e1)
            d["busy_ms"] += dt
            d["busy_by_call"][name] = d["busy_by_call"].get(name, 0.0) + dt
            prev = last.get(st)
            idle = prev.elapsed_time(e0) if prev is not None else t0.elapsed_time(e0)
            if idle > 0:
                d["idle_ms"] += idle
                d["idle_before"][name] = d["idle_before"].get(name, 0.0) + idle
            last[st] = e1
        for d in out.values():
            d["idle_before"] = dict(sorted(d["idle_before"].items(), key=lambda kv: -kv[1])[:top])
            d["busy_by_call"] = dict(sorted(d["busy_by_call"].items(), key=lambda kv: -kv[1])[:2 * top])
        return out

    def durations(self):
        """name -> list of (ms, args); synchronises."""
        import torch
        torch.cuda.synchronize()
        return {k: [(s.elapsed_time(e), a) for s, e, a in v] for k, v in self.records.items()}


_timer: KernelTimer | None = None


def set_timer(timer: KernelTimer | None) -> None:
    global _timer
    _timer = timer


def launch_count() -> int:
    return int(lib().dgnn_launch_count())


def call(name: str, *args) -> None:
    t = _timer
    if t is not None and name in t.names:
        import torch
        s = t.stream(args[-1]) if args[-1] else torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        rc = getattr(lib(), name)(*args)
        e1.record(s)
        t.records.setdefault(name, []).append((e0, e1, args))
        t.order.append((args[-1], name, e0, e1))
    else:
        rc = getattr(lib(), name)(*args)
    if rc:
        msg = lib().dgnn_last_error().decode(errors="replace")
        if rc == 1:
            raise InputError(f"{name}: {msg}")
        if rc == 2:
            raise CorruptDeltaError(f"{name}: {msg}")
        raise DeviceError(f"{name} failed (code {rc}): {msg}")


def query(name: str, *args) -> int:
    return int(getattr(lib(), name)(*args))


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def frame(t, ld: int | None = None, rows_per_slab: int = 0, slab_stride: int = 0) -> Frame:
    if t is None:
        return Frame(None, 0, 0, 0)
    return Frame(t.data_ptr(), int(ld if ld is not None else t.shape[-1]), int(rows_per_slab),
                 int(slab_stride))


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream

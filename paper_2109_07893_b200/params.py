"""Model configuration, seeded parameters and their padded device layout.

`ModelConfig`/`init_params` keep the reference contract (`models.py:49-93`,
`models.py:138-177`): same validation, same parameter names and shapes, and
the same generator draws in the same order, so a seed gives the reference's
parameters bit-for-bit.

On device every feature width is padded (inputs to 4, hidden widths to a
power of two >= 16) so the kernels run on float4 rows and fixed tile
shapes.  Padded weights are zero, which keeps padded activations exactly zero
through ReLU and the LSTM cell (g = tanh(0) = 0 makes c and h stay 0), so
padding never changes a real output or gradient.  The master copy of the
parameters is a flat fp64 vector in sorted-key order (the reference's Adam
order, `training.py:891`); kernels read an fp32 padded image of it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr
from .errors import ConfigError

ARCHITECTURES = ("tm-gcn", "cd-gcn", "egcn-o")


@dataclass(frozen=True)
class ModelConfig:
    architecture: str
    in_features: int = 2
    hidden_features: int = 6
    embed_features: int = 6
    layers: int = 2
    window: int = 2
    edge_life: int = 2
    classes: int = 2

    def __post_init__(self):
        if self.architecture not in ARCHITECTURES:
            raise ConfigError(f"unknown architecture {self.architecture!r}; expected one of {ARCHITECTURES}")
        if self.layers < 1:
            raise ConfigError("layers must be >= 1")
        if self.architecture == "cd-gcn" and self.layers != 2:
            raise ConfigError("cd-gcn is a fixed two-layer architecture")
        if min(self.in_features, self.hidden_features, self.embed_features) < 1:
            raise ConfigError("feature lengths must be positive")
        if self.window < 1:
            raise ConfigError("window must be >= 1")
        if self.edge_life < 1:
            raise ConfigError("edge life must be >= 1")
        if self.classes < 2:
            raise ConfigError("need at least two classification categories")

    def layer_dims(self):
        dims, fin = [], self.in_features
        for layer in range(self.layers):
            last = layer == self.layers - 1
            if self.architecture == "cd-gcn":
                gcn_out = self.hidden_features
                out = self.embed_features if last else self.hidden_features
            else:
                gcn_out = self.embed_features if last else self.hidden_features
                out = gcn_out
            dims.append(LayerDims(fin=fin, gcn_out=gcn_out, out=out))
            fin = out
        return dims


@dataclass(frozen=True)
class LayerDims:
    fin: int
    gcn_out: int
    out: int


def as_config(cfg) -> ModelConfig:
    """Accept the reference's ModelConfig (or any object with its fields)."""
    if isinstance(cfg, ModelConfig):
        return cfg
    return ModelConfig(cfg.architecture, cfg.in_features, cfg.hidden_features, cfg.embed_features,
                       cfg.layers, cfg.window, cfg.edge_life, cfg.classes)


def _glorot(rng, fan_in, fan_out):
    limit = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-limit, limit, size=(fan_in, fan_out))


def init_params(cfg, seed: int) -> dict:
    """Seeded parameters in the reference's key and draw order."""
    cfg = as_config(cfg)
    rng = np.random.default_rng(seed)
    params = {}
    for layer, d in enumerate(cfg.layer_dims()):
        if cfg.architecture == "egcn-o":
            # models.py:157-163: initial weight, four gate matrices, forget bias 1
            params[f"evolve{layer}.w0"] = _glorot(rng, d.fin, d.gcn_out)
            params[f"evolve{layer}.gates"] = np.stack([_glorot(rng, d.fin, d.gcn_out) for _ in range(4)])
            bias = np.zeros((4, d.fin, d.gcn_out))
            bias[1] = 1.0
            params[f"evolve{layer}.bias"] = bias
            continue
        params[f"gcn{layer}.w"] = _glorot(rng, d.fin, d.gcn_out)
        if cfg.architecture == "cd-gcn":
            f_in, hid = d.fin + d.gcn_out, d.out
            params[f"lstm{layer}.wx"] = np.concatenate([_glorot(rng, f_in, hid) for _ in range(4)], axis=1)
            params[f"lstm{layer}.wh"] = np.concatenate([_glorot(rng, hid, hid) for _ in range(4)], axis=1)
            b = np.zeros(4 * hid)
            b[hid:2 * hid] = 1.0
            params[f"lstm{layer}.b"] = b
    params["head.w"] = np.zeros((2 * cfg.embed_features, cfg.classes))
    params["head.b"] = np.zeros(cfg.classes)
    return params


def parameter_count(params: dict) -> int:
    return sum(int(np.prod(np.shape(a))) for a in params.values())


def pad_hidden(x: int) -> int:
    p = 16
    while p < x:
        p *= 2
    if p > 128:
        raise ConfigError(f"feature width {x} exceeds the compiled maximum of 128")
    return p


def pad_input(x: int) -> int:
    return 4 if x <= 4 else pad_hidden(x)


@dataclass(frozen=True)
class PaddedLayer:
    fin: int          # real widths
    gout: int
    out: int
    fp: int           # padded GCN input width
    hg: int           # padded GCN output width
    ho: int           # padded temporal-stage width
    rw: int           # GCN output (= LSTM input) row width
    skip: bool

    @property
    def kx(self) -> int:
        return self.rw


def padded_layers(cfg: ModelConfig):
    out = []
    prev_p = None
    skip = cfg.architecture == "cd-gcn"
    for layer, d in enumerate(cfg.layer_dims()):
        fp = pad_input(d.fin) if layer == 0 else prev_p
        hg = pad_hidden(d.gcn_out)
        ho = pad_hidden(d.out) if skip else hg
        rw = fp + hg if skip else hg
        out.append(PaddedLayer(d.fin, d.gcn_out, d.out, fp, hg, ho, rw, skip))
        prev_p = ho
    return out


class ParamLayout:
    """Offsets of every padded parameter block in one fp32 buffer, and the
    flat (sorted-key, C-order) <-> padded index maps."""

    ALIGN = 64

    def __init__(self, cfg: ModelConfig):
        self.cfg = cfg
        self.layers = padded_layers(cfg)
        self.ep = self.layers[-1].ho
        self.classes = cfg.classes
        self.blocks = {}
        size = 0

        def alloc(name, rows, cols):
            nonlocal size
            self.blocks[name] = (size, rows, cols)
            size += (rows * cols + self.ALIGN - 1) // self.ALIGN * self.ALIGN

        self.evolve = cfg.architecture == "egcn-o"
        for l, L in enumerate(self.layers):
            if self.evolve:
                # the evolving GCN weight: initial matrix, stacked gates / biases
                alloc(f"evolve{l}.w0", L.fp, L.hg)
                alloc(f"evolve{l}.gates", 4 * L.fp, L.hg)
                alloc(f"evolve{l}.bias", 4 * L.fp, L.hg)
                continue
            alloc(f"gcn{l}.w", L.fp, L.hg)
            if L.skip:
                alloc(f"lstm{l}.wcat", L.kx + L.ho, 4 * L.ho)
                alloc(f"lstm{l}.wcat_t", 4 * L.ho, L.kx + L.ho)
                alloc(f"lstm{l}.b", 1, 4 * L.ho)
        alloc("head.w", 2 * self.ep, cfg.classes)
        alloc("head.b", 1, cfg.classes)
        self.size = size

        # flat order = sorted keys, C-order inside each (training.py:891)
        shapes = {k: np.shape(v) for k, v in init_params_shapes(cfg).items()}
        self.keys = sorted(shapes)
        self.shapes = shapes
        pos0, pos1 = [], []
        for k in self.keys:
            p0, p1 = self._positions(k, shapes[k])
            pos0.append(p0)
            pos1.append(p1)
        self.pos0 = np.concatenate(pos0).astype(np.int64)
        self.pos1 = np.concatenate(pos1).astype(np.int64)
        self.count = int(self.pos0.shape[0])

    def _positions(self, key, shape):
        if key.startswith("evolve"):
            l = int(key[6:key.index(".")])
            off, _, cols = self.blocks[key]
            fp = self.layers[l].fp
            if key.endswith(".w0"):
                k, j = np.meshgrid(np.arange(shape[0]), np.arange(shape[1]), indexing="ij")
                return (off + k * cols + j).ravel(), np.full(k.size, -1)
            g, k, j = np.meshgrid(np.arange(4), np.arange(shape[1]), np.arange(shape[2]), indexing="ij")
            return (off + (g * fp + k) * cols + j).ravel(), np.full(k.size, -1)
        if key.startswith("gcn"):
            l = int(key[3:key.index(".")])
            L = self.layers[l]
            off, _, cols = self.blocks[key]
            k, j = np.meshgrid(np.arange(shape[0]), np.arange(shape[1]), indexing="ij")
            return (off + k * cols + j).ravel(), np.full(k.size, -1)
        if key.startswith("lstm"):
            l = int(key[4:key.index(".")])
            L = self.layers[l]
            H = L.out
            ncol = 4 * L.ho
            wcat, _, _ = self.blocks[f"lstm{l}.wcat"]
            wcat_t, _, _ = self.blocks[f"lstm{l}.wcat_t"]
            K = L.kx + L.ho
            if key.endswith(".b"):
                g, u = np.divmod(np.arange(4 * H), H)
                off = self.blocks[key][0]
                return off + g * L.ho + u, np.full(4 * H, -1)
            rows = np.arange(shape[0])
            if key.endswith(".wx"):
                prow = np.where(rows < L.fin, rows, L.fp + (rows - L.fin))
            else:  # wh
                prow = L.kx + rows
            g, u = np.divmod(np.arange(4 * H), H)
            pcol = g * L.ho + u
            R, C = np.meshgrid(prow, pcol, indexing="ij")
            return (wcat + R * ncol + C).ravel(), (wcat_t + C * K + R).ravel()
        if key == "head.w":
            E = self.cfg.embed_features
            off = self.blocks[key][0]
            rows = np.arange(shape[0])
            prow = np.where(rows < E, rows, self.ep + (rows - E))
            R, C = np.meshgrid(prow, np.arange(shape[1]), indexing="ij")
            return (off + R * self.classes + C).ravel(), np.full(R.size, -1)
        if key == "head.b":
            off = self.blocks[key][0]
            return off + np.arange(shape[0]), np.full(shape[0], -1)
        raise ConfigError(f"unexpected parameter {key}")

    def block(self, buf: torch.Tensor, name: str) -> torch.Tensor:
        off, rows, cols = self.blocks[name]
        return buf[off:off + rows * cols].view(rows, cols)

    def flatten(self, params: dict) -> np.ndarray:
        missing = set(self.keys) ^ set(params)
        if missing:
            raise ConfigError(f"parameter dict keys do not match the architecture: {sorted(missing)}")
        parts = []
        for k in self.keys:
            a = np.asarray(params[k], dtype=np.float64)
            if a.shape != tuple(self.shapes[k]):
                raise ConfigError(f"parameter {k} has shape {a.shape}, expected {self.shapes[k]}")
            parts.append(a.ravel())
        return np.concatenate(parts)

    def unflatten(self, flat: np.ndarray) -> dict:
        out, o = {}, 0
        for k in self.keys:
            size = int(np.prod(self.shapes[k]))
            out[k] = np.array(flat[o:o + size], dtype=np.float64).reshape(self.shapes[k])
            o += size
        return out


def init_params_shapes(cfg: ModelConfig) -> dict:
    shapes = {}
    for layer, d in enumerate(cfg.layer_dims()):
        if cfg.architecture == "egcn-o":
            shapes[f"evolve{layer}.w0"] = np.empty((d.fin, d.gcn_out))
            shapes[f"evolve{layer}.gates"] = np.empty((4, d.fin, d.gcn_out))
            shapes[f"evolve{layer}.bias"] = np.empty((4, d.fin, d.gcn_out))
            continue
        shapes[f"gcn{layer}.w"] = np.empty((d.fin, d.gcn_out))
        if cfg.architecture == "cd-gcn":
            shapes[f"lstm{layer}.wx"] = np.empty((d.fin + d.gcn_out, 4 * d.out))
            shapes[f"lstm{layer}.wh"] = np.empty((d.out, 4 * d.out))
            shapes[f"lstm{layer}.b"] = np.empty(4 * d.out)
    shapes["head.w"] = np.empty((2 * cfg.embed_features, cfg.classes))
    shapes["head.b"] = np.empty(cfg.classes)
    return shapes


class DeviceParams:
    """fp64 master parameters + Adam moments (flat), fp32 padded image for
    the kernels, fp64 padded gradient accumulator."""

    def __init__(self, layout: ParamLayout, device):
        self.layout = layout
        dev = torch.device(device)
        self.device = dev
        self.p64 = torch.zeros(layout.count, dtype=torch.float64, device=dev)
        self.m = torch.zeros_like(self.p64)
        self.v = torch.zeros_like(self.p64)
        self.g = torch.zeros_like(self.p64)          # flat gradient (all-reduce / Adam input)
        self.w32 = torch.zeros(layout.size, dtype=torch.float32, device=dev)
        # egcn-o: the weight-evolution chain runs in fp64 (an fp64 padded image)
        self.w64 = torch.zeros(layout.size, dtype=torch.float64, device=dev) if layout.evolve else None
        self.gpad = torch.zeros(layout.size, dtype=torch.float64, device=dev)
        self.pos0 = torch.from_numpy(layout.pos0).to(dev)
        self.pos1 = torch.from_numpy(layout.pos1).to(dev)
        self.step = 0
        # tensor-core operand images of the LSTM weights (tf32 hi/lo, swizzled)
        self.images = {}
        for l, L in enumerate(layout.layers):
            if L.skip:
                nbytes = _lib.query("dgnn_tc_weight_image_bytes", 4 * L.ho, L.kx + L.ho)
                self.images[f"lstm{l}.fwd"] = torch.zeros(nbytes // 4, dtype=torch.float32, device=dev)
                nb = (L.kx + L.ho + 15) // 16 * 16
                nbytes = _lib.query("dgnn_tc_weight_image_bytes", nb, 4 * L.ho)
                self.images[f"lstm{l}.bwd"] = torch.zeros(nbytes // 4, dtype=torch.float32, device=dev)

    def image(self, name: str) -> torch.Tensor:
        return self.images[name]

    def load(self, params: dict, stream=None):
        flat = torch.from_numpy(self.layout.flatten(params))
        self.p64.copy_(flat.to(self.device))
        self.sync_image(stream)

    def sync_image(self, stream=None):
        sh = _lib.stream_handle(stream)
        call("dgnn_params_to_device", self.layout.count, ptr(self.p64), ptr(self.pos0), ptr(self.pos1),
             ptr(self.w32), sh)
        if self.w64 is not None:
            call("dgnn_scatter_f64", self.layout.count, ptr(self.p64), ptr(self.pos0), ptr(self.w64), sh)
        for l, L in enumerate(self.layout.layers):
            if L.skip:
                K = L.kx + L.ho
                call("dgnn_tc_weight_image", 4 * L.ho, K, ptr(self.w(f"lstm{l}.wcat_t")), K,
                     ptr(self.images[f"lstm{l}.fwd"]), sh)
                call("dgnn_tc_weight_image_ex", (K + 15) // 16 * 16, K, 4 * L.ho, ptr(self.w(f"lstm{l}.wcat")),
                     4 * L.ho, L.ho, ptr(self.images[f"lstm{l}.bwd"]), sh)

    def w(self, name: str) -> torch.Tensor:
        return self.layout.block(self.w32, name)

    def w64_block(self, name: str) -> torch.Tensor:
        return self.layout.block(self.w64, name)

    def gw(self, name: str) -> torch.Tensor:
        return self.layout.block(self.gpad, name)

    def zero_grad(self):
        self.gpad.zero_()

    def gather_grads(self, stream=None):
        call("dgnn_grads_gather", self.layout.count, ptr(self.gpad), ptr(self.pos0), ptr(self.g),
             _lib.stream_handle(stream))
        return self.g

    def adam(self, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
        self.step += 1
        t = self.step
        call("dgnn_adam", self.layout.count, ptr(self.p64), ptr(self.g), ptr(self.m), ptr(self.v), lr,
             beta1, 1.0 - beta1, beta2, 1.0 - beta2, 1.0 - beta1 ** t, 1.0 - beta2 ** t, eps,
             _lib.stream_handle(stream))
        self.sync_image(stream)

    def to_host(self) -> dict:
        return self.layout.unflatten(self.p64.cpu().numpy())

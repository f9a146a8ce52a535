"""nlrom.densenet — dense networks over real / multicomplex scalars.

``forward`` / ``backward`` run on the GPU through the C ABI (nlrom_net_forward /
nlrom_net_backward): part-wise FC layers on the fp64 tensor pipe with the real
weight acting per slot (CR block rule, mcx.py:297-300), fused multicomplex sin /
square epilogues, factored filter layers. Weights are uploaded once per net.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .mcx import MCArray, OrderError, MAX_ORDER

KINDS = ("fully_connected", "filter", "activation_sin", "activation_softmax", "activation_square")


@dataclass
class LayerSpec:
    """SPEC.md:111-116."""
    kind: str
    in_dim: int
    out_dim: int
    trainable: bool = True

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown layer kind {self.kind}")
        if self.kind == "filter":
            if self.in_dim != self.out_dim:
                raise ValueError("filter layers are square (SPEC.md:114)")
            self.trainable = False
        if self.kind.startswith("activation"):
            if self.in_dim != self.out_dim:
                raise ValueError("activation layers are square")
            self.trainable = False


@dataclass
class TrainConfig:
    """SPEC.md:123-126 (training itself is offline and out of scope here)."""
    learning_rate: float = 1e-3
    schedule: dict = field(default_factory=lambda: {300: 0.8, 3000: 0.8})
    epochs: int = 1
    batch_size: int = 64
    sample_weights: np.ndarray | None = None


class DenseNet:
    """Layered network: FC weights (out,in) row-major + biases, filter bases."""

    def __init__(self, layers, weights=None, biases=None, bases=None, seed=None):
        self.layers = list(layers)
        for a, b in zip(self.layers, self.layers[1:]):
            if a.out_dim != b.in_dim:
                raise ValueError("consecutive layer dims must chain (SPEC.md:115)")
        self.weights = dict(weights or {})
        self.biases = dict(biases or {})
        self.bases = dict(bases or {})
        self.seed = seed
        self._handle = None
        self._device = None

    @property
    def in_dim(self):
        return self.layers[0].in_dim

    @property
    def out_dim(self):
        return self.layers[-1].out_dim

    # -- device upload ---------------------------------------------------------
    def handle(self):
        if self._handle is None:
            L = _lib.lib()
            descs = (_lib.LayerDesc * len(self.layers))()
            self._keep = []
            for i, spec in enumerate(self.layers):
                d = descs[i]
                d.in_dim, d.out_dim = spec.in_dim, spec.out_dim
                if spec.kind == "fully_connected":
                    W = _lib.f64(self.weights[i])
                    b = _lib.f64(self.biases[i])
                    if W.shape != (spec.out_dim, spec.in_dim):
                        raise ValueError(f"layer {i}: weight shape {W.shape} != {(spec.out_dim, spec.in_dim)}")
                    d.kind, d.W, d.b = _lib.LAYER_FC, _lib.dptr(W), _lib.dptr(b)
                    self._keep += [W, b]
                elif spec.kind == "filter":
                    U = _lib.f64(self.bases[i])
                    d.kind, d.W, d.n_basis = _lib.LAYER_FILTER, _lib.dptr(U), U.shape[1]
                    self._keep.append(U)
                elif spec.kind == "activation_sin":
                    d.kind = _lib.LAYER_SIN
                elif spec.kind == "activation_square":
                    d.kind = _lib.LAYER_SQUARE
                else:
                    raise NotImplementedError("softmax belongs to the selection net S, out of scope (SURVEY.md §2)")
            h = C.c_void_p()
            dev = _lib.device_index()
            _lib.check(L.nlrom_net_create(C.byref(h), dev, len(self.layers), descs),
                       lambda: "nlrom_net_create failed (dimension or argument error)")
            self._handle, self._device = h, dev
            self._keep = None
        return self._handle

    def invalidate(self):
        if self._handle is not None:
            _lib.lib().nlrom_net_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.invalidate()
        except Exception:
            pass

    # -- checkpoint (JSON, row-major weights, bit-exact) -----------
    def to_json(self) -> str:
        doc = {"layers": [vars(s) for s in self.layers], "seed": self.seed,
               "weights": {str(k): np.asarray(v).tolist() for k, v in self.weights.items()},
               "biases": {str(k): np.asarray(v).tolist() for k, v in self.biases.items()},
               "bases": {str(k): np.asarray(v).tolist() for k, v in self.bases.items()}}
        return json.dumps(doc)

    @staticmethod
    def from_json(s: str) -> "DenseNet":
        doc = json.loads(s)
        layers = [LayerSpec(**d) for d in doc["layers"]]
        cv = lambda m: {int(k): np.asarray(v, dtype=float) for k, v in m.items()}
        return DenseNet(layers, cv(doc["weights"]), cv(doc["biases"]), cv(doc["bases"]), doc.get("seed"))


def filter_from_basis(U: np.ndarray):
    """Fixed filter layer I - U U^T. Returns (LayerSpec, U); the
    weights delta_ij - sum_k U_ik U_jk are applied in factored form."""
    U = np.asarray(U, dtype=float)
    err = np.abs(U.T @ U - np.eye(U.shape[1])).max() if U.size else 0.0
    if err > 1e-8:
        raise ValueError(f"basis is not orthonormal (||U^T U - I|| = {err:.2e})")
    return LayerSpec("filter", U.shape[0], U.shape[0], False), U


def init_weights(spec, seed):
    """U(-sqrt(6/fan_in), +sqrt(6/fan_in)) weights and biases."""
    specs = spec if isinstance(spec, (list, tuple)) else [spec]
    rng = np.random.default_rng(seed)
    W, b = {}, {}
    for i, s in enumerate(specs):
        if s.kind == "fully_connected":
            lim = np.sqrt(6.0 / s.in_dim)
            W[i] = rng.uniform(-lim, lim, (s.out_dim, s.in_dim))
            b[i] = rng.uniform(-lim, lim, s.out_dim)
    return (W, b) if isinstance(spec, (list, tuple)) else (W.get(0), b.get(0))


def _as_parts(x, dim):
    """Returns (parts (2^k, dim, B), order, kind) for real vectors/batches or MCArray."""
    if isinstance(x, MCArray):
        p = x.parts
        if p.ndim == 2:
            return _lib.f64(p[:, :, None]), x.order, "mc1"
        return _lib.f64(p), x.order, "mc2"
    a = np.asarray(x, dtype=float)
    if a.ndim == 1:
        return _lib.f64(a[None, :, None]), 0, "r1"
    return _lib.f64(a[None]), 0, "r2"


def _from_parts(p, kind):
    if kind == "r1":
        return p[0, :, 0]
    if kind == "r2":
        return p[0]
    if kind == "mc1":
        return MCArray(p[:, :, 0])
    return MCArray(p)


def forward(net: DenseNet, x):
    """Forward over real (vector or (dim, batch)) or MCArray inputs of order <= 3."""
    parts, order, kind = _as_parts(x, net.in_dim)
    if parts.shape[1] != net.in_dim:
        raise ValueError("dimension mismatch (SPEC.md:143)")
    if order > MAX_ORDER:
        raise OrderError("order > 3")
    B = parts.shape[2]
    out = np.empty((parts.shape[0], net.out_dim, B))
    L = _lib.lib()
    h = net.handle()
    _lib.check(L.nlrom_net_forward(h, order, _lib.dptr(parts), B, _lib.dptr(out)),
               lambda: L.nlrom_net_last_error(h))
    return _from_parts(out, kind)


def backward(net: DenseNet, x, upstream, want_params: bool = False):
    """Reverse mode in real or order-1 complex arithmetic.

    Returns the input cotangent (same container as x) and, if ``want_params``,
    a list of (dW, db) per FC layer (MCArray-style part stacks for complex)."""
    parts, order, kind = _as_parts(x, net.in_dim)
    up, order_u, _ = _as_parts(upstream, net.out_dim)
    if order > 1:
        raise OrderError("backward supports real or order-1 complex scalars (SPEC.md:149)")
    if order_u != order:
        up2 = np.zeros((1 << order,) + up.shape[1:])
        up2[: up.shape[0]] = up
        up = up2
    if up.shape[1] != net.out_dim or up.shape[2] != parts.shape[2]:
        raise ValueError("dimension mismatch")
    S, B = parts.shape[0], parts.shape[2]
    out = np.empty((S, net.in_dim, B))
    n_par = sum(S * s.out_dim * s.in_dim + S * s.out_dim for s in net.layers if s.kind == "fully_connected")
    pc = np.empty(max(n_par, 1)) if want_params else None
    L = _lib.lib()
    h = net.handle()
    _lib.check(L.nlrom_net_backward(h, order, _lib.dptr(parts), _lib.dptr(_lib.f64(up)), B, _lib.dptr(out),
                                    _lib.dptr(pc) if want_params else None),
               lambda: L.nlrom_net_last_error(h))
    res = _from_parts(out, kind)
    if not want_params:
        return res
    grads, off = [], 0
    for s in net.layers:
        if s.kind != "fully_connected":
            continue
        nW, nb = S * s.out_dim * s.in_dim, S * s.out_dim
        dW = pc[off:off + nW].reshape(S, s.out_dim, s.in_dim)
        db = pc[off + nW:off + nW + nb].reshape(S, s.out_dim)
        off += nW + nb
        grads.append((dW[0], db[0]) if S == 1 else (dW, db))
    return res, grads


def lr_at(cfg: TrainConfig, epoch: int) -> float:
    """Learning rate in effect during ``epoch`` (0-based): the base rate times every schedule
    factor whose epoch has been completed ({300: 0.8, 3000: 0.8} from 1e-3 gives
    6.4e-4 after epoch 3000)."""
    lr = float(cfg.learning_rate)
    for e, f in sorted((cfg.schedule or {}).items()):
        if epoch >= int(e):
            lr *= float(f)
    return lr


def _torch_forward(net: DenseNet, params, x):
    """Differentiable forward of a real DenseNet on a (batch, in_dim) tensor (layers as in
    ``forward``; params: {layer index: (W, b)} tensors; filter bases from the net)."""
    import torch
    h = x
    for i, s in enumerate(net.layers):
        if s.kind == "fully_connected":
            W, b = params[i]
            h = h @ W.T + b
        elif s.kind == "filter":
            U = torch.as_tensor(net.bases[i], dtype=h.dtype, device=h.device)
            h = h - (h @ U) @ U.T
        elif s.kind == "activation_sin":
            h = torch.sin(h)
        elif s.kind == "activation_square":
            h = h * h
        elif s.kind == "activation_softmax":
            h = torch.softmax(h, dim=-1)
    return h


def adam_train(net: DenseNet, dataset, loss="mse", cfg: TrainConfig | None = None, device=None, seed=None):
    """Adam training of a DenseNet (§5.2 "use PyTorch and Adam").

    dataset: (X, Y) with X (S, in_dim) and Y (S, out_dim). loss: "mse" -- per-sample mean squared
    error over the output components -- or a callable (pred, target) -> per-sample losses. The
    per-sample losses are multiplied by ``cfg.sample_weights`` (default 1) and averaged; the
    learning rate follows ``cfg.schedule`` (``lr_at``); minibatches are shuffled by ``seed``
    (default net.seed or 0). fp64 torch on CUDA when available. Returns (trained copy of net,
    epoch-loss curve); a NaN loss raises FloatingPointError with the epoch and batch."""
    import torch
    cfg = cfg or TrainConfig()
    X, Y = (np.asarray(a, dtype=float) for a in dataset)
    if X.ndim != 2 or Y.ndim != 2 or X.shape[0] != Y.shape[0] or X.shape[0] == 0:
        raise ValueError("dataset must be (X (S, in), Y (S, out)) with S >= 1")
    if X.shape[1] != net.in_dim or Y.shape[1] != net.out_dim:
        raise ValueError("dimension mismatch (SPEC.md:143)")
    S = X.shape[0]
    w = np.ones(S) if cfg.sample_weights is None else np.asarray(cfg.sample_weights, dtype=float)
    if w.shape != (S,):
        raise ValueError("sample_weights must have one entry per sample")
    dev = torch.device(device) if device is not None else (
        torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    dt = torch.float64
    fcs = [i for i, s in enumerate(net.layers) if s.kind == "fully_connected"]
    params = {i: (torch.tensor(net.weights[i], dtype=dt, device=dev, requires_grad=True),
                  torch.tensor(net.biases[i], dtype=dt, device=dev, requires_grad=True)) for i in fcs}
    opt = torch.optim.Adam([p for i in fcs for p in params[i]], lr=lr_at(cfg, 0))
    Xt, Yt, wt = (torch.as_tensor(a, dtype=dt, device=dev) for a in (X, Y, w))
    per_sample = (lambda p, t: ((p - t) ** 2).mean(dim=1)) if loss == "mse" else loss
    gen = torch.Generator(device="cpu")
    gen.manual_seed(int(seed if seed is not None else (net.seed or 0)))
    bs = max(1, min(int(cfg.batch_size), S))
    curve = []
    for epoch in range(int(cfg.epochs)):
        for g in opt.param_groups:
            g["lr"] = lr_at(cfg, epoch)
        perm = torch.randperm(S, generator=gen).to(dev)
        tot = 0.0
        for b0 in range(0, S, bs):
            idx = perm[b0:b0 + bs]
            l = (per_sample(_torch_forward(net, params, Xt[idx]), Yt[idx]) * wt[idx]).sum() / S
            if not torch.isfinite(l):
                raise FloatingPointError(f"adam_train: non-finite loss at epoch {epoch}, batch {b0 // bs}")
            opt.zero_grad(set_to_none=True)
            l.backward()
            opt.step()
            tot += float(l.detach())
        curve.append(tot)
    out = DenseNet(net.layers, {i: params[i][0].detach().cpu().numpy().copy() for i in fcs},
                   {i: params[i][1].detach().cpu().numpy().copy() for i in fcs}, dict(net.bases), net.seed)
    return out, curve


def make_decoder(Ws, bs, U):
    """Decoder D of the DAE: FC(sin)^(L-1) -> FC -> filter(U) (Fig. 3)."""
    layers, W, b = [], {}, {}
    for l, (Wl, bl) in enumerate(zip(Ws, bs)):
        i = len(layers)
        layers.append(LayerSpec("fully_connected", Wl.shape[1], Wl.shape[0]))
        W[i], b[i] = np.asarray(Wl, dtype=float), np.asarray(bl, dtype=float)
        if l < len(Ws) - 1:
            layers.append(LayerSpec("activation_sin", Wl.shape[0], Wl.shape[0], False))
    spec, Uf = filter_from_basis(U)
    layers.append(spec)
    return DenseNet(layers, W, b, {len(layers) - 1: Uf})


def make_wnet(Ws, bs):
    """Weight net W: 4 FC layers, sin after the first three, square at the end."""
    layers, W, b = [], {}, {}
    for l, (Wl, bl) in enumerate(zip(Ws, bs)):
        i = len(layers)
        layers.append(LayerSpec("fully_connected", Wl.shape[1], Wl.shape[0]))
        W[i], b[i] = np.asarray(Wl, dtype=float), np.asarray(bl, dtype=float)
        kind = "activation_sin" if l < len(Ws) - 1 else "activation_square"
        layers.append(LayerSpec(kind, Wl.shape[0], Wl.shape[0], False))
    return DenseNet(layers, W, b)


def decoder_parts(net: DenseNet):
    """(Ws, bs, U) of a decoder laid out as FC(sin)^(L-1) -> FC -> filter."""
    Ws, bs, U = [], [], None
    for i, s in enumerate(net.layers):
        if s.kind == "fully_connected":
            Ws.append(net.weights[i])
            bs.append(net.biases[i])
        elif s.kind == "filter":
            U = net.bases[i]
    return Ws, bs, U

"""nlrom.daereduce — PCA + PCA-orthogonal DAE subspace (Eq. 9-10)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .densenet import DenseNet


class ReducedModel:
    """U (N x n_p), decoder D (ends with the filter I - U U^T), dims.

    Queries that need only the decoder and U use a device session; the mass matrix
    comes from the ElasticModel attached with ``attach``."""

    def __init__(self, U, decoder: DenseNet, n_p: int, n_q: int, encoder: DenseNet | None = None):
        self.U = np.ascontiguousarray(U, dtype=float)
        self.decoder, self.encoder = decoder, encoder
        self.n_p, self.n_q = int(n_p), int(n_q)
        if self.U.shape[1] != self.n_p:
            raise ValueError("U must be N x n_p")
        self.model = None
        self.cm = None

    @property
    def n(self):
        return self.n_p + self.n_q

    def attach(self, model, cm=None):
        """Bind the FE model (and cubature model) whose mesh the decoder lives on."""
        self.model, self.cm = model, cm
        return self

    def session(self):
        from .session import session_for
        if self.model is None:
            raise ValueError("attach an ElasticModel first (ReducedModel.attach)")
        return session_for(self, self.model, self.cm)


@dataclass
class ReducedState:
    """r = (p, q), rdot, dt."""
    r: np.ndarray
    rdot: np.ndarray
    dt: float = 1.0 / 60.0

    def __post_init__(self):
        self.r = np.asarray(self.r, dtype=float).copy()
        self.rdot = np.asarray(self.rdot, dtype=float).copy()
        _check_state(self.r, self.rdot)

    @classmethod
    def _owned(cls, r, rdot, dt):
        """A state around fresh float64 arrays the caller gives up (no copies): rdsim.step's
        device outputs. Same validation as the constructor."""
        st = object.__new__(cls)
        st.r, st.rdot, st.dt = r, rdot, dt
        _check_state(r, rdot)
        return st


def _check_state(r, rdot):
    if r.shape != rdot.shape or not (np.isfinite(r).all() and np.isfinite(rdot).all()):
        raise ValueError("ReducedState must be finite with matching r / rdot (SPEC.md:452)")


def _split(rm, r):
    r = np.asarray(r, dtype=float)
    return r[: rm.n_p], r[rm.n_p:]


def full_displacement(rm: ReducedModel, r) -> np.ndarray:
    """u = U p + D(q) (Eq. 9)."""
    return rm.session().full_displacement(r)


def jtilde(rm: ReducedModel, q) -> np.ndarray:
    """J~ = [U, J(q)] (N x (n_p + n_q), Eq. 10)."""
    return rm.session().jtilde(q)


def reduced_mass(rm: ReducedModel, q, model=None) -> np.ndarray:
    """J~^T M J~ (Eq. 10): the mass block of the exact_sum system
    Jacobian with dt = 0 and zero state offsets."""
    from .rdsim import SimConfig
    from .session import session_for
    s = rm.session() if model is None else session_for(rm, model, rm.cm)
    r = np.concatenate([np.zeros(rm.n_p), np.asarray(q, dtype=float)])
    # The device system Jacobian at r = r_bar, rdot_bar = 0, f_ext = 0, drop_fict and
    # dt -> 0 is exactly the mass block J~^T M [U, J] (dJ, vhp(a), dt^2 K all vanish).
    cfg = SimConfig(dt=1e-30, integration="exact_sum", drop_fict=True)
    return s.system_jacobian(r, r, np.zeros(rm.n), np.zeros(s.N), cfg)


def encode(rm: ReducedModel, u):
    """(p, q) = (U^T u, encoder(u)); needs a trained encoder."""
    from .densenet import forward
    if rm.encoder is None:
        raise ValueError("no encoder: DAE training is offline (SURVEY.md §2)")
    u = np.asarray(u, dtype=float)
    return rm.U.T @ u, forward(rm.encoder, u)


@dataclass
class DAEArch:
    """Decoder depth (FC layers, >= 4), hidden width (default ceil(4 log2 N)) and
    latent dim n_q; the encoder mirrors the decoder (Fig. 3)."""
    depth: int = 6
    n_q: int = 4
    width: int | None = None


def _dae_layers(N, arch: DAEArch, U, seed):
    """Encoder filter -> FC(sin)^(depth-1) -> FC -> q and decoder FC(sin)^(depth-1) -> FC -> filter
    (filter_from_basis(U) at the input of the encoder and the output of the
    decoder), weights U(+-sqrt(6/fan_in)) from ``seed``."""
    from .densenet import DenseNet, LayerSpec, filter_from_basis, init_weights
    w = arch.width or int(np.ceil(4 * np.log2(max(N, 2))))
    fspec, Uf = filter_from_basis(U)

    def chain(dims, filt_first):
        layers, bases = [], {}
        if filt_first:
            layers.append(fspec)
            bases[0] = Uf
        for l in range(len(dims) - 1):
            layers.append(LayerSpec("fully_connected", dims[l], dims[l + 1]))
            if l < len(dims) - 2:
                layers.append(LayerSpec("activation_sin", dims[l + 1], dims[l + 1], False))
        if not filt_first:
            bases[len(layers)] = Uf
            layers.append(fspec)
        return layers, bases

    enc_l, enc_b = chain([N] + [w] * (arch.depth - 1) + [arch.n_q], True)
    dec_l, dec_b = chain([arch.n_q] + [w] * (arch.depth - 1) + [N], False)
    We, be = init_weights(enc_l, seed)
    Wd, bd = init_weights(dec_l, seed + 1)
    return DenseNet(enc_l, We, be, enc_b, seed), DenseNet(dec_l, Wd, bd, dec_b, seed + 1)


def build_dae(ps, U, arch: DAEArch | None = None, cfg=None, seed: int = 0, device=None):
    """PCA + PCA-orthogonal DAE (Eq. 9, Fig. 3).

    Trains encoder and decoder jointly (untied, SPEC.md open question) with Adam on the
    energy-weighted mean squared error of the PCA residual: for every pose u (column of
    ps.poses), q = E(u) and the loss is ||D(q) - (I - U U^T) u||^2 / N, weighted by ps.weights
    (posegen.energy_weights). Returns a ReducedModel (decoder laid out FC(sin)^(L-1) -> FC ->
    filter, as the device context expects) with ``loss_curve``; NaN training raises."""
    import torch
    from .densenet import TrainConfig, DenseNet, _torch_forward, lr_at
    arch = arch or DAEArch()
    cfg = cfg or TrainConfig(epochs=500, batch_size=64)
    if arch.depth < 4 or arch.n_q < 1:
        raise ValueError("build_dae needs depth >= 4 and n_q >= 1 (SPEC.md:459)")
    Uc = np.ascontiguousarray(U, dtype=float)
    X = np.ascontiguousarray(np.asarray(ps.poses, dtype=float).T)   # (T, N)
    T, N = X.shape
    if Uc.shape[0] != N:
        raise ValueError("dimension mismatch: U must be N x n_p")
    enc, dec = _dae_layers(N, arch, Uc, seed)
    dev = torch.device(device) if device is not None else (
        torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    dt = torch.float64
    pe = {i: (torch.tensor(enc.weights[i], dtype=dt, device=dev, requires_grad=True),
              torch.tensor(enc.biases[i], dtype=dt, device=dev, requires_grad=True)) for i in enc.weights}
    pd = {i: (torch.tensor(dec.weights[i], dtype=dt, device=dev, requires_grad=True),
              torch.tensor(dec.biases[i], dtype=dt, device=dev, requires_grad=True)) for i in dec.weights}
    opt = torch.optim.Adam([p for d in (pe, pd) for v in d.values() for p in v], lr=lr_at(cfg, 0))
    Xt = torch.as_tensor(X, dtype=dt, device=dev)
    Ut = torch.as_tensor(Uc, dtype=dt, device=dev)
    Rt = Xt - (Xt @ Ut) @ Ut.T                       # PCA residual targets
    w = np.asarray(ps.weights if getattr(ps, "weights", None) is not None else np.ones(T), dtype=float)
    if cfg.sample_weights is not None:
        w = w * np.asarray(cfg.sample_weights, dtype=float)
    wt = torch.as_tensor(w, dtype=dt, device=dev)
    gen = torch.Generator(device="cpu")
    gen.manual_seed(int(seed))
    bs = max(1, min(int(cfg.batch_size), T))
    curve = []
    for epoch in range(int(cfg.epochs)):
        for g in opt.param_groups:
            g["lr"] = lr_at(cfg, epoch)
        perm = torch.randperm(T, generator=gen).to(dev)
        tot = 0.0
        for b0 in range(0, T, bs):
            idx = perm[b0:b0 + bs]
            rec = _torch_forward(dec, pd, _torch_forward(enc, pe, Xt[idx]))
            l = ((((rec - Rt[idx]) ** 2).mean(dim=1)) * wt[idx]).sum() / T
            if not torch.isfinite(l):
                raise FloatingPointError(f"build_dae: non-finite loss at epoch {epoch}")
            opt.zero_grad(set_to_none=True)
            l.backward()
            opt.step()
            tot += float(l.detach())
        curve.append(tot)
    enc_t = DenseNet(enc.layers, {i: v[0].detach().cpu().numpy().copy() for i, v in pe.items()},
                     {i: v[1].detach().cpu().numpy().copy() for i, v in pe.items()}, dict(enc.bases), enc.seed)
    dec_t = DenseNet(dec.layers, {i: v[0].detach().cpu().numpy().copy() for i, v in pd.items()},
                     {i: v[1].detach().cpu().numpy().copy() for i, v in pd.items()}, dict(dec.bases), dec.seed)
    rm = ReducedModel(Uc, dec_t, Uc.shape[1], arch.n_q, encoder=enc_t)
    rm.loss_curve = curve
    return rm


def dae_reconstruction(rm: ReducedModel, poses, device=None) -> np.ndarray:
    """Host / torch evaluation of u -> U U^T u + D(E(u)) for poses (N, T) (training checks; the
    simulation path uses the device context)."""
    import torch
    from .densenet import _torch_forward
    dt = torch.float64
    dev = torch.device(device) if device is not None else torch.device("cpu")

    def params(net):
        return {i: (torch.as_tensor(net.weights[i], dtype=dt, device=dev),
                    torch.as_tensor(net.biases[i], dtype=dt, device=dev)) for i in net.weights}
    X = torch.as_tensor(np.asarray(poses, dtype=float).T, dtype=dt, device=dev)
    U = torch.as_tensor(rm.U, dtype=dt, device=dev)
    with torch.no_grad():
        rec = (X @ U) @ U.T + _torch_forward(rm.decoder, params(rm.decoder),
                                             _torch_forward(rm.encoder, params(rm.encoder), X))
    return rec.cpu().numpy().T

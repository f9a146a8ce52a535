"""Synthetic, seeded inputs for the DAE-subspace step.

No trained artifacts or meshes ship with the reference (/examples and /vendor are
stripped, pkg/.gitignore:1-2), so every config is generated here:

* meshes: structured nx x ny x nz boxes of unit cubes of edge ``h``, 6 tets per
  cube (Kuhn/Freudenthal split along the main diagonal, conforming), the x = 0
  face fixed (Dirichlet by DOF elimination);
* decoder: n_q -> w x (L-1) FC(sin) -> FC -> filter(U),
  weights and biases U(+-sqrt(6/fan_in)) from ``default_rng(0)`` (
  nonzero biases); the last FC layer is scaled by ``out_scale`` so the
  decoded displacements are physically small (random init, not a trained model);
* U = Q of QR(default_rng(1).standard_normal((N, n_p)));
* cubature set C = sorted(default_rng(2).choice(T, |C|, replace=False));
* weight net (seed 3): N -> wn -> wn -> wn (sin) -> T, then square;
* states (seed 4): q ~ U(-.5,.5), q_bar = q - U(-.05,.05), qdot_bar ~ U(-1,1),
  p likewise x 1e-2;
* material: E = 5e5 Pa, nu = 0.45, rho = 1000 kg/m^3, alpha = 0.1 1/s; gravity
  f_ext = M (0, -9.81, 0); dt = 1/60 s.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np


# ---------------------------------------------------------------------------
# meshes
# ---------------------------------------------------------------------------

def box_mesh(nx: int, ny: int, nz: int, h: float = 0.1):
    """Vertices (V,3), tets (T,4) int32 with positive volume, fixed mask (x == 0)."""
    gx, gy, gz = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    verts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1).astype(float) * h

    def vid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    corner = [(c & 1, (c >> 1) & 1, (c >> 2) & 1) for c in range(8)]
    paths = []
    for perm in itertools.permutations(range(3)):
        cur = [0, 0, 0]
        path = [0]
        for ax in perm:
            cur[ax] = 1
            path.append(cur[0] | (cur[1] << 1) | (cur[2] << 2))
        paths.append(path)
    tets = []
    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                ids = [vid(i + a, j + b, k + c) for (a, b, c) in corner]
                for p in paths:
                    tets.append([ids[c] for c in p])
    tets = np.asarray(tets, dtype=np.int64)
    X = verts[tets]
    det = np.linalg.det(np.transpose(X[:, 1:] - X[:, :1], (0, 2, 1)))
    neg = det < 0
    tets[neg, 2], tets[neg, 3] = tets[neg, 3].copy(), tets[neg, 2].copy()
    fixed = verts[:, 0] == 0.0
    return verts, tets.astype(np.int32), fixed


# ---------------------------------------------------------------------------
# networks
# ---------------------------------------------------------------------------

def uniform_layer(rng, out_dim, in_dim):
    lim = math.sqrt(6.0 / in_dim)
    return rng.uniform(-lim, lim, (out_dim, in_dim)), rng.uniform(-lim, lim, out_dim)


def decoder_weights(n_q: int, width: int, n_fc: int, N: int, seed: int = 0, out_scale: float = 1e-3,
                    zero_bias: bool = False, rest_at_zero: bool = True):
    """Weights/biases of the n_fc FC layers n_q -> width^(n_fc-1) -> N.

    ``rest_at_zero`` sets the last bias to -W_L h(0) so that D(0) = 0, i.e. r = 0
    is the rest pose, as for a decoder trained on poses that include the rest
    pose."""
    rng = np.random.default_rng(seed)
    dims = [n_q] + [width] * (n_fc - 1) + [N]
    Ws, bs = [], []
    for l in range(n_fc):
        W, b = uniform_layer(rng, dims[l + 1], dims[l])
        if l == n_fc - 1:
            W, b = W * out_scale, b * out_scale
        if zero_bias:
            b = np.zeros_like(b)
        Ws.append(W)
        bs.append(b)
    if rest_at_zero and not zero_bias:
        h = np.zeros(n_q)
        for l in range(n_fc - 1):
            h = np.sin(Ws[l] @ h + bs[l])
        bs[-1] = -(Ws[-1] @ h)
    return Ws, bs


def wnet_weights(N: int, width: int, T: int, seed: int = 3):
    rng = np.random.default_rng(seed)
    dims = [N, width, width, width, T]
    Ws, bs = [], []
    for l in range(4):
        W, b = uniform_layer(rng, dims[l + 1], dims[l])
        Ws.append(W)
        bs.append(b)
    return Ws, bs


def pca_like_basis(N: int, n_p: int, seed: int = 1):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((N, n_p)))
    return np.ascontiguousarray(q)


def decoder_layers(Ws, bs, U):
    """Plain layer-dict list (oracle format): FC(sin)^(L-1) -> FC -> filter."""
    layers = []
    for l, (W, b) in enumerate(zip(Ws, bs)):
        layers.append({"kind": "fc", "W": W, "b": b})
        if l < len(Ws) - 1:
            layers.append({"kind": "sin"})
    layers.append({"kind": "filter", "U": U})
    return layers


def wnet_layers(Ws, bs):
    layers = []
    for l, (W, b) in enumerate(zip(Ws, bs)):
        layers.append({"kind": "fc", "W": W, "b": b})
        layers.append({"kind": "sin"} if l < len(Ws) - 1 else {"kind": "square"})
    return layers


# ---------------------------------------------------------------------------
# configs
# ---------------------------------------------------------------------------

@dataclass
class SynthConfig:
    name: str
    mesh: tuple            # (nx, ny, nz)
    n_q: int
    n_p: int
    n_fc: int              # number of FC layers of the decoder ("L-layer DAE")
    width: int
    n_cub: int
    wnet_width: int
    h: float = 0.1
    out_scale: float = 1e-3
    young: float = 5e5
    poisson: float = 0.45
    density: float = 1000.0
    alpha: float = 0.1
    dt: float = 1.0 / 60.0
    n_sims: int = 1
    extra: dict = field(default_factory=dict)


CONFIGS = {
    # cantilever beam, 5-layer DAE (BASELINE.json configs[0])
    "cfg1": SynthConfig("cfg1", (20, 3, 3), n_q=5, n_p=10, n_fc=5, width=40, n_cub=100, wnet_width=32),
    # ~10k-tet mesh, 10-layer width-256 DAE, n_q=30, 500 cubature points (configs[1]; the metric)
    "cfg2": SynthConfig("cfg2", (35, 7, 7), n_q=30, n_p=30, n_fc=10, width=256, n_cub=500, wnet_width=64),
    # one puffer-ball string (configs[3]); 320 of them per scene
    "cfg4": SynthConfig("cfg4", (36, 3, 3), n_q=5, n_p=10, n_fc=8, width=64, n_cub=36, wnet_width=32),
    # batched independent sims on the cfg1 mesh (configs[4])
    "cfg5": SynthConfig("cfg5", (20, 3, 3), n_q=20, n_p=10, n_fc=10, width=256, n_cub=100, wnet_width=32,
                        n_sims=4096),
    # tiny config for fast CPU tests
    "tiny": SynthConfig("tiny", (4, 2, 2), n_q=3, n_p=4, n_fc=4, width=8, n_cub=12, wnet_width=8),
}


def build(cfg, seed_offset: int = 0):
    """All arrays of one synthetic problem as a dict (host numpy, float64/int32)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    verts, tets, fixed = box_mesh(*cfg.mesh, h=cfg.h)
    N = 3 * int((~fixed).sum())
    T = tets.shape[0]
    Ws, bs = decoder_weights(cfg.n_q, cfg.width, cfg.n_fc, N, seed=0, out_scale=cfg.out_scale)
    U = pca_like_basis(N, cfg.n_p, seed=1)
    cub = np.sort(np.random.default_rng(2).choice(T, min(cfg.n_cub, T), replace=False)).astype(np.int32)
    wW, wb = wnet_weights(N, cfg.wnet_width, T, seed=3)
    return {
        "cfg": cfg, "verts": verts, "tets": tets, "fixed": fixed, "N": N, "T": T,
        "dec_W": Ws, "dec_b": bs, "U": U, "cub": cub, "wnet_W": wW, "wnet_b": wb,
    }


def random_state(n_p: int, n_q: int, seed: int = 4):
    """(q, q_bar, qdot_bar, p, p_bar, pdot_bar) per SURVEY.md §8d."""
    rng = np.random.default_rng(seed)
    q = rng.uniform(-0.5, 0.5, n_q)
    q_bar = q - rng.uniform(-0.05, 0.05, n_q)
    qdot_bar = rng.uniform(-1.0, 1.0, n_q)
    p = 1e-2 * rng.uniform(-0.5, 0.5, n_p)
    p_bar = p - 1e-2 * rng.uniform(-0.05, 0.05, n_p)
    pdot_bar = 1e-2 * rng.uniform(-1.0, 1.0, n_p)
    return q, q_bar, qdot_bar, p, p_bar, pdot_bar


def gravity(mass: np.ndarray, g: float = -9.81):
    """f_ext = M (0, g, 0) on the free DOFs."""
    f = np.zeros_like(mass)
    f[1::3] = mass[1::3] * g
    return f


def string_frames(k: int) -> np.ndarray:
    """(k, 3, 3) rotations string frame -> world for k strings on a sphere (puffer ball,
    PAPER.md:84): local +x (the string axis, fixed face at x = 0) -> the s-th Fibonacci-sphere
    direction; the other two columns complete a right-handed orthonormal frame."""
    i = np.arange(k) + 0.5
    z = 1.0 - 2.0 * i / k
    rho = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = np.pi * (3.0 - np.sqrt(5.0)) * i
    d = np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=1)
    R = np.zeros((k, 3, 3))
    for s in range(k):
        e1 = d[s]
        helper = np.array([0.0, 0.0, 1.0]) if abs(e1[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
        e2 = np.cross(helper, e1)
        e2 /= np.linalg.norm(e2)
        e3 = np.cross(e1, e2)
        R[s] = np.stack([e1, e2, e3], axis=1)
    return R


def coupled_state(k: int, n_p: int, n_q: int, seed: int = 7, scale: float = 0.1):
    """Small seeded per-string states (r_bar, rdot_bar) (k, n) and core (c_bar, cdot_bar)."""
    rng = np.random.default_rng(seed)
    n = n_p + n_q
    rb = scale * rng.uniform(-0.5, 0.5, (k, n))
    rb[:, :n_p] *= 1e-2
    rdb = scale * rng.uniform(-1.0, 1.0, (k, n))
    rdb[:, :n_p] *= 1e-2
    return rb, rdb, 1e-3 * rng.uniform(-1, 1, 3), 1e-2 * rng.uniform(-1, 1, 3)

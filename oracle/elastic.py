"""Oracle tetrahedral StVK model (TEST INFRASTRUCTURE).

Restates SPEC.md [MODULE] elastic: P1 tets with one-point
quadrature, StVK energy density
    Psi = mu ||E||_F^2 + lambda/2 tr(E)^2,   E = (F^T F - I)/2,
internal force f_int = +dE_elastic/du, per-element stiffness
dF_int/du, lumped mass (rho V / 4 per vertex on each coordinate),
Dirichlet constraints by DOF elimination.

Element vectors are vertex-major 12-vectors [v0x v0y v0z v1x ... v3z].
All routines are dtype-generic so they can run on complex displacements (the
outer CSFD direction of rdsim.jacobian_oracle).
"""

from __future__ import annotations

import numpy as np


class OModel:
    """Mesh + material + derived rest data (oracle-side, independent of the product)."""

    def __init__(self, verts, tets, fixed, young, poisson, density, alpha=0.0):
        self.verts = np.asarray(verts, dtype=float)
        self.tets = np.asarray(tets, dtype=np.int64)
        fixed = np.asarray(fixed, dtype=bool)
        self.fixed = fixed
        V = self.verts.shape[0]
        self.dof = -np.ones(V, dtype=np.int64)
        free = np.nonzero(~fixed)[0]
        self.dof[free] = np.arange(free.size)
        self.N = 3 * free.size
        self.mu = young / (2.0 * (1.0 + poisson))
        self.lam = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))
        self.density = density
        self.alpha = alpha
        X = self.verts[self.tets]                       # (T,4,3)
        Dm = np.transpose(X[:, 1:] - X[:, :1], (0, 2, 1))  # columns X_i - X_0
        det = np.linalg.det(Dm)
        if np.any(det <= 0):
            raise ValueError("non-positive tet volume")
        self.Dm_inv = np.linalg.inv(Dm)
        self.vol = det / 6.0
        mv = np.zeros(V)
        np.add.at(mv, self.tets.ravel(), np.repeat(density * self.vol / 4.0, 4))
        self.vertex_mass = mv
        self.mass = np.repeat(mv[free], 3)              # (N,) lumped, free DOFs only
        # 12 free-DOF rows per element (-1 for fixed vertices)
        d = self.dof[self.tets]                          # (T,4)
        rows = 3 * d[:, :, None] + np.arange(3)[None, None, :]
        rows[d < 0] = -1
        self.rows = rows.reshape(-1, 12)
        # gradient vectors g_j (rows of Dm^-1, g_0 = -sum)
        G = np.empty((self.tets.shape[0], 4, 3))
        G[:, 1:] = self.Dm_inv
        G[:, 0] = -self.Dm_inv.sum(axis=1)
        self.G = G

    @property
    def n_tets(self):
        return self.tets.shape[0]

    def vertex_disp(self, u):
        """Free-DOF vector (N,) -> per-vertex displacements (V,3), zeros at fixed."""
        u = np.asarray(u)
        out = np.zeros((self.verts.shape[0], 3), dtype=np.result_type(u.dtype, np.float64))
        free = self.dof >= 0
        out[free] = u.reshape(-1, 3)
        return out


def _deformation(model, u, elems):
    uv = model.vertex_disp(u)[model.tets[elems]]        # (E,4,3)
    Ds = np.transpose(uv[:, 1:] - uv[:, :1], (0, 2, 1))  # (E,3,3) columns u_i - u_0
    return np.eye(3) + Ds @ model.Dm_inv[elems]


def _stress(model, F):
    E = 0.5 * (np.swapaxes(F, -1, -2) @ F - np.eye(3))
    tr = np.trace(E, axis1=-2, axis2=-1)
    S = 2.0 * model.mu * E + model.lam * tr[..., None, None] * np.eye(3)
    return E, tr, S


def stvk_energy(model, u):
    elems = np.arange(model.n_tets)
    F = _deformation(model, u, elems)
    E, tr, _ = _stress(model, F)
    psi = model.mu * np.sum(E * E, axis=(-2, -1)) + 0.5 * model.lam * tr**2
    return np.sum(model.vol * psi)


def element_force_stiffness(model, u, elems=None, want_K=True):
    """Per-element f_e (E,12) and K_e (E,12,12) at free-DOF displacement u."""
    if elems is None:
        elems = np.arange(model.n_tets)
    elems = np.asarray(elems, dtype=np.int64)
    F = _deformation(model, u, elems)
    _, _, S = _stress(model, F)
    P = F @ S
    vol = model.vol[elems]
    G = model.G[elems]                                  # (E,4,3)
    # f_{i,a} = V sum_b P_ab g_i[b]
    f = vol[:, None, None] * np.einsum("eab,eib->eia", P, G)
    f = f.reshape(-1, 12)
    if not want_K:
        return f, None
    nE = elems.size
    # dF for the 12 unit DOF directions (j,d): dF_ab = delta_ad g_j[b]
    dF = np.zeros((nE, 4, 3, 3, 3), dtype=F.dtype)
    for d in range(3):
        dF[:, :, d, d, :] = G
    dF = dF.reshape(nE, 12, 3, 3)
    Fb = F[:, None]
    Sb = S[:, None]
    dE = 0.5 * (np.swapaxes(dF, -1, -2) @ Fb + np.swapaxes(Fb, -1, -2) @ dF)
    trdE = np.trace(dE, axis1=-2, axis2=-1)
    dS = 2.0 * model.mu * dE + model.lam * trdE[..., None, None] * np.eye(3)
    dP = dF @ Sb + Fb @ dS                               # (E,12,3,3)
    K = vol[:, None, None, None] * np.einsum("ejab,eib->eiaj", dP, G)  # (E,4,3,12)
    return f, K.reshape(nE, 12, 12)


def scatter(model, fe, elems, weights=None):
    """Assemble element 12-vectors into the free-DOF vector (N,)."""
    rows = model.rows[elems]
    vals = fe if weights is None else fe * np.asarray(weights)[:, None]
    out = np.zeros(model.N, dtype=np.result_type(vals.dtype, np.float64))
    m = rows >= 0
    np.add.at(out, rows[m], vals[m])
    return out


def internal_force(model, u):
    elems = np.arange(model.n_tets)
    f, _ = element_force_stiffness(model, u, elems, want_K=False)
    return scatter(model, f, elems)


def stiffness_dense(model, u):
    elems = np.arange(model.n_tets)
    _, K = element_force_stiffness(model, u, elems)
    out = np.zeros((model.N, model.N), dtype=K.dtype)
    rows = model.rows
    for e in range(model.n_tets):
        r = rows[e]
        m = r >= 0
        out[np.ix_(r[m], r[m])] += K[e][np.ix_(m, m)]
    return out

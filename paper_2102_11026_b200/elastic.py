"""nlrom.elastic — tetrahedral StVK model.

Mesh / material / lumped-mass setup is host-side (one-time upload). The per-element
StVK force and stiffness used on the hot path run on the GPU (k_cubature in
csrc/sim_kernels.cuh): ``internal_force`` / ``stiffness`` / ``element_reduced_force``
go through the C ABI. ``stvk_energy`` is a test-support utility (SURVEY.md §2:
"OUT OF SCOPE on GPU — test support only").
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class TetMesh:
    """vertices (V,3) m; tets (T,4) int; surface triangles (optional)."""
    vertices: np.ndarray
    tets: np.ndarray
    surface: np.ndarray | None = None

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=float)
        self.tets = np.asarray(self.tets, dtype=np.int32)
        if self.tets.min() < 0 or self.tets.max() >= self.vertices.shape[0]:
            raise ValueError("tet index out of range")


@dataclass
class Material:
    """SPEC.md:309-312."""
    young: float = 5e5
    poisson: float = 0.45
    density: float = 1000.0
    rayleigh_alpha: float = 0.1
    rayleigh_beta: float = 0.0

    def __post_init__(self):
        if not (self.young > 0 and 0 <= self.poisson < 0.5 and self.density > 0
                and self.rayleigh_alpha >= 0 and self.rayleigh_beta >= 0):
            raise ValueError("invalid material (SPEC.md:311)")

    @property
    def mu(self):
        return self.young / (2.0 * (1.0 + self.poisson))

    @property
    def lam(self):
        return self.young * self.poisson / ((1.0 + self.poisson) * (1.0 - 2.0 * self.poisson))


class ElasticModel:
    """Mesh + material + lumped mass on the free DOFs (Dirichlet by elimination)."""

    def __init__(self, mesh: TetMesh, material: Material, fixed):
        self.mesh, self.material = mesh, material
        fixed = np.asarray(fixed)
        if fixed.dtype != bool:
            m = np.zeros(mesh.vertices.shape[0], dtype=bool)
            m[fixed] = True
            fixed = m
        self.fixed = fixed
        V = mesh.vertices.shape[0]
        self.vert_dof = -np.ones(V, dtype=np.int32)
        free = np.nonzero(~fixed)[0]
        self.vert_dof[free] = np.arange(free.size, dtype=np.int32)
        self.N = 3 * free.size
        X = mesh.vertices[mesh.tets]
        Dm = np.transpose(X[:, 1:] - X[:, :1], (0, 2, 1))
        det = np.linalg.det(Dm)
        if np.any(det <= 0):
            raise ValueError("tets must have positive signed volume (SPEC.md:307)")
        self.Dm_inv = np.ascontiguousarray(np.linalg.inv(Dm))
        self.vol = det / 6.0
        vm = np.zeros(V)
        np.add.at(vm, mesh.tets.ravel(), np.repeat(material.density * self.vol / 4.0, 4))
        self.vertex_mass = vm
        self.mass = np.repeat(vm[free], 3)
        self._fe = None
        self._fs = None

    @property
    def n_tets(self):
        return self.mesh.tets.shape[0]

    def element_rows(self):
        d = self.vert_dof[self.mesh.tets]
        rows = 3 * d[:, :, None] + np.arange(3)[None, None, :]
        rows[d < 0] = -1
        return rows.reshape(-1, 12)


def _fe_session(model: ElasticModel):
    """GPU context holding only the FE model (placeholder 1-dim decoder, never evaluated)."""
    if model._fe is None:
        from .daereduce import ReducedModel
        from .densenet import make_decoder
        from .neucubature import CubatureModel
        from .session import Session
        N = model.N
        U = np.zeros((N, 1))
        U[0, 0] = 1.0
        dec = make_decoder([np.zeros((2, 1)), np.zeros((N, 2))], [np.zeros(2), np.zeros(N)], U)
        rm = ReducedModel(U, dec, 1, 1)
        cm = CubatureModel(np.zeros(0, dtype=np.int32), None)
        model._fe = Session(rm, model, cm)
    return model._fe


def stvk_energy(model: ElasticModel, u) -> float:
    """Sum of volume-weighted Psi = mu ||E||_F^2 + lambda/2 tr(E)^2; host, test support."""
    u = np.asarray(u)
    uv = np.zeros((model.mesh.vertices.shape[0], 3), dtype=np.result_type(u.dtype, np.float64))
    uv[model.vert_dof >= 0] = u.reshape(-1, 3)
    ue = uv[model.mesh.tets]
    Ds = np.transpose(ue[:, 1:] - ue[:, :1], (0, 2, 1))
    F = np.eye(3) + Ds @ model.Dm_inv
    E = 0.5 * (np.swapaxes(F, -1, -2) @ F - np.eye(3))
    tr = np.trace(E, axis1=-2, axis2=-1)
    psi = model.material.mu * np.sum(E * E, axis=(-2, -1)) + 0.5 * model.material.lam * tr**2
    return np.sum(model.vol * psi)


def internal_force(model: ElasticModel, u) -> np.ndarray:
    """f_int = +dE/du on the free DOFs, GPU per-element StVK."""
    s = _fe_session(model)
    return s.element_forces(u, want_K=False)[0]


def element_stiffness(model: ElasticModel, u) -> np.ndarray:
    """Per-element K_e (T,12,12), vertex-major DOFs (GPU)."""
    return _fe_session(model).element_forces(u, want_K=True)[1]


def stiffness(model: ElasticModel, u):
    """Sparse N x N stiffness dF_int/du: GPU element blocks, COO assembly."""
    import scipy.sparse as sp
    K = element_stiffness(model, u)
    rows = model.element_rows()
    r = np.repeat(rows[:, :, None], 12, axis=2)
    c = np.repeat(rows[:, None, :], 12, axis=1)
    m = (r >= 0) & (c >= 0)
    return sp.coo_matrix((K[m], (r[m], c[m])), shape=(model.N, model.N)).tocsr()


def element_reduced_force(model: ElasticModel, rm, r, e):
    """J~(r)_e^T f_e(u(r)). ``e`` may be an int or a list of ids."""
    from .session import session_for
    s = session_for(rm, model)
    single = np.isscalar(e)
    out = s.element_reduced_forces(r, np.atleast_1d(e))
    return out[0] if single else out


def fullspace_step(model: ElasticModel, u, v, f_ext, dt, cfg=None, return_info: bool = False):
    """Implicit Euler in the full space: Newton solve of
    M (v' - v)/dt + (alpha M + beta K(u')) v' + f_int(u') = f_ext with u' = u + dt v'.
    GPU (csrc/fullspace.cu): element kernels, CSR assembly, cooperative Jacobi-PCG.
    Returns (u', v') (and a FullspaceInfo if ``return_info``); raises
    _lib.NewtonDivergence after ``cfg.max_iters`` Newton iterations."""
    from .fullspace import session_for as _fs
    uo, vo, info = _fs(model).step(u, v, f_ext, dt, cfg)
    return (uo, vo, info) if return_info else (uo, vo)

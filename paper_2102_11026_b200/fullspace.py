"""Full-space StVK implicit Euler on the GPU (elastic.fullspace_step).

Host-side handle around the ``nlrom_fs_*`` C ABI (csrc/fullspace.cu): the mesh, lumped mass
and material are uploaded once per ElasticModel; each step is a Newton solve whose linear
systems run as one cooperative Jacobi-PCG kernel. There is no CPU fallback: a missing
library raises (``_lib.lib()``).
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class FullspaceConfig:
    """Newton / CG controls for fullspace_step (divergence after max iterations)."""
    newton_tol: float = 1e-8      # ||g||_2 <= newton_tol * max(1, ||f_ext||_2)  [N]
    max_iters: int = 20
    cg_tol: float = 1e-11         # relative preconditioned-CG residual
    cg_max_iters: int = 20000


@dataclass
class FullspaceInfo:
    iters: int
    cg_iters: int
    res_norm: float
    energy: float


class FullspaceSession:
    """GPU state of one ElasticModel for full-space stepping (one per model, not thread-shared)."""

    def __init__(self, model, beta: float | None = None, device: int | None = None):
        L = _lib.lib()
        self.N = model.N
        keep = []

        def arr(a, conv=_lib.f64):
            a = conv(a)
            keep.append(a)
            return a

        d = _lib.FsDesc()
        d.n_verts, d.n_tets = model.mesh.vertices.shape[0], model.n_tets
        d.tets = _lib.iptr(arr(model.mesh.tets, _lib.i32))
        d.vert_dof = _lib.iptr(arr(model.vert_dof, _lib.i32))
        d.Dm_inv = _lib.dptr(arr(model.Dm_inv.reshape(-1, 9)))
        d.vol = _lib.dptr(arr(model.vol))
        d.mass = _lib.dptr(arr(model.mass))
        mat = model.material
        d.mu, d.lam, d.alpha = mat.mu, mat.lam, mat.rayleigh_alpha
        d.beta = mat.rayleigh_beta if beta is None else beta
        h = C.c_void_p()
        self.device = _lib.device_index() if device is None else device
        _lib.check(L.nlrom_fs_create(C.byref(h), self.device, C.byref(d)), lambda: "nlrom_fs_create failed")
        self._h, self._L = h, L
        self._fin = weakref.finalize(self, L.nlrom_fs_destroy, h)

    def _chk(self, code):
        _lib.check(code, lambda: self._L.nlrom_fs_last_error(self._h))

    def step(self, u, v, f_ext, dt, cfg: FullspaceConfig | None = None):
        cfg = cfg or FullspaceConfig()
        u, v, f = (_lib.f64(a) for a in (u, v, f_ext))
        for a in (u, v, f):
            if a.shape != (self.N,):
                raise ValueError(f"dimension mismatch: expected ({self.N},), got {a.shape}")
        c = _lib.FsCfg(float(dt), cfg.newton_tol, cfg.max_iters, cfg.cg_tol, cfg.cg_max_iters)
        uo, vo = np.empty(self.N), np.empty(self.N)
        info = _lib.FsInfo()
        self._chk(self._L.nlrom_fs_step(self._h, _lib.dptr(u), _lib.dptr(v), _lib.dptr(f), C.byref(c),
                                        _lib.dptr(uo), _lib.dptr(vo), C.byref(info)))
        return uo, vo, FullspaceInfo(info.iters, info.cg_iters, info.res_norm, info.energy)

    def energy_force(self, u):
        u = _lib.f64(u)
        e = C.c_double()
        f = np.empty(self.N)
        self._chk(self._L.nlrom_fs_energy_force(self._h, _lib.dptr(u), C.byref(e), _lib.dptr(f)))
        return e.value, f


def session_for(model) -> FullspaceSession:
    s = getattr(model, "_fs", None)
    if s is None:
        s = FullspaceSession(model)
        model._fs = s
    return s

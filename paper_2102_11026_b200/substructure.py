"""Substructured scenes: k DAE strings on a translating core (SURVEY.md §8e, cfg4 puffer ball).

The reference simulates one reduced body per ``rdsim.step`` and has no
coupled scenes; the paper's puffer ball attaches 320
identical strings -- one DAE + cubature training re-used for all -- to a core. The model is
defined in ``oracle/coupled.py``; this module is its multi-GPU host driver:

* strings are partitioned in contiguous ranges over the ranks of the default
  ``torch.distributed`` group (one process per GPU), each rank owns one ``nlrom`` context
  with its strings as sims (shared weights, big-tile batched decoder when there are many);
* the core (3 translational DOFs) is replicated on every rank;
* per Newton iteration every rank runs one CUDA graph (effective loads, decoder bundle,
  cubature, Eq. 11 assembly, vhp, LU with the 3 coupling right-hand sides, local Schur
  terms), then ONE allreduce of 16 doubles (NCCL over NVLink, issued on the context stream,
  no host sync), then the replicated 3 x 3 core solve and the local string updates.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .session import Session, _simcfg

PARTIAL = 16  # doubles exchanged per Newton iteration (sum E_s X_s: 12, core terms: 3, sum ||phi_s||^2: 1)


def shard(k: int, rank: int, world: int):
    """Contiguous string range [lo, hi) of ``rank`` (same partition as oracle/coupled.py)."""
    return rank * k // world, (rank + 1) * k // world


def dist_info(group=None):
    """(rank, world) of the default / given process group, (0, 1) without torch.distributed."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(group), dist.get_world_size(group)
    except ImportError:
        pass
    return 0, 1


def allreduce_sum(t, group=None, stream=None):
    """In-place sum of a tensor over the ranks (no-op at world size 1). ``stream``: the CUDA
    stream the collective is ordered on (the context stream: no host synchronisation)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    if stream is not None:
        with torch.cuda.stream(stream):
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


@dataclass
class Core:
    """The core body: mass, anchoring spring stiffness, constant external force (world frame)."""
    mass: float
    stiffness: float = 0.0
    force: np.ndarray = field(default_factory=lambda: np.zeros(3))


class Scene:
    """One rank's share of a substructured scene.

    R: (k, 3, 3) string frame -> world; f_world: (k, N) external loads (world frame) on every
    string's free DOFs. ``rank`` / ``world`` default to the torch.distributed group; passing
    them explicitly (with ``allreduce=None``) lets a single process drive several shards."""

    def __init__(self, rm, model, cm, R, f_world, core: Core, group=None, rank=None, world=None,
                 device: int | None = None):
        import torch
        R = np.ascontiguousarray(R, dtype=np.float64)
        f_world = np.ascontiguousarray(f_world, dtype=np.float64)
        self.k = R.shape[0]
        if f_world.shape != (self.k, model.N):
            raise ValueError("dimension mismatch: f_world must be (k, N)")
        r0, w0 = dist_info(group)
        self.rank = r0 if rank is None else rank
        self.world = w0 if world is None else world
        self.group = group
        self.lo, self.hi = shard(self.k, self.rank, self.world)
        if self.hi <= self.lo:
            raise ValueError("more ranks than strings")
        self.n = rm.n_p + rm.n_q
        self.sess = Session(rm, model, cm, n_sims=self.hi - self.lo, device=device)
        self._L, self._h = self.sess._L, self.sess._h
        fc = _lib.f64(core.force)
        self.sess._chk(self._L.nlrom_coupled_setup(self._h, _lib.dptr(R[self.lo:self.hi].reshape(-1)),
                                                   _lib.dptr(f_world[self.lo:self.hi].reshape(-1)), self.k,
                                                   float(core.mass), float(core.stiffness), _lib.dptr(fc)))
        sp = C.c_void_p()
        self.sess._chk(self._L.nlrom_stream(self._h, C.byref(sp)))
        self.device = self.sess.device
        self.stream = torch.cuda.ExternalStream(sp.value or 0, device=torch.device("cuda", self.device))
        self.partial = torch.zeros(PARTIAL, dtype=torch.float64, device=torch.device("cuda", self.device))
        self._cfg = None

    # ------------------------------------------------------------------ low-level phases
    def begin(self, r_bar, rdot_bar, c_bar, cdot_bar, cfg):
        rb, rdb = self._local(r_bar), self._local(rdot_bar)
        self._cfg = _simcfg(cfg)
        self.sess._chk(self._L.nlrom_coupled_begin(self._h, _lib.dptr(rb), _lib.dptr(rdb),
                                                   _lib.dptr(_lib.f64(c_bar)), _lib.dptr(_lib.f64(cdot_bar)),
                                                   C.byref(self._cfg)))

    def eval(self, jacobian: bool):
        """Enqueue the local graph: partial <- this rank's 16 Schur / residual terms."""
        self.sess._chk(self._L.nlrom_coupled_eval(self._h, C.byref(self._cfg), int(jacobian),
                                                  C.c_void_p(self.partial.data_ptr())))

    def reduce(self):
        allreduce_sum(self.partial, self.group, self.stream)

    def update(self, mode: int, t: float = 1.0, total=None, want_norm=False):
        tot = self.partial if total is None else total
        out = C.c_double()
        self.sess._chk(self._L.nlrom_coupled_update(self._h, C.byref(self._cfg), C.c_void_p(tot.data_ptr()),
                                                    int(mode), float(t), C.byref(out) if want_norm else None))
        return out.value if want_norm else None

    def read(self, dt):
        S = self.hi - self.lo
        r = np.empty((S, self.n))
        rd = np.empty((S, self.n))
        c = np.empty(3)
        cd = np.empty(3)
        self.sess._chk(self._L.nlrom_coupled_read(self._h, float(dt), _lib.dptr(r), _lib.dptr(rd), _lib.dptr(c),
                                                  _lib.dptr(cd)))
        return r, rd, c, cd

    def launches_per_iteration(self):
        return int(self._L.nlrom_coupled_launches(self._h))

    def _local(self, a):
        a = _lib.f64(a)
        if a.ndim == 2 and a.shape[0] == self.k and self.k != self.hi - self.lo:
            a = a[self.lo:self.hi]
        a = np.ascontiguousarray(a).reshape(-1)
        if a.size != (self.hi - self.lo) * self.n:
            raise ValueError("dimension mismatch: expected (k, n) or this rank's (hi - lo, n) states")
        return a

    # ------------------------------------------------------------------ step
    def step(self, r_bar, rdot_bar, c_bar, cdot_bar, cfg):
        """One coupled implicit timestep (oracle/coupled.py: step). Returns this rank's
        (r, rdot) (hi - lo, n), the core (c, cdot) and (iterations, ||phi||)."""
        self.begin(r_bar, rdot_bar, c_bar, cdot_bar, cfg)
        if cfg.fixed_iters:
            for _ in range(cfg.fixed_iters):
                self.eval(True)
                self.reduce()
                self.update(1, 1.0)
            self.eval(False)
            self.reduce()
            nrm = self.update(0, want_norm=True)
            return (*self.read(cfg.dt), cfg.fixed_iters, nrm)
        self.eval(False)
        self.reduce()
        nrm = self.update(0, want_norm=True)
        it = 0
        while nrm > cfg.newton_tol:
            if it >= cfg.max_iters:
                raise _lib.NewtonDivergence(f"Newton did not converge in {cfg.max_iters} iterations; "
                                            f"last residual norm {nrm:.3e}", nrm)
            self.eval(True)
            self.reduce()
            self.update(1, 1.0)
            t = 1.0
            for trial in range(11):
                if trial:
                    self.update(2, t)
                self.eval(False)
                self.reduce()
                n_try = self.update(0, want_norm=True)
                if not np.isfinite(n_try):
                    raise FloatingPointError("non-finite residual")
                if not cfg.line_search or n_try < nrm:
                    break
                t *= 0.5
            nrm = n_try
            it += 1
        return (*self.read(cfg.dt), it, nrm)

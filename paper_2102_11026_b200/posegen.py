"""nlrom.posegen — training poses by scripted random forcing (§5.1).

Episodes run the GPU full-space integrator (elastic.fullspace_step, csrc/fullspace.cu); the
StVK energy of every frame comes from the same element kernel. Pose weights and the PCA
basis are small host computations.

Script semantics: ``np.random.default_rng(seed)``; the loadable
vertices are the free vertices of the boundary faces (faces of exactly one tet); per
episode one draw of the centre vertex, of a unit direction (normalised standard normal) and
of the magnitude U(lo, hi); the force is split evenly over the free vertices within
``radius`` of the centre (default 10% of the bounding-box diagonal) and held constant for
``steps`` implicit-Euler steps from rest; every frame is recorded. A diverging episode is
skipped with a log entry. The rest pose (u = 0) is appended.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .elastic import ElasticModel, fullspace_step

log = logging.getLogger(__name__)


@dataclass
class ForceScript:
    """SPEC.md:389-392."""
    seed: int = 0
    episodes: int = 10
    radius: float | None = None
    magnitude: tuple = (0.0, 100.0)
    steps: int = 20
    dt: float = 1.0 / 60.0

    def __post_init__(self):
        if self.radius is not None and not self.radius > 0:
            raise ValueError("radius must be > 0 (SPEC.md:391)")
        if self.steps < 1:
            raise ValueError("steps must be >= 1 (SPEC.md:391)")


@dataclass
class PoseSet:
    """poses N x T (m), energies T (J), weights T."""
    poses: np.ndarray
    energies: np.ndarray
    weights: np.ndarray = field(default=None)
    script: dict | None = None

    def __post_init__(self):
        self.poses = np.asarray(self.poses, dtype=float)
        self.energies = np.asarray(self.energies, dtype=float)
        if self.weights is None:
            self.weights = np.ones(self.energies.size)


def surface_vertices(tets) -> np.ndarray:
    """Sorted vertex ids of the boundary faces (faces belonging to exactly one tet)."""
    tets = np.asarray(tets)
    faces = np.sort(np.concatenate([tets[:, [1, 2, 3]], tets[:, [0, 2, 3]], tets[:, [0, 1, 3]],
                                    tets[:, [0, 1, 2]]]), axis=1)
    uniq, cnt = np.unique(faces, axis=0, return_counts=True)
    return np.unique(uniq[cnt == 1].ravel())


def _plan(model: ElasticModel, script: ForceScript):
    verts = model.mesh.vertices
    radius = script.radius
    if radius is None:
        radius = 0.1 * float(np.linalg.norm(verts.max(axis=0) - verts.min(axis=0)))
    rng = np.random.default_rng(script.seed)
    surf = surface_vertices(model.mesh.tets)
    surf = surf[~model.fixed[surf]]
    if surf.size == 0:
        raise ValueError("no free surface vertex to load")
    lo, hi = script.magnitude
    out = []
    for _ in range(script.episodes):
        c = int(rng.choice(surf))
        dist = np.linalg.norm(verts - verts[c], axis=1)
        ids = np.nonzero((dist <= radius) & ~model.fixed)[0]
        d = rng.standard_normal(3)
        d /= max(np.linalg.norm(d), 1e-300)
        out.append((ids, rng.uniform(lo, hi) * d))
    return out


def _load(model: ElasticModel, ids, force):
    f = np.zeros(model.N)
    dof = model.vert_dof[ids]
    dof = dof[dof >= 0]
    if dof.size:
        for c in range(3):
            f[3 * dof + c] = force[c] / dof.size
    return f


def generate_poses(model: ElasticModel, script: ForceScript, cfg=None) -> PoseSet:
    """SPEC.md:395-403. T = episodes x steps + 1 poses (fewer if an episode diverged)."""
    poses, energies = [], []
    for k, (ids, force) in enumerate(_plan(model, script)):
        f = _load(model, ids, force)
        u = np.zeros(model.N)
        v = np.zeros(model.N)
        ep_p, ep_e = [], []
        try:
            for _ in range(script.steps):
                u, v, info = fullspace_step(model, u, v, f, script.dt, cfg=cfg, return_info=True)
                ep_p.append(u)
                ep_e.append(info.energy)
        except (_lib.NewtonDivergence, FloatingPointError) as e:
            log.warning("posegen: episode %d skipped (%s)", k, e)
            continue
        poses += ep_p
        energies += ep_e
    poses.append(np.zeros(model.N))
    energies.append(0.0)
    ps = PoseSet(np.stack(poses, axis=1), np.array(energies),
                 script={"seed": script.seed, "episodes": script.episodes, "radius": script.radius,
                         "magnitude": list(script.magnitude), "steps": script.steps, "dt": script.dt})
    pos = ps.energies[ps.energies > 0]
    floor = 1e-6 * float(np.median(pos)) if pos.size else 1.0
    ps.weights = energy_weights(ps, floor)
    return ps


def energy_weights(ps, floor: float) -> np.ndarray:
    """w_t = 1 / max(E_t, floor), normalised to mean 1."""
    if not floor > 0:
        raise ValueError("floor must be > 0 (SPEC.md:406)")
    e = ps.energies if isinstance(ps, PoseSet) else np.asarray(ps, dtype=float)
    w = 1.0 / np.maximum(e, floor)
    return w / w.mean()


def pca_basis(ps: PoseSet, n_p: int, subset_size: int) -> np.ndarray:
    """Top-n_p left singular vectors of the subset_size lowest-energy poses."""
    T = ps.poses.shape[1]
    if not (n_p <= subset_size <= T):
        raise ValueError("need n_p <= subset_size <= T (SPEC.md:415)")
    idx = np.argsort(ps.energies, kind="stable")[:subset_size]
    U, s, _ = np.linalg.svd(ps.poses[:, idx], full_matrices=False)
    if np.count_nonzero(s > s[0] * 1e-12 if s.size and s[0] > 0 else s > 0) < n_p:
        raise ValueError("rank deficiency: fewer than n_p nonzero singular values (SPEC.md:417)")
    return U[:, :n_p]

"""Oracle full-space implicit Euler and pose generator (TEST INFRASTRUCTURE).

Restates SPEC.md [OP] fullspace_step and [MODULE] posegen
 with numpy / scipy, on top of oracle/elastic.py. Only tests, smoke()
and bench.py's cpu_baseline leg use it.

fullspace_step: Newton on v' for
    g(v') = M (v' - v)/dt + (alpha M + beta K(u')) v' + f_int(u') - f_ext = 0,  u' = u + dt v'
(Rayleigh damping alpha M + beta K). Newton matrix
(1 + alpha dt) M + (beta dt + dt^2) K(u') (the dK/du v' term is dropped, as in the product;
it changes the convergence rate only). Linear systems by a direct sparse solve
(scipy.sparse.linalg.spsolve). Convergence: ||g||_2 <= newton_tol * max(1, ||f_ext||_2).

posegen: scripted random forcing episodes, inverse-energy pose weights,
plain PCA of the lowest-energy poses; surface vertices are the vertices of the boundary
faces of the tet mesh (faces that belong to exactly one tet).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import elastic as oe


def stiffness_sparse(model, u):
    f, K = oe.element_force_stiffness(model, u)
    rows = model.rows
    r = np.repeat(rows[:, :, None], 12, axis=2)
    c = np.repeat(rows[:, None, :], 12, axis=1)
    m = (r >= 0) & (c >= 0)
    Kc = sp.coo_matrix((K[m], (r[m], c[m])), shape=(model.N, model.N)).tocsr()
    fint = oe.scatter(model, f, np.arange(model.n_tets))
    return fint, Kc


def fullspace_step(model, u, v, f_ext, dt, beta=0.0, newton_tol=1e-8, max_iters=20):
    """(u, v) -> (u', v', iterations, ||g||); raises RuntimeError on Newton divergence."""
    if not dt > 0:
        raise ValueError("dt must be > 0")
    M = model.mass
    alpha = model.alpha
    tol = newton_tol * max(1.0, float(np.linalg.norm(f_ext)))
    x = np.array(v, dtype=float)
    it = 0
    while True:
        up = u + dt * x
        fint, K = stiffness_sparse(model, up)
        g = M * (x - v) / dt + alpha * M * x + beta * (K @ x) + fint - f_ext
        gn = float(np.linalg.norm(g))
        if not np.isfinite(gn):
            raise FloatingPointError("non-finite full-space residual")
        if gn <= tol:
            return up, x, it, gn
        if it >= max_iters:
            raise RuntimeError(f"full-space Newton did not converge in {max_iters} iterations; last {gn:.3e}")
        H = sp.diags((1.0 + alpha * dt) * M) + (beta * dt + dt * dt) * K
        x = x + spla.spsolve(H.tocsc(), -dt * g)
        it += 1


def surface_vertices(tets):
    """Vertices of the boundary faces (faces of exactly one tet), sorted."""
    tets = np.asarray(tets)
    faces = np.concatenate([tets[:, [1, 2, 3]], tets[:, [0, 2, 3]], tets[:, [0, 1, 3]], tets[:, [0, 1, 2]]])
    fs = np.sort(faces, axis=1)
    uniq, cnt = np.unique(fs, axis=0, return_counts=True)
    return np.unique(uniq[cnt == 1].ravel())


def episode_plan(verts, tets, fixed, seed, episodes, radius, mag_range):
    """Per episode: (loaded vertex ids, force vector) -- deterministic under seed."""
    rng = np.random.default_rng(seed)
    surf = surface_vertices(tets)
    surf = surf[~np.asarray(fixed)[surf]]
    plan = []
    for _ in range(episodes):
        c = int(rng.choice(surf))
        d = np.linalg.norm(verts - verts[c], axis=1)
        ids = np.nonzero((d <= radius) & ~np.asarray(fixed))[0]
        direction = rng.standard_normal(3)
        direction /= max(np.linalg.norm(direction), 1e-300)
        mag = rng.uniform(mag_range[0], mag_range[1])
        plan.append((ids, mag * direction))
    return plan


def episode_force(model, ids, force):
    """Free-DOF load vector: the force split evenly over the loaded vertices."""
    f = np.zeros(model.N)
    dof = model.dof[ids]
    dof = dof[dof >= 0]
    if dof.size:
        for c in range(3):
            f[3 * dof + c] = force[c] / dof.size
    return f


def generate_poses(model, seed, episodes, steps, dt, radius, mag_range, beta=0.0):
    """PoseSet (poses N x T, energies T): each episode starts from rest, applies its constant
    force for `steps` implicit-Euler steps, records every frame; the rest pose is appended."""
    plan = episode_plan(model.verts, model.tets, model.fixed, seed, episodes, radius, mag_range)
    poses, energies = [], []
    for ids, force in plan:
        fe = episode_force(model, ids, force)
        u = np.zeros(model.N)
        v = np.zeros(model.N)
        for _ in range(steps):
            u, v, _, _ = fullspace_step(model, u, v, fe, dt, beta=beta)
            poses.append(u.copy())
            energies.append(oe.stvk_energy(model, u))
    poses.append(np.zeros(model.N))
    energies.append(0.0)
    return np.stack(poses, axis=1), np.array(energies)


def energy_weights(energies, floor):
    w = 1.0 / np.maximum(np.asarray(energies, dtype=float), floor)
    return w / w.mean()


def pca_basis(poses, energies, n_p, subset_size):
    idx = np.argsort(energies, kind="stable")[:subset_size]
    Uf, s, _ = np.linalg.svd(poses[:, idx], full_matrices=False)
    return Uf[:, :n_p], s

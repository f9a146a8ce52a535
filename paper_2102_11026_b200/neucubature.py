"""nlrom.neucubature — simulation-time neural cubature (§5).

``wnet_forward`` evaluates the weight net W on the GPU (generic net path, all
elements); ``cubature_integrate`` runs the fused device kernel: wnet restricted to
the rows of C, per-element StVK force / stiffness for e in C, projection by the
element's 12 rows of J~ and the weighted sums.
Selection net, alternating training and the greedy NNLS baseline (offline, SURVEY.md §8f
rank 3) are in ``cubature_train`` and re-exported here under the SPEC names.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .densenet import DenseNet, forward


@dataclass
class CubatureModel:
    """C: ordered duplicate-free element ids; wnet: weight net; snet / K per SPEC.md:584-587."""
    C: np.ndarray
    wnet: DenseNet | None = None
    snet: object | None = None
    K: int = 5

    def __post_init__(self):
        self.C = np.asarray(self.C, dtype=np.int32).reshape(-1)
        if self.C.size != np.unique(self.C).size:
            raise ValueError("cubature set has duplicate element ids (SPEC.md:586)")


def wnet_forward(wnet: DenseNet, rm, r) -> np.ndarray:
    """r -> frozen decoder -> u -> W -> square: one nonnegative weight per element."""
    from .daereduce import full_displacement
    u = full_displacement(rm, r)
    return forward(wnet, u)


def cubature_integrate(cm: CubatureModel, rm, model, r, integration: str = "cubature"):
    """(f~, K~) = (sum_{e in C} w_e J~_e^T f_e, sum_e w_e J~_e^T K_e J~_e).
    ``integration="exact_sum"`` uses all elements with w = 1."""
    from .session import session_for
    if integration == "cubature" and cm.C.size == 0:
        n = rm.n
        return np.zeros(n), np.zeros((n, n))
    return session_for(rm, model, cm).cubature_integrate(r, integration)


def select_topk(C, s, K):
    """Add the K highest-scoring non-members, ties by lower id."""
    C = list(np.asarray(C, dtype=int))
    member = set(C)
    s = np.asarray(s, dtype=float)
    order = sorted(range(s.size), key=lambda e: (-s[e], e))
    add = [e for e in order if e not in member][:K]
    return np.asarray(C + add, dtype=np.int32)


# Offline training and the greedy baseline live in cubature_train.py.
def __getattr__(name):
    if name in ("train_alternating", "greedy_cubature", "snet_forward", "nnls", "build_train_set",
                "cubature_error", "CubatureTrainSet", "SelectionNet", "mesh_graph", "farthest_point_elements"):
        from . import cubature_train
        return getattr(cubature_train, name)
    raise AttributeError(name)

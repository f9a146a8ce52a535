"""Build product-side objects (ReducedModel, ElasticModel, CubatureModel, state) for a
synthetic config of synth.py (used by bench.py, smoke() and the tests)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import synth
from .daereduce import ReducedModel, ReducedState
from .densenet import make_decoder, make_wnet
from .elastic import ElasticModel, Material, TetMesh
from .neucubature import CubatureModel


@dataclass
class Problem:
    cfg: synth.SynthConfig
    data: dict
    rm: ReducedModel
    model: ElasticModel
    cm: CubatureModel
    f_ext: np.ndarray

    def random_state(self, seed=4):
        q, qb, qdb, p, pb, pdb = synth.random_state(self.cfg.n_p, self.cfg.n_q, seed)
        return np.concatenate([p, q]), np.concatenate([pb, qb]), np.concatenate([pdb, qdb])

    def rest_state(self):
        n = self.cfg.n_p + self.cfg.n_q
        return ReducedState(np.zeros(n), np.zeros(n), self.cfg.dt)


def build_problem(name="cfg1", **overrides) -> Problem:
    cfg = synth.CONFIGS[name]
    if overrides:
        cfg = synth.SynthConfig(**{**vars(cfg), **overrides})
    P = synth.build(cfg)
    mesh = TetMesh(P["verts"], P["tets"])
    mat = Material(cfg.young, cfg.poisson, cfg.density, cfg.alpha)
    model = ElasticModel(mesh, mat, P["fixed"])
    dec = make_decoder(P["dec_W"], P["dec_b"], P["U"])
    rm = ReducedModel(P["U"], dec, cfg.n_p, cfg.n_q)
    cm = CubatureModel(P["cub"], make_wnet(P["wnet_W"], P["wnet_b"]))
    rm.attach(model, cm)
    return Problem(cfg, P, rm, model, cm, synth.gravity(model.mass))

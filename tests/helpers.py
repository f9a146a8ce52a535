"""Shared builders: the same synthetic problem on the product side (GPU) and the oracle side (CPU)."""

import numpy as np

from oracle import elastic as oe, reduced as orr, rdsim as ors
from paper_2102_11026_b200 import synth


def oracle_sim(P):
    """Oracle OSim from a product Problem (identical arrays)."""
    cfg, d = P.cfg, P.data
    model = oe.OModel(d["verts"], d["tets"], d["fixed"], cfg.young, cfg.poisson, cfg.density, cfg.alpha)
    D = synth.decoder_layers(d["dec_W"], d["dec_b"], d["U"])
    rm = orr.OReduced(d["U"], D, cfg.n_p, cfg.n_q)
    return ors.OSim(rm, model, d["cub"], synth.wnet_layers(d["wnet_W"], d["wnet_b"]))


def ocfg(cfg, **kw):
    return ors.OSimConfig(**{k: getattr(cfg, k) for k in ("dt", "newton_tol", "max_iters", "drop_fict",
                                                          "integration", "line_search", "fixed_iters")}, **kw)


def coupled_setup(P, k, k_core=50.0):
    """Scene arrays shared by the product and the oracle: k strings of problem P on a core."""
    from oracle import coupled as oc
    R = synth.string_frames(k)
    f_world = np.tile(P.f_ext, (k, 1))
    m_core = 2.0 * float(P.model.mass[0::3].sum())
    f_core = np.array([0.0, -9.81 * m_core, 0.0])
    scene = oc.OScene(oracle_sim(P), R, f_world, m_core=m_core, k_core=k_core, f_core=f_core)
    return R, f_world, m_core, k_core, f_core, scene

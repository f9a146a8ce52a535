"""Drive every default kernel of the library once at cfg1 / tiny sizes, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py

Covers: generic nets (forward orders 0-3, backward), reference-structure diffops, the fused
Newton iteration (jet chain, output GEMM, weight net, split cubature, assembly, reductions,
vhp chain, LU) through residual / system_jacobian / fixed and adaptive steps, multi-sim
contexts on the batched kernels (big-tile GEMMs, warp-specialised TMA GEMMs, shared-real vhp,
multi-chunk cubature), the coupled scene and the full-space integrator."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]


def main():
    from paper_2102_11026_b200 import densenet, diffops, rdsim, synth, neucubature
    from paper_2102_11026_b200.daereduce import ReducedState
    from paper_2102_11026_b200.mcx import MCArray
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200.session import Session
    P = build_problem("cfg1")
    for order in range(4):
        q = np.random.default_rng(order).uniform(-0.5, 0.5, (1 << order, P.cfg.n_q, 3))
        densenet.forward(P.rm.decoder, MCArray(q))
    q = np.random.default_rng(1).uniform(-0.5, 0.5, P.cfg.n_q)
    for op in ("jacobian", "hvv", "hv", "svv"):
        getattr(diffops, op)(P.rm, q, q) if op != "jacobian" else diffops.jacobian(P.rm, q)
    a = np.random.default_rng(2).standard_normal(P.model.N)
    diffops.vjp(P.rm, q, a)
    diffops.vhp(P.rm, q, a)
    r, rb, rdb = P.random_state()
    st = ReducedState(rb, rdb, P.cfg.dt)
    for integ in ("cubature", "exact_sum"):
        cfg = rdsim.SimConfig(dt=P.cfg.dt, integration=integ)
        rdsim.residual(P.rm, P.model, st, P.f_ext, cfg, r=r)
        rdsim.system_jacobian(P.rm, P.model, st, P.f_ext, cfg, r=r)
    neucubature.cubature_integrate(P.cm, P.rm, P.model, r)
    P.rm.session().wnet_forward_cub(r)
    rdsim.step(P.rm, P.model, P.rest_state(), P.f_ext, rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2))
    rdsim.step(P.rm, P.model, P.rest_state(), P.f_ext, rdsim.SimConfig(dt=P.cfg.dt))
    # many-sims kernels on 3 sims
    os.environ["NLROM_PATH"] = "batched,cpc=4,shared_real,cpm=4"
    ns = 3
    s = Session(P.rm, P.model, P.cm, n_sims=ns)
    n = P.cfg.n_p + P.cfg.n_q
    s.step(np.zeros(ns * n), np.zeros(ns * n), np.tile(P.f_ext, ns), rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2))
    s.residual(np.tile(r, ns), np.tile(rb, ns), np.tile(rdb, ns), np.tile(P.f_ext, ns), rdsim.SimConfig(dt=P.cfg.dt))
    del os.environ["NLROM_PATH"]
    # coupled scene
    from paper_2102_11026_b200.substructure import Core, Scene
    Pt = build_problem("tiny")
    k = 3
    R = synth.string_frames(k)
    sc = Scene(Pt.rm, Pt.model, Pt.cm, R, np.tile(Pt.f_ext, (k, 1)), Core(1.0, 50.0, np.array([0, -9.81, 0])))
    rb3, rdb3, cb, cdb = synth.coupled_state(k, Pt.cfg.n_p, Pt.cfg.n_q)
    sc.step(rb3, rdb3, cb, cdb, rdsim.SimConfig(dt=Pt.cfg.dt, fixed_iters=2))
    # full-space integrator
    from paper_2102_11026_b200.fullspace import FullspaceConfig, FullspaceSession
    fs = FullspaceSession(P.model)
    z = np.zeros(P.model.N)
    fs.step(z, z, P.f_ext, P.cfg.dt, FullspaceConfig())
    print("sanitize_run: done", flush=True)


if __name__ == "__main__":
    main()

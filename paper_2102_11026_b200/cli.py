"""nlrom.cli -- config-driven commands (pyproject console script nlrom.cli:main).

    nlrom gen-data       --config run.json   scripted full-space poses -> PoseSet (+ mesh)
    nlrom train-dae      --config run.json   PCA basis + DAE (build_dae) -> ReducedModel, loss CSV
    nlrom train-cubature --config run.json   cubature set + weight net (greedy NNLS or neural)
    nlrom simulate       --config run.json   reduced implicit Euler -> per-step JSON lines + OBJ frames
    nlrom validate       --config run.json   invariant checks, pass / fail table (exit 0 / 1)
    nlrom bench          --config run.json   device ms per Newton iteration / adaptive timestep

Flags: --config PATH, --seed INT, --out DIR, --drop-fict, --cubature | --exact; CLI flags override
the config's top-level keys. Exit codes: 0 success, 1 validation failure, 2 input error
(SPEC.md:692-696). Every command is deterministic given the config and its seeds.

RunConfig (JSON), all keys optional except what a command reads:
  out            output directory (artifacts: mesh.txt, poses.bin, reduced/, cubature/,
                 loss_dae.csv, sim.jsonl, frames/frame_NNNN.obj)
  seed           int; data / init / training shuffles derive from it
  mesh           {"box": [nx, ny, nz], "h": 0.1} (x = 0 face fixed) or {"path": "mesh.txt"}
  material       {"young": 5e5, "poisson": 0.45, "density": 1000, "alpha": 0.1}
  script         {"episodes", "steps", "magnitude": [lo, hi], "radius", "dt"} (posegen.ForceScript)
  arch           {"n_p", "n_q", "depth", "width", "pca_subset"}
  train          {"epochs", "batch_size", "learning_rate", "schedule": {epoch: factor}}
  cubature       {"size", "method": "greedy" | "neural", "wnet_width", "rounds", "K"}
  sim            {"steps", "dt", "gravity", "newton_tol", "max_iters", "line_search",
                  "drop_fict", "integration": "cubature" | "exact_sum", "frame_every"}
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

import numpy as np

EXIT_OK, EXIT_VALIDATION, EXIT_INPUT = 0, 1, 2


class InputError(Exception):
    """Bad config / missing artifact (exit code 2)."""


# ----------------------------------------------------------------------------- config & artifacts
def load_config(args) -> dict:
    cfg = {}
    if args.config:
        if not os.path.exists(args.config):
            raise InputError(f"config not found: {args.config}")
        with open(args.config) as f:
            try:
                cfg = json.load(f)
            except json.JSONDecodeError as e:
                raise InputError(f"config is not valid JSON: {e}") from e
    if args.seed is not None:
        cfg["seed"] = args.seed
    if args.out is not None:
        cfg["out"] = args.out
    sim = dict(cfg.get("sim", {}))
    if args.drop_fict:
        sim["drop_fict"] = True
    if args.integration is not None:
        sim["integration"] = args.integration
    cfg["sim"] = sim
    cfg.setdefault("out", "nlrom_run")
    cfg.setdefault("seed", 0)
    return cfg


def _path(cfg, *parts):
    return os.path.join(cfg["out"], *parts)


def build_model(cfg):
    """ElasticModel from cfg["mesh"] / cfg["material"] (saves the mesh to out/mesh.txt)."""
    from . import artifacts, synth
    from .elastic import ElasticModel, Material, TetMesh
    m = cfg.get("mesh", {"box": [10, 2, 2], "h": 0.1})
    mat = cfg.get("material", {})
    material = Material(float(mat.get("young", 5e5)), float(mat.get("poisson", 0.45)),
                        float(mat.get("density", 1000.0)), float(mat.get("alpha", 0.1)))
    if "path" in m:
        if not os.path.exists(m["path"]):
            raise InputError(f"mesh not found: {m['path']}")
        mesh = artifacts.read_mesh(m["path"])
        fixed = np.asarray(m.get("fixed", []), dtype=np.int64)
        if fixed.size == 0:   # default: the x = min face
            fixed = np.nonzero(mesh.vertices[:, 0] <= mesh.vertices[:, 0].min() + 1e-12)[0]
    else:
        box = m.get("box")
        if not (isinstance(box, (list, tuple)) and len(box) == 3 and all(int(b) > 0 for b in box)):
            raise InputError("mesh.box must be [nx, ny, nz] with positive entries")
        verts, tets, fixed = synth.box_mesh(*(int(b) for b in box), h=float(m.get("h", 0.1)))
        mesh = TetMesh(verts, tets)
    os.makedirs(cfg["out"], exist_ok=True)
    artifacts.write_mesh(mesh, _path(cfg, "mesh.txt"))
    return ElasticModel(mesh, material, fixed)


def load_reduced(cfg, model):
    from . import artifacts
    rdir, cdir = _path(cfg, "reduced"), _path(cfg, "cubature")
    if not os.path.exists(os.path.join(rdir, "manifest.json")):
        raise InputError(f"no ReducedModel in {rdir} (run train-dae first)")
    rm = artifacts.load_reduced_model(rdir)
    cm = None
    if os.path.exists(os.path.join(cdir, "manifest.json")):
        cm = artifacts.load_cubature_model(cdir)
    if rm.U.shape[0] != model.N:
        raise InputError("ReducedModel does not match the mesh (N differs)")
    rm.attach(model, cm)
    return rm, cm


def sim_config(cfg):
    from .rdsim import SimConfig
    s = cfg.get("sim", {})
    return SimConfig(dt=float(s.get("dt", cfg.get("dt", 1.0 / 60.0))), newton_tol=float(s.get("newton_tol", 1e-8)),
                     max_iters=int(s.get("max_iters", 20)), drop_fict=bool(s.get("drop_fict", False)),
                     integration=s.get("integration", "cubature"), line_search=bool(s.get("line_search", True)))


def external_force(cfg, model):
    from . import synth
    s = cfg.get("sim", {})
    f = synth.gravity(model.mass, float(s.get("gravity", -9.81)))
    if "force" in s:   # {"vertices": [...], "value": [fx, fy, fz]} split evenly over the vertices
        fv = s["force"]
        ids = np.asarray(fv["vertices"], dtype=np.int64)
        val = np.asarray(fv["value"], dtype=float) / max(1, ids.size)
        for v in ids:
            d = model.vert_dof[v]
            if d >= 0:
                f[3 * d:3 * d + 3] += val
    return f


# ----------------------------------------------------------------------------- surface / OBJ
def surface_faces(tets) -> np.ndarray:
    """Boundary triangles (faces of exactly one tet), oriented outward."""
    tets = np.asarray(tets, dtype=np.int64)
    local = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]])
    faces = tets[:, local].reshape(-1, 3)
    key = np.sort(faces, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    return faces[cnt[inv.ravel()] == 1]


def write_obj(path, vertices, faces):
    with open(path, "w") as f:
        f.write("# nlrom frame\n")
        for v in vertices:
            f.write(f"v {v[0]:.9g} {v[1]:.9g} {v[2]:.9g}\n")
        for t in faces:
            f.write(f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}\n")


def vertex_positions(model, u):
    pos = model.mesh.vertices.copy()
    free = model.vert_dof >= 0
    pos[free] += np.asarray(u).reshape(-1, 3)
    return pos


# ----------------------------------------------------------------------------- commands
def cmd_gen_data(cfg):
    """Scripted random-force poses on the full-space GPU integrator."""
    from . import artifacts
    from .posegen import ForceScript, generate_poses
    model = build_model(cfg)
    sc = cfg.get("script", {})
    script = ForceScript(seed=int(cfg["seed"]), episodes=int(sc.get("episodes", 10)), radius=sc.get("radius"),
                         magnitude=tuple(sc.get("magnitude", (0.0, 100.0))), steps=int(sc.get("steps", 20)),
                         dt=float(sc.get("dt", 1.0 / 60.0)))
    ps = generate_poses(model, script)
    artifacts.save_poseset(_path(cfg, "poses.bin"), ps.poses, ps.energies, ps.script)
    np.save(_path(cfg, "pose_weights.npy"), ps.weights)
    print(json.dumps({"command": "gen-data", "poses": int(ps.poses.shape[1]), "N": int(model.N),
                      "out": _path(cfg, "poses.bin")}))
    return EXIT_OK


def _load_poses(cfg):
    from . import artifacts
    from .posegen import PoseSet, energy_weights
    p = _path(cfg, "poses.bin")
    if not os.path.exists(p):
        raise InputError(f"no PoseSet at {p} (run gen-data first)")
    X, e, script = artifacts.load_poseset(p)
    wpath = _path(cfg, "pose_weights.npy")
    ps = PoseSet(X, e, script=script)
    if os.path.exists(wpath):
        ps.weights = np.load(wpath)
    else:
        pos = e[e > 0]
        ps.weights = energy_weights(ps, 1e-6 * float(np.median(pos)) if pos.size else 1.0)
    return ps


def cmd_train_dae(cfg):
    """PCA basis of the low-energy poses + PCA-orthogonal DAE."""
    from . import artifacts
    from .daereduce import DAEArch, build_dae
    from .densenet import TrainConfig
    from .posegen import pca_basis
    model = build_model(cfg)
    ps = _load_poses(cfg)
    if ps.poses.shape[0] != model.N:
        raise InputError("PoseSet does not match the mesh (N differs)")
    a, t = cfg.get("arch", {}), cfg.get("train", {})
    n_p = int(a.get("n_p", 10))
    T = ps.poses.shape[1]
    U = pca_basis(ps, n_p, min(T, int(a.get("pca_subset", T))))
    tc = TrainConfig(learning_rate=float(t.get("learning_rate", 1e-3)),
                     schedule={int(k): float(v) for k, v in t.get("schedule", {"300": 0.8, "3000": 0.8}).items()},
                     epochs=int(t.get("epochs", 300)), batch_size=int(t.get("batch_size", 64)))
    rm = build_dae(ps, U, DAEArch(depth=int(a.get("depth", 6)), n_q=int(a.get("n_q", 4)), width=a.get("width")), tc,
                   seed=int(cfg["seed"]))
    artifacts.save_reduced_model(rm, _path(cfg, "reduced"))
    with open(_path(cfg, "loss_dae.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["epoch", "loss"])
        for i, v in enumerate(rm.loss_curve):
            w.writerow([i, repr(v)])
    print(json.dumps({"command": "train-dae", "n_p": n_p, "n_q": rm.n_q, "final_loss": rm.loss_curve[-1],
                      "out": _path(cfg, "reduced")}))
    return EXIT_OK


def cmd_train_cubature(cfg):
    """Training set of per-element reduced forces at the encoded poses, then the greedy NNLS set
    (fixed weights, as a constant weight net) or alternating neural training."""
    from . import artifacts
    from .cubature_train import build_train_set, cubature_error, greedy_cubature, train_alternating
    from .daereduce import encode
    from .densenet import make_wnet
    from .neucubature import CubatureModel
    model = build_model(cfg)
    rm, _ = load_reduced(cfg, model)
    ps = _load_poses(cfg)
    c = cfg.get("cubature", {})
    size = int(c.get("size", 50))
    T = model.n_tets
    rs = []
    for k in range(ps.poses.shape[1]):
        p, q = encode(rm, ps.poses[:, k])
        rs.append(np.concatenate([p, q]))
    ts = build_train_set(rm, model, np.array(rs))
    wn = int(c.get("wnet_width", 32))
    rng = np.random.default_rng(int(cfg["seed"]) + 3)
    if c.get("method", "greedy") == "neural":
        C0, w0 = greedy_cubature(rm, model, ts, min(size, 5))
        Ws = [rng.uniform(-1, 1, (wn, model.N)) * np.sqrt(6.0 / model.N), rng.uniform(-1, 1, (wn, wn)) * np.sqrt(6.0 / wn),
              rng.uniform(-1, 1, (wn, wn)) * np.sqrt(6.0 / wn), np.zeros((T, wn))]
        bs = [np.zeros(wn), np.zeros(wn), np.zeros(wn), np.ones(T)]
        cm = train_alternating(rm, model, ts, K=int(c.get("K", 5)), rounds=int(c.get("rounds", 5)),
                               wnet=make_wnet(Ws, bs), seed=int(cfg["seed"]))
        C = cm.C
        err = None
    else:
        C, w = greedy_cubature(rm, model, ts, size)
        err = cubature_error(ts, C, w)
        # fixed weights as a weight net whose last layer is constant: (0 h + sqrt(w_e))^2 = w_e
        b4 = np.zeros(T)
        b4[C] = np.sqrt(w)
        Ws = [np.zeros((wn, model.N)), np.zeros((wn, wn)), np.zeros((wn, wn)), np.zeros((T, wn))]
        bs = [np.zeros(wn), np.zeros(wn), np.zeros(wn), b4]
        cm = CubatureModel(np.sort(C), make_wnet(Ws, bs))
    artifacts.save_cubature_model(cm, _path(cfg, "cubature"))
    print(json.dumps({"command": "train-cubature", "method": c.get("method", "greedy"), "size": int(len(cm.C)),
                      "train_error": err, "out": _path(cfg, "cubature")}))
    return EXIT_OK


def cmd_simulate(cfg):
    """Reduced implicit Euler from rest: one JSON line per step
    {t, r, residual_norm, newton_iters} in out/sim.jsonl, OBJ surface frames in out/frames/."""
    from .daereduce import ReducedState, full_displacement
    from .rdsim import step
    model = build_model(cfg)
    rm, cm = load_reduced(cfg, model)
    sc = sim_config(cfg)
    if sc.integration == "cubature" and cm is None:
        raise InputError("integration 'cubature' needs out/cubature (run train-cubature, or use --exact)")
    s = cfg.get("sim", {})
    steps, every = int(s.get("steps", 60)), int(s.get("frame_every", 1))
    f_ext = external_force(cfg, model)
    faces = surface_faces(model.mesh.tets)
    os.makedirs(_path(cfg, "frames"), exist_ok=True)
    st = ReducedState(np.zeros(rm.n), np.zeros(rm.n), sc.dt)
    t0 = time.perf_counter()
    with open(_path(cfg, "sim.jsonl"), "w") as log:
        for k in range(1, steps + 1):
            st, (it, nrm) = step(rm, model, st, f_ext, sc, cm=cm, return_info=True)
            log.write(json.dumps({"t": k * sc.dt, "r": st.r.tolist(), "residual_norm": nrm, "newton_iters": it}) + "\n")
            if every > 0 and k % every == 0:
                write_obj(_path(cfg, "frames", f"frame_{k:04d}.obj"),
                          vertex_positions(model, full_displacement(rm, st.r)), faces)
    wall = time.perf_counter() - t0
    print(json.dumps({"command": "simulate", "steps": steps, "ms_per_step": 1e3 * wall / max(1, steps),
                      "frames": steps // every if every > 0 else 0, "out": _path(cfg, "sim.jsonl")}))
    return EXIT_OK


def cmd_validate(cfg):
    """Invariant suite on the trained artifacts: orthogonal subspace (#10),
    weight non-negativity (#9), Jacobian vs central differences of the residual, a converging
    short simulation. Prints a pass / fail table; exit 1 on any failure."""
    from .daereduce import ReducedState, full_displacement
    from .densenet import forward
    from .rdsim import residual, step, system_jacobian
    model = build_model(cfg)
    rm, cm = load_reduced(cfg, model)
    sc = sim_config(cfg)
    if cm is None:
        sc.integration = "exact_sum"
    rng = np.random.default_rng(int(cfg["seed"]) + 11)
    rows = []
    worst = 0.0
    for _ in range(50):
        r = np.concatenate([np.zeros(rm.n_p), rng.uniform(-1, 1, rm.n_q)])
        D = full_displacement(rm, r)
        worst = max(worst, np.linalg.norm(rm.U.T @ D) / (np.linalg.norm(D) + 1.0))
    rows.append(("orthogonal subspace ||U^T D(q)|| / (||D|| + 1) <= 1e-8", worst, worst <= 1e-8))
    if cm is not None and cm.wnet is not None:
        u = rng.standard_normal((model.N, 1000)) * 1e-2
        w = forward(cm.wnet, u)
        neg = int((w < 0).sum())
        rows.append(("weight net outputs >= 0 (1000 evaluations)", float(neg), neg == 0))
    r0 = rng.uniform(-0.05, 0.05, rm.n)
    stt = ReducedState(r0, np.zeros(rm.n), sc.dt)
    f_ext = external_force(cfg, model)
    S = system_jacobian(rm, model, stt, f_ext, sc, r=r0, cm=cm)
    h = 1e-6
    Sfd = np.empty_like(S)
    for j in range(rm.n):
        e = np.zeros(rm.n)
        e[j] = h
        Sfd[:, j] = (residual(rm, model, stt, f_ext, sc, r=r0 + e, cm=cm) -
                     residual(rm, model, stt, f_ext, sc, r=r0 - e, cm=cm)) / (2 * h)
    fd = float(np.linalg.norm(S - Sfd) / np.linalg.norm(Sfd))
    rows.append(("system Jacobian vs central differences of the residual <= 1e-4", fd, fd <= 1e-4))
    st = ReducedState(np.zeros(rm.n), np.zeros(rm.n), sc.dt)
    ok = True
    try:
        for _ in range(5):
            st = step(rm, model, st, f_ext, sc, cm=cm)
    except Exception:
        ok = False
    rows.append(("5 adaptive steps from rest converge", 0.0 if ok else 1.0, ok))
    print(f"{'check':70s} {'value':>12s}  result")
    for name, val, good in rows:
        print(f"{name:70s} {val:12.3e}  {'PASS' if good else 'FAIL'}")
    return EXIT_OK if all(g for _, _, g in rows) else EXIT_VALIDATION


def cmd_bench(cfg):
    """Device ms per fixed Newton iteration (CUDA events, L2 flushed) and adaptive timestep wall ms."""
    from .daereduce import ReducedState
    from .rdsim import SimConfig, step
    from .session import session_for
    model = build_model(cfg)
    rm, cm = load_reduced(cfg, model)
    sc = sim_config(cfg)
    f_ext = external_force(cfg, model)
    s = session_for(rm, model, cm)
    z = np.zeros(rm.n)
    s.step(z, z, f_ext, SimConfig(dt=sc.dt, fixed_iters=1, integration=sc.integration, drop_fict=sc.drop_fict))
    s.bench_replays(5)
    each = s.bench_replays(200)
    st = ReducedState(z, z, sc.dt)
    walls, iters = [], []
    for _ in range(20):
        t0 = time.perf_counter()
        st, (it, _) = step(rm, model, st, f_ext, sc, cm=cm, return_info=True)
        walls.append(1e3 * (time.perf_counter() - t0))
        iters.append(it)
    print(json.dumps({"command": "bench", "ms_per_newton_iteration": float(np.mean(each)),
                      "ms_per_newton_iteration_median": float(np.median(each)),
                      "adaptive_ms_per_step_median": float(np.median(walls)), "newton_iters": iters,
                      "N": int(model.N), "n_p": rm.n_p, "n_q": rm.n_q}))
    return EXIT_OK


COMMANDS = {"gen-data": cmd_gen_data, "train-dae": cmd_train_dae, "train-cubature": cmd_train_cubature,
            "simulate": cmd_simulate, "validate": cmd_validate, "bench": cmd_bench}


def parser():
    ap = argparse.ArgumentParser(prog="nlrom", description="DAE-subspace simulation (arXiv 2102.11026), B200 build")
    ap.add_argument("command", choices=sorted(COMMANDS))
    ap.add_argument("--config", help="RunConfig JSON")
    ap.add_argument("--seed", type=int)
    ap.add_argument("--out", help="output directory (overrides the config)")
    ap.add_argument("--drop-fict", action="store_true", help="drop the fictitious force (SPEC.md:509)")
    g = ap.add_mutually_exclusive_group()
    g.add_argument("--cubature", dest="integration", action="store_const", const="cubature")
    g.add_argument("--exact", dest="integration", action="store_const", const="exact_sum")
    ap.set_defaults(integration=None)
    return ap


def main(argv=None) -> int:
    try:
        args = parser().parse_args(argv)
    except SystemExit as e:   # argparse: --help (0) / bad usage (2)
        return int(e.code or 0)
    try:
        return COMMANDS[args.command](load_config(args))
    except InputError as e:
        print(f"nlrom {args.command}: input error: {e}", file=sys.stderr)
        return EXIT_INPUT


if __name__ == "__main__":
    sys.exit(main())

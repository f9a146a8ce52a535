#!/usr/bin/env python
"""Desk-scale Table 2 analogue (Table 2): greedy NNLS cubature vs
neural cubature (alternating W / S training) at equal |C|, relative reduced-force error on
held-out poses, plus the training-set build time on the GPU (per-element reduced forces of
every element, k_cubature) against the numpy oracle on the host.

    python tools/cubature_table.py [--cfg cfg1] [--train 40] [--test 20] [--sizes 10 20 50]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg1")
    ap.add_argument("--train", type=int, default=200)
    ap.add_argument("--test", type=int, default=50)
    ap.add_argument("--sizes", type=int, nargs="+", default=[10, 20, 50])
    ap.add_argument("--K", type=int, nargs="+", default=[5, 10])
    ap.add_argument("--epochs", type=int, default=15)
    ap.add_argument("--lr", type=float, default=1e-2)
    args = ap.parse_args()
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import cubature_train as ct, densenet
    P = build_problem(args.cfg)
    n = P.cfg.n_p + P.cfg.n_q
    rng = np.random.default_rng(21)
    r_tr = rng.uniform(-0.5, 0.5, (args.train, n))
    r_te = rng.uniform(-0.5, 0.5, (args.test, n))
    ct.build_train_set(P.rm, P.model, r_tr[:1])  # context + graph warm-up
    t0 = time.perf_counter()
    ts = ct.build_train_set(P.rm, P.model, r_tr)
    t_gpu = (time.perf_counter() - t0) / args.train
    te = ct.build_train_set(P.rm, P.model, r_te)
    from helpers import oracle_sim
    from oracle import cubature_train as oct_
    S = oracle_sim(P)
    t0 = time.perf_counter()
    oct_.train_arrays(S.model, S.rm, r_tr[:4])
    t_cpu = (time.perf_counter() - t0) / 4
    rows = []
    for size in args.sizes:
        t0 = time.perf_counter()
        C, w = ct.greedy_cubature(P.rm, P.model, ts, size)
        tg = time.perf_counter() - t0
        row = {"size": size, "greedy_test_error": ct.cubature_error(te, C, w),
               "greedy_train_error": ct.cubature_error(ts, C, w), "greedy_s": tg}
        for K in args.K:
            n_init = K
            rounds = max(0, (size - n_init + K - 1) // K)
            t0 = time.perf_counter()
            cm, log = ct.train_alternating(P.rm, P.model, ts, K=K, rounds=rounds, wnet=P.cm.wnet, n_init=n_init,
                                           epochs=args.epochs, lr=args.lr, return_log=True)
            tn = time.perf_counter() - t0
            W = np.stack([densenet.forward(cm.wnet, u) for u in te.u])[:, cm.C]
            Wtr = np.stack([densenet.forward(cm.wnet, u) for u in ts.u])[:, cm.C]
            row[f"neural_K{K}_size"] = int(cm.C.size)
            row[f"neural_K{K}_test_error"] = ct.cubature_error(te, cm.C, W)
            row[f"neural_K{K}_train_error"] = ct.cubature_error(ts, cm.C, Wtr)
            row[f"neural_K{K}_s"] = tn
            # diagnostic: the neural set with fixed NNLS weights (set quality vs weight-net quality)
            A, b = ct._stacked(ts)
            wn, _ = ct.nnls(A[np.asarray(cm.C)].T, b)
            row[f"neural_K{K}_set_nnls_test_error"] = ct.cubature_error(te, cm.C, wn)
        rows.append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps({"cfg": args.cfg, "train_poses": args.train, "test_poses": args.test,
                      "train_set_ms_per_pose_gpu": t_gpu * 1e3, "train_set_ms_per_pose_oracle_cpu": t_cpu * 1e3,
                      "elements": int(P.model.n_tets), "n": n, "epochs": args.epochs, "lr": args.lr}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: ms per implicit Newton step (DAE J/H/3rd-order + cubature) at the 10-layer DAE.

Workload (BASELINE.json configs[1]): 35x7x7-cube tet mesh
(10,290 tets, N = 6,720 free DOFs), 10-layer width-256 sin DAE with n_q = 30 and
n_p = 30, weight-net cubature with |C| = 500, random-init weights (no checkpoints
ship with the reference), gravity load, dt = 1/60.

One step = one Newton iteration of rdsim.step in fixed-iteration mode: decoder
bundle (value, J, hvv, dJ = svv + hv), weight net, StVK cubature + projection,
assembly of phi and the Eq. 11 system matrix including vhp = H~^T a by complex-step
backprop, LU with partial pivoting, r += dr -- one CUDA-graph replay.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: one process per GPU. Under torch.distributed.run the ranks come from the environment;
`bench.py --gpus N` without WORLD_SIZE launches torch.distributed.run itself. cfg2 is a single
mesh that does not shard (SURVEY.md §8e "replicas only"): every rank runs an independent
replica, `value` is the per-replica ms per Newton iteration (max over ranks) and the aggregate
iteration rate of all replicas is reported beside it. The cfg5 leg (4096 independent sims)
shards sims over the ranks; the cfg4 leg shards strings and does one allreduce per iteration.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per implicit Newton step (DAE J/H/3rd-order + cubature) at 10-layer DAE"
WORKLOAD = "cfg2: 10-layer w256 sin DAE, n_q=30, n_p=30, 10290-tet mesh (N=6720), |C|=500 wnet cubature, fp64"


def config_dict(world):
    """The `config` object of BOTH arms (identical for the same N)."""
    return {"workload": WORKLOAD,
            "step": "one Newton iteration (fixed-iteration mode: E + J + LU-pp + r += dr)",
            "l2": "flushed (256 MB write) before every timed replay, outside the timed events",
            "replicas": world,
            "parallelism": (f"replicas x{world} (cfg2 does not shard, SURVEY.md §8e)" if world > 1
                            else "single GPU")}


def peaks():
    """(MEASURED_PEAKS.json, tensor peaks). The tensor peaks come from profiles/r02_tc_peaks.json
    (tools/tc_peaks.py: fp64 DMMA and tcgen05 kind::i8, clocks sampled) or, without it, the
    round-1 fp64 probe (profiles/fp64_peak.json)."""
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    tc = {"fp64": None, "i8": None, "source": "absent"}
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r02_tc_peaks.json")))
        tc = {"fp64": t["dmma_tflops"], "i8": t["i8_best_tops"],
              "source": "profiles/r02_tc_peaks.json (tools/probes/tc_peak.cu, clocks sampled): fp64 DMMA, "
                        "tcgen05 kind::i8 M=128 N>=128 (the Ozaki MMAs are mostly N=128..256 runs of digit "
                        "planes); MEASURED_PEAKS.json has neither"}
    except Exception:
        try:
            tc["fp64"] = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dmma_tflops"]
            tc["source"] = "profiles/fp64_peak.json: measured DMMA.8x8x4 fp64 (MEASURED_PEAKS.json has no fp64 entry)"
        except Exception:
            pass
    return p, tc


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 20 ms while the GPU is loaded."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.005)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------------- process topology
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: run N ranks through torch.distributed.run."""
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
               NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def dist_setup(backend):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "INFO")        # communicator lines show nRanks
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return rank, world, local


def barrier_max(world, value):
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# --------------------------------------------------------------------------- roofline helpers
def jet_groups(n_q, batched):
    """Mirror of ctx.cu choose_groups: (columns per group G, groups per sim)."""
    if batched:
        g = min((1, 3, 7, 15), key=lambda c: ((4 + 4 * c) * (-(-n_q // c)), c))
    else:
        g = next((c for c in (1, 3, 5, 7, 15) if c >= n_q), 3) if n_q <= 15 else 3
    return 4 + 4 * g, -(-n_q // g)


def decoder_flops(P, n_sims=1):
    """(F_dec per sim per §8d, executed flops per sim of our collapsed passes)."""
    c = P.cfg
    N, w, n_p, n_q, L = P.model.N, c.width, c.n_p, c.n_q, c.n_fc
    widths = [n_q] + [w] * (L - 1) + [N]
    mac = sum(a * b for a, b in zip(widths[:-1], widths[1:]))
    hidden_mac = mac - w * N
    F = (18 * n_q + 6) * (2.0 * mac + 4.0 * N * n_p)
    batched = n_sims * (4 + 4 * n_q) >= 2048
    G, gps = jet_groups(n_q, batched)
    hid_cols = gps * G                               # grouped jet columns through the sin layers
    out_cols = 2 + 2 * n_q                           # [D_1, 2 D_ss | (D_t, 2 D_tss + D_tr) x n_q] per sim
    ctas2 = -(-(n_sims * 2 * n_q) // 128) * -(-w // 64)
    shared = batched and ctas2 >= 4 * 148            # mirror of ctx.cu decoder_backward
    bwd_cols = (1 + n_q) if shared else 2 * n_q      # vhp backward: shared real part at >= 4 waves
    executed = 2.0 * hid_cols * hidden_mac + 2.0 * out_cols * N * w + 2.0 * N * w + 2.0 * bwd_cols * hidden_mac
    return F, executed


def decoder_roofline(P, stage_ms, n_sims, tc, tc_info=(0, 0, 0)):
    """Roofline of the decoder bundle (hidden jet chain + output layer + vhp backward chain).

    `achieved` counts the work the kernels EXECUTE on their pipe; the §8d algorithmic figure of
    the reference pass structure is reported separately as the work the collapsed bundle
    replaces (it is not a pipe fraction). Batched contexts run most of the bundle's GEMMs on the
    tcgen05 Ozaki GEMM (tc_info = hidden layers, output layer, vhp backward layers on it): those
    are counted in executed kind::i8 ops (28 digit-pair MMAs per 32-deep K chunk over the
    128-row / 64-column padded tiles) against the measured kind::i8 peak, the remaining DMMA
    GEMMs in fp64 flops against the DMMA peak, and `frac` is the time-weighted mean of the
    stages' pipe fractions (the share of the bundle's time its pipes would be busy at peak)."""
    fp64 = tc["fp64"]
    F, ex = decoder_flops(P, n_sims)
    dec_ms = stage_ms[0] + stage_ms[1] + stage_ms[2]
    executed = ex * n_sims / (dec_ms * 1e-3) / 1e12
    algorithmic = F * n_sims / (dec_ms * 1e-3) / 1e12
    out = {"bound": "tensor",
           "kernel": "decoder bundle: hidden jet layers + output GEMM (EpiJetOutC) + vhp backprop layers, fp64 DMMA",
           "achieved": executed, "peak": fp64, "unit": "TFLOP/s",
           "frac": (executed / fp64) if fp64 else None, "traffic": None, "peak_source": tc["source"],
           "kernel_ms": dec_ms, "executed_flops_per_launch": ex * n_sims,
           "algorithmic": {"flops_per_launch": F * n_sims, "tflops_equivalent": algorithmic,
                           "def": "SURVEY.md §8d F_dec = (18 n_q+6)(2 sum in*out + 4 N n_p) per sim: the "
                                  "reference's 4 n_q + 2 passes; the jet bundle executes fewer columns"},
           "stages_ms": {"hidden_jet": stage_ms[0], "output_gemm": stage_ms[1], "vhp_bwd": stage_ms[2]}}
    n_hid, n_out, n_bwd = tc_info
    if n_hid or n_out or n_bwd:
        c = P.cfg
        w, n_q, N = c.width, c.n_q, P.model.N
        G, gps = jet_groups(n_q, True)
        up = lambda x, m: -(-x // m) * m
        P1 = 1 + n_q
        ocs = (64 // P1) * P1
        i8 = [n_hid * 28 * 2.0 * w * w * up(n_sims * G * gps, 64),
              n_out * 28 * 2.0 * up(N, 128) * w * up(n_sims * (2 + 2 * n_q), 64),
              n_bwd * 28 * 2.0 * w * w * (-(-(n_sims * P1) // ocs) * 64) if ocs else 0.0]
        # fp64 flops of the stages' remaining DMMA GEMMs: each stage's executed flops minus the
        # GEMMs on tcgen05 (the seed layer K = n_q, the vhp seed (P W_L)^T a and the last backward
        # layer M = n_q always stay on DMMA)
        L = c.n_fc
        hidden_mac = n_q * w + (L - 2) * w * w
        batched = n_sims * (4 + 4 * n_q) >= 2048
        bwd_cols = (1 + n_q) if n_bwd else None
        if bwd_cols is None:
            ctas2 = -(-(n_sims * 2 * n_q) // 128) * -(-w // 64)
            bwd_cols = (1 + n_q) if (batched and ctas2 >= 4 * 148) else 2 * n_q
        ex_stage = [2.0 * G * gps * n_sims * hidden_mac,
                    2.0 * (2 + 2 * n_q) * n_sims * N * w,
                    2.0 * n_sims * N * w + 2.0 * bwd_cols * n_sims * hidden_mac]
        tc_f64 = [2.0 * G * gps * n_sims * w * w * n_hid,
                  ex_stage[1] if n_out else 0.0,
                  2.0 * (1 + n_q) * n_sims * w * w * n_bwd]
        dm = [max(0.0, e - t) for e, t in zip(ex_stage, tc_f64)]
        stages = []
        for k, name in enumerate(("hidden_jet", "output_gemm", "vhp_bwd")):
            t = stage_ms[k] * 1e-3
            f_i8 = i8[k] / t / 1e12 / tc["i8"] if tc["i8"] else None
            f_dm = dm[k] / t / 1e12 / fp64 if fp64 else None
            stages.append({"stage": name, "ms": stage_ms[k], "i8_ops": i8[k], "i8_tops": i8[k] / t / 1e12,
                           "fp64_flops": dm[k], "fp64_tflops": dm[k] / t / 1e12,
                           "pipe_frac": (f_i8 or 0.0) + (f_dm or 0.0)})
        frac = sum(st["pipe_frac"] * st["ms"] for st in stages) / dec_ms
        out["kernel"] = ("decoder bundle on tcgen05 kind::i8 (Ozaki fp64, 7 digits): %d hidden jet layers, "
                         "%s, %d vhp backward layers; seed / vhp-seed / last backward GEMMs on fp64 DMMA"
                         % (n_hid, "output layer" if n_out else "output layer on DMMA", n_bwd))
        out["unit"] = "pipe fraction (time-weighted)"
        out["achieved"] = frac
        out["peak"] = 1.0
        out["frac"] = frac
        out["pipes"] = {"i8_peak_tops": tc["i8"], "fp64_peak_tflops": fp64, "stages": stages,
                        "i8_ops_per_launch": sum(i8), "i8_tops": sum(i8) / (dec_ms * 1e-3) / 1e12,
                        "fp64_equivalent_tflops": executed}
    return out


# --------------------------------------------------------------------------- extra legs
def coupled_leg(args, rank, world):
    """cfg4: the 320-string puffer ball, strings sharded over the ranks, the core
    replicated; per Newton iteration one graph per rank + ONE allreduce of 16 doubles (NCCL on
    the context stream) + the core solve / string update. Device time per iteration with CUDA
    events on the context stream, L2 flushed before every iteration, max over ranks."""
    import torch
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim, synth
    from paper_2102_11026_b200.substructure import Core, Scene
    P = build_problem("cfg4")
    k = args.strings
    R = synth.string_frames(k)
    f_world = np.tile(P.f_ext, (k, 1))
    m_core = 2.0 * float(P.model.mass[0::3].sum())
    sc = Scene(P.rm, P.model, P.cm, R, f_world, Core(m_core, 50.0, np.array([0.0, -9.81 * m_core, 0.0])))
    rb, rdb, cb, cdb = synth.coupled_state(k, P.cfg.n_p, P.cfg.n_q)
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1)
    sc.step(rb, rdb, cb, cdb, cfg)          # captures the graphs
    sc.begin(rb, rdb, cb, cdb, cfg)
    flush = torch.empty(32 << 20, dtype=torch.float64, device=sc.partial.device)
    iters = 20
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for _ in range(3):
        sc.eval(True); sc.reduce(); sc.update(1, 1.0)
    barrier(world)
    torch.cuda.synchronize()
    with torch.cuda.stream(sc.stream):
        for e0, e1 in evs:
            flush.fill_(1.0)
            e0.record(sc.stream)
            sc.eval(True)
            sc.reduce()
            sc.update(1, 1.0)
            e1.record(sc.stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = barrier_max(world, sum(e0.elapsed_time(e1) for e0, e1 in evs) / iters)
    _, _, _, _, _, nrm = sc.step(rb, rdb, cb, cdb, rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=3))
    return {"workload": "cfg4: puffer ball, %d strings x (36x3x3 tets, N=1728, n_p=10, n_q=5, 8-layer w64 DAE, "
                        "|C|=36) on a translating core, %d strings on rank 0" % (k, sc.hi - sc.lo),
            "scaling": "strong (total strings fixed)", "ms_per_newton_iteration": ms,
            "string_iterations_per_s": k * 1e3 / ms, "exchange": "1 allreduce of 16 fp64 per iteration"
            + (" (NCCL)" if world > 1 else " (single rank: none)"),
            "residual_after_3_iters": nrm, "l2": "flushed before every iteration",
            "gpu_launches_per_iteration": sc.launches_per_iteration()}


def batched_leg(args, rank, world):
    """cfg5: 4096 independent 10-layer DAE sims, sharded over the ranks with
    no data-path collective (sim ranges of paper_2102_11026_b200.shard); one graph replay = one
    Newton iteration of every local sim."""
    import torch
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.shard import SimShard
    P = build_problem("cfg5")
    total = args.batched_sims
    sh = SimShard(P.rm, P.model, P.cm, total, rank, world)
    ns = sh.n_local
    n = P.cfg.n_p + P.cfg.n_q
    rng = np.random.default_rng(4 + sh.lo)
    rb = rng.uniform(-0.05, 0.05, ns * n)
    rdb = rng.uniform(-0.1, 0.1, ns * n)
    s = sh.session
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1)
    s.step(rb, rdb, np.tile(P.f_ext, ns), cfg)
    iters = 10
    s.bench_replays(3, flush_l2=True)
    barrier(world)
    torch.cuda.synchronize()
    each = s.bench_replays(iters, flush_l2=True)
    torch.cuda.synchronize()
    barrier(world)
    ms = barrier_max(world, float(each.mean()))
    pk, tc = peaks()
    fp64 = tc["fp64"]
    stage_ms = s.bench_kernels(3, flush_l2=True)
    roof = decoder_roofline(P, stage_ms, ns, tc, s.tc_info())
    cub_ms, cub_bytes = s.bench_cubature(5, flush_l2=True)
    hbm = pk.get("hbm_gbs")
    cub_gbs = cub_bytes / (cub_ms * 1e-3) / 1e9
    traffic = None
    try:
        if ns == 4096:  # the captured configuration
            traffic = json.load(open(os.path.join(ROOT, "profiles", "dominant_traffic.json")))[
                "k_cubature_cfg5"]["dram_bytes_per_launch"]
    except Exception:
        pass
    cub_roof = {"bound": "hbm", "kernel": "k_cubature (all %d local sims, |C| elements each)" % ns,
                "achieved": cub_gbs, "peak": hbm, "unit": "GB/s", "frac": (cub_gbs / hbm) if hbm else None,
                "traffic": traffic, "kernel_ms": cub_ms, "algorithmic_bytes_per_launch": cub_bytes,
                "algorithmic_def": "SURVEY.md 8d B_cub = |C| (96 n + 200) + 8 (n + n^2) per sim",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else "absent"}
    # ~(24 n^2 + 312 n + 3000) flop per element: 10.7 flop/B at cfg5, above the
    # fp64 ridge (37 TFLOP/s / 6.55 TB/s = 5.7 flop/B), so the fp64 pipe, not HBM, bounds it
    n_c = P.cm.C.size if hasattr(P.cm.C, "size") else len(P.cm.C)
    cub_flops = ns * n_c * (24.0 * n * n + 312.0 * n + 3000.0)
    cub_roof["fp64_view"] = {"bound": "tensor", "achieved": cub_flops / (cub_ms * 1e-3) / 1e12, "peak": fp64,
                             "unit": "TFLOP/s", "frac": (cub_flops / (cub_ms * 1e-3) / 1e12 / fp64) if fp64 else None,
                             "algorithmic_flops_per_launch": cub_flops,
                             "min_time_ms_at_fp64_peak": (cub_flops / (fp64 * 1e12) * 1e3) if fp64 else None}
    launches = s.launches_per_iteration()
    del s, sh
    return {"workload": "cfg5: %d independent sims (10-layer w256 DAE, n_q=20, n_p=10, N=960, |C|=100), "
                        "%d per GPU, no per-iteration collective" % (total, ns),
            "scaling": "strong (total sims fixed)", "ms_per_iteration": ms,
            "ms_per_iteration_median_rank0": float(np.median(each)),
            "sim_iterations_per_s": total * 1e3 / ms, "iterations": iters,
            "l2": "flushed between timed iterations", "decoder_roofline_rank0": roof,
            "cubature_roofline_rank0": cub_roof, "gpu_launches_per_iteration": launches}


def fullspace_leg(args, rank, world):
    """elastic.fullspace_step on the cfg2 mesh (N = 6720):
    gravity from rest, wall clock per step through the public API (host arrays in and out),
    beside one step of the scipy-direct oracle -- the ground-truth integrator the reduced step
    replaces."""
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200.fullspace import FullspaceConfig, FullspaceSession
    P = build_problem("cfg2", n_fc=2, width=16)
    fs = FullspaceSession(P.model)
    cfg = FullspaceConfig()
    u = v = np.zeros(P.model.N)
    u, v, _ = fs.step(u, v, P.f_ext, P.cfg.dt, cfg)
    ts, its, cgs = [], [], []
    for _ in range(4):
        t0 = time.perf_counter()
        u, v, info = fs.step(u, v, P.f_ext, P.cfg.dt, cfg)
        ts.append(time.perf_counter() - t0)
        its.append(info.iters)
        cgs.append(info.cg_iters)
    out = {"workload": "cfg2 mesh (10290 tets, N = 6720), StVK implicit Euler, gravity, dt = 1/60",
           "ms_per_step": barrier_max(world, 1e3 * sorted(ts)[len(ts) // 2]),
           "newton_iters": its, "pcg_iters": cgs}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = fullspace_cpu_baseline(P, u, v)
    return out


def fullspace_cpu_baseline(P, u, v):
    """cpu_baseline of the full-space leg: one step of the scipy-direct oracle on the host."""
    from oracle import elastic as oe, fullspace as ofs
    c = P.cfg
    om = oe.OModel(P.data["verts"], P.data["tets"], P.data["fixed"], c.young, c.poisson, c.density, c.alpha)
    t0 = time.perf_counter()
    ofs.fullspace_step(om, u, v, P.f_ext, c.dt)
    return {"value": 1e3 * (time.perf_counter() - t0), "unit": "ms per step", "kind": "port",
            "sample": "1 step of oracle/fullspace.py (numpy + scipy spsolve) at the same state"}


# --------------------------------------------------------------------------- CPU arms (oracle = checker / baseline)
def blas_threads(n):
    """Pin the host BLAS pool to n threads (torchrun exports OMP_NUM_THREADS=1); returns the
    thread count the pools actually report."""
    from threadpoolctl import threadpool_info, threadpool_limits
    threadpool_limits(limits=n)
    info = threadpool_info()
    return max([d.get("num_threads", 1) for d in info] or [1])


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_iteration_runner(P):
    """One Newton iteration of the reference algorithm (numpy fp64 restatement of SPEC
    rdsim: residual + analytic system Jacobian with the reference pass structure + LU)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import scipy.linalg
    from helpers import oracle_sim
    from oracle import rdsim as ors
    S = oracle_sim(P)
    r, rb, rdb = P.random_state()
    oc = ors.OSimConfig(dt=P.cfg.dt)
    state = (rb, rdb)
    cur = {"r": r.copy()}

    def one():
        phi = ors.residual(S, cur["r"], state, P.f_ext, oc)
        J = ors.system_jacobian(S, cur["r"], state, P.f_ext, oc)
        cur["r"] = cur["r"] + scipy.linalg.lu_solve(scipy.linalg.lu_factor(J), -phi)
    return one


def timed_oracle(one, n_min, budget_s):
    one()  # warm-up
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < n_min or (time.perf_counter() < t_end and len(times) < 30):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    return times


def cpu_baseline(P, budget_s=10.0):
    """The oracle on the box's host cores: all cores (the reported baseline) and 1 thread (the
    paper's single-core convention)."""
    one = oracle_iteration_runner(P)
    cores = blas_threads(host_cores())
    times = timed_oracle(one, 3, budget_s)
    t1 = blas_threads(1)
    times1 = timed_oracle(one, 2, budget_s / 2)
    blas_threads(host_cores())
    return {"value": 1e3 * float(np.median(times)), "unit": "ms", "cores": cores, "kind": "port",
            "cpu": cpu_model(),
            "sample": f"{len(times)} Newton iterations of the numpy-fp64 oracle (SPEC rdsim residual + "
                      f"system_jacobian with the 4n_q+2 reference passes + LU) at cfg2, median",
            "single_thread": {"value": 1e3 * float(np.median(times1)), "unit": "ms", "cores": t1,
                              "sample": f"{len(times1)} iterations, median"}}


def parity_check(s, P, rb, rdb, iters=3):
    """The exact benchmarked graph vs the oracle (checker): from the step's predictor
    r0 = r_bar + dt rdot_bar, `iters` replays of the timed one-iteration graph against `iters`
    oracle Newton iterations. r: norm-relative max error after each update;
    phi: max error at each iterate relative to ||phi(r0)||_inf (the step's residual scale: phi
    itself converges to roundoff, where a relative error is meaningless)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import scipy.linalg
    from helpers import oracle_sim
    from oracle import rdsim as ors
    S = oracle_sim(P)
    oc = ors.OSimConfig(dt=P.cfg.dt)
    ro = rb + P.cfg.dt * rdb
    s.set_iterate(ro)
    err_r = err_phi = 0.0
    phi_scale = None
    per_iter = []
    for _ in range(iters):
        s.iterate(1)
        rg, phig, _ = s.get_iterate()
        phio = ors.residual(S, ro, (rb, rdb), P.f_ext, oc)
        J = ors.system_jacobian(S, ro, (rb, rdb), P.f_ext, oc)
        ro = ro + scipy.linalg.lu_solve(scipy.linalg.lu_factor(J), -phio)
        if phi_scale is None:
            phi_scale = float(np.abs(phio).max())
        e_phi = float(np.abs(phig - phio).max() / phi_scale)
        e_r = float(np.abs(rg - ro).max() / np.abs(ro).max())
        per_iter.append({"rel_err_r": e_r, "err_phi_over_phi0": e_phi, "phi_norm": float(np.linalg.norm(phio))})
        err_phi, err_r = max(err_phi, e_phi), max(err_r, e_r)
    return {"iterations": iters, "max_rel_err_r": err_r, "max_err_phi_over_phi0": err_phi, "tol": 1e-10,
            "ok": bool(err_r <= 1e-10 and err_phi <= 1e-10), "per_iteration": per_iter,
            "def": "the timed graph replayed from the step predictor vs oracle/rdsim.py fixed Newton iterations; "
                   "r: ||r - r_oracle||_inf / ||r_oracle||_inf, phi: ||phi - phi_oracle||_inf / ||phi_oracle(r0)||_inf"}


def run_reference(args):
    """Reference arm: the reference algorithm's CPU implementation (the oracle port; the
    reference ships no executable code above mcx) on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from paper_2102_11026_b200.problem import build_problem
    cores = blas_threads(host_cores())
    P = build_problem("cfg2")
    one = oracle_iteration_runner(P)
    for _ in range(args.warmup):
        one()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded random-init weights, SURVEY.md §8d)",
        "config": config_dict(world),
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port", "cpu": cpu_model(),
                         "sample": f"{args.steps} Newton iterations of the numpy-fp64 oracle at cfg2 (mean), "
                                   f"BLAS pool pinned to {cores} threads"},
        "ms_median": 1e3 * float(np.median(times)),
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------- GPU arm
def load_gpu(s, seconds):
    """Keep the GPU busy with flushed replays for `seconds` (clock sampling window)."""
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        s.bench_replays(50, flush_l2=True)


def run_ours(args):
    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl ours needs a CUDA device (the product path has no CPU fallback)")
    rank, world, local = dist_setup("nccl")
    os.environ["NLROM_DEVICE"] = str(local)
    torch.cuda.set_device(local)
    barrier(world)   # creates the NCCL communicator (NCCL_DEBUG=INFO prints nRanks)
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.session import session_for
    P = build_problem("cfg2")
    s = session_for(P.rm, P.model, P.cm)
    n = P.cfg.n_p + P.cfg.n_q
    # a physically evolving state: 5 timesteps under gravity from rest (3 Newton iterations
    # each), so the timed Newton iterations converge as in a simulation (an arbitrary random
    # state makes undamped fixed-iteration Newton diverge and feeds sin / cos garbage)
    rb, rdb = np.zeros(n), np.zeros(n)
    for _ in range(5):
        rb, rdb, _, _ = s.step(rb, rdb, P.f_ext, rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=3))
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1)

    def arm():
        """(Re)load the benchmark state: r_bar, rdot_bar, f_ext and the iterate the timed
        region starts from (other API calls below move the context's state)."""
        s.step(rb, rdb, P.f_ext, cfg)          # captures the graphs on first use
        return s.get_iterate()[0]

    r_start = arm()
    s.bench_replays(max(args.warmup, 3), flush_l2=True)
    s.set_iterate(r_start)

    with ClockSampler(local) as clk:
        load_gpu(s, 0.5)                       # clocks are sampled under the same load
        s.set_iterate(r_start)
        barrier(world)
        torch.cuda.synchronize()
        each = s.bench_replays(args.steps, flush_l2=True)
        torch.cuda.synchronize()
        barrier(world)
        load_gpu(s, 0.5)
    ms_iter = barrier_max(world, float(each.mean()))

    # e2e through the public API (rdsim.step, host buffers, H2D/D2H inside), 3 fixed iterations/step
    from paper_2102_11026_b200.daereduce import ReducedState
    cfg3 = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=3)
    st = ReducedState(rb, rdb, cfg3.dt)
    for _ in range(2):
        rdsim.step(P.rm, P.model, st, P.f_ext, cfg3)
    n_e2e = max(5, args.steps // 3)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        st = rdsim.step(P.rm, P.model, st, P.f_ext, cfg3)
    e2e_ms = barrier_max(world, 1e3 * (time.perf_counter() - t0) / (n_e2e * 3))
    h2d = (2 * n + P.model.N) * 8
    d2h = 2 * n * 8 + 8

    # adaptive timesteps (||phi|| <= newton_tol = 1e-8, line search on): the
    # Newton and line-search loops run on the device as conditional graph nodes, one launch and
    # one host sync per timestep (wall clock through the public API, host buffers)
    cfgA = rdsim.SimConfig(dt=P.cfg.dt)
    stA = ReducedState(rb, rdb, cfgA.dt)
    for _ in range(2):
        stA = rdsim.step(P.rm, P.model, stA, P.f_ext, cfgA)
    ad_ms, ad_it = [], []
    for _ in range(max(10, args.steps // 20)):
        t0 = time.perf_counter()
        stA, (itA, _) = rdsim.step(P.rm, P.model, stA, P.f_ext, cfgA, return_info=True)
        ad_ms.append(1e3 * (time.perf_counter() - t0))
        ad_it.append(itA)
    adaptive = {"ms_per_timestep_median": float(np.median(ad_ms)), "newton_iters": ad_it,
                "newton_iters_mean": float(np.mean(ad_it)), "hz": 1e3 / float(np.median(ad_ms)),
                "how": "nlrom.rdsim.step, adaptive (newton_tol 1e-8, line search), host numpy in/out, "
                       "Newton + line-search loops as device conditional graph nodes, wall clock per step"}

    # roofline: stages timed live with CUDA events on the context stream (L2 flushed before each
    # launch); in-graph share of the decoder bundle from the prefix-graph profile
    pk, tc = peaks()
    fp64 = tc["fp64"]
    stage_ms = s.bench_kernels(max(20, args.steps // 4), flush_l2=True)
    roof = decoder_roofline(P, stage_ms, 1, tc)
    roof["share_of_step_isolated"] = roof["kernel_ms"] / ms_iter
    roof["lu_ms_isolated"] = stage_ms[3]
    try:
        marg, _ = s.bench_prefix(n_iters=20, flush_l2=True)
        dec_names = ("k_mlp_jet_fwd", "gemm_ws_kernel", "gemm_tn_kernel", "k_mlp_dual_bwd", "k_gemv_t2")
        in_graph = sum(v for nm, v in marg if any(k in nm for k in dec_names))
        roof["share_of_step_in_graph"] = in_graph / max(sum(v for _, v in marg), 1e-9)
        roof["in_graph_marginal_ms"] = {nm.split("(")[0][:60]: round(v, 5) for nm, v in marg}
    except Exception as e:  # profiling aid only
        roof["share_of_step_in_graph"] = f"unavailable: {e}"
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "dominant_traffic.json")))
        roof["traffic"] = sum(tr.get(k, {}).get("dram_bytes_per_launch", 0) for k in
                              ("k_mlp_jet_fwd", "gemm_tn_kernel<CfgOutC,EpiJetOutC>", "k_mlp_dual_bwd")) or None
    except Exception:
        pass

    batched = None if args.no_batched else batched_leg(args, rank, world)
    coupled = None if args.no_coupled else coupled_leg(args, rank, world)
    fullspace = None if args.no_fullspace else fullspace_leg(args, rank, world)

    cpu = parity = None
    if rank == 0:
        arm()
        parity = parity_check(s, P, rb, rdb)
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(P)

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_iter, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_iter, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded random-init weights, SURVEY.md §8d)",
            "config": config_dict(world),
            "timing": {"mean_ms": float(each.mean()), "median_ms": float(np.median(each)),
                       "p90_ms": float(np.percentile(each, 90)), "min_ms": float(each.min()), "replays": len(each),
                       "how": "CUDA events around each graph replay on the context stream, max over ranks of "
                              "the mean"},
            "aggregate": {"newton_iterations_per_s": world * 1e3 / ms_iter,
                          "def": "all replicas' iterations per second (each replica at value ms per iteration)"},
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d * 1, "d2h_bytes_per_step": d2h,
                    "how": "nlrom.rdsim.step (host numpy in/out), fixed_iters=3, wall clock / 3, max over ranks"},
            "gpu_launches": s.launches_per_iteration() * args.steps,
            "roofline": roof,
            "parity": parity,
            "batched_cfg5": batched,
            "coupled_cfg4": coupled,
            "fullspace_cfg2": fullspace,
            "cpu_baseline": cpu,
            "clocks": dict(clk.summary(), window="0.5 s load + timed replays + 0.5 s load"),
            "hz_at_3_iters": 1000.0 / (3 * ms_iter),
            "adaptive_step": adaptive,
        }
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batched", action="store_true", help="skip the cfg5 4096-sim throughput leg")
    ap.add_argument("--batched-sims", type=int, default=4096)
    ap.add_argument("--no-coupled", action="store_true", help="skip the cfg4 320-string coupled leg")
    ap.add_argument("--strings", type=int, default=320)
    ap.add_argument("--no-fullspace", action="store_true", help="skip the full-space implicit Euler leg")
    args = ap.parse_args()
    if os.environ.get("NLROM_DEBUG_SKIP"):
        raise SystemExit("bench.py refuses to run with NLROM_DEBUG_SKIP set (kernels would be dropped)")
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

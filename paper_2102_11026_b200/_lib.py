"""ctypes binding of the C ABI in include/nlrom_b200.h (libnlrom_b200.so, built in-tree).

This is the reference-side binding a maintainer of `nlrom` would add:
the shared library is loaded from the package directory; if it is missing the
import fails loudly -- there is no CPU fallback for the hot path.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnlrom_b200.so")

OK, ERR_ORDER, ERR_DIM, ERR_NONFINITE, ERR_NEWTON, ERR_CUDA, ERR_ARG, ERR_NOCACHE = range(8)
LAYER_FC, LAYER_FILTER, LAYER_SIN, LAYER_SQUARE = range(4)
OP_VALUE, OP_JVP, OP_JACOBIAN, OP_HVV, OP_HV, OP_SVV, OP_VJP, OP_VHP = range(8)

EXPORTED = [
    "nlrom_net_create", "nlrom_net_destroy", "nlrom_net_last_error", "nlrom_net_forward", "nlrom_net_backward",
    "nlrom_create", "nlrom_destroy", "nlrom_last_error", "nlrom_diffop", "nlrom_residual",
    "nlrom_system_jacobian", "nlrom_delta_j", "nlrom_fictitious_force", "nlrom_wnet_forward",
    "nlrom_cubature_integrate", "nlrom_full_displacement", "nlrom_jtilde", "nlrom_step", "nlrom_step_device",
    "nlrom_bench_iterations", "nlrom_bench_replays", "nlrom_iterate", "nlrom_get_iterate", "nlrom_set_iterate",
    "nlrom_launches_per_iteration", "nlrom_tc_layers", "nlrom_tc_info", "nlrom_element_forces",
    "nlrom_element_reduced_forces", "nlrom_bench_kernels", "nlrom_bench_cubature", "nlrom_train_forces", "nlrom_stream", "nlrom_coupled_setup",
    "nlrom_coupled_begin", "nlrom_coupled_eval", "nlrom_coupled_update", "nlrom_coupled_read",
    "nlrom_coupled_launches", "nlrom_bench_prefix", "nlrom_debug_poison_shared_memory",
    "nlrom_fs_create", "nlrom_fs_destroy", "nlrom_fs_last_error", "nlrom_fs_step", "nlrom_fs_energy_force",
]


class LayerDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("in_dim", C.c_int), ("out_dim", C.c_int),
                ("W", C.POINTER(C.c_double)), ("b", C.POINTER(C.c_double)), ("n_basis", C.c_int)]


class ModelDesc(C.Structure):
    _fields_ = [
        ("N", C.c_int), ("n_p", C.c_int), ("n_q", C.c_int),
        ("n_fc", C.c_int), ("widths", C.POINTER(C.c_int)),
        ("W", C.POINTER(C.POINTER(C.c_double))), ("b", C.POINTER(C.POINTER(C.c_double))),
        ("U", C.POINTER(C.c_double)), ("mass", C.POINTER(C.c_double)),
        ("n_verts", C.c_int), ("n_tets", C.c_int), ("tets", C.POINTER(C.c_int)), ("vert_dof", C.POINTER(C.c_int)),
        ("Dm_inv", C.POINTER(C.c_double)), ("vol", C.POINTER(C.c_double)),
        ("mu", C.c_double), ("lam", C.c_double), ("alpha", C.c_double),
        ("n_cub", C.c_int), ("cub_elems", C.POINTER(C.c_int)),
        ("wnet_width", C.c_int),
        ("wnet_W", C.POINTER(C.POINTER(C.c_double))), ("wnet_b", C.POINTER(C.POINTER(C.c_double))),
        ("n_sims", C.c_int),
    ]


class SimCfg(C.Structure):
    _fields_ = [("dt", C.c_double), ("newton_tol", C.c_double), ("max_iters", C.c_int), ("drop_fict", C.c_int),
                ("integration", C.c_int), ("line_search", C.c_int), ("fixed_iters", C.c_int)]


class StepInfo(C.Structure):
    _fields_ = [("iters", C.c_int), ("res_norm", C.c_double), ("status", C.c_int)]


class FsDesc(C.Structure):
    _fields_ = [("n_verts", C.c_int), ("n_tets", C.c_int), ("tets", C.POINTER(C.c_int)),
                ("vert_dof", C.POINTER(C.c_int)), ("Dm_inv", C.POINTER(C.c_double)), ("vol", C.POINTER(C.c_double)),
                ("mass", C.POINTER(C.c_double)), ("mu", C.c_double), ("lam", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double)]


class FsCfg(C.Structure):
    _fields_ = [("dt", C.c_double), ("newton_tol", C.c_double), ("max_iters", C.c_int), ("cg_tol", C.c_double),
                ("cg_max_iters", C.c_int)]


class FsInfo(C.Structure):
    _fields_ = [("iters", C.c_int), ("cg_iters", C.c_int), ("res_norm", C.c_double), ("energy", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        sig = {
            "nlrom_net_create": (C.c_int, [C.POINTER(vp), C.c_int, C.c_int, C.POINTER(LayerDesc)]),
            "nlrom_net_destroy": (None, [vp]),
            "nlrom_net_last_error": (C.c_char_p, [vp]),
            "nlrom_net_forward": (C.c_int, [vp, C.c_int, dp, C.c_int, dp]),
            "nlrom_net_backward": (C.c_int, [vp, C.c_int, dp, dp, C.c_int, dp, dp]),
            "nlrom_create": (C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(ModelDesc)]),
            "nlrom_destroy": (None, [vp]),
            "nlrom_last_error": (C.c_char_p, [vp]),
            "nlrom_diffop": (C.c_int, [vp, C.c_int, dp, dp, C.c_double, C.c_int, dp]),
            "nlrom_residual": (C.c_int, [vp, dp, dp, dp, dp, C.POINTER(SimCfg), dp]),
            "nlrom_system_jacobian": (C.c_int, [vp, dp, dp, dp, dp, C.POINTER(SimCfg), dp]),
            "nlrom_delta_j": (C.c_int, [vp, dp, dp, dp, C.c_double, C.c_int, dp]),
            "nlrom_fictitious_force": (C.c_int, [vp, dp, dp, dp]),
            "nlrom_wnet_forward": (C.c_int, [vp, dp, dp, C.c_int64]),
            "nlrom_cubature_integrate": (C.c_int, [vp, dp, C.c_int, dp, dp]),
            "nlrom_full_displacement": (C.c_int, [vp, dp, dp]),
            "nlrom_jtilde": (C.c_int, [vp, dp, dp]),
            "nlrom_step": (C.c_int, [vp, vp, vp, vp, C.POINTER(SimCfg), vp, vp, C.POINTER(StepInfo)]),
            "nlrom_step_device": (C.c_int, [vp, vp, vp, vp, C.POINTER(SimCfg), vp, vp, vp]),
            "nlrom_bench_iterations": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
            "nlrom_launches_per_iteration": (C.c_int, [vp]),
            "nlrom_tc_layers": (C.c_int, [vp]),
            "nlrom_tc_info": (C.c_int, [vp, ip]),
            "nlrom_bench_replays": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_float)]),
            "nlrom_iterate": (C.c_int, [vp, C.c_int]),
            "nlrom_get_iterate": (C.c_int, [vp, dp, dp, dp]),
            "nlrom_set_iterate": (C.c_int, [vp, dp]),
            "nlrom_bench_kernels": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_float)]),
            "nlrom_bench_cubature": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_float), dp]),
            "nlrom_train_forces": (C.c_int, [vp, dp, C.c_int, dp, dp]),
            "nlrom_element_forces": (C.c_int, [vp, dp, C.c_int, dp, dp]),
            "nlrom_element_reduced_forces": (C.c_int, [vp, dp, ip, C.c_int, dp]),
            "nlrom_stream": (C.c_int, [vp, C.POINTER(vp)]),
            "nlrom_coupled_setup": (C.c_int, [vp, dp, dp, C.c_int, C.c_double, C.c_double, dp]),
            "nlrom_coupled_begin": (C.c_int, [vp, dp, dp, dp, dp, C.POINTER(SimCfg)]),
            "nlrom_coupled_eval": (C.c_int, [vp, C.POINTER(SimCfg), C.c_int, vp]),
            "nlrom_coupled_update": (C.c_int, [vp, C.POINTER(SimCfg), vp, C.c_int, C.c_double, dp]),
            "nlrom_coupled_read": (C.c_int, [vp, C.c_double, dp, dp, dp, dp]),
            "nlrom_coupled_launches": (C.c_int, [vp]),
            "nlrom_bench_prefix": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float), C.c_char_p,
                                             C.c_int, ip]),
            "nlrom_debug_poison_shared_memory": (C.c_int, [C.c_int]),
            "nlrom_fs_create": (C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(FsDesc)]),
            "nlrom_fs_destroy": (None, [vp]),
            "nlrom_fs_last_error": (C.c_char_p, [vp]),
            "nlrom_fs_step": (C.c_int, [vp, dp, dp, dp, C.POINTER(FsCfg), dp, dp, C.POINTER(FsInfo)]),
            "nlrom_fs_energy_force": (C.c_int, [vp, dp, dp, dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def iptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


class NewtonDivergence(RuntimeError):
    """Newton exceeded max_iters; carries the last residual norm."""

    def __init__(self, msg, last_norm=float("nan")):
        super().__init__(msg)
        self.last_norm = last_norm


def check(code: int, msg_fn):
    if code == OK:
        return
    msg = msg_fn()
    if isinstance(msg, bytes):
        msg = msg.decode(errors="replace")
    if code == ERR_ORDER:
        from .mcx import OrderError
        raise OrderError(msg)
    if code == ERR_DIM:
        raise ValueError(f"dimension mismatch: {msg}")
    if code == ERR_NONFINITE:
        raise FloatingPointError(f"non-finite result: {msg}")
    if code == ERR_NEWTON:
        import re
        m = re.search(r"norm ([0-9.eE+-]+)", msg)
        raise NewtonDivergence(msg, float(m.group(1)) if m else float("nan"))
    if code == ERR_NOCACHE:
        raise RuntimeError(f"no cached forward: {msg}")
    if code == ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"nlrom_b200 CUDA error: {msg}")


def device_index() -> int:
    return int(os.environ.get("NLROM_DEVICE", "0"))

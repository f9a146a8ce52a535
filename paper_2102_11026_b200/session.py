"""Device session: one ``nlrom_ctx`` (C ABI) per (ReducedModel, ElasticModel, CubatureModel).

Uploads decoder / basis / mesh / cubature set / weight net once, then serves every
hot-path query (diffops, residual, system Jacobian, cubature, step) from device
memory with host buffers copied in and out per call.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib


def _simcfg(cfg) -> _lib.SimCfg:
    s = _lib.SimCfg()
    s.dt = float(cfg.dt)
    s.newton_tol = float(cfg.newton_tol)
    s.max_iters = int(cfg.max_iters)
    s.drop_fict = int(bool(cfg.drop_fict))
    s.integration = 1 if cfg.integration == "exact_sum" else 0
    s.line_search = int(bool(cfg.line_search))
    s.fixed_iters = int(cfg.fixed_iters or 0)
    return s


class Session:
    def __init__(self, rm, model, cm=None, n_sims: int = 1, device: int | None = None):
        from .densenet import decoder_parts
        L = _lib.lib()
        Ws, bs, U = decoder_parts(rm.decoder)
        if U is None:
            raise ValueError("decoder must end with the PCA filter layer (PAPER.md:230)")
        self.N, self.n_p, self.n_q = model.N, rm.n_p, rm.n_q
        self.n = self.n_p + self.n_q
        self.n_sims = n_sims
        self.T = model.n_tets
        if U.shape != (self.N, self.n_p):
            raise ValueError("dimension mismatch: U must be (N, n_p)")
        keep = []

        def arr(a, conv=_lib.f64):
            a = conv(a)
            keep.append(a)
            return a

        d = _lib.ModelDesc()
        d.N, d.n_p, d.n_q, d.n_fc = self.N, self.n_p, self.n_q, len(Ws)
        widths = arr([self.n_q] + [W.shape[0] for W in Ws], _lib.i32)
        d.widths = _lib.iptr(widths)
        Wp = (C.POINTER(C.c_double) * len(Ws))(*[_lib.dptr(arr(W)) for W in Ws])
        bp = (C.POINTER(C.c_double) * len(Ws))(*[_lib.dptr(arr(b)) for b in bs])
        d.W, d.b = Wp, bp
        d.U = _lib.dptr(arr(U))
        d.mass = _lib.dptr(arr(model.mass))
        d.n_verts, d.n_tets = model.mesh.vertices.shape[0], self.T
        d.tets = _lib.iptr(arr(model.mesh.tets, _lib.i32))
        d.vert_dof = _lib.iptr(arr(model.vert_dof, _lib.i32))
        d.Dm_inv = _lib.dptr(arr(model.Dm_inv.reshape(-1, 9)))
        d.vol = _lib.dptr(arr(model.vol))
        d.mu, d.lam, d.alpha = model.material.mu, model.material.lam, model.material.rayleigh_alpha
        C_ids = np.zeros(0, dtype=np.int32) if cm is None else np.asarray(cm.C, dtype=np.int32)
        if C_ids.size != np.unique(C_ids).size:
            raise ValueError("cubature set has duplicates (SPEC.md:586)")
        d.n_cub = int(C_ids.size)
        self.n_cub = d.n_cub
        d.cub_elems = _lib.iptr(arr(C_ids if C_ids.size else np.zeros(1, np.int32), _lib.i32))
        if cm is not None and cm.wnet is not None:
            from .densenet import decoder_parts as _dp
            wW, wb, _ = _dp(cm.wnet)
        else:
            wW = [np.zeros((1, self.N)), np.zeros((1, 1)), np.zeros((1, 1)), np.zeros((self.T, 1))]
            wb = [np.zeros(1), np.zeros(1), np.zeros(1), np.zeros(self.T)]
        if len(wW) != 4 or wW[-1].shape[0] != self.T:
            raise ValueError("weight net must be N -> w -> w -> w -> T (4 FC layers, PAPER.md:406)")
        d.wnet_width = wW[0].shape[0]
        d.wnet_W = (C.POINTER(C.c_double) * 4)(*[_lib.dptr(arr(W)) for W in wW])
        d.wnet_b = (C.POINTER(C.c_double) * 4)(*[_lib.dptr(arr(b)) for b in wb])
        d.n_sims = n_sims
        h = C.c_void_p()
        self.device = _lib.device_index() if device is None else device
        code = L.nlrom_create(C.byref(h), self.device, C.byref(d))
        _lib.check(code, lambda: "nlrom_create failed")
        self._h = h
        self._L = L
        self._fin = weakref.finalize(self, L.nlrom_destroy, h)

    # ------------------------------------------------------------------ helpers
    def _chk(self, code):
        _lib.check(code, lambda: self._L.nlrom_last_error(self._h))

    @staticmethod
    def _v(a, n=None):
        a = _lib.f64(a).reshape(-1)
        if n is not None and a.size != n:
            raise ValueError(f"dimension mismatch: expected {n} values, got {a.size}")
        return a

    # ------------------------------------------------------------------ diffops
    def diffop(self, op, q, vec=None, eps=1e-10, mode=0):
        q = self._v(q, self.n_q)
        shapes = {_lib.OP_VALUE: (self.N,), _lib.OP_JVP: (self.N,), _lib.OP_HVV: (self.N,),
                  _lib.OP_JACOBIAN: (self.N, self.n_q), _lib.OP_HV: (self.N, self.n_q),
                  _lib.OP_SVV: (self.N, self.n_q), _lib.OP_VJP: (self.n_q,), _lib.OP_VHP: (self.n_q, self.n_q)}
        vn = self.N if op in (_lib.OP_VJP, _lib.OP_VHP) else self.n_q
        v = None if vec is None else self._v(vec, vn)
        out = np.empty(shapes[op])
        self._chk(self._L.nlrom_diffop(self._h, op, _lib.dptr(q), None if v is None else _lib.dptr(v),
                                       float(eps), int(mode), _lib.dptr(out)))
        return out

    # ------------------------------------------------------------------ reduced queries
    def full_displacement(self, r):
        out = np.empty(self.N)
        self._chk(self._L.nlrom_full_displacement(self._h, _lib.dptr(self._v(r, self.n)), _lib.dptr(out)))
        return out

    def jtilde(self, q):
        out = np.empty((self.N, self.n))
        self._chk(self._L.nlrom_jtilde(self._h, _lib.dptr(self._v(q, self.n_q)), _lib.dptr(out)))
        return out

    def delta_j(self, q, q_bar, qdot_bar, dt, drop_fict=False):
        out = np.empty((self.N, self.n_q))
        self._chk(self._L.nlrom_delta_j(self._h, _lib.dptr(self._v(q, self.n_q)), _lib.dptr(self._v(q_bar, self.n_q)),
                                        _lib.dptr(self._v(qdot_bar, self.n_q)), float(dt), int(drop_fict),
                                        _lib.dptr(out)))
        return out

    def fictitious_force(self, q, q_bar):
        out = np.empty(self.N)
        self._chk(self._L.nlrom_fictitious_force(self._h, _lib.dptr(self._v(q, self.n_q)),
                                                 _lib.dptr(self._v(q_bar, self.n_q)), _lib.dptr(out)))
        return out

    def wnet_forward_cub(self, r):
        """Weight-net outputs on the cubature set C (length |C|)."""
        out = np.empty(self.n_cub)
        self._chk(self._L.nlrom_wnet_forward(self._h, _lib.dptr(self._v(r, self.n)), _lib.dptr(out), out.size))
        return out

    def cubature_integrate(self, r, integration="cubature"):
        f = np.empty(self.n)
        K = np.empty((self.n, self.n))
        self._chk(self._L.nlrom_cubature_integrate(self._h, _lib.dptr(self._v(r, self.n)),
                                                   1 if integration == "exact_sum" else 0, _lib.dptr(f), _lib.dptr(K)))
        return f, K

    def element_forces(self, u, want_K=False):
        f = np.empty(self.N)
        K = np.empty((self.T, 12, 12)) if want_K else None
        self._chk(self._L.nlrom_element_forces(self._h, _lib.dptr(self._v(u, self.N)), int(want_K), _lib.dptr(f),
                                               _lib.dptr(K) if want_K else None))
        return f, K

    def element_reduced_forces(self, r, elems):
        e = _lib.i32(elems)
        out = np.empty((e.size, self.n))
        self._chk(self._L.nlrom_element_reduced_forces(self._h, _lib.dptr(self._v(r, self.n)), _lib.iptr(e), e.size,
                                                       _lib.dptr(out)))
        return out

    def train_forces(self, rs):
        """(F (S, T, n), u (S, N)): per-element reduced forces of all elements at poses rs."""
        rs = np.ascontiguousarray(np.atleast_2d(rs), dtype=np.float64)
        S = rs.shape[0]
        F = np.empty((S, self.T, self.n))
        u = np.empty((S, self.N))
        self._chk(self._L.nlrom_train_forces(self._h, _lib.dptr(rs), S, _lib.dptr(F), _lib.dptr(u)))
        return F, u

    # ------------------------------------------------------------------ rdsim
    def _state(self, r_bar, rdot_bar, f_ext):
        S = self.n_sims
        return (self._v(r_bar, S * self.n), self._v(rdot_bar, S * self.n), self._v(f_ext, S * self.N))

    def residual(self, r, r_bar, rdot_bar, f_ext, cfg):
        rb, rd, fe = self._state(r_bar, rdot_bar, f_ext)
        out = np.empty(self.n_sims * self.n)
        c = _simcfg(cfg)
        self._chk(self._L.nlrom_residual(self._h, _lib.dptr(self._v(r, self.n_sims * self.n)), _lib.dptr(rb),
                                         _lib.dptr(rd), _lib.dptr(fe), C.byref(c), _lib.dptr(out)))
        return out if self.n_sims > 1 else out

    def system_jacobian(self, r, r_bar, rdot_bar, f_ext, cfg):
        rb, rd, fe = self._state(r_bar, rdot_bar, f_ext)
        out = np.empty((self.n_sims, self.n, self.n))
        c = _simcfg(cfg)
        self._chk(self._L.nlrom_system_jacobian(self._h, _lib.dptr(self._v(r, self.n_sims * self.n)), _lib.dptr(rb),
                                                _lib.dptr(rd), _lib.dptr(fe), C.byref(c), _lib.dptr(out)))
        return out[0] if self.n_sims == 1 else out

    def step(self, r_bar, rdot_bar, f_ext, cfg, want_norm=True):
        """One timestep of every sim: (r, rdot, iterations, ||phi||). With fixed iterations and
        want_norm=False the final residual is not evaluated and ||phi|| is returned as None."""
        rb, rd, fe = self._state(r_bar, rdot_bar, f_ext)
        r = np.empty(self.n_sims * self.n)
        rdot = np.empty(self.n_sims * self.n)
        info = _lib.StepInfo()
        c = _simcfg(cfg)
        skip = (not want_norm) and c.fixed_iters > 0
        # raw addresses (c_void_p arguments): the per-call ctypes pointer objects are the largest
        # host cost of a step call after the device work
        self._chk(self._L.nlrom_step(self._h, rb.ctypes.data, rd.ctypes.data, fe.ctypes.data, C.byref(c),
                                     r.ctypes.data, rdot.ctypes.data, None if skip else C.byref(info)))
        if skip:
            return r, rdot, c.fixed_iters, None
        return r, rdot, info.iters, info.res_norm

    def step_device(self, r_bar, rdot_bar, f_ext, cfg, r_out, rdot_out, stream_ptr):
        """Device pointers (ints, e.g. torch tensor.data_ptr()) on a CUDA stream handle."""
        c = _simcfg(cfg)
        self._chk(self._L.nlrom_step_device(self._h, C.c_void_p(r_bar), C.c_void_p(rdot_bar), C.c_void_p(f_ext),
                                            C.byref(c), C.c_void_p(r_out), C.c_void_p(rdot_out),
                                            C.c_void_p(stream_ptr)))

    def bench_iterations(self, n_iters, flush_l2=True):
        tot, dom = C.c_float(), C.c_float()
        self._chk(self._L.nlrom_bench_iterations(self._h, int(n_iters), int(flush_l2), C.byref(tot), C.byref(dom)))
        return tot.value, dom.value

    def bench_replays(self, n_iters, flush_l2=True):
        """Device ms of each of n_iters replays of the one-Newton-iteration graph."""
        out = (C.c_float * int(n_iters))()
        self._chk(self._L.nlrom_bench_replays(self._h, int(n_iters), int(flush_l2), out))
        return np.array(out[:], dtype=float)

    def iterate(self, n_iters=1):
        """n_iters replays of the benchmarked one-Newton-iteration graph (no timing)."""
        self._chk(self._L.nlrom_iterate(self._h, int(n_iters)))

    def get_iterate(self):
        """(r, phi at the iterate the last E phase evaluated, ||phi||_2) per sim, flattened."""
        nn = self.n_sims * self.n
        r, phi, nrm = np.empty(nn), np.empty(nn), np.empty(self.n_sims)
        self._chk(self._L.nlrom_get_iterate(self._h, _lib.dptr(r), _lib.dptr(phi), _lib.dptr(nrm)))
        return r, phi, nrm

    def set_iterate(self, r):
        self._chk(self._L.nlrom_set_iterate(self._h, _lib.dptr(self._v(r, self.n_sims * self.n))))

    def bench_kernels(self, n_iters, flush_l2=True):
        """Device ms per launch of [hidden jet chain, output layer, vhp backward chain, LU]."""
        out = (C.c_float * 4)()
        self._chk(self._L.nlrom_bench_kernels(self._h, int(n_iters), int(flush_l2), out))
        return list(out)

    def bench_cubature(self, n_iters, flush_l2=True):
        """(device ms, algorithmic bytes) of one cubature launch over all sims."""
        ms, by = C.c_float(), C.c_double()
        self._chk(self._L.nlrom_bench_cubature(self._h, int(n_iters), int(flush_l2), C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def bench_prefix(self, n_iters=50, flush_l2=True, cap=64):
        """[(kernel name, marginal in-graph ms)] for the launches of one Newton iteration."""
        ms = (C.c_float * cap)()
        buf = C.create_string_buffer(8192)
        cnt = C.c_int()
        self._chk(self._L.nlrom_bench_prefix(self._h, int(n_iters), int(flush_l2), cap, ms, buf, 8192, C.byref(cnt)))
        names = buf.value.decode().split("\n")[:cnt.value]
        vals = list(ms)[:cnt.value]
        return [(nm, v - (vals[i - 1] if i else 0.0)) for i, (nm, v) in enumerate(zip(names, vals))], vals

    def launches_per_iteration(self):
        return int(self._L.nlrom_launches_per_iteration(self._h))

    def tc_layers(self):
        """Decoder hidden layers on the tcgen05 Ozaki GEMM (0: all on fp64 DMMA)."""
        return int(self._L.nlrom_tc_layers(self._h))

    def tc_info(self):
        """(hidden layers, output layer 0/1, vhp backward layers) on the tcgen05 Ozaki GEMM."""
        out = np.zeros(3, dtype=np.int32)
        self._chk(self._L.nlrom_tc_info(self._h, out.ctypes.data_as(C.POINTER(C.c_int))))
        return tuple(int(x) for x in out)


def _uploaded_arrays(rm, model, cm):
    """Every host array a Session copies to the device (decoder, basis, mesh, set, weight net)."""
    arrs = [rm.U, model.mass, model.mesh.tets, model.vert_dof, model.Dm_inv, model.vol]
    nets = [rm.decoder] + ([cm.wnet] if cm is not None and cm.wnet is not None else [])
    for net in nets:
        for table in (net.weights, net.biases, net.bases):
            # insertion order: stable across calls (a key added / removed changes the fingerprint)
            arrs.extend(table.values())
    if cm is not None:
        arrs.append(cm.C)
    return [a for a in arrs if isinstance(a, np.ndarray)]


def _fingerprint(arrs):
    # identity: the uploaded arrays are frozen read-only, so an array object keeps its buffer and
    # contents (an in-place resize needs a writeable array) and its id identifies the data
    # (reading the data pointer per array costs ~1 us each on every step call)
    return tuple(map(id, arrs))


_MAX_SESSIONS_PER_MODEL = 4


def session_for(rm, model, cm=None, n_sims: int = 1) -> Session:
    """The device session of (rm, model, cm), cached on ``rm``.

    The cache entry holds strong references to ``model`` and ``cm`` (so their ids cannot
    be recycled while it exists) and a fingerprint of every uploaded array (identity, data
    pointer, shape): replacing an array (``net.weights[i] = W2``, a new mesh, a new set)
    rebuilds the session. The uploaded arrays are made read-only, so an in-place edit of
    weights that a device context holds raises instead of silently using stale values;
    call ``invalidate(rm)`` first to edit in place. At most a few sessions per model are
    kept (oldest evicted and its device memory freed)."""
    cache = rm.__dict__.setdefault("_nlrom_sessions", {})
    key = (id(model), id(cm), int(n_sims))
    arrs = _uploaded_arrays(rm, model, cm)
    fp = _fingerprint(arrs)
    hit = cache.get(key)
    if hit is not None and hit[0] is model and hit[1] is cm and hit[2] == fp:
        return hit[3]
    if hit is not None:
        _drop(cache, key)
    while len(cache) >= _MAX_SESSIONS_PER_MODEL:
        _drop(cache, next(iter(cache)))
    s = Session(rm, model, cm, n_sims)
    frozen = []
    for a in arrs:
        if a.flags.writeable:
            a.flags.writeable = False
            frozen.append(a)
    cache[key] = (model, cm, fp, s, frozen)
    return s


def _drop(cache, key):
    model, cm, fp, s, frozen = cache.pop(key)
    for a in frozen:
        try:
            a.flags.writeable = True
        except ValueError:
            pass
    s._fin()  # free the device context now, not at garbage collection


def invalidate(rm):
    """Drop every cached device session of ``rm`` (and make its arrays writeable again)."""
    cache = rm.__dict__.get("_nlrom_sessions", {})
    for key in list(cache):
        _drop(cache, key)

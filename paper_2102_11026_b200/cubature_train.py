"""Neural-cubature training (§5, Eqs. 17-19) and the greedy NNLS
baseline.

Offline work around the simulation-time cubature of ``neucubature``:

* ``build_train_set`` evaluates the per-element reduced forces ``f~_e(r) = J~_e(r)^T f_e(u(r))``
  for every element at every training pose on the GPU, with the same cubature kernel the
  Newton step uses (``k_cubature``, per-element projection epilogue; Eq. 18's f~_e).
* ``greedy_cubature`` is the classic baseline: add the element whose
  normalised reduced-force column best matches the residual, re-solve all weights by
  Lawson-Hanson NNLS (``nnls``) after each addition.
* ``snet_forward`` is the selection GCN S (Eq. 17: two graph convolutions with 8 channels and
  sin, degree normalisation 1/sqrt(d_i d_j), vertex-to-element mean pooling, two FC layers,
  softmax over elements); ``train_alternating`` alternates W and S (Fig. 4, Eq. 19) starting
  from farthest-point ("Voronoi") samples, adding the K best-scoring non-members per round.

Network training follows the reference's stated tooling (SPEC.md cmd_train: "use PyTorch and
Adam for all our network training"): torch fp64 autograd, on the GPU when one is present.
The per-timestep path never runs through this module.

Builder decisions where the paper / SPEC leave a choice (documented in DESIGN.md §4e):
the GCN uses the one-ring plus a self loop, degrees counted with the self loop; L_S (whose
printed form does not depend on s) is ``mean_s || fbar_s - a_s sum_e s_e f~_e(r_s) ||`` with
the per-pose scale ``a_s >= 0`` solved in closed form, so the scores learn which elements'
forces explain the cubature residual; losses are mean L2 norms over samples;
the greedy match normalises every pose's block by ||f~(r_s)|| so poses weigh equally.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


# ---------------------------------------------------------------------------- training set
@dataclass
class CubatureTrainSet:
    """Poses r (S, n), full reduced forces f~(r) (S, n), per-element reduced forces
    f~_e(r) (S, T, n) and the poses' full-space displacements u (S, N)."""
    r: np.ndarray
    f: np.ndarray
    F: np.ndarray
    u: np.ndarray

    def __post_init__(self):
        S, T, n = self.F.shape
        if self.r.shape != (S, n) or self.f.shape != (S, n) or self.u.shape[0] != S:
            raise ValueError("CubatureTrainSet dimensions are inconsistent (SPEC.md:590)")
        if S == 0:
            raise ValueError("empty training set (SPEC.md:639)")

    @property
    def n_elems(self) -> int:
        return self.F.shape[1]


def build_train_set(rm, model, rs) -> CubatureTrainSet:
    """Per-element reduced forces of every element at every pose r_s, on the GPU (one decoder
    bundle + one cubature launch over all T elements per pose). f~(r_s) = sum_e f~_e(r_s)."""
    from .session import session_for
    rs = np.atleast_2d(np.asarray(rs, dtype=np.float64))
    F, u = session_for(rm, model).train_forces(rs)  # nlrom_train_forces
    return CubatureTrainSet(rs.copy(), F.sum(axis=1), F, u)


# ---------------------------------------------------------------------------- NNLS + greedy
def nnls(A, b, max_iter=None, tol=None):
    """min ||A x - b||_2 s.t. x >= 0 by the Lawson-Hanson active-set method.
    Returns (x, residual norm). Raises RuntimeError if it does not converge."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, k = A.shape
    x = np.zeros(k)
    if k == 0:
        return x, float(np.linalg.norm(b))
    passive = np.zeros(k, dtype=bool)
    tol = 10 * np.finfo(float).eps * np.linalg.norm(A, 1) * max(m, k) if tol is None else tol
    max_iter = 3 * k if max_iter is None else max_iter
    w = A.T @ (b - A @ x)
    it = 0
    while (~passive).any() and np.max(np.where(~passive, w, -np.inf)) > tol:
        j = int(np.argmax(np.where(~passive, w, -np.inf)))
        passive[j] = True
        while True:
            it += 1
            if it > max_iter:
                raise RuntimeError("NNLS did not converge (SPEC.md:636)")
            z = np.zeros(k)
            z[passive] = np.linalg.lstsq(A[:, passive], b, rcond=None)[0]
            if np.all(z[passive] > 0):
                x = z
                break
            neg = passive & (z <= 0)
            alpha = np.min(x[neg] / (x[neg] - z[neg]))
            x = x + alpha * (z - x)
            passive &= x > tol
            x[~passive] = 0.0
        w = A.T @ (b - A @ x)
    return x, float(np.linalg.norm(A @ x - b))


def _stacked(ts: CubatureTrainSet):
    """Element-major design matrix A (T, S n) and target b (S n), every pose's block scaled by
    1 / ||f~(r_s)||."""
    S, T, n = ts.F.shape
    scale = 1.0 / np.maximum(np.linalg.norm(ts.f, axis=1), 1e-300)
    A = (ts.F * scale[:, None, None]).transpose(1, 0, 2).reshape(T, S * n)
    b = (ts.f * scale[:, None]).reshape(S * n)
    return A, b


def greedy_cubature(rm, model, ts: CubatureTrainSet, target_size: int):
    """Greedy residual matching + NNLS -> (C, w) with w >= 0 fixed weights."""
    if target_size > ts.n_elems:
        raise ValueError("target_size exceeds the element count (SPEC.md:633)")
    A, b = _stacked(ts)
    norms = np.linalg.norm(A, axis=1)
    live = norms > 0
    C: list[int] = []
    w = np.zeros(0)
    res = b.copy()
    while len(C) < target_size:
        score = np.full(A.shape[0], -np.inf)
        score[live] = (A[live] @ res) / norms[live]
        score[C] = -np.inf
        e = int(np.argmax(score))
        if not np.isfinite(score[e]):
            break
        C.append(e)
        w, _ = nnls(A[C].T, b)
        res = b - A[C].T @ w
    return np.asarray(C, dtype=np.int32), w


def cubature_error(ts: CubatureTrainSet, C, w) -> float:
    """Table 2 metric: mean over poses of ||f~ - sum_{e in C} w_e f~_e|| / ||f~||.
    ``w`` is (|C|,) fixed weights or (S, |C|) per-pose weights."""
    C = np.asarray(C, dtype=np.int64)
    if C.size == 0:
        return 1.0
    w = np.asarray(w, dtype=np.float64)
    approx = np.einsum("sc,scn->sn", np.broadcast_to(w, (ts.F.shape[0], C.size)), ts.F[:, C])
    return float(np.mean(np.linalg.norm(ts.f - approx, axis=1) / np.linalg.norm(ts.f, axis=1)))


# ---------------------------------------------------------------------------- selection net
@dataclass
class SelectionNet:
    """S of Eq. 17: gamma1 (3 x 8), gamma2 (8 x 8) graph convolutions, then per-element FC
    layers fc1 (8 -> 8, sin) and fc2 (8 -> 1), softmax over elements."""
    gamma1: np.ndarray
    gamma2: np.ndarray
    fc1_W: np.ndarray
    fc1_b: np.ndarray
    fc2_W: np.ndarray
    fc2_b: np.ndarray

    @staticmethod
    def init(seed=0, channels=8, hidden=8):
        rng = np.random.default_rng(seed)

        def uni(o, i):
            return rng.uniform(-np.sqrt(6.0 / i), np.sqrt(6.0 / i), (o, i))
        # gamma acts on the right (h_j gamma): shape (in channels, out channels)
        return SelectionNet(uni(channels, 3).T.copy(), uni(channels, channels).T.copy(),
                            uni(hidden, channels), np.zeros(hidden), uni(1, hidden), np.zeros(1))

    @staticmethod
    def zeros(channels=8, hidden=8):
        z = np.zeros
        return SelectionNet(z((3, channels)), z((channels, channels)), z((hidden, channels)), z(hidden),
                            z((1, hidden)), z(1))

    def params(self):
        return [self.gamma1, self.gamma2, self.fc1_W, self.fc1_b, self.fc2_W, self.fc2_b]


@dataclass
class MeshGraph:
    """Normalised one-ring adjacency with self loops (Eq. 17: 1 / c_ij, c_ij = sqrt(d_i d_j))
    as COO (rows, cols, vals) over vertices, plus the tets for vertex-to-element pooling."""
    n_verts: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    tets: np.ndarray
    vert_dof: np.ndarray = field(default=None)


def mesh_graph(model) -> MeshGraph:
    tets = np.asarray(model.mesh.tets, dtype=np.int64)
    V = int(np.asarray(model.mesh.vertices).shape[0])
    pairs = set()
    for t in tets:
        for a in range(4):
            for b in range(4):
                pairs.add((int(t[a]), int(t[b])))  # a == b: the self loop
    rc = np.array(sorted(pairs), dtype=np.int64)
    deg = np.bincount(rc[:, 0], minlength=V).astype(np.float64)
    vals = 1.0 / np.sqrt(deg[rc[:, 0]] * deg[rc[:, 1]])
    return MeshGraph(V, rc[:, 0], rc[:, 1], vals, tets, _vertex_dofs(model, V))


def _vertex_dofs(model, V):
    """(V, 3) free-DOF index per vertex coordinate, -1 for fixed vertices (model.vert_dof)."""
    vd = np.asarray(model.vert_dof, dtype=np.int64)
    return np.where(vd[:, None] >= 0, 3 * vd[:, None] + np.arange(3)[None, :], -1)


def vertex_displacements(graph: MeshGraph, u):
    """Free-DOF vector(s) u (..., N) -> per-vertex displacements (..., V, 3), fixed vertices 0."""
    u = np.asarray(u, dtype=np.float64)
    pad = np.concatenate([u, np.zeros(u.shape[:-1] + (1,))], axis=-1)
    return pad[..., np.where(graph.vert_dof >= 0, graph.vert_dof, u.shape[-1])]


def _snet_torch(torch, graph, params, X):
    """Batched S forward in torch: X (B, V, 3) -> scores (B, T)."""
    g1, g2, W1, b1, W2, b2 = params
    rows = torch.as_tensor(graph.rows, device=X.device)
    cols = torch.as_tensor(graph.cols, device=X.device)
    vals = torch.as_tensor(graph.vals, dtype=X.dtype, device=X.device)[:, None]

    def conv(H, g):  # sin(sum_j (1/c_ij) h_j gamma), the sum as a fixed-order index_add over edges
        HG = H @ g
        out = torch.zeros(HG.shape, dtype=HG.dtype, device=HG.device)
        return torch.sin(out.index_add(1, rows, vals * HG[:, cols]))
    H = conv(conv(X, g1), g2)
    tets = torch.as_tensor(graph.tets, device=X.device)
    E = H[:, tets].mean(dim=2)  # (B, T, 8): mean over each tet's 4 vertices
    z = (torch.sin(E @ W1.T + b1) @ W2.T + b2)[..., 0]
    return torch.softmax(z, dim=-1)


def snet_forward(snet: SelectionNet, graph: MeshGraph, u) -> np.ndarray:
    """Scores s (one per element, sum 1, >= 0) for displacement(s) u."""
    import torch
    u = np.asarray(u, dtype=np.float64)
    X = torch.as_tensor(vertex_displacements(graph, np.atleast_2d(u)))
    with torch.no_grad():
        s = _snet_torch(torch, graph, [torch.as_tensor(p) for p in snet.params()], X).numpy()
    return s[0] if u.ndim == 1 else s


# ---------------------------------------------------------------------------- alternating training
def farthest_point_elements(model, k: int, seed: int = 0) -> np.ndarray:
    """k element ids spread over the mesh by farthest-point sampling of the tet centroids
    (the "few Voronoi samples" initialisation)."""
    verts = np.asarray(model.mesh.vertices, dtype=np.float64)
    cen = verts[np.asarray(model.mesh.tets)].mean(axis=1)
    T = cen.shape[0]
    k = min(k, T)
    if k <= 0:
        return np.zeros(0, dtype=np.int32)
    first = int(np.random.default_rng(seed).integers(T))
    C = [first]
    d = np.linalg.norm(cen - cen[first], axis=1)
    while len(C) < k:
        e = int(np.argmax(d))
        C.append(e)
        d = np.minimum(d, np.linalg.norm(cen - cen[e], axis=1))
    return np.asarray(C, dtype=np.int32)


@dataclass
class TrainLog:
    loss_w: list = field(default_factory=list)   # L_W at the end of each round's W phase
    loss_s: list = field(default_factory=list)   # L_S at the end of each round's S phase
    sizes: list = field(default_factory=list)    # |C| after each round
    errors: list = field(default_factory=list)   # Table 2 metric with the trained W per round


def _select_topk(C, s, K):
    from .neucubature import select_topk
    return select_topk(C, s, K)


def train_alternating(rm, model, ts: CubatureTrainSet, K: int = 5, rounds: int = 10, *, wnet=None,
                      snet: SelectionNet | None = None, n_init: int = 5, epochs: int = 15, lr: float = 1e-3,
                      seed: int = 0, device=None, return_log: bool = False, nnls_init: bool = True,
                      epochs_s: int | None = None,
                      new_row_scale: float = 1e-2):
    """Fig. 4: C <- farthest-point samples; per round train W for ``epochs`` on L_W, compute the
    residuals fbar (Eq. 18), train S for ``epochs`` on L_S (W frozen), add the K best-scoring
    non-members (select_topk). Both nets warm-start across rounds (§6.3). With
    ``nnls_init`` every newly added element's output starts at its fixed-weight NNLS value
    (bias sqrt(w_e), weight row scaled by ``new_row_scale``). Returns a CubatureModel
    (C, trained wnet, snet, K) [and a TrainLog]."""
    import torch
    from .densenet import make_wnet
    from .neucubature import CubatureModel
    dev = torch.device(device) if device is not None else (
        torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    dt = torch.float64
    S, T, n = ts.F.shape
    graph = mesh_graph(model)
    if wnet is None:
        wnet = rm.cubature.wnet if getattr(rm, "cubature", None) is not None else None
    if wnet is None:
        raise ValueError("train_alternating needs an initial weight net (wnet=...)")
    fcs = [i for i, L in enumerate(wnet.layers) if L.kind == "fully_connected"]
    if wnet.layers[fcs[-1]].out_dim != T:
        raise ValueError("the weight net must output one weight per element")
    Wp = [torch.tensor(wnet.weights[i], dtype=dt, device=dev, requires_grad=True) for i in fcs]
    bp = [torch.tensor(wnet.biases[i], dtype=dt, device=dev, requires_grad=True) for i in fcs]
    snet = snet or SelectionNet.init(seed)
    Sp = [torch.tensor(p, dtype=dt, device=dev, requires_grad=True) for p in snet.params()]
    U = torch.as_tensor(ts.u, dtype=dt, device=dev)
    # losses on per-pose normalised forces (every pose weighs equally, as in the Table 2 metric)
    fs = np.maximum(np.linalg.norm(ts.f, axis=1), 1e-300)
    F = torch.as_tensor(ts.F / fs[:, None, None], dtype=dt, device=dev)
    f = torch.as_tensor(ts.f / fs[:, None], dtype=dt, device=dev)
    A_np, b_np = _stacked(ts)
    X = torch.as_tensor(vertex_displacements(graph, ts.u), dtype=dt, device=dev)

    def w_all():
        h = U
        for l, (W, b) in enumerate(zip(Wp, bp)):
            h = h @ W.T + b
            h = torch.sin(h) if l < len(Wp) - 1 else h * h
        return h  # (S, T) nonnegative

    def masked(w, C):
        m = torch.zeros(T, dtype=dt, device=dev)
        if len(C):
            m[torch.as_tensor(np.asarray(C, dtype=np.int64), device=dev)] = 1.0
        return w * m

    def loss_w(C):  # Eq. 19, L_W
        return torch.linalg.norm(f - torch.einsum("st,stn->sn", masked(w_all(), C), F), dim=1).mean()

    def loss_s(fbar):  # builder-defined L_S (module docstring)
        g = torch.einsum("st,stn->sn", _snet_torch(torch, graph, Sp, X), F)
        a = torch.clamp((fbar * g).sum(1) / torch.clamp((g * g).sum(1), min=1e-300), min=0.0)
        return torch.linalg.norm(fbar - a[:, None] * g, dim=1).mean()

    def seed_new(C, new):
        """Newly added members start from the fixed-weight NNLS fit on C: output bias
        sqrt(w_e), output row scaled by ``new_row_scale`` (W then learns the pose dependence)."""
        if not nnls_init or not len(new):
            return
        w, _ = nnls(A_np[np.asarray(C)].T, b_np)
        pos = {int(e): i for i, e in enumerate(C)}
        with torch.no_grad():
            for e in new:
                bp[-1][int(e)] = float(np.sqrt(w[pos[int(e)]]))
                Wp[-1][int(e)] *= new_row_scale

    C = farthest_point_elements(model, n_init, seed)
    seed_new(C, list(C))
    log = TrainLog()
    optW = torch.optim.Adam(Wp + bp, lr=lr)
    optS = torch.optim.Adam(Sp, lr=lr)
    for _ in range(rounds):
        for _ in range(epochs):
            optW.zero_grad()
            L = loss_w(C)
            if not torch.isfinite(L):
                raise FloatingPointError("NaN loss in the W phase (SPEC.md:640)")
            L.backward()
            optW.step()
        with torch.no_grad():
            Lw = loss_w(C)
            wC = masked(w_all(), C)
            fbar = f - torch.einsum("st,stn->sn", wC, F)
            log.loss_w.append(float(Lw))
            log.errors.append(float((torch.linalg.norm(fbar, dim=1) / torch.linalg.norm(f, dim=1)).mean()))
        for _ in range(epochs if epochs_s is None else epochs_s):
            optS.zero_grad()
            L = loss_s(fbar)
            if not torch.isfinite(L):
                raise FloatingPointError("NaN loss in the S phase (SPEC.md:640)")
            L.backward()
            optS.step()
        with torch.no_grad():
            log.loss_s.append(float(loss_s(fbar)))
            s_mean = _snet_torch(torch, graph, Sp, X).mean(0).cpu().numpy()
        C_old = set(int(e) for e in C)
        C = _select_topk(C, s_mean, K)
        seed_new(C, [e for e in C if int(e) not in C_old])
        log.sizes.append(int(len(C)))
    Ws = [W.detach().cpu().numpy() for W in Wp]
    bs = [b.detach().cpu().numpy() for b in bp]
    sn = SelectionNet(*[p.detach().cpu().numpy() for p in Sp])
    cm = CubatureModel(np.asarray(C, dtype=np.int32), make_wnet(Ws, bs), sn, K)
    return (cm, log) if return_log else cm

"""Independent simulations sharded over GPUs (4096 sims on 1/2/4/8 B200).

The reference steps one reduced body per ``rdsim.step`` call ("one simulation per thread",
SPEC.md:570). Many independent sims that share one trained DAE + cubature model partition
naturally: each rank (one process per GPU) owns a contiguous range of sims as the sims of ONE
``nlrom`` context (weights replicated, big-tile batched decoder when the range is large), and
no data crosses ranks while stepping. The only exchange is an optional gather of per-sim
results at the end (``gather``), e.g. for logging.
"""

from __future__ import annotations

import numpy as np

from .session import Session
from .substructure import dist_info


def shard_range(total: int, rank: int, world: int):
    """Contiguous sim range [lo, hi) of ``rank``; sizes differ by at most one."""
    if total < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("need total >= 0, world >= 1 and 0 <= rank < world")
    return rank * total // world, (rank + 1) * total // world


class SimShard:
    """This rank's share of ``total`` independent sims of one (rm, model, cm).

    States are passed either for all sims ((total, n) / (total, N) arrays, sliced here) or for
    the local range only ((hi - lo, n)). ``rank`` / ``world`` default to torch.distributed's
    default group (0 / 1 without it)."""

    def __init__(self, rm, model, cm, total: int, rank=None, world=None, device: int | None = None):
        r0, w0 = dist_info()
        self.rank = r0 if rank is None else int(rank)
        self.world = w0 if world is None else int(world)
        self.total = int(total)
        self.lo, self.hi = shard_range(self.total, self.rank, self.world)
        self.n = rm.n_p + rm.n_q
        self.N = model.N
        self.session = Session(rm, model, cm, n_sims=self.n_local, device=device) if self.n_local else None

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    def local(self, a, width):
        """Rows of this rank from a (total, width) array, or a local (n_local, width) array."""
        a = np.asarray(a, dtype=np.float64)
        if a.ndim == 1:
            a = a.reshape(-1, width)
        if a.shape == (self.total, width) and self.total != self.n_local:
            a = a[self.lo:self.hi]
        if a.shape != (self.n_local, width):
            raise ValueError(f"dimension mismatch: expected ({self.total} or {self.n_local}, {width}) rows")
        return np.ascontiguousarray(a)

    def step(self, r_bar, rdot_bar, f_ext, cfg):
        """One implicit timestep of every local sim (fixed-iteration mode for many sims).
        Returns local (r, rdot) as (n_local, n) arrays and the iteration count."""
        if self.session is None:
            z = np.zeros((0, self.n))
            return z, z.copy(), 0
        rb, rdb = self.local(r_bar, self.n), self.local(rdot_bar, self.n)
        fe = np.asarray(f_ext, dtype=np.float64)
        if fe.ndim == 1 and fe.size == self.N:       # one load shared by every sim
            fe = np.tile(fe, (self.n_local, 1))
        fe = self.local(fe, self.N)
        r, rd, iters, _ = self.session.step(rb.reshape(-1), rdb.reshape(-1), fe.reshape(-1), cfg)
        return r.reshape(self.n_local, self.n), rd.reshape(self.n_local, self.n), iters

    def gather(self, local_rows, group=None):
        """All sims' rows in global order on every rank (host all_gather; no-op at world 1)."""
        return gather_rows(self.lo, local_rows, self.world, group)


def gather_rows(lo: int, local_rows, world: int, group=None):
    """Concatenate every rank's (lo, rows) in sim order (torch.distributed all_gather_object)."""
    local_rows = np.asarray(local_rows)
    if world == 1:
        return local_rows
    import torch.distributed as dist
    parts = [None] * world
    dist.all_gather_object(parts, (int(lo), local_rows), group=group)
    parts.sort(key=lambda p: p[0])
    return np.concatenate([p[1] for p in parts], axis=0)

"""The rotating-star step across devices: z-slabs of the leaf lattice, one
per rank (the north_star's "octree leaves partitioned across the GPUs of one
box, with ghost-layer and multipole-moment exchange").

PARITY UNPINNED (self-authored spec, oracle/star_oracle.py). The partitioned
step is arithmetic-for-arithmetic the single-device step, so any number of
ranks reproduces ``RotatingStarStep`` bit for bit (tests/test_gpu_star_dist.py).

Per right-hand-side evaluation a rank exchanges, with its z-neighbours only:
* 4 planes of the conserved state each way (periodic): the hydro ghost layer
  (2 planes) and the leaf monopole stencil's reach (4 planes of rho; zero
  beyond the isolated domain);
* 4 planes of reduced multipole records per partitioned FMM level each way
  (non-periodic), into the halo planes the M2L's TMA boxes read;
and with all ranks: the raw and reduced records of the one gathered level
(all-gather; the coarser levels are then computed redundantly) and the CFL
dt (all-reduce MIN: min over ranks of cfl*dx/max_local == cfl*dx/max_global).

The step is a generator of exchange requests; a driver services them:
``VirtualCluster`` runs R slabs on one device in lockstep (device copies),
``DistDriver`` is one rank of a torch.distributed job (NCCL on GPUs; gloo
through host staging for CPU-side tests).
"""

from __future__ import annotations

import ctypes
from typing import Iterator, List, Optional, Tuple

import torch

from . import _native as N
from .hydro import NF, NI


def slab_layout(max_level: int, ranks: int, rank: int, level: int) -> dict:
    info = (ctypes.c_uint64 * 8)()
    N.call("tb_fmm_slab_layout", max_level, ranks, rank, level, info)
    keys = ("raw_off", "red_off", "loc_off", "n", "nz", "z0", "halo", "lp")
    return dict(zip(keys, list(info)))


class StarSlab:
    """One rank's z-slab of the rotating-star lattice (state [5, nz, N, N])."""

    def __init__(self, max_level: int, ranks: int, rank: int, state: torch.Tensor,
                 gamma: float = 5.0 / 3.0, cfl: float = 0.4):
        self.L, self.R, self.r = max_level, ranks, rank
        self.n = 8 << max_level
        self.nz = self.n // ranks
        if self.nz < 16 or self.n % (16 * ranks):
            raise ValueError("need N/ranks a multiple of 16")
        if tuple(state.shape) != (NF, self.nz, self.n, self.n):
            raise ValueError("state must be this rank's [5, nz, N, N] slab")
        self.device = state.device
        self.gamma, self.cfl, self.dx = float(gamma), float(cfl), 1.0 / self.n
        n, nz = self.n, self.nz
        f64 = dict(dtype=torch.float64, device=self.device)
        self.U = state.contiguous().clone()
        self.U1 = torch.empty_like(self.U)
        self.send_lo = torch.empty((NF, 4, n, n), **f64)
        self.send_hi = torch.empty((NF, 4, n, n), **f64)
        self.recv_lo = torch.zeros((NF, 4, n, n), **f64)
        self.recv_hi = torch.zeros((NF, 4, n, n), **f64)
        self.Up = torch.empty((NF, nz + 4, n + 4, n + 4), **f64)
        self.rho_h = torch.zeros((nz + 8, n, n), **f64)
        self.nsub = (n // NI) ** 2 * (nz // NI)
        self.dudt = torch.empty((self.nsub, NF, NI, NI, NI), **f64)
        self.amax = torch.empty(self.nsub, **f64)
        self.dt = torch.zeros(1, **f64)
        self.time = torch.zeros(1, **f64)
        nbytes = ctypes.c_uint64()
        N.call("tb_fmm_slab_workspace_bytes", max_level, ranks, ctypes.byref(nbytes))
        self.work = torch.zeros(nbytes.value // 8, **f64)     # halo planes start at zero
        self.out = torch.empty((4, nz, n, n), **f64)
        self.levels = [slab_layout(max_level, ranks, rank, l) for l in range(max_level)]
        self.lp = self.levels[0]["lp"]

    # ------------------------------------------------------------- views --
    def _records(self, level: int) -> Tuple[torch.Tensor, int, int]:
        """Reduced records of a partitioned level as [planes, N*N*18] and (halo, nz)."""
        d = self.levels[level]
        per = d["n"] * d["n"] * 18
        planes = d["nz"] + 2 * d["halo"]
        t = self.work[d["red_off"] // 8:d["red_off"] // 8 + planes * per]
        return t.view(planes, per), d["halo"], d["nz"]

    def _gathered(self) -> List[Tuple[torch.Tensor, int, int]]:
        """(full array, first, last) element ranges of this rank's slab of the
        gathered level's raw and reduced records."""
        g = self.lp - 1
        d = self.levels[g]
        n = d["n"]
        z0 = self.levels[self.lp]["z0"] // 2
        nzg = self.levels[self.lp]["nz"] // 2
        out = []
        for off, rec in ((d["raw_off"], 20), (d["red_off"], 18)):
            full = self.work[off // 8:off // 8 + n ** 3 * rec]
            out.append((full, z0 * n * n * rec, (z0 + nzg) * n * n * rec))
        return out

    def _s(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    # ------------------------------------------------------------- phases --
    def _rhs(self, Uc: torch.Tensor) -> Iterator[tuple]:
        """One right-hand side. Exchanges are posted ("halo", "allgather") and
        awaited ("wait") only where their data is consumed, so on NCCL the
        state halo flies under the FMM upward pass and the multipole halos /
        gather under the hydro pad + flux."""
        s, n, nz = self._s(), self.n, self.nz
        self.send_lo.copy_(Uc[:, :4])
        self.send_hi.copy_(Uc[:, nz - 4:])
        yield ("halo", self.send_lo, self.send_hi, self.recv_lo, self.recv_hi, True)
        # gravity upward pass: local planes only
        self.rho_h[4:4 + nz].copy_(Uc[0])
        rho = self.rho_h.data_ptr() + 4 * n * n * 8
        N.call("tb_fmm_slab_upward", s, self.L, self.R, self.r, rho, self.work.data_ptr())
        for level in range(self.lp, self.L):
            rec, halo, lnz = self._records(level)
            yield ("halo", rec[halo:2 * halo], rec[lnz:lnz + halo], rec[:halo],
                   rec[lnz + halo:], False)
        if self.R > 1:
            for full, a, b in self._gathered():
                yield ("allgather", full, a, b)
        yield ("wait", 0)                 # the state halo (posted first)
        # hydro on the slab: 2 ghost planes from each neighbour (periodic)
        lo2 = self.recv_lo[:, 2:].contiguous()
        hi2 = self.recv_hi[:, :2].contiguous()
        N.call("tb_star_pad_slab", s, Uc.data_ptr(), n, nz, lo2.data_ptr(), hi2.data_ptr(),
               self.Up.data_ptr())
        N.call("tb_hydro_flux_lattice", s, self.Up.data_ptr(), n, nz, self.dudt.data_ptr(),
               self.amax.data_ptr(), self.dx, self.gamma)
        # rho halo for the leaf stencil (zero beyond the isolated domain)
        if self.r > 0:
            self.rho_h[:4].copy_(self.recv_lo[0])
        if self.r < self.R - 1:
            self.rho_h[4 + nz:].copy_(self.recv_hi[0])
        yield ("wait", None)              # everything else
        if self.R > 1:
            N.call("tb_fmm_slab_coarse", s, self.L, self.R, self.r, self.work.data_ptr())
        N.call("tb_fmm_slab_m2l", s, self.L, self.R, self.r, self.work.data_ptr())
        N.call("tb_fmm_slab_downward", s, self.L, self.R, self.r, self.work.data_ptr())
        N.call("tb_fmm_slab_leaf", s, self.L, self.R, self.r, rho, -4, nz + 4,
               self.work.data_ptr(), self.out.data_ptr())

    def step_gen(self) -> Iterator[tuple]:
        """One SSP-RK2 step, yielding the exchanges it needs."""
        s, n, nz = self._s(), self.n, self.nz
        g = self.out.data_ptr() + nz * n * n * 8            # force rows of [4][nz][N][N]
        yield from self._rhs(self.U)
        N.call("tb_star_cfl", s, self.amax.data_ptr(), self.nsub, self.dx, self.cfl,
               self.dt.data_ptr())
        yield ("min", self.dt)
        yield ("wait", None)
        N.call("tb_star_stage", s, 1, None, self.U.data_ptr(), self.dudt.data_ptr(), g,
               self.dt.data_ptr(), n, nz, self.U1.data_ptr())
        yield from self._rhs(self.U1)
        N.call("tb_star_stage", s, 2, self.U.data_ptr(), self.U1.data_ptr(),
               self.dudt.data_ptr(), g, self.dt.data_ptr(), n, nz, self.U.data_ptr())
        self.time.add_(self.dt)


def split_state(U: torch.Tensor, ranks: int) -> List[torch.Tensor]:
    """Global [5, N, N, N] state -> the ranks' [5, N/ranks, N, N] slabs."""
    nz = U.shape[1] // ranks
    return [U[:, r * nz:(r + 1) * nz].contiguous() for r in range(ranks)]


class VirtualCluster:
    """R slabs on one device stepped in lockstep; exchanges are device copies
    on the current stream. Validates the decomposition without R GPUs."""

    def __init__(self, max_level: int, ranks: int, state: torch.Tensor, **kw):
        self.ranks = ranks
        self.slabs = [StarSlab(max_level, ranks, r, s, **kw)
                      for r, s in enumerate(split_state(state, ranks))]

    def _service(self, reqs: List[tuple]) -> None:
        kind = reqs[0][0]
        assert all(q[0] == kind for q in reqs), "ranks out of lockstep"
        R = self.ranks
        if kind == "halo":
            periodic = reqs[0][5]
            for r in range(R):
                _, send_lo, send_hi, recv_lo, recv_hi, _ = reqs[r]
                if periodic or r > 0:          # from the rank below: its top planes
                    recv_lo.copy_(reqs[(r - 1) % R][2])
                if periodic or r < R - 1:      # from the rank above: its bottom planes
                    recv_hi.copy_(reqs[(r + 1) % R][1])
        elif kind == "allgather":
            for r in range(R):
                for q in range(R):
                    if q != r:
                        _, full, a, b = reqs[q]
                        reqs[r][1][a:b].copy_(full[a:b])
        elif kind == "min":
            m = torch.stack([q[1] for q in reqs]).min(dim=0).values
            for q in reqs:
                q[1].copy_(m)
        elif kind != "wait":              # copies above complete in stream order
            raise ValueError(kind)

    def step(self) -> None:
        gens = [s.step_gen() for s in self.slabs]
        while True:
            reqs = []
            for g in gens:
                reqs.append(next(g, None))
            if all(q is None for q in reqs):
                return
            if any(q is None for q in reqs):
                raise RuntimeError("ranks out of lockstep")
            self._service(reqs)

    def state(self) -> torch.Tensor:
        return torch.cat([s.U for s in self.slabs], dim=1)


class DistDriver:
    """One rank of a torch.distributed job stepping its slab. NCCL exchanges
    device tensors directly; other backends (gloo: CPU-side tests) go through
    host copies."""

    def __init__(self, slab: StarSlab, group=None):
        import torch.distributed as dist
        self.dist, self.slab, self.group = dist, slab, group
        self.R, self.r = slab.R, slab.r
        self.host = dist.get_backend(group) != "nccl"
        self.pending: list = []

    def _h(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.host else t

    def _halo(self, send_lo, send_hi, recv_lo, recv_hi, periodic) -> None:
        dist, R, r = self.dist, self.R, self.r
        if R == 1:
            if periodic:
                recv_lo.copy_(send_hi)
                recv_hi.copy_(send_lo)
            return
        below, above = (r - 1) % R, (r + 1) % R
        has_below, has_above = periodic or r > 0, periodic or r < R - 1
        s_lo, s_hi = self._h(send_lo.contiguous()), self._h(send_hi.contiguous())
        # NCCL receives straight into the (contiguous) targets; host staging
        # copies them in when the exchange is awaited
        r_lo = (recv_lo if not self.host else torch.empty_like(s_lo)) if has_below else None
        r_hi = (recv_hi if not self.host else torch.empty_like(s_hi)) if has_above else None
        ops = []
        # sends (lo down, hi up), receives (hi from above, lo from below): with
        # two ranks both neighbours coincide and issue order pairs them up
        if has_below:
            ops.append(dist.P2POp(dist.isend, s_lo, below, self.group))
        if has_above:
            ops.append(dist.P2POp(dist.isend, s_hi, above, self.group))
        if has_above:
            ops.append(dist.P2POp(dist.irecv, r_hi, above, self.group))
        if has_below:
            ops.append(dist.P2POp(dist.irecv, r_lo, below, self.group))
        works = dist.batch_isend_irecv(ops)
        copies = []
        if self.host:
            if has_below:
                copies.append((recv_lo, r_lo))
            if has_above:
                copies.append((recv_hi, r_hi))
        self.pending.append((works, copies, (s_lo, s_hi)))

    def _allgather(self, full, a, b) -> None:
        if self.R == 1:
            return
        dist = self.dist
        if not self.host:
            src = full[a:b].clone()
            w = dist.all_gather_into_tensor(full, src, group=self.group, async_op=True)
            self.pending.append(([w], [], (src,)))
            return
        parts = [torch.empty(b - a, dtype=full.dtype) for _ in range(self.R)]
        w = dist.all_gather(parts, full[a:b].cpu(), group=self.group, async_op=True)
        self.pending.append(([w], [(full, parts)], ()))

    def _wait(self, first_only: bool) -> None:
        todo = self.pending[:1] if first_only else self.pending
        for works, copies, _ in todo:
            for w in works:
                w.wait()
            for dst, src in copies:
                dst.copy_(torch.cat(src) if isinstance(src, list) else src)
        self.pending = self.pending[1:] if first_only else []

    def _min(self, t) -> None:
        if self.R == 1:
            return
        h = self._h(t)
        self.dist.all_reduce(h, op=self.dist.ReduceOp.MIN, group=self.group)
        if self.host:
            t.copy_(h)

    def step(self) -> None:
        self.pending = []
        for req in self.slab.step_gen():
            kind = req[0]
            if kind == "halo":
                self._halo(*req[1:])
            elif kind == "allgather":
                self._allgather(*req[1:])
            elif kind == "min":
                self._min(req[1])
            elif kind == "wait":
                self._wait(first_only=req[1] == 0)
        self._wait(first_only=False)

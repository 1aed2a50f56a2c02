"""Device-resident sub-grid ring: the whole time step on the GPU.

Data layout in HBM (per rank): two contiguous ``double[n_local][512]`` state
generations (4 KiB per sub-grid, 256-B aligned — the reference keeps one
numpy array per sub-grid, src/miniapp.py:77,87), a 72-word int64 step
accumulator (include/tb.h TB_ACC_*), a 2x8 halo of ring-neighbour faces and
per-step ``(piece, dt)`` records plus the running checksum.

One step = K2 (``tb_step``: ghost fold + 15 transforms + per-sub-grid min and
pairwise sum folded into the exact accumulator) + K4 (correctly rounded
piece, dt, ``checksum += piece``) — on one device K4 runs in K2's last CTA
(``tb_step_final``): one launch per step. Bit-identical to ``run_reference``
(src/reference.py:23-50) at any rank count.

Multi-GPU (one process per GPU, torch.distributed/NCCL): the ring is split
into contiguous ranges; per step each rank posts the send of its first
sub-grid's left face to rank-1 and its last sub-grid's right face to rank+1
(64 B each, from the previous generation — Jacobi, src/miniapp.py:89-93),
runs K2 on its interior sub-grids while the faces are in flight, then the two
boundary sub-grids; the accumulator's limbs are then all-reduced with SUM and
its min word with MIN (int64): exact, so every partition gives the
single-device checksum.

Host-buffer path (``step_host``): the drop-in for callers that keep the
cells on the host (the reference's Scenario.grids). The H2D of the input
generation, K2 and the D2H of the new generation are pipelined in chunks of
sub-grids on three streams, so the PCIe transfers in both directions overlap
each other and the compute.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Tuple

import torch

from . import _native as N

CELLS = N.TB_CELLS
FACE = N.TB_FACE


def ring_partition(subgrids: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced [lo, hi) range of sub-grid ids owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if subgrids < world:
        raise ValueError(f"{subgrids} sub-grids cannot be split over {world} ranks")
    base, extra = divmod(subgrids, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def chunk_bounds(n: int, chunks: int) -> List[Tuple[int, int]]:
    """Split [0, n) into at most ``chunks`` contiguous non-empty ranges."""
    chunks = max(1, min(chunks, n))
    base, extra = divmod(n, chunks)
    out, lo = [], 0
    for c in range(chunks):
        hi = lo + base + (1 if c < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def _ptr(t):
    """Device address of a tensor (or a raw address already, e.g. peer HBM)."""
    if t is None or isinstance(t, int):
        return t
    return t.data_ptr()


class CudaRingOps:
    """The product kernels (libtb) behind the stepper's primitives."""

    def __init__(self, device: torch.device):
        if device.type != "cuda":
            raise RuntimeError("CudaRingOps needs a CUDA device (no CPU fallback)")
        N.init(device.index or 0)
        self.device = device

    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def init_cells(self, cells: torch.Tensor, subgrids: int, lo: int) -> None:
        N.call("tb_init_cells", self.stream(), _ptr(cells), subgrids, lo, cells.shape[0])

    def step(self, old, out, left_face, right_face, chains, kpc, acc,
             mins=None, sums=None) -> None:
        N.call("tb_step", self.stream(), _ptr(old), _ptr(out), old.shape[0],
               _ptr(left_face), _ptr(right_face), chains, kpc, _ptr(mins), _ptr(sums),
               _ptr(acc))

    def step_final(self, old, out, left_face, right_face, chains, kpc, acc, piece, dt,
                   checksum, mins=None, sums=None) -> None:
        N.call("tb_step_final", self.stream(), _ptr(old), _ptr(out), old.shape[0],
               _ptr(left_face), _ptr(right_face), chains, kpc, _ptr(mins), _ptr(sums),
               _ptr(acc), _ptr(piece), _ptr(dt), _ptr(checksum))

    def step_deferred(self, old, out, left_face, right_face, chains, kpc, sums, mins,
                      prev_sums, prev_mins, acc, prev_piece, prev_dt, checksum) -> None:
        N.call("tb_step_deferred", self.stream(), _ptr(old), _ptr(out), old.shape[0],
               _ptr(left_face), _ptr(right_face), chains, kpc, _ptr(sums), _ptr(mins),
               _ptr(prev_sums), _ptr(prev_mins), _ptr(acc), _ptr(prev_piece), _ptr(prev_dt),
               _ptr(checksum))

    def step_close(self, sums, mins, acc, piece, dt, checksum) -> None:
        N.call("tb_step_close", self.stream(), _ptr(sums), _ptr(mins), sums.shape[0],
               _ptr(acc), _ptr(piece), _ptr(dt), _ptr(checksum))

    def acc_reset(self, acc) -> None:
        N.call("tb_acc_reset", self.stream(), _ptr(acc))

    def acc_finalize(self, acc, piece, dt, checksum) -> None:
        N.call("tb_acc_finalize", self.stream(), _ptr(acc), _ptr(piece), _ptr(dt),
               _ptr(checksum), 1)


@dataclass
class RingResult:
    checksum: float
    dts: List[float]
    pieces: List[float]


class RingStepper:
    """Runs the sub-grid ring for ``steps`` time steps on this rank's device.

    ``group`` is a torch.distributed process group (None: single device, or
    the default group when ``world > 1``). ``ops`` defaults to the libtb
    kernels; tests substitute a CPU double to cover the multi-rank host logic
    under gloo.
    """

    def __init__(self, subgrids: int, device: Optional[torch.device] = None,
                 rank: int = 0, world: int = 1, chains: int = 3,
                 kernels_per_chain: int = 5, max_steps: int = 1 << 16,
                 ops=None, group=None, collect_subgrid_stats: bool = False,
                 halo: str = "auto"):
        if subgrids < 1:
            raise ValueError("subgrids must be >= 1")
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.ops = ops if ops is not None else CudaRingOps(device)
        self.subgrids, self.rank, self.world = subgrids, rank, world
        self.chains, self.kpc = chains, kernels_per_chain
        self.group = group
        self.lo, self.hi = ring_partition(subgrids, world, rank)
        n = self.n = self.hi - self.lo
        f64 = dict(dtype=torch.float64, device=device)
        self.state = [torch.empty((n, CELLS), **f64), torch.empty((n, CELLS), **f64)]
        self.cur = 0
        self.acc = torch.zeros(N.TB_ACC_WORDS, dtype=torch.int64, device=device)
        self.halo = torch.zeros((2, FACE), **f64)        # [left ghost, right ghost]
        self.myfaces = torch.zeros((2, FACE), **f64)     # [my left face, my right face]
        self.max_steps = max_steps
        self.pieces = torch.zeros(max_steps, **f64)
        self.dts = torch.zeros(max_steps, **f64)
        self.checksum = torch.zeros(1, **f64)
        self.mins = torch.empty(n, **f64) if collect_subgrid_stats else None
        self.sums = torch.empty(n, **f64) if collect_subgrid_stats else None
        self.steps_done = 0
        self._streams = None
        # (chunk bounds, D2H events, steps_done, unjoined in-place, host_out)
        self._host_prev = None
        self.ops.init_cells(self.state[0], subgrids, self.lo)
        self.ops.acc_reset(self.acc)
        # single device, back to back: step k writes per-sub-grid (sum, min)
        # into parity k & 1 and step k+1's launch closes it exactly
        # (tb_step_deferred); `pending` = the step still awaiting that
        self.dsums = torch.zeros((2, n), **f64)
        self.dmins = torch.zeros((2, n), **f64)
        self._pending: Optional[int] = None
        self._collect = collect_subgrid_stats
        # Multi-GPU halo: "p2p" maps the ring neighbours' state buffers (CUDA
        # IPC) so K2 reads the ghost faces straight from their HBM; "nccl"
        # sends them with NCCL P2P; "auto" tries p2p, else nccl.
        self.halo_mode = "local" if world == 1 else "nccl"
        self._peers = None
        if world > 1 and halo not in ("auto", "p2p", "nccl"):
            raise ValueError(f"unknown halo mode {halo!r}")
        if world > 1 and halo != "nccl" and isinstance(self.ops, CudaRingOps):
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                self._peers, err = self._map_peers()
            else:
                err = "no process group to exchange IPC handles over"
            if self._peers is not None:
                self.halo_mode = "p2p"
                self._alloc_diag()
            elif halo == "p2p":
                raise RuntimeError(f"peer-memory halo unavailable: {err}")

    @staticmethod
    def _export(t: torch.Tensor):
        """(IPC handle of the allocation holding t, byte offset of t in it)."""
        import ctypes
        handle = (ctypes.c_uint8 * N.TB_IPC_HANDLE_BYTES)()
        offset = ctypes.c_uint64(0)
        N.call("tb_ipc_get_handle", t.data_ptr(), handle, ctypes.byref(offset))
        return bytes(handle), offset.value

    def _map_peers(self):
        """Exchange IPC handles with every rank; map the ring neighbours' two
        state generations (peer-memory halo) and every rank's reduction
        accumulators (peer-memory all-reduce).

        Collective and all-or-nothing: every rank runs the same two
        all-gathers whatever fails locally, and the mapping is kept only when
        every rank succeeded, so all ranks take the same halo path. Returns
        (peers, None) or (None, the first local error)."""
        import ctypes

        import torch.distributed as dist
        err = None
        mine = None
        try:
            # two parities of the cross-rank accumulator (tb_acc_allreduce_p2p)
            self.gacc = torch.zeros((2, N.TB_ACC_WORDS), dtype=torch.int64,
                                    device=self.device)
            self.gacc[:, N.TB_ACC_MIN_WORD] = 0x7FF0000000000000      # key(+inf)
            mine = ([self._export(t) for t in self.state], self.n, self._export(self.gacc))
        except Exception as e:          # noqa: BLE001 — reported after agreement
            err = e
        table = [None] * self.world
        dist.all_gather_object(table, mine, group=self.group)
        if any(t is None for t in table):
            return None, err or "a peer could not export its buffers"
        opened = {}

        def open_handle(handle, offset):
            # cudaIpcOpenMemHandle reference-counts repeated opens of one
            # allocation (small rings put several tensors in one caching-
            # allocator segment): count them, close() closes each open
            base = ctypes.c_void_p()
            buf = (ctypes.c_uint8 * N.TB_IPC_HANDLE_BYTES).from_buffer_copy(handle)
            N.call("tb_ipc_open_handle", buf, ctypes.byref(base))
            opened[base.value] = opened.get(base.value, 0) + 1
            return base.value, base.value + offset

        peers = None
        try:
            left, right = (self.rank - 1) % self.world, (self.rank + 1) % self.world
            state = {}
            for peer in sorted({left, right}):
                state[peer] = ([open_handle(h, off) for h, off in table[peer][0]],
                               table[peer][1])
            row = self.gacc.stride(0) * self.gacc.element_size()
            tab = [[0] * self.world for _ in range(2)]
            for p in range(self.world):
                if p == self.rank:
                    base_ptr = self.gacc.data_ptr()
                else:
                    base_ptr = open_handle(*table[p][2])[1]
                for parity in range(2):
                    tab[parity][p] = base_ptr + parity * row
            self.peer_tab = torch.tensor(tab, dtype=torch.int64, device=self.device)
            peers = {"left": state[left], "right": state[right], "bases": dict(opened)}
        except Exception as e:          # noqa: BLE001 — reported after agreement
            err = e
        ok = [None] * self.world
        dist.all_gather_object(ok, peers is not None, group=self.group)
        if not all(ok):
            for base, count in opened.items():
                for _ in range(count):
                    N.call("tb_ipc_close", base)
            return None, err or "a peer could not map its neighbours' buffers"
        return peers, None

    def _alloc_diag(self) -> None:
        """The arrival watchdog's diagnostic words: mapped pinned host memory,
        still readable after a trap has taken the CUDA context down."""
        p = ctypes.c_void_p()
        N.call("tb_host_alloc", ctypes.byref(p), 32)
        self._diag_ptr = p.value
        self._diag = (ctypes.c_int64 * 4).from_address(p.value)
        for i in range(4):
            self._diag[i] = 0

    def close(self) -> None:
        """Unmap neighbours' buffers (p2p halo): every open of each mapped
        allocation is closed."""
        if self._peers is not None:
            torch.cuda.synchronize(self.device)
            for base, count in self._peers["bases"].items():
                for _ in range(count):
                    N.call("tb_ipc_close", base)
            self._peers = None
            N.call("tb_host_free", ctypes.c_void_p(self._diag_ptr))
            self._diag = None

    P2P_DIAG_MAGIC = 0x7470325774696d65
    P2P_TIMEOUT_S = float(os.environ.get("TB_P2P_TIMEOUT_S", "30"))

    def peer_timeout(self) -> Optional[str]:
        """After a failed step: which rank's peer-memory arrival wait timed
        out, at which step, with how many of the ranks arrived (None if the
        watchdog did not fire)."""
        d = getattr(self, "_diag", None)
        if d is None or d[0] != self.P2P_DIAG_MAGIC:
            return None
        return (f"rank {d[1]} waited more than {self.P2P_TIMEOUT_S:g} s at step {d[2]} "
                f"for the step's arrivals: {d[3]} of {self.world} ranks arrived")

    # -------------------------------------------------------------- state --
    def reset(self) -> None:
        """Begin a new run on this stepper's buffers: step count, checksum
        and exact accumulator zeroed (the cells are left to load_cells)."""
        self.flush()
        self.steps_done = 0
        self.checksum.zero_()
        self.ops.acc_reset(self.acc)
        self._pending = None
        self._host_prev = None

    @property
    def cells(self) -> torch.Tensor:
        """This rank's current generation, [n_local, 512] (device)."""
        return self.state[self.cur]

    def load_cells(self, host: torch.Tensor) -> None:
        """Replace the current generation with ``host`` ([n_local, 512])."""
        self.state[self.cur].copy_(host, non_blocking=True)

    # --------------------------------------------------------------- step --
    def _exchange_start(self, send_left: torch.Tensor, send_right: torch.Tensor):
        """Post the ring halo exchange into self.halo = [left ghost, right
        ghost]; returns the requests (wait them before reading the halo)."""
        import torch.distributed as dist
        left = (self.rank - 1) % self.world
        right = (self.rank + 1) % self.world
        # Issue order makes N=2 (left == right) unambiguous: the first message
        # from a peer is its LEFT face (-> my right ghost), the second its
        # RIGHT face (-> my left ghost).
        ops = [dist.P2POp(dist.isend, send_left, left, self.group),
               dist.P2POp(dist.irecv, self.halo[1], right, self.group),
               dist.P2POp(dist.isend, send_right, right, self.group),
               dist.P2POp(dist.irecv, self.halo[0], left, self.group)]
        return dist.batch_isend_irecv(ops)

    def _exchange(self, send_left: torch.Tensor, send_right: torch.Tensor) -> None:
        import torch.distributed as dist
        if send_left.is_cuda and dist.get_backend(self.group) != "nccl":
            # gloo cannot send device memory: stage the 64-byte faces on the host
            left = (self.rank - 1) % self.world
            right = (self.rank + 1) % self.world
            sl, sr = send_left.cpu(), send_right.cpu()
            h0, h1 = torch.empty_like(sl), torch.empty_like(sr)
            ops = [dist.P2POp(dist.isend, sl, left, self.group),
                   dist.P2POp(dist.irecv, h1, right, self.group),
                   dist.P2POp(dist.isend, sr, right, self.group),
                   dist.P2POp(dist.irecv, h0, left, self.group)]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            self.halo[0].copy_(h0)
            self.halo[1].copy_(h1)
            return
        for req in self._exchange_start(send_left, send_right):
            req.wait()

    def _reduce_acc(self) -> None:
        import torch.distributed as dist
        dist.all_reduce(self.acc[:N.TB_ACC_LIMBS], op=dist.ReduceOp.SUM, group=self.group)
        dist.all_reduce(self.acc[N.TB_ACC_MIN_WORD:N.TB_ACC_MIN_WORD + 1],
                        op=dist.ReduceOp.MIN, group=self.group)

    def _close(self, k: int) -> None:
        if self.world > 1:
            self._reduce_acc()
        self.ops.acc_finalize(self.acc, self.pieces[k:k + 1], self.dts[k:k + 1],
                              self.checksum)

    def step(self, kernel_events=None) -> None:
        """Advance one time step (asynchronous on the current stream).

        ``kernel_events``: optional (start, end) CUDA events recorded around
        the fused step launch alone (bench.py uses them for the roofline).
        """
        if self.steps_done >= self.max_steps:
            raise RuntimeError("max_steps exceeded; raise max_steps")
        if self._host_prev is not None:
            self.join_host()        # downloads of a host step still read state
            self._host_prev = None
        k = self.steps_done
        old, out = self.state[self.cur], self.state[1 - self.cur]
        n = self.n
        if self.world > 1:
            self._step_partitioned(old, out, kernel_events)
            if self._peers is not None:
                # exact cross-rank reduction + step barrier over peer memory
                N.call("tb_acc_allreduce_p2p_ex", self.ops.stream(), _ptr(self.acc),
                       self.peer_tab[k & 1].data_ptr(), self.world,
                       self.gacc[k & 1].data_ptr(), _ptr(self.pieces[k:k + 1]),
                       _ptr(self.dts[k:k + 1]), _ptr(self.checksum),
                       int(self.P2P_TIMEOUT_S * 1e9), self.rank, k, self._diag_ptr)
            else:
                self._close(k)
        else:
            lf, rf = old[n - 1, CELLS - FACE:], old[0, :FACE]   # ring wraps locally
            if kernel_events is not None:
                kernel_events[0].record()
            if hasattr(self.ops, "step_deferred"):
                p = self._pending
                self.ops.step_deferred(
                    old, out, lf, rf, self.chains, self.kpc, self.dsums[k & 1],
                    self.dmins[k & 1], None if p is None else self.dsums[p & 1],
                    None if p is None else self.dmins[p & 1], self.acc,
                    None if p is None else self.pieces[p:p + 1],
                    None if p is None else self.dts[p:p + 1], self.checksum)
                self._pending = k
                if self._collect:
                    self.sums, self.mins = self.dsums[k & 1], self.dmins[k & 1]
            elif hasattr(self.ops, "step_final"):
                self.ops.step_final(old, out, lf, rf, self.chains, self.kpc, self.acc,
                                    self.pieces[k:k + 1], self.dts[k:k + 1],
                                    self.checksum, self.mins, self.sums)
            else:
                self.ops.step(old, out, lf, rf, self.chains, self.kpc, self.acc,
                              self.mins, self.sums)
                self._close(k)
            if kernel_events is not None:
                kernel_events[1].record()
        self.cur = 1 - self.cur
        self.steps_done += 1

    def _step_partitioned(self, old, out, kernel_events) -> None:
        """N>1. p2p halo: one K2 launch whose two ghost-face pointers point
        into the neighbours' HBM (the previous step's all-reduce orders every
        rank's K2(t-1) before any K2(t), and K2(t) before any K2(t+1), so no
        extra synchronisation is needed). nccl halo: post the exchange, run K2
        on the interior sub-grids while the 2 x 64 B faces are in flight, then
        the two boundary sub-grids."""
        n = self.n
        if self._peers is not None:
            (lptrs, ln), (rptrs, _) = self._peers["left"], self._peers["right"]
            lf = lptrs[self.cur][1] + ((ln - 1) * CELLS + CELLS - FACE) * 8
            rf = rptrs[self.cur][1]
            if kernel_events is not None:
                kernel_events[0].record()
            self.ops.step(old, out, lf, rf, self.chains, self.kpc, self.acc,
                          self.mins, self.sums)
            if kernel_events is not None:
                kernel_events[1].record()
            return
        import torch.distributed as dist
        if old.is_cuda and dist.is_initialized() and dist.get_backend(self.group) != "nccl":
            # gloo cannot post device memory: the host-staged blocking exchange
            # (a code-path test configuration, e.g. several ranks on one GPU)
            self._exchange(old[0, :FACE], old[n - 1, CELLS - FACE:])
            reqs = []
        else:
            reqs = self._exchange_start(old[0, :FACE], old[n - 1, CELLS - FACE:])
        if kernel_events is not None:
            kernel_events[0].record()
        mins, sums = self.mins, self.sums

        def part(lo, hi, lf, rf):
            self.ops.step(old[lo:hi], out[lo:hi], lf, rf, self.chains, self.kpc, self.acc,
                          None if mins is None else mins[lo:hi],
                          None if sums is None else sums[lo:hi])

        if n > 2:       # interior: every ghost face is local
            part(1, n - 1, old[0, CELLS - FACE:], old[n - 1, :FACE])
        for req in reqs:
            req.wait()
        if n == 1:
            part(0, 1, self.halo[0], self.halo[1])
        else:
            part(0, 1, self.halo[0], old[1, :FACE])
            part(n - 1, n, old[n - 2, CELLS - FACE:], self.halo[1])
        if kernel_events is not None:
            kernel_events[1].record()

    def flush(self) -> None:
        """Close the last device step's deferred accumulator (its piece, dt
        and checksum contribution are then final)."""
        p = self._pending
        if p is not None:
            self.ops.step_close(self.dsums[p & 1], self.dmins[p & 1], self.acc,
                                self.pieces[p:p + 1], self.dts[p:p + 1], self.checksum)
            self._pending = None

    def run(self, steps: int) -> RingResult:
        k0 = self.steps_done
        for _ in range(steps):
            self.step()
        return self.result(k0)

    # ------------------------------------------------------ host buffers --
    def step_host(self, host_in: torch.Tensor, host_out: Optional[torch.Tensor],
                  host_stats: torch.Tensor, chunks: int = 16, join: bool = True) -> None:
        """One step on host-resident cells (the host-buffer drop-in path).

        ``host_in``/``host_out``: pinned [n_local, 512] float64 (may alias;
        ``host_out=None`` keeps the new generation on the device and returns
        only the step result); ``host_stats``: pinned float64[2] receiving
        (piece, dt). Work goes to the current stream plus an upload and a
        download stream. Per chunk c of sub-grids: H2D(c) on the upload
        stream; K2(c) once H2D(c) and H2D(c+1) landed (c's right ghost lives
        in c+1); D2H(c) on the download stream once K2(c) is done.

        Consecutive calls pipeline across steps: H2D(c) of the next step only
        waits for this step's D2H(c) (the host rows and device rows it
        overwrites), so uploads and downloads stream continuously in both
        PCIe directions. ``join=False`` leaves the download stream un-joined
        (call :meth:`join_host` before reading the outputs on the host or
        timing on the current stream); ``join=True`` joins every step.
        """
        if self.steps_done >= self.max_steps:
            raise RuntimeError("max_steps exceeded; raise max_steps")
        if not isinstance(self.ops, CudaRingOps):
            raise RuntimeError("step_host needs the CUDA ops")
        self.flush()          # a preceding device step's checksum piece comes first
        dev = self.device
        main = torch.cuda.current_stream(dev)
        if self._streams is None:
            self._streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        up, down = self._streams
        k = self.steps_done
        old, out = self.state[self.cur], self.state[1 - self.cur]
        bounds = chunk_bounds(self.n, chunks)
        ev_h2d = [torch.cuda.Event() for _ in bounds]
        ev_k2 = [torch.cuda.Event() for _ in bounds]
        ev_d2h = [torch.cuda.Event() for _ in bounds]
        ev_faces = torch.cuda.Event()
        n = self.n
        last = len(bounds) - 1
        prev = self._host_prev
        chained = (prev is not None and prev[0] == bounds and prev[2] == self.steps_done)
        # In an un-joined in-place chain the host rows this step reads are
        # exactly the previous step's device output: take the wrap faces from
        # HBM instead of waiting for the previous step's last download.
        faces_on_device = chained and prev[3] and host_in is prev[4]
        if not chained:
            # previous work on these buffers came from elsewhere: full order
            up.wait_stream(main)
            up.wait_stream(down)
        faces = self.myfaces if self.world > 1 else self.halo
        src_rows = (0, n - 1) if self.world > 1 else (n - 1, 0)
        if faces_on_device:
            # `old` holds the previous step's output (= the host rows being
            # re-uploaded into it, byte-identical in an in-place chain)
            prev_out = old
            faces[0].copy_(prev_out[src_rows[0], :FACE] if self.world > 1
                           else prev_out[src_rows[0], CELLS - FACE:])
            faces[1].copy_(prev_out[src_rows[1], CELLS - FACE:] if self.world > 1
                           else prev_out[src_rows[1], :FACE])
            ev_faces.record(main)
        with torch.cuda.stream(up):
            if not faces_on_device:
                if chained:
                    up.wait_event(prev[1][0])
                    up.wait_event(prev[1][last])
                if self.world > 1:
                    faces[0].copy_(host_in[0, :FACE], non_blocking=True)
                    faces[1].copy_(host_in[n - 1, CELLS - FACE:], non_blocking=True)
                else:
                    faces[0].copy_(host_in[n - 1, CELLS - FACE:], non_blocking=True)
                    faces[1].copy_(host_in[0, :FACE], non_blocking=True)
                ev_faces.record(up)
            for c, ((lo, hi), ev) in enumerate(zip(bounds, ev_h2d)):
                if chained:
                    up.wait_event(prev[1][c])
                old[lo:hi].copy_(host_in[lo:hi], non_blocking=True)
                ev.record(up)
        main.wait_event(ev_faces)
        if self.world > 1:
            self._exchange(self.myfaces[0], self.myfaces[1])
        for c, (lo, hi) in enumerate(bounds):
            main.wait_event(ev_h2d[c])
            if c < last:
                main.wait_event(ev_h2d[c + 1])
            lf = self.halo[0] if c == 0 else old[lo - 1, CELLS - FACE:]
            rf = self.halo[1] if c == last else old[hi, :FACE]
            self.ops.step(old[lo:hi], out[lo:hi], lf, rf, self.chains, self.kpc, self.acc)
            ev_k2[c].record(main)
        self._close(k)
        ev_done = torch.cuda.Event()
        ev_done.record(main)
        with torch.cuda.stream(down):
            for c, (lo, hi) in enumerate(bounds):
                down.wait_event(ev_k2[c])
                if host_out is not None:
                    host_out[lo:hi].copy_(out[lo:hi], non_blocking=True)
                ev_d2h[c].record(down)
            down.wait_event(ev_done)
            host_stats[0:1].copy_(self.pieces[k:k + 1], non_blocking=True)
            host_stats[1:2].copy_(self.dts[k:k + 1], non_blocking=True)
        self.cur = 1 - self.cur
        self.steps_done += 1
        self._host_prev = (bounds, ev_d2h, self.steps_done, not join and host_out is not None,
                           host_out)
        if join:
            self.join_host()

    def join_host(self) -> None:
        """Make the current stream wait for all enqueued host-buffer downloads."""
        if self._streams is not None:
            torch.cuda.current_stream(self.device).wait_stream(self._streams[1])

    def result(self, first_step: int = 0) -> RingResult:
        self.flush()
        k = self.steps_done
        return RingResult(checksum=float(self.checksum.item()),
                          dts=self.dts[first_step:k].tolist(),
                          pieces=self.pieces[first_step:k].tolist())


def run_reference_gpu(subgrids: int, steps: int, chains: int = 3,
                      kernels_per_chain: int = 5,
                      device: Optional[torch.device] = None) -> Tuple[float, List[float]]:
    """Drop-in for ``run_reference(subgrids, steps)`` (src/reference.py:23)
    computed on the GPU: returns (checksum, dts)."""
    st = RingStepper(subgrids, device=device, chains=chains,
                     kernels_per_chain=kernels_per_chain, max_steps=max(steps, 1))
    res = st.run(steps)
    return res.checksum, res.dts

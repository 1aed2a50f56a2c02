"""numpy restatement of the reference mini-app data path — TEST INFRASTRUCTURE.

See ``oracle/__init__.py`` for who may import this. Every function cites the
reference lines it restates (paths relative to ``/root/reference``; ``src/``
is ``pkg/src/taskbridge/``).
"""

from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

CELLS = 512          # src/miniapp.py:30
FACE = 8             # src/miniapp.py:31
KINDS = 5            # src/miniapp.py:32
C1 = (1.0000003, 0.9999998, 1.0000001, 0.9999997, 1.0000002)   # src/miniapp.py:36
C2 = (1e-07, -1e-07, 2e-07, 5e-08, -2e-07)                     # src/miniapp.py:37


def initial_cells(subgrids: int, lo: int = 0, hi: int | None = None) -> np.ndarray:
    """``cells[g][i] = (g*1000 + i) / (S*1000 + 512)`` as one [n, 512] array.

    Restates ``SubGrid.__init__`` (src/miniapp.py:72-77) and
    src/reference.py:26-28 (same expression, same rounding: the numerator
    ``g*1000.0 + i`` is exact, the division rounds once).
    """
    hi = subgrids if hi is None else hi
    scale = float(subgrids * 1000 + CELLS)
    base = np.arange(CELLS, dtype=np.float64)
    ids = np.arange(lo, hi, dtype=np.float64)[:, None]
    return (ids * 1000.0 + base[None, :]) / scale


def transform(view: np.ndarray, kind: int) -> None:
    """In-place ``view *= c1[k]; view += c2[k]`` (src/miniapp.py:49-51):
    two separately rounded IEEE operations, never a fused multiply-add."""
    view *= C1[kind]
    view += C2[kind]


def pairwise_sum(a: Sequence[float]) -> float:
    """numpy's float64 ``add.reduce`` order for a contiguous 1-D array
    (``ndarray.sum`` as used at src/miniapp.py:133 and src/reference.py:47).

    Blocks of <=128 use 8 strided accumulators combined as
    ``((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))``; longer runs split at
    ``n/2`` rounded down to a multiple of 8. Pure Python: for small cases.
    """
    n = len(a)
    if n < 8:
        res = 0.0
        for x in a:
            res += float(x)
        return res
    if n <= 128:
        r = [float(x) for x in a[:8]]
        for i in range(8, n - (n % 8), 8):
            for j in range(8):
                r[j] += float(a[i + j])
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for i in range(n - (n % 8), n):
            res += float(a[i])
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def subgrid_sums_512(work: np.ndarray) -> np.ndarray:
    """Vectorised :func:`pairwise_sum` for an [n, 512] array (one row per
    sub-grid), identical bits to ``row.sum()`` per row."""
    assert work.shape[1] == CELLS
    blocks = work.reshape(work.shape[0], 4, 16, 8)   # [g, block, i, r]
    r = blocks[:, :, 0, :].copy()
    for i in range(1, 16):
        r += blocks[:, :, i, :]
    b = ((r[..., 0] + r[..., 1]) + (r[..., 2] + r[..., 3])) + \
        ((r[..., 4] + r[..., 5]) + (r[..., 6] + r[..., 7]))
    return (b[:, 0] + b[:, 1]) + (b[:, 2] + b[:, 3])


def step_cells(old: np.ndarray, left_face: np.ndarray | None = None,
               right_face: np.ndarray | None = None,
               chains: int = 3, kernels_per_chain: int = 5
               ) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """One time step over sub-grids ``old`` ([n, 512], consecutive ids).

    Restates src/reference.py:31-47 (= src/miniapp.py:119-133 per grid):
    ghost faces are read from the *previous* generation (face snapshot,
    src/reference.py:32 / src/miniapp.py:89-93); ``left_face`` is the right
    face of the sub-grid before ``old[0]`` and ``right_face`` the left face
    of the one after ``old[-1]`` — for a full ring (the default) these wrap.
    Returns ``(new, mins, sums)``.
    """
    n = old.shape[0]
    if left_face is None:
        left_face = old[-1, -FACE:]
    if right_face is None:
        right_face = old[0, :FACE]
    lefts = np.empty((n, FACE))
    rights = np.empty((n, FACE))
    lefts[0] = left_face
    lefts[1:] = old[:-1, -FACE:]
    rights[-1] = right_face
    rights[:-1] = old[1:, :FACE]
    work = old.copy()
    work[:, :FACE] = 0.5 * (work[:, :FACE] + lefts)       # src/reference.py:37
    work[:, -FACE:] = 0.5 * (work[:, -FACE:] + rights)    # src/reference.py:38
    for _chain in range(chains):                          # src/reference.py:39-42
        for kind in range(kernels_per_chain):
            transform(work, kind)
    return work, work.min(axis=1), subgrid_sums_512(work)


def run_reference_cells(subgrids: int, steps: int, chains: int = 3,
                        kernels_per_chain: int = 5
                        ) -> Tuple[float, List[float], np.ndarray]:
    """``run_reference`` (src/reference.py:23-50) that also returns the cells.

    dt is the min over sub-grid mins (src/reference.py:48); the step piece
    is ``math.fsum`` over per-sub-grid sums in id order and accumulates
    sequentially into the checksum (src/reference.py:49).
    """
    cells = initial_cells(subgrids)
    checksum = 0.0
    dts: List[float] = []
    for _ in range(steps):
        cells, mins, sums = step_cells(cells, chains=chains,
                                       kernels_per_chain=kernels_per_chain)
        dts.append(float(mins.min()))
        checksum += math.fsum(sums.tolist())
    return checksum, dts, cells


def run_reference_per_subgrid(subgrids: int, steps: int, chains: int = 3,
                               kernels_per_chain: int = 5) -> Tuple[float, List[float]]:
    """``run_reference`` with the reference's execution shape — a Python loop
    over sub-grids, each a separate 512-value numpy array (src/reference.py:
    26-47) — for timing the Python reference on the GPU box's host, where
    the reference package itself is absent (bench.py python_reference).
    Same results as :func:`run_reference` (tests/test_oracle.py)."""
    rows = list(initial_cells(subgrids))
    checksum = 0.0
    dts: List[float] = []
    for _ in range(steps):
        ghosts = [(r[:FACE].copy(), r[-FACE:].copy()) for r in rows]   # Jacobi snapshot
        mins, sums = [], []
        for g in range(subgrids):
            w = rows[g].copy()
            w[:FACE] = 0.5 * (w[:FACE] + ghosts[g - 1][1])
            w[-FACE:] = 0.5 * (w[-FACE:] + ghosts[(g + 1) % subgrids][0])
            for _chain in range(chains):
                for kind in range(kernels_per_chain):
                    transform(w, kind)
            rows[g] = w
            mins.append(float(w.min()))
            sums.append(float(w.sum()))
        dts.append(min(mins))
        checksum += math.fsum(sums)
    return checksum, dts


def run_reference(subgrids: int, steps: int, chains: int = 3,
                  kernels_per_chain: int = 5) -> Tuple[float, List[float]]:
    """Same signature and result as src/reference.py:23."""
    checksum, dts, _ = run_reference_cells(subgrids, steps, chains, kernels_per_chain)
    return checksum, dts


# ---------------------------------------------------------------- exact sum
# The product computes the per-step checksum piece on the GPU with an
# integer superaccumulator (32-bit digits in int64 limbs). This restatement
# of that decomposition lets CPU tests check the digit layout against
# math.fsum without a GPU. Layout constants mirror include/tb.h.

ACC_DIGIT_BITS = 32
ACC_LIMBS = 68            # TB_ACC_LIMBS: covers bit 0 (2^-1074) .. 2^1024 + carries
ACC_BIAS = 1074


def acc_add(acc: List[int], x: float) -> None:
    """Add ``x`` exactly into ``acc`` (list of Python ints, one per limb)."""
    if x == 0.0:
        return
    m, e = math.frexp(abs(x))              # x = m * 2^e, 0.5 <= m < 1
    mant = int(m * (1 << 53))              # 53-bit integer
    p = e - 53 + ACC_BIAS                  # bit position of mant's LSB
    if p < 0:                              # subnormal inputs: mant has trailing zeros
        mant >>= -p
        p = 0
    sign = -1 if x < 0 else 1
    limb, off = divmod(p, ACC_DIGIT_BITS)
    v = mant << off
    while v:
        acc[limb] += sign * (v & 0xFFFFFFFF)
        v >>= 32
        limb += 1


def acc_round(acc: List[int]) -> float:
    """Correctly rounded (half-even) double of the exact sum in ``acc``."""
    total = 0
    for i, d in enumerate(acc):
        total += d << (ACC_DIGIT_BITS * i)
    if total == 0:
        return 0.0
    sign = -1.0 if total < 0 else 1.0
    mag = abs(total)
    nbits = mag.bit_length()
    if nbits <= 53:
        return sign * math.ldexp(float(mag), -ACC_BIAS)
    shift = nbits - 53
    top = mag >> shift
    rem = mag & ((1 << shift) - 1)
    half = 1 << (shift - 1)
    if rem > half or (rem == half and (top & 1)):
        top += 1
    return sign * math.ldexp(float(top), shift - ACC_BIAS)


def exact_sum(values: Sequence[float]) -> float:
    acc = [0] * ACC_LIMBS
    for v in values:
        acc_add(acc, float(v))
    return acc_round(acc)

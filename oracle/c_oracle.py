"""ctypes binding of oracle/libtb_oracle.so — TEST INFRASTRUCTURE / CPU BASELINE.

See oracle/__init__.py for who may import this. ``build()`` runs
``make -C oracle``; the .so is git-ignored but travels to the GPU box.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtb_oracle.so")

_lib = None
_dp = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, ci = ctypes.c_int64, ctypes.c_int
        L.tbo_init.argtypes = [_dp, i64, i64, i64]
        L.tbo_step.argtypes = [_dp, _dp, i64, _dp, _dp, ci, ci, _dp, _dp, ci]
        L.tbo_fsum.argtypes = [_dp, i64]
        L.tbo_fsum.restype = ctypes.c_double
        L.tbo_run.argtypes = [i64, ci, ci, ci, ci, _dp, _dp]
        L.tbo_run.restype = ci
        L.tbo_max_threads.restype = ci
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def max_threads() -> int:
    return lib().tbo_max_threads()


def init_cells(subgrids: int, lo: int = 0, n: int | None = None) -> np.ndarray:
    n = subgrids - lo if n is None else n
    out = np.empty((n, 512))
    lib().tbo_init(_p(out), subgrids, lo, n)
    return out


def step(old: np.ndarray, out: np.ndarray, left_face: np.ndarray,
         right_face: np.ndarray, mins: np.ndarray, sums: np.ndarray,
         chains: int = 3, kernels_per_chain: int = 5, threads: int = 0) -> None:
    lib().tbo_step(_p(old), _p(out), old.shape[0], _p(left_face), _p(right_face),
                   chains, kernels_per_chain, _p(mins), _p(sums), threads)


def fsum(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().tbo_fsum(_p(x), x.size)


def run_reference(subgrids: int, steps: int, chains: int = 3,
                  kernels_per_chain: int = 5, threads: int = 0
                  ) -> Tuple[float, List[float]]:
    cs = ctypes.c_double()
    dts = np.empty(steps)
    rc = lib().tbo_run(subgrids, steps, chains, kernels_per_chain, threads,
                       ctypes.byref(cs), _p(dts))
    if rc != 0:
        raise MemoryError("tbo_run: allocation failed")
    return cs.value, dts.tolist()

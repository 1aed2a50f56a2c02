"""ctypes binding of libtb.so (include/tb.h).

There is no CPU fallback: if the library is missing or fails to load, every
entry point raises :class:`NativeUnavailable`. Two views of the same library
are kept: ``fast`` (``ctypes.PyDLL``: the GIL stays held — for calls that only
enqueue work and return in microseconds) and ``blocking`` (``ctypes.CDLL``:
the GIL is released — for calls that may wait on the device).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceGoneError, TaskBridgeError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TB_LIBTB", os.path.join(PKG, "libtb.so"))

TB_OK = 0
TB_NOT_READY = 1
TB_E_INVALID = -10000
TB_E_NOMEM = -10001
TB_E_CLOSED = -10002

TB_CELLS = 512
TB_FACE = 8
TB_KINDS = 5
TB_ACC_LIMBS = 68
TB_ACC_BIAS = 1074
TB_ACC_MIN_WORD = 68
TB_ACC_COUNT_WORD = 70
TB_ACC_WORDS = 72
TB_IPC_HANDLE_BYTES = 64

TB_OPT_STEP_IMPL = 1
TB_STEP_AUTO = 0
TB_STEP_REG = 1
TB_STEP_BULK = 2
TB_STEP_REGPF = 3
TB_STEP_LEAN = 4
TB_STEP_PAIR = 5
TB_STEP_BULK1 = 6
TB_OPT_STEP_SPW = 2

TB_MODE_POLLING = 0
TB_MODE_HOSTTASK = 1
TB_MODE_FENCE = 2

TB_COMPLETION_EVENTS = 0
TB_COMPLETION_WORDS = 1

TB_PROBE_DADD = 0
TB_PROBE_DMUL = 1
TB_PROBE_DFMA = 2
TB_PROBE_DMUL_DADD = 3

TB_OP_NONE = 0
TB_OP_KIND = 1
TB_OP_AFFINE = 2
TB_OP_TRAP = 3          # fault injection: the kernel traps
TB_GATHER_MAX = 256

ABI_VERSION = 1


class NativeUnavailable(TaskBridgeError):
    """libtb.so is missing or cannot be loaded (no CPU fallback exists)."""


class CudaError(TaskBridgeError):
    """A libtb call failed; ``rc`` is the negative return code."""

    def __init__(self, rc: int, what: str):
        self.rc = rc
        super().__init__(f"{what} failed: rc={rc} ({error_string(rc)})")


_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_szt = ctypes.c_size_t
_pu64 = ctypes.POINTER(ctypes.c_uint64)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pint = ctypes.POINTER(ctypes.c_int)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pu8 = ctypes.POINTER(ctypes.c_uint8)
_pvp = ctypes.POINTER(ctypes.c_void_p)

# name -> argtypes (restype is int unless noted); "blocking" calls may wait.
SIGNATURES = {
    "tb_abi_version": [],
    "tb_error_string": [_int],
    "tb_init": [_int],
    "tb_device_count": [_pint],
    "tb_sm_count": [_int, _pint],
    "tb_device_sync": [],
    "tb_set_option": [_int, _int],
    "tb_stream_create": [_pu64],
    "tb_stream_destroy": [_u64],
    "tb_stream_query": [_u64],
    "tb_stream_sync": [_u64],
    "tb_event_record": [_u64, _pu64],
    "tb_event_query": [_u64],
    "tb_event_wait": [_u64],
    "tb_event_release": [_u64],
    "tb_tevent_record": [_u64, _pu64],
    "tb_tevent_elapsed": [_u64, _u64, ctypes.POINTER(ctypes.c_double)],
    "tb_tevent_release": [_u64],
    "tb_stream_wait_event": [_u64, _u64],
    "tb_event_pool_set": [_int],
    "tb_event_pool_stats": [_pi64, _pi64, _pi64],
    "tb_malloc": [_pvp, _szt],
    "tb_free": [_vp],
    "tb_host_alloc": [_pvp, _szt],
    "tb_host_free": [_vp],
    "tb_memcpy_h2d": [_u64, _vp, _vp, _szt],
    "tb_memcpy_d2h": [_u64, _vp, _vp, _szt],
    "tb_memcpy_d2d": [_u64, _vp, _vp, _szt],
    "tb_memset": [_u64, _vp, _int, _szt],
    "tb_transform": [_u64, _int, _vp, _i64],
    "tb_launch": [_u64, _int, _int, _dbl, _dbl, _vp, _i64],
    "tb_barrier": [_u64],
    "tb_spin": [_u64, _i64],
    "tb_init_cells": [_u64, _vp, _i64, _i64, _i64],
    "tb_agg_launch": [_u64, _int, _int, _dbl, _dbl, _vp, _vp, _szt, _int, _pu64],
    "tb_step": [_u64, _vp, _vp, _i64, _vp, _vp, _int, _int, _vp, _vp, _vp],
    "tb_step_final": [_u64, _vp, _vp, _i64, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp, _vp,
                      _vp],
    "tb_step_deferred": [_u64, _vp, _vp, _i64, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp, _vp,
                         _vp, _vp, _vp],
    "tb_step_close": [_u64, _vp, _vp, _i64, _vp, _vp, _vp, _vp],
    "tb_acc_reset": [_u64, _vp],
    "tb_acc_add": [_u64, _vp, _i64, _vp],
    "tb_acc_finalize": [_u64, _vp, _vp, _vp, _vp, _int],
    "tb_poll_create": [_pu64],
    "tb_poll_destroy": [_u64],
    "tb_poll_add": [_u64, _u64, _u64, _u64],
    "tb_poll_add_seq": [_u64, _u64, _u64, _u64, _u64],
    "tb_poll": [_u64, _pu64, _pi32, _int, _pint],
    "tb_poll_pending": [_u64, _pi64],
    "tb_poll_drain": [_u64, _pu64, _pu8, _int, _pint],
    "tb_poll_entry_high_water": [_u64, _pint],
    "tb_htq_create": [_int, _pu64],
    "tb_host_task": [_u64, _u64, _u64],
    "tb_htq_next": [_u64, _pu64, _pint, _i64],
    "tb_htq_close": [_u64],
    "tb_htq_destroy": [_u64],
    "tb_machine_run": [_vp, _vp, _vp, _vp],
    "tb_machine_run_cells": [_vp, _vp, _vp, _vp, _vp],
    "tb_launch_gather": [_u64, _int, _int, _dbl, _dbl, _vp, _vp, _vp, _int],
    "tb_launch_gather_edge": [_u64, _int, _vp, _vp, _vp, _vp, _vp, _int, _vp, _vp, _vp, _i64,
                              _vp],
    "tb_launch_gather_done": [_u64, _int, _int, _dbl, _dbl, _vp, _vp, _vp, _int, _vp],
    "tb_agg_launch_hydro": [_u64, _vp, _vp, _i64, _vp, _vp, _dbl, _dbl, _pu64],
    "tb_machine_run_hydro": [_vp, _vp, _vp, _dbl, _dbl, _vp],
    "tb_ipc_get_handle": [_vp, _vp, _pu64],
    "tb_ipc_open_handle": [_vp, _pvp],
    "tb_ipc_close": [_vp],
    "tb_acc_allreduce_p2p": [_u64, _vp, _vp, _int, _vp, _vp, _vp, _vp],
    "tb_acc_allreduce_p2p_ex": [_u64, _vp, _vp, _int, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                                _vp],
    "tb_hydro_flux": [_u64, _vp, _vp, _vp, _i64, _dbl, _dbl],
    "tb_fp64_probe": [_int, _i64, _vp, _vp],
    "tb_divsqrt_fast": [_u64, _vp, _vp, _i64, _vp, _vp, _vp],
    "tb_hydro_flux_lattice": [_u64, _vp, _i64, _i64, _vp, _vp, _dbl, _dbl],
    "tb_hydro_stamps": [_vp, _int],
    "tb_star_pad": [_u64, _vp, _i64, _vp],
    "tb_star_pad_slab": [_u64, _vp, _i64, _i64, _vp, _vp, _vp],
    "tb_star_cfl": [_u64, _vp, _i64, _dbl, _dbl, _vp],
    "tb_star_stage": [_u64, _int, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp],
    "tb_fmm_workspace_bytes": [_int, _pu64],
    "tb_fmm_upward": [_u64, _int, _vp, _vp],
    "tb_fmm_m2l": [_u64, _int, _vp],
    "tb_fmm_downward": [_u64, _int, _vp],
    "tb_fmm_leaf": [_u64, _int, _vp, _vp, _vp],
    "tb_fmm_solve": [_u64, _int, _vp, _vp, _vp],
    "tb_fmm_slab_workspace_bytes": [_int, _int, _pu64],
    "tb_fmm_slab_layout": [_int, _int, _int, _int, _pu64],
    "tb_fmm_slab_upward": [_u64, _int, _int, _int, _vp, _vp],
    "tb_fmm_slab_coarse": [_u64, _int, _int, _int, _vp],
    "tb_fmm_slab_m2l": [_u64, _int, _int, _int, _vp],
    "tb_fmm_slab_downward": [_u64, _int, _int, _int, _vp],
    "tb_fmm_slab_leaf": [_u64, _int, _int, _int, _vp, _int, _int, _vp, _vp],
}
BLOCKING = {"tb_init", "tb_device_sync", "tb_stream_sync", "tb_event_wait",
            "tb_htq_next", "tb_htq_destroy", "tb_malloc", "tb_free",
            "tb_host_alloc", "tb_host_free", "tb_stream_destroy",
            "tb_memcpy_h2d", "tb_memcpy_d2h", "tb_poll_drain", "tb_machine_run", "tb_machine_run_cells",
            "tb_machine_run_hydro",
            "tb_fp64_probe"}

_lock = threading.Lock()
_libs = None


def _configure(lib):
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_char_p if name == "tb_error_string" else _int
    return lib


def _load():
    global _libs
    with _lock:
        if _libs is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} is not built; run `python -m paper_2303_08058_b200.build` "
                    "(there is no CPU fallback)")
            try:
                blocking = _configure(ctypes.CDLL(LIB_PATH))
                fast = _configure(ctypes.PyDLL(LIB_PATH))
            except OSError as e:  # pragma: no cover - load failure path
                raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
            if fast.tb_abi_version() != ABI_VERSION:
                raise NativeUnavailable("libtb ABI version mismatch; rebuild")
            _libs = (fast, blocking)
    return _libs


def fast():
    libs = _libs
    return libs[0] if libs is not None else _load()[0]


def blocking():
    libs = _libs
    return libs[1] if libs is not None else _load()[1]


def call(name: str, *args) -> int:
    """Call ``name``; raise CudaError on a negative return code."""
    lib = blocking() if name in BLOCKING else fast()
    rc = getattr(lib, name)(*args)
    if rc < 0:
        raise CudaError(rc, name)
    return rc


def error_string(rc: int) -> str:
    try:
        return fast().tb_error_string(rc).decode()
    except NativeUnavailable:
        return "libtb unavailable"


def exported_symbols():
    return list(SIGNATURES)


_initialised = {}


def init(device: int = 0) -> None:
    """Bind libtb to ``device`` (idempotent per device)."""
    if _initialised.get("device") == device:
        return
    call("tb_init", device)
    _initialised["device"] = device


def device_count() -> int:
    n = ctypes.c_int(0)
    call("tb_device_count", ctypes.byref(n))
    return n.value


def sm_count(device: int = 0) -> int:
    n = ctypes.c_int(0)
    call("tb_sm_count", device, ctypes.byref(n))
    return n.value


__all__ = ["NativeUnavailable", "CudaError", "DeviceGoneError", "call", "fast",
           "blocking", "init"]

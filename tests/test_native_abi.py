"""libtb.so loads without a GPU and exports every symbol include/tb.h declares
(no compute calls here: CPU-only checks)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2303_08058_b200 import _native as N
from paper_2303_08058_b200.build import LIB, build

HEADER = os.path.join(ROOT, "include", "tb.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(tb_\w+)\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_binding_table():
    assert declared_symbols() == sorted(N.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing


def test_abi_version_and_constants(lib):
    assert N.fast().tb_abi_version() == N.ABI_VERSION
    text = open(HEADER).read()
    for name in ("TB_CELLS", "TB_FACE", "TB_KINDS", "TB_ACC_LIMBS", "TB_ACC_BIAS",
                 "TB_ACC_MIN_WORD", "TB_ACC_COUNT_WORD", "TB_ACC_WORDS", "TB_OPT_STEP_IMPL",
                 "TB_STEP_AUTO", "TB_STEP_REG", "TB_STEP_BULK", "TB_STEP_REGPF", "TB_STEP_LEAN", "TB_STEP_PAIR", "TB_STEP_BULK1", "TB_OPT_STEP_SPW", "TB_OP_NONE", "TB_OP_KIND",
                 "TB_OP_AFFINE", "TB_OK", "TB_NOT_READY", "TB_MODE_POLLING", "TB_MODE_HOSTTASK",
                 "TB_MODE_FENCE", "TB_IPC_HANDLE_BYTES", "TB_COMPLETION_EVENTS",
                 "TB_COMPLETION_WORDS"):
        m = re.search(rf"#define {name} \(?(-?\d+)\)?", text)
        assert m and int(m.group(1)) == getattr(N, name), name


def test_error_strings(lib):
    assert N.error_string(0) == "ok"
    assert N.error_string(N.TB_E_INVALID) == "invalid argument"
    assert N.error_string(N.TB_E_CLOSED) == "closed"


def test_argument_validation_without_gpu(lib):
    f = N.fast()
    assert f.tb_step(0, None, None, 4, None, None, 3, 5, None, None, None) == N.TB_E_INVALID
    assert f.tb_transform(0, 7, None, 4) == N.TB_E_INVALID
    assert f.tb_init_cells(0, None, 4, 0, 4) == N.TB_E_INVALID
    assert f.tb_acc_finalize(0, None, None, None, None, 1) == N.TB_E_INVALID


def test_poll_registry_lifecycle_without_gpu(lib):
    f = N.fast()
    h = ctypes.c_uint64(0)
    assert f.tb_poll_create(ctypes.byref(h)) == 0
    n = ctypes.c_int64(-1)
    assert f.tb_poll_pending(h.value, ctypes.byref(n)) == 0 and n.value == 0
    fired = (ctypes.c_uint64 * 4)()
    k = ctypes.c_int(-1)
    assert f.tb_poll(h.value, fired, None, 4, ctypes.byref(k)) == 0 and k.value == 0
    hw = ctypes.c_int(0)
    assert f.tb_poll_entry_high_water(h.value, ctypes.byref(hw)) == 0 and hw.value == 1
    assert f.tb_poll_destroy(h.value) == 0


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2303_08058_b200 import CudaDevice
    with pytest.raises(N.CudaError):
        CudaDevice()


def test_machine_struct_layout_matches_header():
    from paper_2303_08058_b200.native_machine import MachineConfig, MachineStep
    text = open(HEADER).read()
    cfg = re.search(r"typedef struct \{(.*?)\} tb_machine_config;", text, re.S).group(1)
    fields = re.findall(r"int64_t (\w+);", cfg)
    assert fields == [f for f, _ in MachineConfig._fields_]
    assert ctypes.sizeof(MachineStep) == 3 * 8 + 6 * 8


def test_machine_rejects_bad_config_without_gpu():
    from paper_2303_08058_b200.native_machine import MachineConfig
    cfg = MachineConfig(0, 1, 3, 5, 1, 1, 1, 0, 1, 0, 1, 2)     # subgrids = 0
    cs = ctypes.c_double()
    assert N.fast().tb_machine_run(ctypes.addressof(cfg), ctypes.addressof(cs), None,
                                   None) == N.TB_E_INVALID

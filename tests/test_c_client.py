"""The C-ABI from plain C (no Python in the consumer): tests/c/ring_client.c
compiles against include/tb.h with a C99 compiler and links libtb.so (CPU);
on the GPU it reproduces GOLDEN_4X2 bit for bit, polls events and runs one
aggregation batch (see the program's header)."""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT
from paper_2303_08058_b200.build import LIB, build

SRC = os.path.join(ROOT, "tests", "c", "ring_client.c")


def compile_client(out_dir):
    cc = shutil.which("cc") or shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    build()
    exe = os.path.join(out_dir, "ring_client")
    libdir = os.path.dirname(LIB)
    cmd = [cc, "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-ffp-contract=off",
           "-I", os.path.join(ROOT, "include"), SRC, "-L", libdir, "-ltb",
           f"-Wl,-rpath,{libdir}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_client_compiles_and_links(tmp_path):
    assert os.path.exists(compile_client(str(tmp_path)))


@pytest.mark.gpu
def test_c_client_runs_golden(tmp_path):
    exe = compile_client(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("OK")

"""The C ABI from plain C (tests/c/abi_roundtrip.c): include/kvc.h compiles
as C99 with -Wall -Wextra and links against libkvc.so + the CUDA runtime only
(CPU); the program's encode / decode round trips, determinism, truncation and
bad-id checks pass on the B200 (GPU)."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2605_13734_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    if shutil.which("gcc") is None or not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime.h")):
        pytest.skip("gcc or the CUDA headers are not available")
    if not os.path.exists(os.path.join(LIBDIR, "libkvc.so")):
        pytest.skip("libkvc.so not built")
    exe = str(tmp_path / "abi_roundtrip")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-O2", "-o", exe,
           os.path.join(ROOT, "tests", "c", "abi_roundtrip.c"), "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(CUDA, "include"), "-L" + LIBDIR, "-L" + os.path.join(CUDA, "lib64"),
           "-lkvc", "-lcudart", "-lm", "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_header_compiles_as_c99_and_links(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_program_round_trips(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi ok" in r.stdout, r.stdout

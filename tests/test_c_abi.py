"""The header is plain C: a C99 program compiled with gcc against
include/fgb200.h and linked to libfgb200.so calls the host-only entry points
(no GPU needed) and checks the reference's values and error codes."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1704_05231_b200", "lib")


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_c99_program_against_the_header(tmp_path):
    exe = str(tmp_path / "abi_host")
    cc = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                         os.path.join(ROOT, "tests", "c", "abi_host.c"), "-L", LIB, "-lfgb200",
                         "-Wl,-rpath," + LIB, "-lm", "-o", exe], capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "abi_host ok" in r.stdout

"""The C++ drop-in header (include/rcp_b200/rcp.hpp) compiles against the C ABI
(CPU) and, on a GPU, a reference-style program decomposes through it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp")
LIBDIR = os.path.join(ROOT, "paper_1703_09074_b200")


def build(tmp_path):
    exe = tmp_path / "dropin"
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lrcpg", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def test_dropin_header_compiles_and_links(rcp, tmp_path):
    assert build(tmp_path).exists()


@pytest.mark.gpu
def test_dropin_program_runs(rcp, tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "converged=1" in out.stdout and "compressed 13x13x13" in out.stdout

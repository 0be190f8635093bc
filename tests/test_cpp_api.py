"""The C++ host mirror (include/mixedstep_b200.hpp) compiles against the C-ABI
library (CPU) and passes the reference KATs on the device (GPU)."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIBDIR = ROOT / "paper_2605_23727_b200"


def _build(tmp_path):
    exe = tmp_path / "test_cpp_api"
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "test_cpp_api.cpp"), "-L", str(LIBDIR), "-lmixedstep_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def test_cpp_header_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_api_on_device(gpu, tmp_path):
    r = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpp api ok" in r.stdout

"""The C++ lsr:: API (include/lsr/*.hpp) compiles like the reference's
headers and its sl_step runs on the GPU (tests/cpp/test_api.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT


def _build(tmp_path):
    exe = str(tmp_path / "test_api")
    lib_dir = os.path.join(ROOT, "paper_2410_22205_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-L", lib_dir, "-llsr_b200",
                    f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    return exe


def test_cpp_api_compiles_and_links(built, tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_runs_on_gpu(gpu, tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout

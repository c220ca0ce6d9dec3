"""INTEGRATION.md Options A and B as written: the reference's own translation
units compiled against include/ (whose lsr/*.hpp shadow the reference
headers with a superset, include/lsr/lsr_b200.hpp) and linked with
liblsr_b200.so in place of the units it replaces (oracle/Makefile target
`integration`), driving the reference's own run_schedule
(driver.cpp:139-230) via tests/cpp/run_schedule_main.cpp.

  Option A: minus evolve.cpp                          (sl_step on the GPU)
  Option B: minus evolve.cpp, grid.cpp, distance.cpp, reinit.cpp
            (band, clamp, distance field, reinitialisation on the GPU too)
  Option C: all reference units and headers + include/lsr_cuda.h, the
            snippet's lsr_cuda_sl_step_host call beside lsr::sl_step
            (tests/cpp/capi_snippet_main.cpp)

CPU tests: all three programs build and link, and liblsr_b200.so defines
every external lsr:: symbol the replaced reference units define. GPU test:
the three programs produce byte-identical output (every run's final phi,
E_2, Err_S and the per-iteration log)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

REF_DIR = os.path.join(ROOT, "oracle", "_ref")
EXES = {k: os.path.join(REF_DIR, f"run_schedule_{k}") for k in ("ref", "optA", "optB")}
LIB = os.path.join(ROOT, "paper_2410_22205_b200", "liblsr_b200.so")


def _need_builds():
    if not all(os.path.exists(p) for p in EXES.values()):
        pytest.skip("integration programs not built (no reference tree on this machine)")


def _defined(path, dynamic=False):
    """External lsr:: functions a file defines (demangled, namespace lsr
    only, not lsr::ref:: nor anonymous namespaces; an object file's weak
    inline instantiations do not count)."""
    args = ["nm", "-C", "--defined-only"] + (["-D"] if dynamic else []) + [path]
    out = subprocess.run(args, capture_output=True, text=True, check=True).stdout
    syms = set()
    for line in out.splitlines():
        parts = line.split(" ", 2)
        if len(parts) == 3 and parts[1] in (("T", "W") if dynamic else ("T",)) and parts[2].startswith("lsr::") \
                and not parts[2].startswith("lsr::ref::") and "(anonymous namespace)" not in parts[2]:
            syms.add(re.sub(r"\s+", " ", parts[2]))
    return syms


def test_integration_programs_build_and_link(built):
    _need_builds()
    for k in ("optA", "optB"):
        r = subprocess.run(["ldd", EXES[k]], capture_output=True, text=True, check=True)
        assert "liblsr_b200.so" in r.stdout and "not found" not in r.stdout, r.stdout


@pytest.mark.parametrize("unit", ["evolve", "grid", "distance", "reinit"])
def test_library_replaces_reference_unit(built, unit):
    """Every external lsr:: function of the reference unit is exported by
    liblsr_b200.so with the same signature."""
    obj = os.path.join(REF_DIR, "obj", f"{unit}.o")
    if not os.path.exists(obj):
        pytest.skip("reference objects not built")
    need = {s for s in _defined(obj) if not s.startswith("lsr::(anonymous")}
    have = _defined(LIB, dynamic=True)
    assert need, unit
    assert need <= have, sorted(need - have)


@pytest.mark.gpu
def test_run_schedule_bit_identical_in_all_builds(gpu, tmp_path):
    _need_builds()
    out = {}
    for k, exe in EXES.items():
        dst = tmp_path / f"{k}.bin"
        r = subprocess.run([exe, str(dst)], capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, (k, r.stdout, r.stderr)
        out[k] = dst.read_bytes()
    assert len(out["ref"]) > 1_000_000
    assert out["optA"] == out["ref"]
    assert out["optB"] == out["ref"]


@pytest.mark.gpu
def test_option_c_snippet_matches_reference_sl_step(gpu):
    """INTEGRATION.md Option C (the C-ABI call in place of lsr::sl_step,
    compiled against the reference's own headers) writes the same bytes into
    `next` as the reference's lsr::sl_step: 2d and 3d, Q1 and WENO, (p, delta)
    in {(1, 0), (2, 1), (2, 1/2)}, including a 72^3 grid that takes the
    pipelined one-shot path."""
    exe = os.path.join(REF_DIR, "capi_snippet")
    if not os.path.exists(exe):
        pytest.skip("integration programs not built (no reference tree on this machine)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (r.stdout, r.stderr)
    assert r.stdout.count(" 0 differ") == 5, r.stdout

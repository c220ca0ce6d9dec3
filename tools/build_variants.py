"""Build experimental variants of the CUDA library with different launch
bounds (-D LSR_SL_THREADS / LSR_SL_MIN_BLOCKS) into build/variants/, for
side-by-side timing on the GPU (tools/microbench.py with LSR_B200_LIB=...)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as ge  # noqa: E402


def build(name, defines):
    out = os.path.join(ge.ROOT, "build", "variants", f"lib_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = [os.path.join(ge.CSRC, s) for s in ge.CU_SOURCES + ge.CPP_SOURCES]
    cmd = [ge.NVCC, *ge.NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ge.ROOT, "include"), "-I",
           ge.CSRC, "-shared", "-o", out, *srcs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-3000:])
        raise SystemExit(1)
    regs = [l for l in r.stderr.splitlines() if "Used" in l]
    print(name, out)
    return out


if __name__ == "__main__":
    for spec in sys.argv[1:]:  # e.g. t128b3=LSR_SL_THREADS=128,LSR_SL_MIN_BLOCKS=3
        name, d = spec.split("=", 1)
        build(name, d.split(",") if d else [])

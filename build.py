"""Build the in-tree CUDA library paper_2103_14990_b200/libdlmpc.so (sm_100a).

    python build.py            # incremental: rebuild when a source is newer
    python build.py --force

nvcc cross-compiles without a GPU. The .so is git-ignored but travels to the
GPU box with the repo snapshot.
"""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2103_14990_b200")
SRC_DIR = os.path.join(PKG, "csrc")
SOURCES = [os.path.join(SRC_DIR, "dlmpc.cu")]
DEPS = SOURCES + [os.path.join(SRC_DIR, "dlmpc_device.cuh"), os.path.join(SRC_DIR, "dlmpc_schedules.cuh"),
        os.path.join(ROOT, "include", "dlmpc.h")]
OUT = os.path.join(PKG, "libdlmpc.so")
# bounds-checked variant (-DDLMPC_CHECKED): the pool has no compute-sanitizer,
# so the tests run the kernels once more with every risky access checked
OUT_CHECKED = os.path.join(PKG, "libdlmpc_checked.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build(out=OUT):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force=False, verbose=False, checked=False):
    out = OUT_CHECKED if checked else OUT
    if not force and not needs_build(out):
        return out
    cmd = [nvcc()] + NVCC_FLAGS + (["-DDLMPC_CHECKED"] if checked else []) + ["-o", out] + SOURCES
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed: " + " ".join(cmd))
    if verbose:
        for line in (res.stdout + res.stderr).splitlines():
            if "registers" in line or "spill" in line or "error" in line:
                print(line)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))

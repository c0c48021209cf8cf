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
SOURCES = [os.path.join(SRC_DIR, "dlmpc.cu"), os.path.join(SRC_DIR, "dlmpc_multi.cu")]
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
    """Compile the translation units in parallel (one nvcc per source, -c),
    then link the shared library."""
    from concurrent.futures import ThreadPoolExecutor
    out = OUT_CHECKED if checked else OUT
    if not force and not needs_build(out):
        return out
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-DDLMPC_CHECKED"] if checked else [])
    obj_dir = os.path.join(ROOT, "build", "checked" if checked else "release")
    os.makedirs(obj_dir, exist_ok=True)
    objs = [os.path.join(obj_dir, os.path.basename(src) + ".o") for src in SOURCES]

    def compile_one(src, obj):
        cmd = [nvcc()] + flags + ["-c", "-o", obj, src]
        return cmd, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as pool:
        results = list(pool.map(lambda so: compile_one(*so), zip(SOURCES, objs)))
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out] + objs
    for cmd, res in results + [(link, subprocess.run(link, capture_output=True, text=True))]:
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

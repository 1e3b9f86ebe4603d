"""Build libsage2.so (the product) and libsage2_dev.so (-DSAGE2_DEV: + measurement entry points of
include/sage2_dev.h) in-tree with nvcc for sm_100a (no JIT cache; the .so files travel with the repo).

    python -m paper_2411_10958_b200.build [--force] [--verbose] [--dev]
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsage2.so")
DEV_LIB = os.path.join(HERE, "libsage2_dev.so")
SOURCES = ["sage2_api.cu"]
DEPS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    # never --use_fast_math: the quantizers must use IEEE division / RNE (C-2)
]


def needs_build(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", h)
                                                    for h in ("sage2.h", "sage2_dev.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False, out=None, defines=(), dev=False):
    """dev=True builds libsage2_dev.so.  out/defines: A/B builds for experiments (e.g.
    out=libsage2_x.so, defines=["SAGE2_KSTAGES=4"])."""
    if dev:
        defines = tuple(defines) + ("SAGE2_DEV",)
    lib = out or (DEV_LIB if dev else LIB)
    if out is None and not force and not needs_build(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC] + FLAGS + [f"-D{x}" for x in defines] + ["-I", os.path.join(ROOT, "include"), "-o", tmp] + \
        [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode:
        raise RuntimeError(f"nvcc failed building {os.path.basename(lib)}")
    os.replace(tmp, lib)
    return lib


def build_all(force=False, verbose=False):
    """Both libraries, compiled in parallel."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(2) as ex:
        fs = [ex.submit(build, force, verbose, None, (), d) for d in (False, True)]
        return [f.result() for f in fs]


if __name__ == "__main__":
    if "--dev" in sys.argv:
        print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, dev=True))
    else:
        print("\n".join(build_all(force="--force" in sys.argv, verbose="--verbose" in sys.argv)))

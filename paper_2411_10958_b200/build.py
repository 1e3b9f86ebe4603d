"""Build libsage2.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo).

    python -m paper_2411_10958_b200.build [--force] [--verbose]
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsage2.so")
SOURCES = ["sage2_api.cu"]
DEPS = ["sage2_api.cu", "attn.cuh", "attn2.cuh", "attn4.cuh", "attn5.cuh", "attn6.cuh", "attn8.cuh", "attn10.cuh", "dsg.cuh", "prep.cuh", "probe.cuh", "ptx.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    # never --use_fast_math: the quantizers must use IEEE division / RNE (C-2)
]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "sage2.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False, out=None, defines=()):
    """out/defines: A/B builds for experiments (e.g. out=libsage2_x.so, defines=["SAGE2_WAIT_CLOOP"])."""
    lib = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC] + FLAGS + [f"-D{x}" for x in defines] + ["-I", os.path.join(ROOT, "include"), "-o", tmp] + \
        [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode:
        raise RuntimeError("nvcc failed building libsage2.so")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)

"""The C-ABI library loads on a CPU-only box and exports every symbol include/sage2.h declares
(no compute calls: those need a B200)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="sage2.h"):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sage2_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("sage2_attn", "sage2_attn_ws", "sage2_workspace_bytes", "sage2_prepare", "sage2_attention",
              "sage2_debug_qk_int32", "sage2_strerror", "sage2_version", "sage2_attn_host"):
        assert s in syms


def test_library_builds_loads_and_exports_all_symbols():
    from paper_2411_10958_b200 import build
    path = build.build()
    L = ctypes.CDLL(path)
    for s in declared_symbols():
        assert hasattr(L, s), s
    L.sage2_version.restype = ctypes.c_int
    assert L.sage2_version() >= 1
    L.sage2_strerror.restype = ctypes.c_char_p
    assert b"sm_100" in L.sage2_strerror(-2)
    L.sage2_workspace_bytes.restype = ctypes.c_size_t
    assert L.sage2_workspace_bytes(1, 1, 1, 256, 64, 0) > 0
    assert L.sage2_workspace_bytes(1, 1, 1, 256, 96, 0) == 0          # d = 96 invalid
    assert L.sage2_workspace_bytes(2, 40000, 40000, 256, 64, 0) == 0  # B * H_q > 65535 invalid
    # the product library carries no measurement entry points
    for s in declared_symbols("sage2_dev.h"):
        assert not hasattr(L, s), f"{s} must live in libsage2_dev.so only"


def test_dev_library_exports_the_dev_header():
    from paper_2411_10958_b200 import build
    L = ctypes.CDLL(build.build(dev=True))
    for s in declared_symbols() + declared_symbols("sage2_dev.h"):
        assert hasattr(L, s), s


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2411_10958_b200 import sage2
    q = torch.zeros((1, 1, 128, 64), dtype=torch.float16)
    try:
        sage2.attn(q, q, q)
    except (ValueError, sage2.Sage2Error):
        return
    raise AssertionError("attn on CPU tensors must raise (no CPU fallback)")


def test_default_kernel_dispatch_rule():
    """Host-only query of the kernel sage2_attention runs (include/sage2.h sage2_attention_kernel):
    v12 for d = 64 non-causal, v8 otherwise (d = 128, causal, the carrier / granularity / single-level
    variants)."""
    from paper_2411_10958_b200 import sage2
    ak = sage2.attention_kernel
    assert ak(4096, 128) == 8 and ak(8192, 128) == 8 and ak(200, 128) == 8
    assert ak(8193, 128) == 8 and ak(32768, 128) == 8 and ak(4096, 64, kernel="one") == 8
    assert ak(4096, 128, causal=True) == 8 and ak(4096, 64) == 12 and ak(100000, 64) == 12
    assert ak(4096, 64, causal=True) == 8 and ak(4096, 64, qk_e4m3=True) == 8
    assert ak(4096, 64, kernel="v8") == 8 and ak(4096, 64, kernel="v12") == 12
    assert ak(4096, 128, qk_e4m3=True) == 8 and ak(4096, 128, gran="block") == 8
    assert ak(1024, 128, kernel="v8") == 8
    # the experimental v14 runs only when selected (csrc/attn14.cuh)
    assert ak(4096, 128, kernel="v14") == 14 and ak(4096, 64, kernel="v14") == 14

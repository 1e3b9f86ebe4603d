"""Thin ctypes binding over libsage2.so (include/sage2.h).  Argument marshalling only: every step
of the SageAttention2 forward runs in the library's CUDA kernels.  PyTorch is used only for device
memory and streams.  There is no CPU fallback: if libsage2.so is missing or the GPU is not sm_100,
these functions raise.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SAGE2_LIB overrides the path for A/B experiments (scripts/); the default is the in-tree build.
LIB_PATH = os.environ.get("SAGE2_LIB") or os.path.join(_HERE, "libsage2.so")
# measurement-only library (include/sage2_dev.h): phase traces, probes, microbenchmarks
DEV_LIB_PATH = os.environ.get("SAGE2_DEV_LIB") or os.path.join(_HERE, "libsage2_dev.so")

F_CAUSAL = 1
F_INT8 = 2
WS_NREGIONS = 15
REGIONS = ("ksum", "vmax", "vsum", "kbar", "dv", "vmean", "qhat", "dq", "qbar", "khat", "dk", "vhat", "qbt", "ds", "end")

_lib = None
_dev = None


class Sage2Error(RuntimeError):
    pass


def _declare(L):
    P, I, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.sage2_version.restype = I
    L.sage2_strerror.restype = ctypes.c_char_p
    L.sage2_strerror.argtypes = [I]
    L.sage2_last_cuda_error.restype = ctypes.c_char_p
    L.sage2_workspace_bytes.restype = S
    L.sage2_workspace_bytes.argtypes = [I] * 6
    L.sage2_attn.argtypes = [P, P, P, P] + [I] * 6 + [P]
    L.sage2_attn_ws.argtypes = [P, P, P, P] + [I] * 6 + [P, S, P]
    L.sage2_attn_ex.argtypes = [P, P, P, P] + [I] * 6 + [P, S, P]
    L.sage2_workspace_layout.argtypes = [I] * 5 + [ctypes.POINTER(S)]
    L.sage2_prepare.argtypes = [P, P, P] + [I] * 6 + [P, S, P]
    L.sage2_attention.argtypes = [P] + [I] * 6 + [P, S, P]
    L.sage2_debug_qk_int32.argtypes = [P, P, P] + [I] * 6 + [P, S, P]
    L.sage2_attn_host.argtypes = [P, P, P, P] + [I] * 6 + [P]
    L.sage2_attention_kernel.argtypes = [I, I, I]
    L.sage2_attention_kernel.restype = I
    L.sage2_release_memory.argtypes = []
    for n in ("sage2_attn", "sage2_attn_ws", "sage2_attn_ex", "sage2_workspace_layout", "sage2_prepare",
              "sage2_attention", "sage2_debug_qk_int32", "sage2_attn_host", "sage2_release_memory"):
        getattr(L, n).restype = I
    return L


def lib():
    """Load libsage2.so (built in-tree by paper_2411_10958_b200.build).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise Sage2Error(f"{LIB_PATH} is missing: run `python -m paper_2411_10958_b200.build` "
                             "(there is no CPU fallback)")
        _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


def dev_lib():
    """Load libsage2_dev.so (measurement entry points, include/sage2_dev.h).  Raises if absent."""
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB_PATH):
            raise Sage2Error(f"{DEV_LIB_PATH} is missing: run `python -m paper_2411_10958_b200.build`")
        L = _declare(ctypes.CDLL(DEV_LIB_PATH))
        P, I = ctypes.c_void_p, ctypes.c_int
        L.sage2_dev_trace.argtypes = [P, P] + [I] * 6 + [P, ctypes.c_size_t, P]
        L.sage2_probe_accumulator.argtypes = [P, P, I, P, P]
        L.sage2_bench_mma.argtypes = [I, I, ctypes.POINTER(ctypes.c_double)]
        L.sage2_microbench.argtypes = [I, I, ctypes.POINTER(ctypes.c_double)]
        for n in ("sage2_dev_trace", "sage2_probe_accumulator", "sage2_bench_mma", "sage2_microbench"):
            getattr(L, n).restype = I
        _dev = L
    return _dev


def _lib_for(kernel):
    """The experimental v14 kernel lives in the dev library only (include/sage2_dev.h)."""
    return dev_lib() if kernel == "v14" else lib()


def _check(rc, L=None):
    if rc != 0:
        L = L or lib()
        msg = L.sage2_strerror(rc).decode()
        if rc == -4:
            msg += ": " + L.sage2_last_cuda_error().decode()
        raise Sage2Error(f"libsage2 error {rc}: {msg}")


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _shape(q, k):
    B, Hq, N, d = q.shape
    Hkv = k.shape[1]
    return B, Hq, Hkv, N, d


def _check_inputs(q, k, v):
    for t in (q, k, v):
        if t.dtype != torch.float16 or not t.is_cuda or not t.is_contiguous() or t.dim() != 4:
            raise ValueError("q, k, v must be contiguous fp16 CUDA tensors [B, H, N, d]")
    if k.shape != v.shape or q.shape[0] != k.shape[0] or q.shape[2:] != k.shape[2:]:
        raise ValueError("shape mismatch: q [B,Hq,N,d], k/v [B,Hkv,N,d]")


F_QK_E4M3 = 2048    # include/sage2.h SAGE2_F_QK_E4M3 (E4M3-carrier QK^T variant)
F_SMOOTH_V = 32768  # include/sage2.h SAGE2_F_SMOOTH_V (optional smooth V)
F_GRAN = {"thread": 0, "block": 262144, "token": 524288, "tensor": 2097152}   # SAGE2_F_GRAN_* (NEXT#4 ablation)


def flags(causal=False, int8=False, qk_e4m3=False, smooth_v=False, gran="thread"):
    return ((F_CAUSAL if causal else 0) | (F_INT8 if int8 else 0) | (F_QK_E4M3 if qk_e4m3 else 0) |
            (F_SMOOTH_V if smooth_v else 0) | F_GRAN[gran])


def workspace_bytes(B, Hq, Hkv, N, d, causal=False):
    """Workspace size; causal=True sizes Delta S in the triangular causal layout (half the bytes) --
    such a workspace only serves causal prepare/attention calls.  The non-causal size serves both."""
    return int(lib().sage2_workspace_bytes(B, Hq, Hkv, N, d, int(causal)))


def layout(B, Hq, Hkv, N, d):
    offs = (ctypes.c_size_t * WS_NREGIONS)()
    _check(lib().sage2_workspace_layout(B, Hq, Hkv, N, d, offs))
    return dict(zip(REGIONS, [int(o) for o in offs]))


def alloc_workspace(B, Hq, Hkv, N, d, device="cuda", causal=False):
    return torch.empty(workspace_bytes(B, Hq, Hkv, N, d, causal), dtype=torch.uint8, device=device)


def attn(q, k, v, causal=False, int8=False, out=None, workspace=None, qk_e4m3=False, smooth_v=False,
         gran="thread", kernel="default"):
    """SageAttn2 forward: q [B,Hq,N,d], k/v [B,Hkv,N,d] fp16 CUDA -> out [B,Hq,N,d] fp16.
    qk_e4m3=True runs QK^T through the E4M3 carrier (kind::f8f6f4) instead of kind::i8;
    smooth_v=True subtracts V's column mean before the FP8 quantization and adds it back;
    gran="block"/"token" selects the granularity-ablation quantization groups (d = 128 only);
    kernel forces an attention kernel / the single-level ablation ("v8", "v12", "v14", "one")."""
    _check_inputs(q, k, v)
    B, Hq, Hkv, N, d = _shape(q, k)
    if out is None:
        out = torch.empty_like(q)
    if workspace is None and not int8 and not qk_e4m3 and not smooth_v and gran == "thread" and kernel == "default":
        _check(lib().sage2_attn(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), B, Hq, Hkv, N, d,
                                int(causal), _stream()))
        return out
    if workspace is None:
        workspace = alloc_workspace(B, Hq, Hkv, N, d, q.device)
    _check(_lib_for(kernel).sage2_attn_ex(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), B, Hq, Hkv, N, d,
                               flags(causal, int8, qk_e4m3, smooth_v, gran) | KERNEL_FLAGS[kernel], workspace.data_ptr(),
                               workspace.numel(), _stream()))
    return out


DS_SIMT = 1024      # include/sage2.h SAGE2_F_DS_SIMT


def prepare(q, k, v, workspace, causal=False, int8=False, ds_simt=False, qk_e4m3=False, smooth_v=False,
            gran="thread", kernel="default"):
    """Preprocessing kernels only (smoothing, quantization, Delta S) into `workspace`, laid out for
    the attention kernel `kernel` will select (pass the same kernel to attention()).

    ds_simt=True computes Delta S with the SIMT fp32 kernel instead of the tf32 tensor-core GEMM
    (A/B checks)."""
    _check_inputs(q, k, v)
    B, Hq, Hkv, N, d = _shape(q, k)
    fl = flags(causal, int8, qk_e4m3, smooth_v, gran) | (DS_SIMT if ds_simt else 0) | KERNEL_FLAGS[kernel]
    _check(_lib_for(kernel).sage2_prepare(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, Hq, Hkv, N, d, fl,
                               workspace.data_ptr(), workspace.numel(), _stream()))


KERNEL_FLAGS = {"default": 0, "v8": 4096, "v12": 131072, "one": 1048576, "v14": 4194304}   # SAGE2_F_KERNEL_* (v14: sage2_dev.h, dev library); "one": v8 single-level ablation


def attention(out, workspace, B, Hq, Hkv, N, d, causal=False, int8=False, kernel="default", qk_e4m3=False,
              smooth_v=False, gran="thread"):
    """The tcgen05 attention kernel only, on a prepared workspace (kernel: "default" = the dispatch
    rule of sage2_attention_kernel, or "v8" / "v12" / "one"; data flags must match the prepare() call)."""
    _check(_lib_for(kernel).sage2_attention(out.data_ptr(), B, Hq, Hkv, N, d,
                                 flags(causal, int8, qk_e4m3, smooth_v, gran) | KERNEL_FLAGS[kernel],
                                 workspace.data_ptr(), workspace.numel(), _stream()))
    return out


def attention_kernel(N, d, causal=False, kernel="default", qk_e4m3=False, gran="thread"):
    """Version number of the attention kernel sage2_attention runs for these arguments (host only)."""
    return int(_lib_for(kernel).sage2_attention_kernel(N, d, flags(causal, False, qk_e4m3, False, gran) | KERNEL_FLAGS[kernel]))


def debug_qk_int32(out, workspace, B, Hq, Hkv, N, d, int8=False, with_p=False, qk_e4m3=False, kernel="default",
                   smooth_v=False):
    """Runs the attention kernel (non-causal; kernel: "default" dispatch rule, "v8" or "v12") and
    returns the raw INT32 S = Q^ K^T read from TMEM, [B*Hq, N_pad, N_pad] (and, with_p=True, also
    the P^ E4M3 codes the kernel produced)."""
    Np = (N + 127) // 128 * 128
    s = torch.zeros((B * Hq, Np, Np), dtype=torch.int32, device=out.device)
    ph = torch.zeros((B * Hq, Np, Np), dtype=torch.uint8, device=out.device) if with_p else None
    _check(_lib_for(kernel).sage2_debug_qk_int32(out.data_ptr(), s.data_ptr(), ph.data_ptr() if with_p else None, B, Hq, Hkv,
                                      N, d, flags(False, int8, qk_e4m3, smooth_v) | KERNEL_FLAGS[kernel], workspace.data_ptr(), workspace.numel(),
                                      _stream()))
    return (s, ph) if with_p else s


def attn_host(q, k, v, out, causal=False):
    """End-to-end C-ABI call on HOST buffers (pinned recommended): H2D copies, preprocessing,
    attention and the D2H copy of out all happen inside sage2_attn_host on `stream`."""
    for t in (q, k, v, out):
        if t.is_cuda or t.dtype != torch.float16 or not t.is_contiguous():
            raise ValueError("attn_host expects contiguous fp16 host tensors")
    B, Hq, Hkv, N, d = _shape(q, k)
    _check(lib().sage2_attn_host(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), B, Hq, Hkv, N, d,
                                 int(causal), _stream()))
    return out


def probe_accumulator(d_bits, prod_vals):
    """FP22 probe on tcgen05 kind::f8f6f4.  d_bits: uint32 numpy, prod_vals: uint8 (E4M3)."""
    import numpy as np
    d_bits = np.ascontiguousarray(d_bits, dtype=np.uint32)
    prod_vals = np.ascontiguousarray(prod_vals, dtype=np.uint8)
    n = d_bits.size
    cz = np.zeros(n, np.uint32)
    cp = np.zeros(n, np.uint32)
    _check(dev_lib().sage2_probe_accumulator(d_bits.ctypes.data, prod_vals.ctypes.data, n, cz.ctypes.data,
                                             cp.ctypes.data), dev_lib())
    return cz, cp


def bench_mma(kind, iters=20000):
    """Dense tcgen05 throughput, ops/s.  kind 0 = kind::i8, 1 = kind::f8f6f4 (E4M3)."""
    r = ctypes.c_double()
    _check(dev_lib().sage2_bench_mma(int(kind), int(iters), ctypes.byref(r)), dev_lib())
    return r.value


MICRO = {0: "tmem_ld_bytes_per_clk_sm", 1: "tmem_st_bytes_per_clk_sm", 2: "mufu_ex2_per_clk_sm",
         3: "i2f_per_clk_sm", 4: "ffma2_lanes_per_clk_sm", 5: "mma_sync_s4_ops_per_clk_sm",
         6: "mma_sync_s8_ops_per_clk_sm", 7: "f2fp_e4m3x2_elems_per_clk_sm", 8: "fmnmx3_per_clk_sm",
         9: "softmax_mix_elems_per_clk_sm", 10: "tmem_ld16x64_bytes_per_clk_sm",
         11: "tmem_st16x64_bytes_per_clk_sm"}


def microbench(which, iters=4096):
    r = ctypes.c_double()
    _check(dev_lib().sage2_microbench(int(which), int(iters), ctypes.byref(r)), dev_lib())
    return r.value


def trace(out, workspace, B, Hq, Hkv, N, d, kernel="default"):
    """clock64 phase stamps of CTA (0,0,0) (dev library): uint64 [32, 64, 16] (role, KV step, slot)."""
    st = torch.zeros(32 * 64 * 16, dtype=torch.int64, device=out.device)
    _check(dev_lib().sage2_dev_trace(out.data_ptr(), st.data_ptr(), B, Hq, Hkv, N, d, KERNEL_FLAGS[kernel],
                                     workspace.data_ptr(), workspace.numel(), _stream()), dev_lib())
    return st.view(32, 64, 16)


def release_memory():
    """Return the library pool's retained device memory (sage2_release_memory)."""
    _check(lib().sage2_release_memory())


def version():
    return int(lib().sage2_version())

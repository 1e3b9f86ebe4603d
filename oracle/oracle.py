"""ctypes marshalling for the C oracle (sage2_oracle.c).  TEST INFRASTRUCTURE ONLY.

No arithmetic of the method lives here: every number the oracle produces is computed in C.
"""
import ctypes
import dataclasses
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sage2_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force=False):
    """Compile the oracle with gcc: -O2, no fast-math, no FP contraction, OpenMP."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
            "-ffp-contract=off", "-fno-fast-math", "-Wall",
            "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "b_q", "kv_tile", "causal", "quant", "qk_max", "smooth_q", "smooth_k",
        "pv_mode", "two_level", "smooth_v", "p_fp32", "qk_gran")] + [("amb_eta", ctypes.c_double),
                                                                       ("q_delta", ctypes.c_float)]


@dataclass
class OracleConfig:
    """SageAttn2-4b defaults (Table 3): INT4 per-thread Q/K, FP8 P~ and V."""
    b_q: int = 128
    kv_tile: int = 128        # the kernel's b_kv (C-9): 128 (default kernel v6); 64 for v5
    causal: bool = False
    quant: bool = True        # False: P~ not quantized (P^ = 448 P~) in attn_block (lossless pin)
    qk_max: int = 7
    smooth_q: bool = True
    smooth_k: bool = True
    pv_mode: int = 0          # 0 fp64 R, 1 fp32 R, 2 FP22-truncated R
    two_level: bool = True
    smooth_v: bool = False
    p_fp32: bool = False      # True: P^ decision in fp32 (diagnostic of C-21); default fp64 (paper verbatim)
    qk_gran: int = 0          # 0 per-thread (SageAttn2), 1 per-block, 2 per-token, 3 per-tensor (NEXT#4)
    amb_eta: float = 2.0 ** -21    # floor of the per-element ambiguity window (ex2.approx, C-21)
    q_delta: float = 0.0      # qk_gran == 3: the head's delta_Q (set by sage2_forward_blocks / q_head_delta)

    def c(self):
        return _Cfg(self.b_q, self.kv_tile, int(self.causal), int(self.quant), self.qk_max,
                    int(self.smooth_q), int(self.smooth_k), self.pv_mode, int(self.two_level),
                    int(self.smooth_v), int(self.p_fp32), int(self.qk_gran), float(self.amb_eta),
                    float(self.q_delta))


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            I = ctypes.c_int
            L.orc_fp16_decode.restype = ctypes.c_double
            L.orc_fp16_decode.argtypes = [ctypes.c_uint16]
            L.orc_e4m3_encode.restype = ctypes.c_uint8
            L.orc_e4m3_encode.argtypes = [ctypes.c_double]
            L.orc_e4m3_decode.restype = ctypes.c_double
            L.orc_e4m3_decode.argtypes = [ctypes.c_uint8]
            L.orc_group_q.argtypes = [I]
            L.orc_group_k.argtypes = [I]
            L.orc_group_q_g.argtypes = [I, I]
            L.orc_group_k_g.argtypes = [I, I]
            L.orc_ngroups_q.argtypes = [I]
            L.orc_ngroups_k128.argtypes = [I]
            for n in ("orc_e4m3_encode_array", "orc_e4m3_decode_array", "orc_fp16_decode_array",
                      "orc_fp16_round_array", "orc_fp22_truncate_array"):
                getattr(L, n).argtypes = [P, ctypes.c_long, P]
                getattr(L, n).restype = None
            L.orc_kv_head.argtypes = [P, P, I, I, ctypes.POINTER(_Cfg), P, P, P, P, P, P, P]
            L.orc_q_block.argtypes = [P, I, I, ctypes.POINTER(_Cfg), P, P, P]
            L.orc_q_head_delta.argtypes = [P, I, I, ctypes.POINTER(_Cfg)]
            L.orc_q_head_delta.restype = ctypes.c_float
            L.orc_delta_s.argtypes = [P, P, I, I, P]
            L.orc_delta_s2.argtypes = [P, P, I, I, P, P]
            L.orc_s_int_block.argtypes = [P, P, I, I, P]
            L.orc_attn_block_q.argtypes = [P, P, P, P, P, P, P, P, I, I, I, ctypes.POINTER(_Cfg), P, P]
            L.orc_attn_block_dbg.argtypes = [P, P, P, P, P, P, P, P, I, I, I, ctypes.POINTER(_Cfg), P, P,
                                             P, P, P]
            L.orc_attn_block_dbg2.argtypes = [P, P, P, P, P, P, P, P, P, I, I, I, ctypes.POINTER(_Cfg), P, P,
                                              P, P, P]
            L.orc_attn_exact_tiled.argtypes = [P, P, P, I, I, ctypes.POINTER(_Cfg), I, I, P]
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def num_threads():
    return lib().orc_num_threads()


# ---- number formats ---------------------------------------------------------------------------
def e4m3_encode(x):
    x = _c(x, np.float64)
    out = np.empty(x.shape, np.uint8)
    lib().orc_e4m3_encode_array(_p(x), x.size, _p(out))
    return out


def e4m3_decode(c):
    c = _c(c, np.uint8)
    out = np.empty(c.shape, np.float64)
    lib().orc_e4m3_decode_array(_p(c), c.size, _p(out))
    return out


def fp16_decode(bits):
    bits = _c(bits, np.uint16)
    out = np.empty(bits.shape, np.float64)
    lib().orc_fp16_decode_array(_p(bits), bits.size, _p(out))
    return out


def fp16_round(x):
    x = _c(x, np.float64)
    out = np.empty(x.shape, np.float64)
    lib().orc_fp16_round_array(_p(x), x.size, _p(out))
    return out


def fp22_truncate(x):
    x = _c(x, np.float32)
    out = np.empty(x.shape, np.float32)
    lib().orc_fp22_truncate_array(_p(x), x.size, _p(out))
    return out


def group_q(t):
    return lib().orc_group_q(int(t))


def group_k(t):
    return lib().orc_group_k(int(t))


def group_q_g(t, gran):
    return lib().orc_group_q_g(int(t), int(gran))


def group_k_g(t, gran):
    return lib().orc_group_k_g(int(t), int(gran))


def ngroups(gran):
    """(Q groups per 128-token block, K groups per 128 keys) of a granularity."""
    return lib().orc_ngroups_q(int(gran)), lib().orc_ngroups_k128(int(gran))


def _bits(x):
    x = np.ascontiguousarray(x)
    if x.dtype == np.float16:
        return x.view(np.uint16)
    assert x.dtype == np.uint16
    return x


# ---- preprocessing ----------------------------------------------------------------------------
def kv_head(K, V, cfg=OracleConfig()):
    """One KV head (K, V: [N, d] fp16).  Returns dict kbar, kprime, khat, dk, vhat, dv, vmean."""
    K, V = _bits(K), _bits(V)
    N, d = K.shape
    Np = (N + 127) // 128 * 128
    r = dict(kbar=np.zeros(d, np.float32), kprime=np.zeros((N, d), np.float32),
             khat=np.zeros((Np, d), np.int8), dk=np.zeros(Np // 128 * ngroups(cfg.qk_gran)[1], np.float32),
             vhat=np.zeros((Np, d), np.uint8), dv=np.zeros(d, np.float32),
             vmean=np.zeros(d, np.float32))
    c = cfg.c()
    lib().orc_kv_head(_p(K), _p(V), N, d, ctypes.byref(c), _p(r["kbar"]), _p(r["kprime"]),
                      _p(r["khat"]), _p(r["dk"]), _p(r["vhat"]), _p(r["dv"]), _p(r["vmean"]))
    return r


def q_block(Qblk, cfg=OracleConfig()):
    """One Q block (rows present, <= 128, fp16).  Returns dict qbar, qhat[128,d], dq[groups]
    (32 per-thread groups by default)."""
    Qb = _bits(Qblk)
    n, d = Qb.shape
    r = dict(qbar=np.zeros(d, np.float32), qhat=np.zeros((128, d), np.int8),
             dq=np.zeros(ngroups(cfg.qk_gran)[0], np.float32))
    c = cfg.c()
    lib().orc_q_block(_p(Qb), n, d, ctypes.byref(c), _p(r["qbar"]), _p(r["qhat"]), _p(r["dq"]))
    return r


def q_head_delta(Q, cfg=OracleConfig()):
    """Per-tensor granularity (qk_gran = 3): the head's delta_Q = max |gamma(Q_i)| over every block / qmax."""
    Qb = _bits(Q)
    N, d = Qb.shape
    c = cfg.c()
    return float(lib().orc_q_head_delta(_p(Qb), N, d, ctypes.byref(c)))


def delta_s(qbar, kprime, with_abs=False):
    """Delta S_i = q_bar_i gamma(K)^T (O-7), fp64.  with_abs=True also returns sum_c |q_bar_c||K'_tc|."""
    qbar = _c(qbar, np.float32)
    kprime = _c(kprime, np.float32)
    N, d = kprime.shape
    out = np.zeros(N, np.float64)
    if not with_abs:
        lib().orc_delta_s(_p(qbar), _p(kprime), N, d, _p(out))
        return out
    ab = np.zeros(N, np.float64)
    lib().orc_delta_s2(_p(qbar), _p(kprime), N, d, _p(out), _p(ab))
    return out, ab


def s_int_block(qhat, khat):
    qhat = _c(qhat, np.int8)
    khat = _c(khat, np.int8)
    Np, d = khat.shape
    out = np.zeros((128, Np), np.int64)
    lib().orc_s_int_block(_p(qhat), _p(khat), Np, d, _p(out))
    return out


def attn_block(qb, ds, kv, N, i, cfg=OracleConfig(), debug=False, ds_abs=None):
    """Alg. 1 inner loop for Q block i. Returns (O[128,d] fp64, l[128]) and, with debug=True,
    a dict with the P^ codes [128, N_pad], ambiguity flags and per-row flip bounds (the window of
    each decision is the fp32 error bound of its score; ds_abs = sum_c |q_bar_c||K'_tc| feeds the
    Delta S part of it, C-21)."""
    d = qb["qhat"].shape[1]
    Np = (N + 127) // 128 * 128
    O = np.zeros((128, d), np.float64)
    l = np.zeros(128, np.float64)
    ds = _c(ds, np.float64)
    c = cfg.c()
    if not debug:
        lib().orc_attn_block_q(_p(qb["qhat"]), _p(qb["dq"]), _p(ds), _p(kv["khat"]), _p(kv["dk"]),
                               _p(kv["vhat"]), _p(kv["dv"]), _p(kv["vmean"]), N, d, i,
                               ctypes.byref(c), _p(O), _p(l))
        return O, l
    ph = np.zeros((128, Np), np.uint8)
    amb = np.zeros((128, Np), np.uint8)
    flip = np.zeros(128, np.float64)
    dsa = None if ds_abs is None else _c(ds_abs, np.float64)
    lib().orc_attn_block_dbg2(_p(qb["qhat"]), _p(qb["dq"]), _p(ds), None if dsa is None else _p(dsa),
                              _p(kv["khat"]), _p(kv["dk"]), _p(kv["vhat"]), _p(kv["dv"]), _p(kv["vmean"]), N, d, i,
                              ctypes.byref(c), _p(O), _p(l), _p(ph), _p(amb), _p(flip))
    return O, l, dict(phat=ph, amb=amb, flip=flip)


def attn_exact_tiled(Q, K, V, cfg=OracleConfig(quant=False), row0=0, row1=None):
    """Exact mode (no quantization): tiled online softmax in fp64 with smoothing per cfg."""
    Q, K, V = _bits(Q), _bits(K), _bits(V)
    N, d = Q.shape
    row1 = N if row1 is None else row1
    O = np.zeros((row1 - row0, d), np.float64)
    c = cfg.c()
    lib().orc_attn_exact_tiled(_p(Q), _p(K), _p(V), N, d, ctypes.byref(c), row0, row1, _p(O))
    return O


def sage2_forward_blocks(q, k, v, units, cfg=OracleConfig(), keep=False, debug=False):
    """SageAttn2 forward on selected Q blocks.

    q: [B, Hq, N, d] fp16 numpy; k, v: [B, Hkv, N, d].  units: iterable of (b, h_q, i).
    Returns dict with 'O' [n_units, 128, d] fp64 (pre-rounding), 'O16' (fp16-rounded, fp64
    array), 'flip' [n_units, 128] (debug=True: per-row bound on the effect of ambiguous P^
    decisions, C-21) and when keep=True the per-unit intermediates (incl. P^ codes).
    """
    B, Hq, N, d = q.shape
    Hkv = k.shape[1]
    grp = Hq // Hkv
    kv_cache, qdelta = {}, {}
    outO, outO16, inter, flips = [], [], [], []
    for (b, h, i) in units:
        hk = h // grp
        if (b, hk) not in kv_cache:
            kv_cache[(b, hk)] = kv_head(k[b, hk], v[b, hk], cfg)
        kv = kv_cache[(b, hk)]
        r0, r1 = 128 * i, min(128 * i + 128, N)
        if cfg.qk_gran == 3:                         # per-tensor: the head's delta_Q first
            if (b, h) not in qdelta:
                qdelta[(b, h)] = q_head_delta(q[b, h], cfg)
            qb = q_block(q[b, h, r0:r1], dataclasses.replace(cfg, q_delta=qdelta[(b, h)]))
        else:
            qb = q_block(q[b, h, r0:r1], cfg)
        if debug:
            ds, dsa = delta_s(qb["qbar"], kv["kprime"], with_abs=True)
            O, l, dbg = attn_block(qb, ds, kv, N, i, cfg, debug=True, ds_abs=dsa)
            flips.append(dbg["flip"])
        else:
            ds = delta_s(qb["qbar"], kv["kprime"])
            O, l = attn_block(qb, ds, kv, N, i, cfg)
            dbg = None
        outO.append(O)
        outO16.append(fp16_round(O))
        if keep:
            inter.append(dict(qb=qb, ds=ds, l=l, dbg=dbg))
    res = dict(O=np.stack(outO), O16=np.stack(outO16))
    if debug:
        res["flip"] = np.stack(flips)
    if keep:
        res["inter"] = inter
        res["kv"] = kv_cache
    return res

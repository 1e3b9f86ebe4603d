"""Test-side helpers for the GPU parity tests: read the workspace regions the CUDA path writes and
undo its tile-image storage layout (K-major, 128B / 64B swizzled; include/sage2.h) so the values
can be compared with the oracle's natural [tokens, channels] arrays.  No method arithmetic."""
import numpy as np
import torch


def swz_offsets(rows, row_bytes):
    """Byte offset of (row, byte col) in a swizzled K-major tile image (see ptx.cuh swz_off)."""
    r = np.arange(rows)[:, None]
    c = np.arange(row_bytes)[None, :]
    sw = (r & 7) if row_bytes == 128 else ((r & 7) >> 1)
    return (r >> 3) * (8 * row_bytes) + (r & 7) * row_bytes + (((c >> 4) ^ sw) << 4) + (c & 15)


def region(ws, lay, name, dtype, count):
    off = lay[name]
    nbytes = count * np.dtype(dtype).itemsize
    return ws[off:off + nbytes].cpu().numpy().view(dtype)


def untile_rows(raw, n_tiles_total, d):
    """[n_tiles, 128*d] tile images (row = token) -> [n_tiles*128, d]."""
    off = swz_offsets(128, d)
    t = raw.reshape(n_tiles_total, 128 * d)
    return t[:, off].reshape(n_tiles_total * 128, d)


def untile_vt(raw, n_tiles_total, d):
    """[n_tiles, d*128] V^T tile images (row = channel, byte = token) -> [n_tiles*128, d]."""
    off = swz_offsets(d, 128)                    # [d, 128]
    t = raw.reshape(n_tiles_total, d * 128)[:, off]   # [n_tiles, d, 128]
    return np.ascontiguousarray(t.transpose(0, 2, 1)).reshape(n_tiles_total * 128, d)


def read_prepared(ws, lay, B, Hq, Hkv, N, d):
    nT = (N + 127) // 128
    Np = nT * 128
    out = {}
    out["kbar"] = region(ws, lay, "kbar", np.float32, B * Hkv * d).reshape(B * Hkv, d)
    out["dv"] = region(ws, lay, "dv", np.float32, B * Hkv * d).reshape(B * Hkv, d)
    out["vmean"] = region(ws, lay, "vmean", np.float32, B * Hkv * d).reshape(B * Hkv, d)
    out["qbar"] = region(ws, lay, "qbar", np.float32, B * Hq * nT * d).reshape(B * Hq, nT, d)
    out["dq"] = region(ws, lay, "dq", np.float32, B * Hq * Np // 4).reshape(B * Hq, Np // 4)
    out["dk"] = region(ws, lay, "dk", np.float32, B * Hkv * Np // 16).reshape(B * Hkv, Np // 16)
    out["qhat"] = untile_rows(region(ws, lay, "qhat", np.int8, B * Hq * Np * d), B * Hq * nT, d).reshape(B * Hq, Np, d)
    out["khat"] = untile_rows(region(ws, lay, "khat", np.int8, B * Hkv * Np * d), B * Hkv * nT, d).reshape(B * Hkv, Np, d)
    out["vhat"] = untile_vt(region(ws, lay, "vhat", np.uint8, B * Hkv * Np * d), B * Hkv * nT, d).reshape(B * Hkv, Np, d)
    out["ds"] = region(ws, lay, "ds", np.float32, B * Hq * nT * Np).reshape(B * Hq, nT, Np)
    return out


def fp16_ulp(x):
    """Spacing of fp16 at |x| (subnormal spacing 2^-24 near 0)."""
    a = np.abs(np.asarray(x, np.float64))
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -14)))
    return 2.0 ** (e - 10)


def to_np16(t):
    return t.detach().cpu().numpy().astype(np.float16)


def kv_tile_for(N, d, causal=False, kernel="default", **flags):
    """The b_kv of the attention kernel the library runs for these arguments (reading C-9: the
    oracle's kv_tile must equal it): 64 for v12, 128 otherwise."""
    from paper_2411_10958_b200 import sage2
    return 64 if sage2.attention_kernel(N, d, causal=causal, kernel=kernel, **flags) == 12 else 128

"""Per-phase clock64 stamps of one CTA of the v8 (default) or, with V10=1, the persistent v10 kernel (its last item; softmax stamps only for v10).
Softmax tile k (thread 0 of its half-0 warpgroup), slots: 0 loop start, 1 S ready, 9 S loaded,
2 dequant, 3 max exchanged, 4 MUFU turn, 5 P^ written, 6 R ready, 7 R read, 8 promotion done.
MMA issuer k: 0 kv_full seen, 1 s_free seen, 2 QK committed, 3 P^ seen, 4 PV committed.
Tile 0, every warp (4 + wq + 4h): slot 7 = its R read (s_free arrival)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

B, H = 1, 4
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
flags = 64 + (16384 if os.environ.get("V10") else 4096)
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
buf = torch.zeros(12 * 64 * 16, dtype=torch.int64, device="cuda")
L = sage2.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    rc = L.sage2_debug_qk_int32(out.data_ptr(), buf.data_ptr(), None, B, H, H, N, d, flags, ws.data_ptr(),
                                ctypes.c_size_t(ws.numel()), st)
    assert rc == 0, L.sage2_last_cuda_error()
torch.cuda.synchronize()
t = buf.view(12, 64, 16).cpu().numpy().astype(np.int64)
for j in range(8, 12):
    b = t[0, j, 0]
    print(f"j={j} iter(t0) {t[0, j + 1, 0] - b:5d}")
    for kk in (0, 1):
        s = t[kk, j]
        print(f"  sm{kk}: start {s[0] - b:6d} Sready {s[1] - b:6d} Sld {s[9] - b:6d} deq {s[2] - b:6d} max {s[3] - b:6d} "
              f"turn {s[4] - b:6d} P {s[5] - b:6d} Rready {s[6] - b:6d} Rread {s[7] - b:6d} prom {s[8] - b:6d}")
        if os.environ.get("V10"):            # v10: rows 2, 3 hold the key-half-1 softmax stamps
            s1 = t[2 + kk, j]
            print(f"  h1 {kk}: start {s1[0] - b:6d} Sready {s1[1] - b:6d} Sld {s1[9] - b:6d} deq {s1[2] - b:6d} "
                  f"max {s1[3] - b:6d} turn {s1[4] - b:6d} P {s1[5] - b:6d} Rready {s1[6] - b:6d} "
                  f"Rread {s1[7] - b:6d} prom {s1[8] - b:6d}")
            continue
        m = t[2 + kk, j]
        m1 = t[2 + kk, j + 1]
        print(f"  mma{kk}: kvfull {m[0] - b:6d} sfree {m[1] - b:6d} QK {m[2] - b:6d} Pseen {m[3] - b:6d} PV {m[4] - b:6d} "
              f"| next kvfull {m1[0] - b:6d} sfree {m1[1] - b:6d} QK {m1[2] - b:6d}")
    print("  tile0 warps Rread:", [int(t[4 + w, j, 7] - b) for w in range(8)])

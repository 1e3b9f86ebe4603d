"""Per-phase clock64 stamps of one CTA of the v6 / v8 attention kernel (SAGE2_F_DEBUG_TIMING;
flags argument 64 + 8192 = v6 (default), 64 + 4096 = v8; scripts/kernel_timing_v8.py has the v8 layout).

Slots (softmax tile k, lane 0 of its first warp): 0 loop start, 1 S ready, 2 S loaded + dequant,
3 max done, 4 MUFU turn acquired, 5 P^ written, 6 R ready, 7 R read (S/R freed), 8 promotion done.
MMA issuer k: 0 QK committed, 1 P^ seen, 2 PV committed.  Producer: 0 stage j issued."""
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
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 64 + 8192   # DEBUG_TIMING | KERNEL_V6
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
buf = torch.zeros(6 * 64 * 16, dtype=torch.int64, device="cuda")
L = sage2.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    rc = L.sage2_debug_qk_int32(out.data_ptr(), buf.data_ptr(), None, B, H, H, N, d, flags, ws.data_ptr(),
                                ctypes.c_size_t(ws.numel()), st)
    assert rc == 0, L.sage2_last_cuda_error()
torch.cuda.synchronize()
t = buf.view(6, 64, 16).cpu().numpy().astype(np.int64)
for j in range(8, 14):
    b = t[0, j, 0]
    print(f"j={j} iter(t0) {t[0, j + 1, 0] - b:5d}")
    for kk in (0, 1):
        s = t[kk, j]
        print(f"  sm{kk}: start {s[0] - b:6d} Sready {s[1] - b:6d} Sld {s[9] - b:6d} deq {s[2] - b:6d} max {s[3] - b:6d} "
              f"turn {s[4] - b:6d} P {s[5] - b:6d} Rready {s[6] - b:6d} Rread {s[7] - b:6d} prom {s[8] - b:6d}")
        m = t[2 + kk, j]
        print(f"  mma{kk}: top {m[3] - b:6d} kvfull {m[4] - b:6d} sfree {m[5] - b:6d} mma1 {m[6] - b:6d} "
              f"QK {m[0] - b:6d} Pseen {m[1] - b:6d} PV {m[2] - b:6d}   prod j: {t[4, j, 0] - b:6d}")

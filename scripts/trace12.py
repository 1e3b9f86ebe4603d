"""clock64 phase stamps of CTA (0,0,0) of the v12 kernel (dev library).  Softmax tile k (thread 0 of
its quarter-0 warp), slots: 0 loop start, 1 S ready, 9 S loaded, 2 dequant, 3 max, 4 MUFU turn,
5 P^ written, 6 R ready, 7 R read, 8 promotion done.  MMA (who 4+k): 1 QK issued(s_free seen), 2 QK
committed, 3 P^ first half seen, 4 PV committed.   python scripts/trace12.py [N] [causal]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

B, H, d = 1, 4, 64
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws, kernel="v12")
out = torch.empty_like(q)
for _ in range(3):
    buf = sage2.trace(out, ws, B, H, H, N, d, kernel="v12")
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.int64)
names = {0: "start", 1: "Srdy", 9: "Sld", 2: "deq", 3: "max", 4: "turn", 5: "P", 6: "Rrdy", 7: "Rread", 8: "prom"}
for j in range(16, 20):
    b = t[0, j, 0]
    print(f"j={j} step(t0) {t[0, j + 1, 0] - b:5d}")
    for kk in range(4):
        s = t[kk, j]
        print(f"  sm{kk}: " + " ".join(f"{names[x]} {s[x] - b:6d}" for x in (0, 1, 9, 2, 3, 4, 5, 6, 7, 8)))
        m = t[4 + kk, j]
        print(f"  mma{kk}: QKgo {m[1] - b:6d} QK {m[2] - b:6d} Pa {m[3] - b:6d} PV {m[4] - b:6d}")
print("per-warp MUFU turn / P-written stamps (warps 0-15 = tile warp // 4), step 17:")
b = t[0, 17, 0]
for w in range(16):
    print(f"  warp {w:2d} tile {w // 4}: turn {t[16 + w, 17, 4] - b:6d}  P {t[16 + w, 17, 5] - b:6d}")

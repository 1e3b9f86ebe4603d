"""clock64 phase stamps of one CTA of the v13 attention kernel (dev library).  python scripts/trace13.py [N] [d]
Softmax tile k iteration j: 2 loop top (S(j) dequantized), 3 max exchanged, 4 MUFU turn, 5 P^(j) written,
1 S(j+1) ready, 9 S(j+1) loaded, 6 S(j+1) dequantized, 7 R(j) ready, 8 promotion done.
MMA issuer k: 3 P^ halves + S(j+1) read seen, 4 PV(j) committed, 5 R(j) freed seen, 6 QK(j+2) committed."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

B, H = 1, 4
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
kern = os.environ.get("KERNEL", "v13")
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
for _ in range(3):
    buf = sage2.trace(out, ws, B, H, H, N, d, kernel=kern)
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.int64)
for j in range(8, 13):
    b = t[0, j, 4]
    print(f"j={j} iter(t0 turn->turn) {t[0, j + 1, 4] - b:5d}")
    for kk in (0, 1):
        s = t[kk, j]
        print(f"  sm{kk}: top {s[2] - b:6d} max {s[3] - b:6d} turn {s[4] - b:6d} P {s[5] - b:6d} S+1rdy {s[1] - b:6d} "
              f"S+1ld {s[9] - b:6d} S+1deq {s[6] - b:6d} Rrdy {s[7] - b:6d} prom {s[8] - b:6d}")
        m = t[2 + kk, j]
        print(f"  mma{kk}: Pseen {m[3] - b:6d} PV {m[4] - b:6d} Rfree {m[5] - b:6d} QK+2 {m[6] - b:6d}")

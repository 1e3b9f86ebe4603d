"""Per-phase clock64 stamps of one CTA of the v8 (or KERNEL=v12) attention kernel (dev library:
sage2.trace).  python scripts/trace.py [N] [d]
Softmax tile k (thread 0 of its half-0 warpgroup), slots: 0 loop start, 1 S ready, 9 S loaded,
2 dequant, 3 max exchanged, 4 MUFU turn, 5 P^ written, 6 R ready, 7 R read, 8 promotion done.
MMA issuer k: 0 kv_full seen, 1 s_free seen, 2 QK committed, 3 P^ seen, 4 PV committed.
Tile 0, every warp (4 + wq + 4h): slot 7 = its R read (s_free arrival)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

B, H = 1, 4
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
for _ in range(3):
    buf = sage2.trace(out, ws, B, H, H, N, d, kernel=os.environ.get("KERNEL", "v8"))
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.int64)
for j in range(8, 12):
    b = t[0, j, 0]
    print(f"j={j} iter(t0) {t[0, j + 1, 0] - b:5d}")
    for kk in (0, 1):
        s = t[kk, j]
        print(f"  sm{kk}: start {s[0] - b:6d} Sready {s[1] - b:6d} Sld {s[9] - b:6d} deq {s[2] - b:6d} max {s[3] - b:6d} "
              f"turn {s[4] - b:6d} P {s[5] - b:6d} Rready {s[6] - b:6d} Rread {s[7] - b:6d} prom {s[8] - b:6d}")
        m = t[2 + kk, j]
        m1 = t[2 + kk, j + 1]
        print(f"  mma{kk}: kvfull {m[0] - b:6d} sfree {m[1] - b:6d} QK {m[2] - b:6d} Pseen {m[3] - b:6d} PV {m[4] - b:6d} "
              f"| next kvfull {m1[0] - b:6d} sfree {m1[1] - b:6d} QK {m1[2] - b:6d}")
    print("  tile0 warps Rread:", [int(t[4 + w, j, 7] - b) for w in range(8)])

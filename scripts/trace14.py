"""clock64 phase stamps of one CTA of the v14 attention kernel (dev library: sage2.trace, KERNEL v14).
    python scripts/trace14.py [N] [d] [B] [H]
Pair P (row-0 thread of its half-0 warpgroup), per KV tile j, slots: 0 loop start, 1 S ready, 2 S loaded,
3 dequant + partial max done, 4 max exchanged, 5 MUFU turn, 6 P^ written, 7 R ready, 8 previous
promotion seen, 9 promotion done.  MMA issuer, per j: 0 loop, 1 s_free(j) seen, 2 QK(j+2) issued,
3 first P^ half seen, 4 R free, 5 all of P^ seen, 6 PV(j) committed (1, 2: the QK issuer: kv_full(j) seen, QK(j) committed)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
B = int(sys.argv[3]) if len(sys.argv) > 3 else 4
H = int(sys.argv[4]) if len(sys.argv) > 4 else 32
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws, kernel="v14")
out = torch.empty_like(q)
for _ in range(3):
    buf = sage2.trace(out, ws, B, H, H, N, d, kernel="v14")
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.int64)
names = ["start", "Srdy", "Sld", "deq", "xchg", "turn", "Pdone", "Rrdy", "prevpr", "prom"]
mnames = ["loop", "sfree", "QK", "Pa", "Rfree", "Pall", "PV"]
js = range(20, 30)
b0 = t[0, 20, 5]
for j in js:
    P = j & 1
    s = t[P, j]
    m = t[2, j]
    print(f"j={j:2d} pair{P}: " + " ".join(f"{n} {int(s[i] - b0):6d}" for i, n in enumerate(names)))
    print(f"       mma:   " + " ".join(f"{n} {int(m[i] - b0):6d}" for i, n in enumerate(mnames)))
ex = [t[j & 1, j, 6] - t[j & 1, j, 5] for j in js]
per = [(t[j & 1, j + 2, 5] - t[j & 1, j, 5]) / 2 for j in js]
print("exp phase cycles:", [int(x) for x in ex])
print("cycles per tile (turn to turn / 2):", [int(x) for x in per])

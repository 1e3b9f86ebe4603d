"""Per-phase clock64 stamps of one CTA of the v4 attention kernel (SAGE2_F_DEBUG_TIMING)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth

B, H, N, d = 1, 4, int(sys.argv[1]) if len(sys.argv) > 1 else 8192, int(sys.argv[2]) if len(sys.argv) > 2 else 128
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
buf = torch.zeros(3 * 64 * 16, dtype=torch.int64, device="cuda")
L = sage2.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    rc = L.sage2_debug_qk_int32(out.data_ptr(), buf.data_ptr(), None, B, H, H, N, d, 64 + 8, ws.data_ptr(),
                                ctypes.c_size_t(ws.numel()), st)
    assert rc == 0, L.sage2_last_cuda_error()
torch.cuda.synchronize()
t = buf.view(3, 64, 16).cpu().numpy().astype(np.int64)
names = {0: "start", 1: "S ready", 2: "S loaded", 3: "dequant+max", 4: "barrier", 5: "exp/pack", 6: "p arrive",
         7: "R ready", 8: "corrected"}
for who in (0, 1):
    print(f"--- softmax half {who}: cycles relative to iteration start")
    for j in range(8, 16):
        row = t[who, j]
        base = row[0]
        print(j, " ".join(f"{names[k]}={row[k]-base:5d}" for k in range(9) if row[k] != 0 or k == 0),
              f" iter={t[who, j+1, 0]-base}")
print("--- MMA thread: issue_qk(j+1) start / end / p_full(j) seen, relative to softmax half0 start of j")
for j in range(8, 16):
    base = t[0, j, 0]
    print(j, [int(t[2, j, kk] - base) for kk in range(3)])

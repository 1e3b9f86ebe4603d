"""Per-phase clock64 stamps of one CTA of the v5 attention kernel (SAGE2_F_DEBUG_TIMING)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth

B, H, N, d = 1, 4, int(sys.argv[1]) if len(sys.argv) > 1 else 8192, int(sys.argv[2]) if len(sys.argv) > 2 else 128
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
buf = torch.zeros(6 * 64 * 16, dtype=torch.int64, device="cuda")
L = sage2.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    rc = L.sage2_debug_qk_int32(out.data_ptr(), buf.data_ptr(), None, B, H, H, N, d, 64 + 512, ws.data_ptr(),
                                ctypes.c_size_t(ws.numel()), st)
    assert rc == 0, L.sage2_last_cuda_error()
torch.cuda.synchronize()
t = buf.view(6, 64, 16).cpu().numpy().astype(np.int64)
for u in range(16, 24):
    b = t[0, u, 0]
    sm = lambda w, kk: int(t[w, u, kk] - b)
    print(f"u={u} t0: Sload {sm(0,1):5d} max {sm(0,2):5d} pfree {sm(0,3):5d} turn {sm(0,4):5d} exp {sm(0,5):5d} arrive {sm(0,6):5d} next {int(t[0,u+1,0]-b):5d}"
          f" | t1 start {sm(1,0):5d} turn {sm(1,4):5d} exp {sm(1,5):5d}")
    print(f"      corr0: p {sm(2,1):5d} rlo {sm(2,2):5d}/{sm(2,3):5d} rhi {sm(2,4):5d}/{sm(2,5):5d} | mma0: qk(u+1) {sm(4,1):5d} p {sm(4,2):5d} pvlo {sm(4,3):5d} pvhi {sm(4,4):5d}")

"""Per-phase clock64 stamps of one CTA of the v1 attention kernel (SAGE2_F_DEBUG_TIMING)."""
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
    rc = L.sage2_debug_qk_int32(out.data_ptr(), buf.data_ptr(), None, B, H, H, N, d, 64 + 128, ws.data_ptr(),
                                ctypes.c_size_t(ws.numel()), st)
    assert rc == 0, L.sage2_last_cuda_error()
torch.cuda.synchronize()
t = buf.view(6, 64, 16).cpu().numpy().astype(np.int64)
base0 = t[0, 8, 0]
for j in range(8, 14):
    b = t[0, j, 0]
    print(f"j={j} t0-softmax start={b-base0:6d} | S ready {t[0,j,1]-b:5d} S loaded {t[0,j,2]-b:5d} max {t[0,j,3]-b:5d} exp/pack {t[0,j,4]-b:5d} next {t[0,j+1,0]-b:5d}")
    print(f"      t1-softmax start={t[1,j,0]-b:6d} | S ready {t[1,j,1]-t[1,j,0]:5d} max {t[1,j,3]-t[1,j,0]:5d} exp/pack {t[1,j,4]-t[1,j,0]:5d} next {t[1,j+1,0]-t[1,j,0]:5d}")
    for kk in (0, 1):
        c = t[2 + kk, j]
        m = t[4 + kk, j]
        print(f"      corr t{kk}: p_full {c[1]-b:6d} r_full {c[2]-b:6d} done {c[3]-b:6d} | mma t{kk}: QK issued {m[0]-b:6d} p seen {m[1]-b:6d}")

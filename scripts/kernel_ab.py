"""A/B timing of attention-kernel variants on one config (CUDA events, kernel only)."""
import ctypes
import json
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth

B, H, N, d = 4, 32, int(sys.argv[1]) if len(sys.argv) > 1 else 32768, int(sys.argv[2]) if len(sys.argv) > 2 else 128
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
L = sage2.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ops = 4.0 * B * H * N * N * d
res = {}
VARIANTS = [("v6", 0), ("v1", 128), ("v5", 512), ("v6_causal", 1), ("v5_causal", 513), ("v4", 8), ("v0", 4), ("v4_nullsm", 24), ("v4_nullmma", 40),
            ("v1_nullmma", 160), ("v1_causal", 129), ("v4_causal", 9)]
if len(sys.argv) > 3:
    VARIANTS = [v for v in VARIANTS if v[0] in sys.argv[3].split(",")]
for name, fl in VARIANTS:
    def run():
        rc = L.sage2_attention(out.data_ptr(), B, H, H, N, d, fl, ws.data_ptr(), ctypes.c_size_t(ws.numel()), st)
        assert rc == 0, (name, rc, L.sage2_last_cuda_error())
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    o = ops / 2 if fl & 1 else ops
    res[name] = (round(ms, 3), round(o / ms / 1e9, 1))
    print(name, res[name], flush=True)

"""A/B of a whole step (sage2_prepare + sage2_attention, back to back, 10 steps, CUDA events) between
library builds.  python scripts/step_ab.py LIB1,LIB2 B Hq Hkv N d [causal]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

libs = sys.argv[1].split(",")
B, Hq, Hkv, N, d = (int(x) for x in sys.argv[2:7])
causal = len(sys.argv) > 7 and sys.argv[7] == "1"
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, device="cuda")
out = torch.empty_like(q)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ops = 4.0 * B * Hq * N * N * d / (2 if causal else 1)
res = {}
for r in range(3):
    for lp in libs:
        L = sage2._declare(ctypes.CDLL(lp))
        ws = torch.empty(L.sage2_workspace_bytes(B, Hq, Hkv, N, d, int(causal)), dtype=torch.uint8, device="cuda")

        def step():
            assert L.sage2_prepare(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, Hq, Hkv, N, d, int(causal),
                                   ws.data_ptr(), ctypes.c_size_t(ws.numel()), st) == 0
            assert L.sage2_attention(out.data_ptr(), B, Hq, Hkv, N, d, int(causal), ws.data_ptr(),
                                     ctypes.c_size_t(ws.numel()), st) == 0
        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            step()
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(lp, []).append(e0.elapsed_time(e1) / 10)
        del ws
for lp, t in res.items():
    print(f"B={B} Hq={Hq} N={N} d={d} causal={causal} {os.path.basename(lp):22s} step {min(t)*1e3:8.1f} us "
          f"{ops / min(t) / 1e9:7.1f} TOPS")

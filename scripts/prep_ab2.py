"""A/B of sage2_prepare between library builds (CUDA events, 10 calls).  python scripts/prep_ab2.py LIB1,LIB2 B Hq Hkv N d [causal]"""
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
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
for r in range(3):
    for lp in libs:
        L = sage2._declare(ctypes.CDLL(lp))
        ws = torch.empty(L.sage2_workspace_bytes(B, Hq, Hkv, N, d, int(causal)), dtype=torch.uint8, device="cuda")
        run = lambda: L.sage2_prepare(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, Hq, Hkv, N, d, int(causal),
                                      ws.data_ptr(), ctypes.c_size_t(ws.numel()), st)
        assert run() == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(lp, []).append(e0.elapsed_time(e1) / 10)
        del ws
for lp, t in res.items():
    print(f"B={B} Hq={Hq} Hkv={Hkv} N={N} d={d} causal={causal} {os.path.basename(lp):20s} prepare min {min(t)*1e3:8.1f} us")

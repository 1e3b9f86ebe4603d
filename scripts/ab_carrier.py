"""A/B: kind::i8 QK^T vs the E4M3 carrier (SAGE2_F_QK_E4M3), default kernel, C2 shapes."""
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

B, H = 4, 32
N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ops = 4.0 * B * H * N * N * d
res = {}
for name, e4 in (("i8", False), ("e4m3", True)):
    ws = sage2.alloc_workspace(B, H, H, N, d)
    sage2.prepare(q, k, v, ws, qk_e4m3=e4)
    out = torch.empty_like(q)
    ts = []
    for causal in (False, True):
        sage2.attention(out, ws, B, H, H, N, d, causal=causal, qk_e4m3=e4)
        torch.cuda.synchronize()
        for r in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                sage2.attention(out, ws, B, H, H, N, d, causal=causal, qk_e4m3=e4)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 3)
        ms = statistics.median(ts[-3:])
        o = ops / 2 if causal else ops
        print(f"{os.environ.get('SAGE2_LIB', 'default')} N={N} d={d} {name} causal={causal}: {ms:.3f} ms "
              f"{o / ms / 1e9:.1f} TOPS", flush=True)
    del ws

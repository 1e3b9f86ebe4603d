"""A/B of the E4M3-carrier QK^T (SAGE2_F_QK_E4M3) against kind::i8, each on its own correctly
prepared workspace (kernel only, CUDA events, round-robin median).

    python scripts/carrier_ab.py N d [rounds]"""
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
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
L = sage2.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
out = torch.empty_like(q)
ops = 4.0 * B * H * N * N * d
cases = {}
for causal in (False, True):
    for f8 in (False, True):
        ws = sage2.alloc_workspace(B, H, H, N, d, causal=causal)
        sage2.prepare(q, k, v, ws, causal=causal, qk_e4m3=f8)
        fl = sage2.flags(causal, False, f8, False, "thread")
        cases[f"{'causal ' if causal else ''}{'e4m3' if f8 else 'i8'}"] = (ws, fl, ops / 2 if causal else ops)
times = {n: [] for n in cases}
for r in range(rounds):
    for name, (ws, fl, o) in cases.items():
        def run():
            rc = L.sage2_attention(out.data_ptr(), B, H, H, N, d, fl, ws.data_ptr(), ctypes.c_size_t(ws.numel()), st)
            assert rc == 0, rc
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        times[name].append(e0.elapsed_time(e1) / 5)
for name, (ws, fl, o) in cases.items():
    med = statistics.median(times[name])
    print(f"N={N} d={d} {name:14s} median {med:8.3f} ms {o / med / 1e9:7.1f} TOPS", flush=True)

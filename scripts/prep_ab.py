"""Time sage2_prepare (all preprocessing kernels) with CUDA events: causal vs non-causal workspaces,
tf32 tensor-core Delta S vs the SIMT kernel.  python scripts/prep_ab.py B Hq Hkv N d"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

B, Hq, Hkv, N, d = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (4, 32, 32, 32768, 128)
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, device="cuda")
for causal in (False, True):
    for simt in (False, True):
        ws = sage2.alloc_workspace(B, Hq, Hkv, N, d, causal=causal)
        for _ in range(2):
            sage2.prepare(q, k, v, ws, causal=causal, ds_simt=simt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sage2.prepare(q, k, v, ws, causal=causal, ds_simt=simt)
        e1.record()
        torch.cuda.synchronize()
        print(f"B={B} Hq={Hq} Hkv={Hkv} N={N} d={d} causal={causal} ds_simt={simt}: "
              f"prepare {e0.elapsed_time(e1) / 5:.3f} ms, workspace {ws.numel() / 1e9:.2f} GB", flush=True)
        del ws

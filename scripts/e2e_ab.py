"""e2e (sage2_attn_host, pinned host buffers) timing at C2-32K d=128: median of 5 calls after 2 warm-ups."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

B, H, N, d = 4, 32, 32768, 128
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
qh, kh, vh = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
oh = torch.empty(q.shape, dtype=torch.float16).pin_memory()
for _ in range(2):
    sage2.attn_host(qh, kh, vh, oh)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sage2.attn_host(qh, kh, vh, oh)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(f"{os.environ.get('SAGE2_LIB', 'default')}: e2e {ms:.2f} ms = {4.0 * B * H * N * N * d / ms / 1e9:.1f} TOPS")

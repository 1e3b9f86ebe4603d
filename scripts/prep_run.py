"""Run sage2.prepare a few times on one config (for ncu captures of the preprocessing kernels)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_10958_b200 import sage2, synth

B, H, N, d = [int(x) for x in sys.argv[1:5]]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
q, k, v = synth.make_qkv(B, H, H, N, d, "iid", seed=1, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
for _ in range(reps):
    sage2.prepare(q, k, v, ws)
torch.cuda.synchronize()
print("ok")

"""Small forward passes for compute-sanitizer (memcheck / racecheck / synccheck): config C1 and a
ragged causal GQA case, through every product kernel (v8, v12, the single-level ablation, the
experimental v14) and the preprocessing kernels (SIMT and tensor-core Delta S, the side-stream Q
quantizer of short sequences).
    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

CASES = [  # B, Hq, Hkv, N, d, causal, kernel, extra prepare flags
    (1, 1, 1, 256, 64, False, "default", {}),            # C1 (v12)
    (1, 1, 1, 256, 64, False, "v8", {}),
    (1, 4, 2, 300, 128, True, "default", {}),            # ragged causal GQA (v8)
    (1, 4, 2, 300, 128, False, "v8", {}),
    (1, 4, 2, 300, 64, True, "v12", {}),
    (1, 4, 2, 300, 128, True, "one", {}),
    (1, 2, 1, 2200, 128, False, "default", {}),          # tensor-core Delta S (N > 2048)
    (1, 2, 2, 333, 128, False, "default", {"smooth_v": True, "int8": True}),
    (1, 2, 1, 700, 128, False, "v14", {}),               # v14 (experimental): 6 KV tiles, ragged
    (1, 2, 2, 128, 128, False, "v14", {}),               # v14 with one KV tile (pair B idle)
    (1, 2, 1, 333, 64, False, "v14", {"smooth_v": True}),
]
for B, Hq, Hkv, N, d, causal, kern, fl in CASES:
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, kind="structured", seed=2, device="cuda")
    ws = sage2.alloc_workspace(B, Hq, Hkv, N, d, causal=causal)
    sage2.prepare(q, k, v, ws, causal=causal, kernel=kern, **fl)
    out = torch.empty_like(q)
    sage2.attention(out, ws, B, Hq, Hkv, N, d, causal=causal, kernel=kern, **fl)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    print("ok", B, Hq, Hkv, N, d, causal, kern, fl, flush=True)
o = sage2.attn(*synth.make_qkv(1, 2, 1, 200, 128, seed=4, device="cuda"), causal=True)   # sage2_attn (pool)
torch.cuda.synchronize()
print("all cases done")

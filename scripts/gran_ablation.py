"""NEXT#4: QK quantization granularity ablation on B200 (the paper's P:1089-1106 speed table and
P:540-547 accuracy table, re-measured): per-thread (SageAttn2 default) / per-block / per-token.

  (per-tensor added in round 2: one scale per head)
  speed:    attention kernel TOPS at C2-32K d=128 (B=4, H=32, N=32768), non-causal and causal
  accuracy: CosSim / Rel-L1 / RMSE against fp32 attention (torch SDPA, TF32 off) on the
            'structured' synthetic inputs (channel outliers) at B=1, H=8, N=4096
Prints one JSON object."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
res = {"speed": {}, "accuracy": {}}
B, H, N, d = 4, 32, 32768, 128
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ops = 4.0 * B * H * N * N * d
for gran in ("thread", "block", "token", "tensor"):
    for causal in (False, True):
        ws = sage2.alloc_workspace(B, H, H, N, d)
        sage2.prepare(q, k, v, ws, causal=causal, gran=gran)
        out = torch.empty_like(q)
        sage2.attention(out, ws, B, H, H, N, d, causal=causal, gran=gran)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                sage2.attention(out, ws, B, H, H, N, d, causal=causal, gran=gran)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 3)
        ms = statistics.median(ts)
        res["speed"][f"{gran}{'_causal' if causal else ''}"] = round((ops / 2 if causal else ops) / ms / 1e9, 1)
        del ws
del q, k, v
B, H, N = 1, 8, 4096
q, k, v = synth.make_qkv(B, H, H, N, d, kind="structured", seed=3, device="cuda")
ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float())
for gran in ("thread", "block", "token", "tensor"):
    o = sage2.attn(q, k, v, gran=gran).float()
    cos = torch.nn.functional.cosine_similarity(o.flatten(), ref.flatten(), dim=0).item()
    rl1 = ((o - ref).abs().sum() / ref.abs().sum()).item()
    rmse = (o - ref).pow(2).mean().sqrt().item()
    res["accuracy"][gran] = {"cos_sim": round(cos, 6), "rel_l1": round(rl1, 5), "rmse": round(rmse, 5)}
print(json.dumps(res))

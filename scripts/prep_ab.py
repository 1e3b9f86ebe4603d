"""A/B of the Delta S kernels (tf32 tensor-core GEMM vs SIMT fp32) on one config: timing + agreement."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_10958_b200 import sage2, synth

B, H, N, d = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4, 32, 32768, 128))]
q, k, v = synth.make_qkv(B, H, H, N, d, "structured" if "--structured" in sys.argv else "iid", seed=1, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
lay = sage2.layout(B, H, H, N, d)
nT = (N + 127) // 128
Np = nT * 128


def ds_view():
    return ws[lay["ds"]:lay["ds"] + B * H * nT * Np * 4].view(torch.float32).view(B * H, nT, Np)


res = {}
for simt in (True, False):
    for _ in range(2):
        sage2.prepare(q, k, v, ws, ds_simt=simt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        sage2.prepare(q, k, v, ws, ds_simt=simt)
    e1.record()
    torch.cuda.synchronize()
    res[simt] = (e0.elapsed_time(e1) / 5, ds_view()[:, :, :N].clone())
a, b = res[True][1], res[False][1]
err = (a.double() - b.double()).abs()
print(f"prepare ms: simt {res[True][0]:.3f}  tc {res[False][0]:.3f}; max|diff| {err.max().item():.3e} "
      f"max|ds| {a.abs().max().item():.3e} rel {(err / (a.double().abs() + 1e-3)).max().item():.3e}")

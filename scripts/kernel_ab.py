"""A/B timing of attention-kernel variants on one config (CUDA events, kernel only).

    python scripts/kernel_ab.py N d [variants,comma,separated] [rounds]

Variants are timed round-robin (5 launches each per round, `rounds` rounds) so clock drift hits
all of them alike; prints the median and best TOPS per variant."""
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
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
ws = sage2.alloc_workspace(B, H, H, N, d)
sage2.prepare(q, k, v, ws)
out = torch.empty_like(q)
L = sage2.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ops = 4.0 * B * H * N * N * d
VARIANTS = [("default", 0), ("v10", 16384), ("v10_causal", 16385), ("v6", 8192), ("v6_causal", 8193), ("v8", 4096), ("v8_causal", 4097), ("v8f8", 4096 + 2048),
            ("v6f8", 8192 + 2048), ("v1", 128), ("v1_causal", 129), ("v5", 512), ("v5_causal", 513),
            ("v4", 8), ("v4_causal", 9), ("v0", 4), ("v4_nullsm", 24), ("v4_nullmma", 40), ("v1_nullmma", 160)]
if len(sys.argv) > 3 and sys.argv[3]:
    VARIANTS = [x for x in VARIANTS if x[0] in sys.argv[3].split(",")]
times = {name: [] for name, _ in VARIANTS}
for r in range(rounds):
    for name, fl in VARIANTS:
        def run():
            rc = L.sage2_attention(out.data_ptr(), B, H, H, N, d, fl, ws.data_ptr(), ctypes.c_size_t(ws.numel()), st)
            assert rc == 0, (name, rc, L.sage2_last_cuda_error())
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        times[name].append(e0.elapsed_time(e1) / 5)
for name, fl in VARIANTS:
    o = ops / 2 if fl & 1 else ops
    med, best = statistics.median(times[name]), min(times[name])
    print(f"N={N} d={d} {name:12s} median {med:8.3f} ms {o / med / 1e9:7.1f} TOPS | best {o / best / 1e9:7.1f} TOPS",
          flush=True)

"""A/B timing of attention kernels on one config (CUDA events, kernel only, warm L2).

    python scripts/kernel_ab.py N d [variants] [rounds] [B] [H]

variants: comma list of NAME or NAME@LIB, where NAME is default / v8 / v12 / one (suffix _causal for the
causal mask, _f8 for the E4M3 carrier) and LIB the path of an A/B build of the library
(paper_2411_10958_b200.build.build(out=..., defines=...)); default: the in-tree libsage2.so.  Each
library prepares its own workspace.  Variants are timed round-robin (5 launches each per round) so
clock drift hits all of them alike; prints the median and best TOPS per variant."""
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
names = (sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] else "default").split(",")
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
B = int(sys.argv[5]) if len(sys.argv) > 5 else 4
H = int(sys.argv[6]) if len(sys.argv) > 6 else 32
KF = {"default": 0, "v8": 4096, "v12": 131072, "one": 1048576, "v14": 4194304}
q, k, v = synth.make_qkv(B, H, H, N, d, device="cuda")
out = torch.empty_like(q)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ops = 4.0 * B * H * N * N * d
libs, wss, variants = {}, {}, []
for nm in names:
    base, _, lib = nm.partition("@")
    lib = lib or (sage2.DEV_LIB_PATH if base.startswith("v14") else sage2.LIB_PATH)   # v14: dev library only
    if lib not in libs:
        libs[lib] = sage2._declare(ctypes.CDLL(lib))
    parts = base.split("_")
    fl = KF[parts[0]] | (1 if "causal" in parts else 0) | (2048 if "f8" in parts else 0)
    prep_fl = fl
    key = (lib, prep_fl)
    if key not in wss:
        L = libs[lib]
        ws = torch.empty(L.sage2_workspace_bytes(B, H, H, N, d, prep_fl & 1), dtype=torch.uint8, device="cuda")
        rc = L.sage2_prepare(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, H, H, N, d, prep_fl, ws.data_ptr(),
                             ctypes.c_size_t(ws.numel()), st)
        assert rc == 0, (nm, rc)
        wss[key] = ws
    variants.append((nm, libs[lib], fl, wss[key]))
times = {nm: [] for nm, *_ in variants}
for r in range(rounds):
    for nm, L, fl, ws in variants:
        def run():
            rc = L.sage2_attention(out.data_ptr(), B, H, H, N, d, fl, ws.data_ptr(), ctypes.c_size_t(ws.numel()), st)
            assert rc == 0, (nm, rc, L.sage2_last_cuda_error())
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        times[nm].append(e0.elapsed_time(e1) / 5)
for nm, L, fl, ws in variants:
    o = ops / 2 if fl & 1 else ops
    med, best = statistics.median(times[nm]), min(times[nm])
    print(f"B={B} H={H} N={N} d={d} {nm:40s} median {med:8.3f} ms {o / med / 1e9:7.1f} TOPS | best {o / best / 1e9:7.1f} TOPS",
          flush=True)

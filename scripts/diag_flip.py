"""Diagnose an O-parity excess: dump the kernel's P^ codes for one case and list, for the worst
row, every code that differs from the oracle's with the oracle's ambiguity flag."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as orc  # noqa: E402
from oracle import OracleConfig  # noqa: E402
from paper_2411_10958_b200 import sage2, synth  # noqa: E402

B, Hq, Hkv, N, d = 2, 4, 1, 1000, 128
smooth_v = len(sys.argv) > 1 and sys.argv[1] == "sv"
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, kind="structured", seed=5)
qg, kg, vg = q.cuda(), k.cuda(), v.cuda()
ws = sage2.alloc_workspace(B, Hq, Hkv, N, d)
sage2.prepare(qg, kg, vg, ws, smooth_v=smooth_v)
out = torch.empty_like(qg)
s, ph = sage2.debug_qk_int32(out, ws, B, Hq, Hkv, N, d, with_p=True, smooth_v=smooth_v)
torch.cuda.synchronize()
ph = ph.cpu().numpy()
o = out.cpu().numpy().astype(np.float64)
nT = (N + 127) // 128
for b in range(B):
    for h in range(Hq):
        units = [(b, h, i) for i in range(nT)]
        res = orc.sage2_forward_blocks(q.numpy(), k.numpy(), v.numpy(), units,
                                       OracleConfig(smooth_v=smooth_v), keep=True, debug=True)
        for u, (_, _, i) in enumerate(units):
            r1 = min(N, 128 * i + 128) - 128 * i
            ref16 = res["O16"][u, :r1]
            err = np.abs(o[b, h, 128 * i:128 * i + r1] - ref16)
            ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(ref16), 2.0 ** -14))) - 10)
            bar = np.maximum(2e-3, ulp)
            dbg = res["inter"][u]["dbg"]
            g = ph[b * Hq + h, 128 * i:128 * i + r1, :N]
            oc = dbg["phat"][:r1, :N]
            amb = dbg["amb"][:r1, :N].astype(bool)
            diff = g != oc
            for r in np.flatnonzero((err > bar).any(1)):
                cols = np.flatnonzero(diff[r])
                print(f"b={b} h={h} blk={i} row={r}: max err {err[r].max():.3e} bar {bar[r].max():.2e} "
                      f"flip allowance {dbg['flip'][r]:.3e}; codes differing at {cols.tolist()} "
                      f"(gpu {g[r, cols].tolist()} oracle {oc[r, cols].tolist()} ambiguous {amb[r, cols].tolist()})")
            if (diff & ~amb).any():
                print(f"b={b} h={h} blk={i}: {(diff & ~amb).sum()} UNAMBIGUOUS code differences")
print("done")

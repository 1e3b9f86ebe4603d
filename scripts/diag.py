"""Stage-by-stage diagnostics of the CUDA path vs the oracle on small configs (prints, no asserts).
Run under gpurun; output is the first thing to read when a parity test fails."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as orc  # noqa: E402
from oracle import OracleConfig  # noqa: E402
from paper_2411_10958_b200 import sage2, synth  # noqa: E402
from tests._gpu_helpers import read_prepared, to_np16  # noqa: E402


def run(B, Hq, Hkv, N, d, kind, causal):
    print(f"=== B={B} Hq={Hq} Hkv={Hkv} N={N} d={d} {kind} causal={causal}")
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, kind=kind, seed=0)
    qg, kg, vg = q.cuda(), k.cuda(), v.cuda()
    ws = sage2.alloc_workspace(B, Hq, Hkv, N, d)
    sage2.prepare(qg, kg, vg, ws)
    torch.cuda.synchronize()
    g = read_prepared(ws, sage2.layout(B, Hq, Hkv, N, d), B, Hq, Hkv, N, d)
    kv = orc.kv_head(k.numpy()[0, 0], v.numpy()[0, 0])
    qb = orc.q_block(q.numpy()[0, 0, :min(N, 128)])
    print(" kbar eq", np.array_equal(g["kbar"][0], kv["kbar"]), " dv eq", np.array_equal(g["dv"][0], kv["dv"]))
    print(" dk eq", np.array_equal(g["dk"][0], kv["dk"]), " khat mism", int((g["khat"][0] != kv["khat"]).sum()),
          " vhat mism", int((g["vhat"][0] != kv["vhat"]).sum()))
    print(" qbar eq", np.array_equal(g["qbar"][0, 0], qb["qbar"]), " dq eq", np.array_equal(g["dq"][0, :32], qb["dq"]),
          " qhat mism", int((g["qhat"][0, :128] != qb["qhat"]).sum()))
    ds = orc.delta_s(qb["qbar"], kv["kprime"])
    gds = g["ds"][0, 0, :N] / (1.4426950408889634 / math.sqrt(d))
    print(" ds max abs diff", float(np.max(np.abs(gds - ds))), " ds scale", float(np.max(np.abs(ds))))
    out = torch.empty_like(qg)
    try:
        s = sage2.debug_qk_int32(out, ws, B, Hq, Hkv, N, d)
        torch.cuda.synchronize()
        s = s.cpu().numpy()[0, :128].astype(np.int64)
        ref = orc.s_int_block(qb["qhat"], kv["khat"])
        bad = s != ref
        print(" S_int mism", int(bad.sum()), "of", bad.size)
        if bad.any():
            r, c = np.nonzero(bad)
            print("  first bad", list(zip(r[:8], c[:8])), s[r[:4], c[:4]], ref[r[:4], c[:4]])
    except Exception as e:
        print(" S_int dump failed:", e)
        return
    out = sage2.attn(qg, kg, vg, causal=causal)
    torch.cuda.synchronize()
    o = to_np16(out).astype(np.float64)
    res = orc.sage2_forward_blocks(q.numpy(), k.numpy(), v.numpy(), [(0, 0, 0)], OracleConfig(causal=causal))
    n0 = min(N, 128)
    err = np.abs(o[0, 0, :n0] - res["O16"][0, :n0])
    print(" O max abs err", float(err.max()), " cos", orc.cos_sim(res["O"][0, :n0], o[0, 0, :n0]),
          " |O| max", float(np.abs(res["O"][0, :n0]).max()))


if __name__ == "__main__":
    torch.cuda.init()
    for args in [(1, 1, 1, 256, 64, "iid", False), (1, 1, 1, 256, 128, "iid", False),
                 (1, 1, 1, 300, 128, "structured", True)]:
        try:
            run(*args)
        except Exception as e:
            print("FAILED", args, repr(e))

"""Accuracy of the SageAttn2-4b forward (the default kernel of every config) against full-precision
attention, with the paper's three metrics: CosSim, Rel-L1, RMSE.  BASELINE.json metric
"cos-sim vs FP32 attention", per config: C1, all 16 C2 points, C3, C4, each on the iid and
the structured (channel-outlier, DESIGN.md Inputs) synthetic inputs.

The reference is softmax attention in fp64 (paper_2411_10958_b200/accuracy.py, pinned to the oracle's
exact mode by tests/test_accuracy_ref.py) on sampled heads: every query row up to N = 4096, the
first / middle / last Q block above.  Variants (INT8 8b, smooth V, per-block / per-token groups,
single-level) are reported on C2-4K d=128 structured.

    python scripts/accuracy.py [--out profiles/r02_accuracy.json] [--quick]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (config table)
from paper_2411_10958_b200 import accuracy, sage2, synth  # noqa: E402


def heads_of(B, Hq, n=4):
    """Sampled (b, h_q) pairs: first, last and two in between."""
    allh = [(b, h) for b in range(B) for h in range(Hq)]
    if len(allh) <= n:
        return allh
    idx = sorted({0, len(allh) - 1, len(allh) // 3, (2 * len(allh)) // 3})
    return [allh[i] for i in idx]


def run(name, kind, **variant):
    B, Hq, Hkv, N, d, causal, _ = bench.CONFIGS[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, kind=kind, seed=11, device="cuda")
    out = sage2.attn(q, k, v, causal=causal, **variant)
    torch.cuda.synchronize()
    rows = accuracy.sample_rows(N)
    m = accuracy.evaluate(out, q, k, v, causal, heads_of(B, Hq), rows)
    m["rows_per_head"] = int(rows.numel())
    m["heads"] = len(heads_of(B, Hq))
    del q, k, v, out
    torch.cuda.empty_cache()
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true", help="C1, C2-1K/4K only")
    a = ap.parse_args()
    names = ["c1_256_d64"] + sorted(n for n in bench.CONFIGS if n.startswith("c2_")) + ["c3_cogvideox", "c4_llama_gqa"]
    if a.quick:
        names = [n for n in names if n.startswith("c1") or "_1k_" in n or "_4k_" in n]
    res = {"reference": "softmax attention in fp64 (P:77), sampled heads/rows; metrics P:895",
           "kernel": {}, "configs": {}, "variants_c2_4k_d128_structured": {}}
    t0 = time.time()
    for n in names:
        B, Hq, Hkv, N, d, causal, _ = bench.CONFIGS[n]
        res["kernel"][n] = f"v{sage2.attention_kernel(N, d, causal=causal)}"
        res["configs"][n] = {kind: run(n, kind) for kind in ("iid", "structured")}
        print(n, json.dumps(res["configs"][n]), flush=True)
    for vn, kw in (("sage2_8b", {"int8": True}), ("smooth_v", {"smooth_v": True}), ("per_block", {"gran": "block"}),
                   ("per_token", {"gran": "token"}), ("single_level", {"kernel": "one"})):
        res["variants_c2_4k_d128_structured"][vn] = run("c2_4k_d128", "structured", **kw)
        print(vn, json.dumps(res["variants_c2_4k_d128_structured"][vn]), flush=True)
    res["wall_s"] = round(time.time() - t0, 1)
    s = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(s)
    print(s)


if __name__ == "__main__":
    main()

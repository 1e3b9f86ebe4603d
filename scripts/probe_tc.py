"""Hardware probes on a B200 (run under gpurun):
  1. The paper's FP22 experiment on tcgen05.mma.kind::f8f6f4: does C = 0*0 + D keep D?
     does x*1 + D round like fp32?  (decides whether two-level accumulation buys accuracy here)
  2. Dense tcgen05 kind::i8 and kind::f8f6f4 throughput (the tensor roofline denominators).
Writes gpurun_out/probe.json."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2  # noqa: E402


def main():
    g = np.random.default_rng(0)
    # D patterns: 1 + k*2^-23 (every low mantissa bit), random normals, wide exponents
    base = np.float32(1.0).view(np.uint32)
    d = [base + k for k in range(0, 1024, 7)]
    d += list(g.standard_normal(2000).astype(np.float32).view(np.uint32))
    d += list((g.standard_normal(1000) * 10.0 ** g.integers(-20, 20, 1000)).astype(np.float32).view(np.uint32))
    d = np.array(d, np.uint32)
    prod = g.choice(np.array([0x38, 0x30, 0x40, 0x7E, 0x01, 0x3A, 0xB8], np.uint8), size=d.size)
    cz, cp = sage2.probe_accumulator(d, prod)
    trunc10 = d & np.uint32(0xFFFFFC00)
    res = {}
    res["zero_product_keeps_D"] = float(np.mean(cz == d))
    res["zero_product_equals_trunc10"] = float(np.mean(cz == trunc10))
    # low mantissa bits retained by C = 0*0 + D
    diff = (cz ^ d)
    res["zero_product_max_lost_bits"] = int(np.max([int(x).bit_length() for x in diff]))
    import torch
    x = torch.from_numpy(prod.copy()).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    df = d.view(np.float32).astype(np.float64)
    exact = x + df
    rn = exact.astype(np.float32)                      # fp32 round-to-nearest of the exact sum
    fin = np.isfinite(rn)
    cpf = cp.view(np.float32)
    res["prod_equals_fp32_rn"] = float(np.mean(cpf[fin] == rn[fin]))
    # truncation toward zero of exact sum to 23 / 13 mantissa bits
    def trunc_to(v, mbits):
        m, e = np.frexp(v)
        return np.ldexp(np.trunc(m * 2.0 ** (mbits + 1)) / 2.0 ** (mbits + 1), e)
    res["prod_equals_trunc23"] = float(np.mean(cpf[fin] == trunc_to(exact, 23)[fin].astype(np.float32)))
    res["prod_equals_trunc13"] = float(np.mean(cpf[fin] == trunc_to(exact, 13)[fin].astype(np.float32)))
    rel = np.abs(cpf[fin].astype(np.float64) - exact[fin]) / np.maximum(np.abs(exact[fin]), 1e-30)
    res["prod_max_rel_err"] = float(rel.max())
    res["prod_max_rel_err_log2"] = float(np.log2(rel.max())) if rel.max() > 0 else None
    res["n"] = int(d.size)
    res["mma_i8_ops_per_s"] = sage2.bench_mma(0, 20000)
    res["mma_f8f6f4_ops_per_s"] = sage2.bench_mma(1, 20000)
    for w, name in sage2.MICRO.items():
        try:
            res[name] = sage2.microbench(w, 4096)
        except Exception as e:
            res[name] = repr(e)
    print(json.dumps(res, indent=1))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/probe.json", "w"), indent=1)


if __name__ == "__main__":
    main()

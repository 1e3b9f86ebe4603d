#!/usr/bin/env python
"""Benchmark: SageAttention2 (arXiv 2411.10958) forward on B200, BASELINE.json's metric
("attention TOPS hd64/128 seq 1K-32K causal/non-causal").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

One step = one whole pass of the hot path over one batch: preprocessing (smooth + per-thread INT4
Q/K + per-channel FP8 V + Delta S) and the tcgen05 attention kernel, on inputs resident in HBM.
Ops counted with the FlashAttention convention 4*B*H_q*N^2*d (x1/2 causal) -- DESIGN.md C-19.
Multi-GPU (torchrun): every rank runs the same per-GPU workload on its own (batch, head) units
(weak scaling, no collective on the data path); time = max over ranks of CUDA-event time.
--impl reference times the CPU oracle (oracle/) on a bounded sample of the same workload.
Prints ONE JSON line (rank 0).
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (B, H_q, H_kv, N, d, causal, kind)
    "c1_256_d64": (1, 1, 1, 256, 64, False, "structured"),
    "c3_cogvideox": (1, 48, 48, 17776, 64, False, "structured"),
    "c4_llama_gqa": (1, 32, 8, 100000, 128, True, "iid"),
    "c5_b8": (8, 32, 32, 32768, 128, False, "iid"),
}
# C2 kernel sweep (BASELINE.json configs[1]): B=4, H=32, d in {64, 128}, N in {1K, 4K, 16K, 32K},
# causal and non-causal, N(0,1) inputs (the paper's kernel-benchmark protocol)
for _n, _tag in ((1024, "1k"), (4096, "4k"), (16384, "16k"), (32768, "32k")):
    for _d in (64, 128):
        for _c in (False, True):
            CONFIGS[f"c2_{_tag}_d{_d}" + ("_causal" if _c else "")] = (4, 32, 32, _n, _d, _c, "iid")
DEFAULT = "c2_32k_d128"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_BF16_TFLOPS = 1590.0          # B200_PROFILING.md fallback (burst)


def ops_of(B, Hq, N, d, causal):
    o = 4.0 * B * Hq * N * N * d
    return o / 2 if causal else o


def tensor_peak():
    """INT8/FP8 dense peak = 2 x the measured bf16 GEMM (the guide's nominal fp8:bf16 ratio).
    The attention kernel is timed inside a long step -> the sustained figure."""
    try:
        pk = json.load(open(PEAKS_FILE))
        return 2.0 * float(pk["bf16_tflops_sustained"]), "2 x bf16_tflops_sustained of measured (MEASURED_PEAKS.json)"
    except Exception:
        return 2.0 * FALLBACK_BF16_TFLOPS, "2 x bf16 fallback 1590 TFLOP/s (B200_PROFILING.md), of fallback"


class ClockSampler:
    """Samples SM clock and clock-event reasons via NVML while the timed region runs."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def dist_setup(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    from paper_2411_10958_b200.shard import max_over_ranks as mx
    return mx(x, world, device="cuda")


# ------------------------------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle, as it stands, on a bounded sample
# ------------------------------------------------------------------------------------------------
def oracle_sample(cfg_name, budget_s, max_blocks=None):
    """Time the CPU oracle on whole Q blocks of the workload (its KV-head preprocessing included)
    until `budget_s` seconds of work are done.  Returns (ops/s, ops, seconds, blocks, threads)."""
    import numpy as np
    import oracle as orc
    from oracle import OracleConfig
    from paper_2411_10958_b200 import synth
    B, Hq, Hkv, N, d, causal, kind = CONFIGS[cfg_name]
    orc.build()
    q, k, v = synth.make_qkv(1, Hq // Hkv, 1, N, d, kind=kind, seed=0, units=[(0, 0)])
    q, k, v = q.numpy(), k.numpy()[:, None], v.numpy()[:, None]
    nT = (N + 127) // 128
    order = [nT - 1, nT // 2, 0] + [t for t in range(nT - 2, 0, -1) if t != nT // 2]
    cfg = OracleConfig(causal=causal)
    done_ops, t0, blocks = 0.0, time.perf_counter(), 0
    for i in order:
        r0, r1 = 128 * i, min(N, 128 * i + 128)
        orc.sage2_forward_blocks(q, k, v, [(0, 0, i)], cfg)
        # same convention as the GPU count: 4 d per (query, visible key) pair
        pairs = sum(r + 1 for r in range(r0, r1)) if causal else (r1 - r0) * N
        done_ops += 4.0 * pairs * d
        blocks += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (max_blocks and blocks >= max_blocks):
            break
    el = time.perf_counter() - t0
    return done_ops / el, done_ops, el, blocks, orc.num_threads()


def run_reference(args, world, rank):
    if rank != 0:
        return
    name = args.config
    B, Hq, Hkv, N, d, causal, kind = CONFIGS[name]
    per = []
    for s in range(args.warmup + args.steps):
        ops_s, ops, el, blocks, thr = oracle_sample(name, budget_s=0.0, max_blocks=1)
        if s >= args.warmup:
            per.append((ops, el))
    tot_ops = sum(o for o, _ in per)
    tot_t = sum(t for _, t in per)
    v = tot_ops / tot_t / 1e12
    line = {
        "impl": "reference", "metric": "attention TOPS (SageAttn2-4b forward)", "value": v, "unit": "TOPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / len(per),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)",
        "data": "synthetic", "config": workload_config(name),
        "cpu_baseline": {"value": v, "unit": "TOPS", "cores": thr, "kind": "oracle",
                         "sample": f"1 Q block (128 query rows x all {N} keys, its KV head preprocessed) per step"},
        "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(name):
    B, Hq, Hkv, N, d, causal, kind = CONFIGS[name]
    return {"workload": name, "B": B, "H_q": Hq, "H_kv": Hkv, "N": N, "d": d, "causal": causal,
            "inputs": f"{kind} fp16 (DESIGN.md Inputs), seeded per (b, h_kv) unit",
            "l2": "inputs larger than L2 (no flush needed)" if 3 * B * Hq * N * d * 2 > 200e6 else
                  "small inputs: L2 flushed between steps (outside the timed events)",
            "variant": "SageAttn2-4b: INT4 per-thread QK (int8 lanes, tcgen05 kind::i8), FP8 E4M3 PV (kind::f8f6f4), two-level accumulation"}


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def run_ours(args, world, rank, local):
    import torch
    from paper_2411_10958_b200 import sage2, synth
    name = args.config
    B, Hq, Hkv, N, d, causal, kind = CONFIGS[name]
    dev = torch.device("cuda", local if world > 1 else 0)
    # this rank's (b, h_kv) units: batch index offset by rank (weak scaling, independent units)
    from paper_2411_10958_b200.shard import rank_units
    units = rank_units(rank, world, B, Hkv)
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, kind=kind, seed=0, device=dev, units=units)
    grp = Hq // Hkv
    q = q.view(B, Hkv, grp, N, d).reshape(B, Hq, N, d).contiguous()
    k = k.view(B, Hkv, N, d).contiguous()
    v = v.view(B, Hkv, N, d).contiguous()
    out = torch.empty_like(q)
    ws = sage2.alloc_workspace(B, Hq, Hkv, N, d, dev, causal=causal)
    small = 3 * B * Hq * N * d * 2 <= 200e6
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev) if small else None
    stream = torch.cuda.current_stream()

    def step(ev=None):
        # ev = (step start, attention start, attention end): the L2 flush of small configs sits
        # BETWEEN timed steps, outside every event pair
        if flush is not None:
            flush.zero_()
        if ev:
            ev[0].record(stream)
        sage2.prepare(q, k, v, ws, causal=causal)
        if ev:
            ev[1].record(stream)
        sage2.attention(out, ws, B, Hq, Hkv, N, d, causal=causal)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    kev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        e0.record(stream)
        for s in range(args.steps):
            step(kev[s])
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    if flush is None:      # back-to-back steps: one event pair around all of them
        ms = e0.elapsed_time(e1) / args.steps
    else:                  # flushed steps: the sum of the per-step event pairs (flush excluded)
        ms = sum(a.elapsed_time(c) for a, _, c in kev) / args.steps
    kms = statistics.mean(b.elapsed_time(c) for _, b, c in kev)
    prep_ms = statistics.mean(a.elapsed_time(b) for a, b, _ in kev)
    ms_max = max_over_ranks(ms, world)
    kms_max = max_over_ranks(kms, world)
    ops = ops_of(B, Hq, N, d, causal)
    value = world * ops / (ms_max * 1e-3) / 1e12
    # roofline of the dominant kernel (the tcgen05 attention kernel)
    peak, peak_src = tensor_peak()
    achieved = ops / (kms_max * 1e-3) / 1e12
    traffic = None
    try:   # DRAM bytes per launch of this kernel from the committed ncu --set full capture
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[name]["dram_bytes_per_launch"]
    except Exception:
        pass
    # end to end through the public C ABI on host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        qh, kh, vh = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
        oh = torch.empty(q.shape, dtype=torch.float16).pin_memory()
        for _ in range(2):                       # warm-up (pool growth, first-touch of pinned pages)
            sage2.attn_host(qh, kh, vh, oh, causal=causal)
        torch.cuda.synchronize()
        n_e2e = max(3, min(args.steps, 5))
        barrier(world)
        times = []
        for _ in range(n_e2e):
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            sage2.attn_host(qh, kh, vh, oh, causal=causal)
            t1.record(stream)
            torch.cuda.synchronize()
            times.append(t0.elapsed_time(t1))
        e2e_ms = max_over_ranks(statistics.median(times), world)
        e2e = {"value": world * ops / (e2e_ms * 1e-3) / 1e12, "unit": "TOPS",
               "h2d_bytes_per_step": int((q.numel() + 2 * k.numel()) * 2),
               "d2h_bytes_per_step": int(oh.numel() * 2), "ms_per_step": e2e_ms,
               "api": "sage2_attn_host (C ABI, pinned host buffers)"}
    # validation (outside every timed region): NCCL all-gather of the outputs over NVLink, rank 0
    # re-runs each rank's first (b, h_kv) unit alone and checks the gathered slice bit for bit
    validation = None
    if world > 1 and not args.no_validate:
        from paper_2411_10958_b200.shard import gather_outputs, first_unit_check
        g0 = time.perf_counter()
        parts = gather_outputs(out, world)
        torch.cuda.synchronize()
        g_ms = (time.perf_counter() - g0) * 1e3
        bad = None
        if rank == 0:
            def recompute(r):
                u0 = rank_units(r, world, B, Hkv)[0]
                qu, ku, vu = synth.make_qkv(B, Hq, Hkv, N, d, kind=kind, seed=0, device=dev, units=[u0])
                return sage2.attn(qu.view(1, grp, N, d), ku.view(1, 1, N, d), vu.view(1, 1, N, d),
                                  causal=causal)[0]
            bad = first_unit_check(parts, recompute)
        del parts
        validation = {"collective": "all_gather (NCCL)", "gathered_bytes": int(out.numel() * 2 * world),
                      "gather_ms_wall": g_ms, "ranks_mismatched": bad,
                      "check": "rank 0 recomputes every rank's first unit alone: bitwise equal"}
    kver = sage2.attention_kernel(N, d, causal=causal)
    line = {
        "metric": "attention TOPS (SageAttn2-4b forward)", "value": value, "unit": "TOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int4-in-int8 (QK^T) + e4m3 (PV), fp32 softmax",
        "data": "synthetic", "config": workload_config(name),
        "gpu_launches": 5 * args.steps,
        "roofline": {"bound": "tensor", "kernel": f"k_attn{kver} (tcgen05 attention, v{kver})", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src, "kernel_ms": kms_max,
                     "kernel_share_of_step": kms_max / ms_max},
        "clocks": clk.summary(),
        "e2e": e2e,
        "phases_ms": {"preprocessing": prep_ms, "attention": kms},
    }
    if validation is not None:
        line["validation"] = validation
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            ops_s, o, el, blocks, thr = oracle_sample(name, budget_s=args.cpu_budget)
            line["cpu_baseline"] = {"value": ops_s / 1e12, "unit": "TOPS", "cores": thr, "kind": "oracle",
                                    "sample": f"{blocks} Q blocks (128 rows x all keys each, KV head preprocessing "
                                              f"included), {el:.1f} s"}
        except Exception as e:  # reported, never silently replaced
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT, choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-validate", action="store_true", help="skip the N>1 NCCL gather validation")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

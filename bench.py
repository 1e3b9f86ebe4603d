#!/usr/bin/env python
"""Benchmark: SageAttention2 (arXiv 2411.10958) forward on B200, BASELINE.json's metric
("attention TOPS hd64/128 seq 1K-32K causal/non-causal").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

One step = one whole pass of the hot path over one batch: preprocessing (smooth + per-thread INT4
Q/K + per-channel FP8 V + Delta S) and the tcgen05 attention kernel, on inputs resident in HBM.
Ops counted with the FlashAttention convention 4*B*H_q*N^2*d (x1/2 causal) -- DESIGN.md C-19.

Multi-GPU: `--gpus N` with N > 1 starts N ranks itself (torch.distributed.run, 127.0.0.1) unless it
already runs under torchrun (WORLD_SIZE set); one process per GPU, NCCL.  The default config is then
north-star C5 (B=8, H=32, N=32K, d=128), STRONG scaling: its 256 (b, h_kv) units are split evenly
over the ranks and each rank runs its share (no collective on the data path); time = max over ranks
of the CUDA-event time; value = the whole batch's ops / that time.  Other configs under torchrun run
weak scaling (every rank a full copy of the config on its own batch slice).  After the timed region
the outputs are all-gathered over NVLink (NCCL) and rank 0 checks every rank's first unit bitwise
against a recomputation (`validation`).
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
    """INT8/FP8 dense peak = 2 x the measured bf16 GEMM burst figure (the guide's nominal fp8:bf16
    ratio).  The burst figure: the attention kernel runs at the boost clock (the bench's clock record
    shows ~1.9-2.0 GHz), while the sustained figure embeds a 1.3 GHz median."""
    try:
        pk = json.load(open(PEAKS_FILE))
        return 2.0 * float(pk["bf16_tflops"]), "2 x bf16_tflops (burst) of measured (MEASURED_PEAKS.json)"
    except Exception:
        return 2.0 * FALLBACK_BF16_TFLOPS, "2 x bf16 fallback 1590 TFLOP/s (B200_PROFILING.md), of fallback"


def binding_roofs(achieved, d, clocks):
    """The two other ceilings DESIGN.md section 9 derives for this kernel, at the measured SM clock:
    the tcgen05 kind::i8 rate measured by the dev library's microbenchmark (profiles/
    r01_probe_tc.json: 4.49e15 ops/s at 1965 MHz = 15 250 ops/clk/SM) and the MUFU ex2 rate (16 exp/clk/SM; one exp per (query, key) pair carrying
    4 d ops)."""
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    i8 = 15250.0 * 148 * mhz * 1e6 / 1e12
    mufu = 16.0 * 4 * d * 148 * mhz * 1e6 / 1e12
    return {"i8_measured_peak": i8, "frac_of_i8_measured": achieved / i8,
            "mufu_roof": mufu, "frac_of_mufu_roof": achieved / mufu, "roof_clock_mhz": mhz}


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
        if torch.cuda.is_available():
            # SAGE2_DIST_BACKEND=gloo (test hook): several ranks on fewer GPUs (rank -> device
            # local % count) so the multi-rank path can be exercised on a one-GPU box; NCCL otherwise
            backend = os.environ.get("SAGE2_DIST_BACKEND", "nccl")
            torch.cuda.set_device(local % torch.cuda.device_count())
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(backend)
        else:                               # CPU dry runs of the launch path (tests: --dist-check)
            dist.init_process_group("gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def torchrun_cmd(argv, n):
    """The command bench.py re-executes itself with for `--gpus n` outside torchrun."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


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
    from paper_2411_10958_b200 import sage2
    # the oracle's KV tile is the kernel's b_kv (reading C-9): 64 for the d = 64 kernel v12
    cfg = OracleConfig(causal=causal, kv_tile=64 if sage2.attention_kernel(N, d, causal=causal) == 12 else 128)
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
        "cpu_baseline": {"value": v, "unit": "TOPS", "cores": thr, "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"1 Q block (128 query rows x all {N} keys, its KV head preprocessed) per step",
                         "extrapolated_full_step_s": ops_of(B, Hq, N, d, causal) / (v * 1e12)},
        "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(name, scaling="weak", world=1):
    B, Hq, Hkv, N, d, causal, kind = CONFIGS[name]
    c = {"workload": name, "B": B, "H_q": Hq, "H_kv": Hkv, "N": N, "d": d, "causal": causal,
         "inputs": f"{kind} fp16 (DESIGN.md Inputs), seeded per (b, h_kv) unit",
         "l2": "inputs larger than L2 (no flush needed)" if 3 * B * Hq * N * d * 2 / (world if scaling == "strong" else 1) > 200e6 else
               "small inputs: L2 flushed between steps (outside the timed events)",
         "variant": "SageAttn2-4b: INT4 per-thread QK (int8 lanes, tcgen05 kind::i8), FP8 E4M3 PV (kind::f8f6f4), two-level accumulation"}
    if world > 1:
        c["parallelism"] = (f"(b, h_kv)-unit sharding over {world} GPUs: " +
                            ("the config's B*H_kv units split evenly (strong)" if scaling == "strong" else
                             "every rank a full copy on its own batch slice (weak)"))
    return c


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def run_ours(args, world, rank, local):
    import torch
    from paper_2411_10958_b200 import sage2, shard, synth
    name = args.config
    B, Hq, Hkv, N, d, causal, kind = CONFIGS[name]
    grp = Hq // Hkv
    dev = torch.device("cuda", (local % torch.cuda.device_count()) if world > 1 else 0)
    strong = args.scaling == "strong"
    if strong:
        # this rank's share of the config's fixed unit list, run as [n_units, grp, N, d] (H_kv = 1 per unit)
        units = shard.split_units(shard.all_units(B, Hkv), rank, world)
        lB, lHq, lHkv = len(units), grp, 1
    else:
        # weak: a full copy of the config on this rank's own batch slice
        units = shard.rank_units(rank, world, B, Hkv)
        lB, lHq, lHkv = B, Hq, Hkv
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, kind=kind, seed=0, device=dev, units=units)
    q = q.reshape(lB, lHq, N, d).contiguous()
    k = k.reshape(lB, lHkv, N, d).contiguous()
    v = v.reshape(lB, lHkv, N, d).contiguous()
    out = torch.empty_like(q)
    ws = sage2.alloc_workspace(lB, lHq, lHkv, N, d, dev, causal=causal)
    small = 3 * lB * lHq * N * d * 2 <= 200e6
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
        sage2.attention(out, ws, lB, lHq, lHkv, N, d, causal=causal)
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
    # accuracy of this workload's output against fp64 softmax attention (BASELINE metric "cos-sim vs
    # FP32 attention"; the paper's metrics), outside every timed region: sampled heads / rows
    acc = None
    if rank == 0:
        from paper_2411_10958_b200 import accuracy
        heads = sorted({(0, 0), (lB - 1, lHq - 1)})
        acc = accuracy.evaluate(out, q, k, v, causal, heads, accuracy.sample_rows(N, full_up_to=1024))
        acc.update({"reference": "softmax attention in fp64", "heads": len(heads),
                    "rows_per_head": int(accuracy.sample_rows(N, full_up_to=1024).numel())})
    prep_ms = statistics.mean(a.elapsed_time(b) for a, b, _ in kev)
    ms_max = max_over_ranks(ms, world)
    kms_max = max_over_ranks(kms, world)
    my_ops = ops_of(lB, lHq, N, d, causal)
    total_ops = shard.sum_over_ranks(my_ops, world, device=dev)      # = the config's ops when strong
    value = total_ops / (ms_max * 1e-3) / 1e12
    # roofline of the dominant kernel (the tcgen05 attention kernel), on the slowest rank's share
    peak, peak_src = tensor_peak()
    achieved = (total_ops / world) / (kms_max * 1e-3) / 1e12
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
        e2e = {"value": total_ops / (e2e_ms * 1e-3) / 1e12, "unit": "TOPS",
               "h2d_bytes_per_step": int(shard.sum_over_ranks((q.numel() + 2 * k.numel()) * 2, world, device=dev)),
               "d2h_bytes_per_step": int(shard.sum_over_ranks(oh.numel() * 2, world, device=dev)),
               "ms_per_step": e2e_ms, "api": "sage2_attn_host (C ABI, pinned host buffers)"}
        del qh, kh, vh, oh
    # validation (outside every timed region): NCCL all-gather of the outputs over NVLink, rank 0
    # re-runs each rank's first (b, h_kv) unit alone and checks the gathered slice bit for bit
    validation = None
    if world > 1 and not args.no_validate:
        del ws
        torch.cuda.empty_cache()
        g0 = time.perf_counter()
        parts = shard.gather_units(out, lB, world)
        torch.cuda.synchronize()
        g_ms = (time.perf_counter() - g0) * 1e3
        bad = None
        if rank == 0:
            def recompute(r):
                if strong:
                    u0 = shard.split_units(shard.all_units(B, Hkv), r, world)[0]
                else:
                    u0 = shard.rank_units(r, world, B, Hkv)[0]
                qu, ku, vu = synth.make_qkv(B, Hq, Hkv, N, d, kind=kind, seed=0, device=dev, units=[u0])
                return sage2.attn(qu.view(1, grp, N, d), ku.view(1, 1, N, d), vu.view(1, 1, N, d),
                                  causal=causal)[0]
            bad = shard.first_unit_check(parts, recompute)
        del parts
        import torch.distributed as dist
        validation = {"collective": f"all_gather ({dist.get_backend()})", "gathered_bytes": int(out.numel() * 2 * world),
                      "gather_ms_wall": g_ms, "ranks_mismatched": bad,
                      "check": "rank 0 recomputes every rank's first unit alone: bitwise equal"}
    kver = sage2.attention_kernel(N, d, causal=causal)
    line = {
        "metric": "attention TOPS (SageAttn2-4b forward)", "value": value, "unit": "TOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "int4-in-int8 (QK^T) + e4m3 (PV), fp32 softmax",
        "data": "synthetic", "config": workload_config(name, args.scaling, world),
        # our kernels per step (sage2_api.cu launch_prepare + the attention kernel): k_kv_stats, k_q_quant,
        # Delta S, k_kv_quant (two launches: K and V halves), attention
        "gpu_launches": 6 * args.steps,
        "roofline": {"bound": "tensor", "kernel": f"k_attn{kver} (tcgen05 attention, v{kver})", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src, "kernel_ms": kms_max,
                     "kernel_share_of_step": kms_max / ms_max},
        "clocks": clk.summary(),
        "e2e": e2e,
        "phases_ms": {"preprocessing": prep_ms, "attention": kms},
    }
    if acc is not None:
        line["accuracy"] = acc
    line["roofline"].update(binding_roofs(achieved, d, clk.summary()))
    if validation is not None:
        line["validation"] = validation
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            ops_s, o, el, blocks, thr = oracle_sample(name, budget_s=args.cpu_budget)
            full_s = ops_of(B, Hq, N, d, causal) / ops_s
            line["cpu_baseline"] = {"value": ops_s / 1e12, "unit": "TOPS", "cores": thr, "kind": "oracle",
                                    "cpu": cpu_model(),
                                    "sample": f"{blocks} Q blocks (128 rows x all keys each, KV head preprocessing "
                                              f"included), {el:.1f} s",
                                    "extrapolated_full_step_s": full_s,
                                    "extrapolated_note": "the whole config at the sampled rate (extrapolated, not run)"}
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
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help=f"default: {DEFAULT} on one GPU, c5_b8 (strong scaling) on several")
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="default: strong for c5_b8, weak otherwise")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-validate", action="store_true", help="skip the N>1 NCCL gather validation")
    ap.add_argument("--dist-check", action="store_true",
                    help="start the ranks, initialise the process group, print one JSON line per rank, exit")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-execute this script under torchrun (127.0.0.1 rendezvous)
        import subprocess
        sys.exit(subprocess.call(torchrun_cmd(sys.argv[1:], args.gpus)))
    world, rank, local = dist_setup(args.gpus)
    if args.config is None:
        args.config = "c5_b8" if world > 1 else DEFAULT
    if args.scaling is None:
        args.scaling = "strong" if args.config.startswith("c5") else "weak"
    if args.dist_check:
        import torch.distributed as dist
        ok = True
        if world > 1:
            from paper_2411_10958_b200 import shard
            ok = shard.max_over_ranks(rank, world) == world - 1
        B, Hq, Hkv = CONFIGS[args.config][:3]
        from paper_2411_10958_b200 import shard
        units = shard.split_units(shard.all_units(B, Hkv), rank, world) if args.scaling == "strong" else \
            shard.rank_units(rank, world, B, Hkv)
        print(json.dumps({"rank": rank, "world": world, "gpus_arg": args.gpus, "config": args.config,
                          "scaling": args.scaling, "n_units": len(units), "first_unit": units[0] if units else None,
                          "reduce_ok": ok}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}; measuring {world} ranks", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

/*
 * sage2_dev.h -- measurement-only entry points of libsage2_dev.so (the same source as libsage2.so
 * built with -DSAGE2_DEV).  Not part of the product ABI (include/sage2.h): scripts/ and the
 * measurement tests load the dev library explicitly; the product path never does.
 *
 * Same conventions as sage2.h: 0 or a negative SAGE2_E* code, nothing printed, no CPU fallback.
 */
#ifndef SAGE2_DEV_H_
#define SAGE2_DEV_H_

#include "sage2.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SAGE2_F_DEBUG_TIMING 64 /* internal: clock64 phase-stamp builds of the attention kernels */
/* Experimental attention kernel v14 (csrc/attn14.cuh), dev library only: one Q
 * tile per CTA, S double-buffered in TMEM, KV tiles alternating over two softmax pairs, promotion in a
 * correction warpgroup; b_kv = 128.  Measured slower than v8.  Accepted by sage2_prepare /
 * sage2_attention / sage2_attention_kernel of libsage2_dev.so; non-causal; not with GRAN / ONE_LEVEL. */
#define SAGE2_F_KERNEL_V14 4194304

/* clock64 phase trace of the attention kernel sage2_attention would run (non-causal; a KERNEL flag
 * selects v8 / v12): stamps of CTA (0,0,0) written to `stamps` (device, caller-owned, zeroed,
 * uint64 [32 roles][64 KV steps][16 slots]; the slot meaning is in the kernel source (ts / tss
 * calls)).  out receives the output. */
int sage2_dev_trace(void* out, uint64_t* stamps, int B, int H_q, int H_kv, int N, int d, int flags,
                    const void* workspace, size_t ws_bytes, void* stream);

/* Probe (the experiment of P:284-285 repeated on tcgen05).  For each of n
 * fp32 bit patterns D[i] (host array) the accumulator of tcgen05.mma.kind::f8f6f4 (M=128, N=32,
 * K=32, E4M3 x E4M3 -> F32) is initialised to D[i] and one MMA with enable-input-d is issued:
 *   c_zero[i] = bits of (A B + D) with A = B = 0                       (the paper's test)
 *   c_prod[i] = bits of (x[i] * 1.0 + D[i]), x[i] = E4M3 value of prod_vals[i] (one non-zero product)
 * Host arrays, synchronous. */
int sage2_probe_accumulator(const uint32_t* d_bits, const uint8_t* prod_vals, int n, uint32_t* c_zero,
                            uint32_t* c_prod);

/* Dense tcgen05 throughput: `iters` back-to-back MMAs of kind 0 = i8 (M128 N256 K32) or 1 = f8f6f4
 * E4M3 (M128 N256 K32) on every SM; measured ops/s in *ops_per_s.  Synchronous. */
int sage2_bench_mma(int kind, int iters, double* ops_per_s);

/* Unit microbenchmarks (per-SM rates per SM clock; synchronous):
 *   0 tcgen05.ld 32x32b bytes/clk, 1 tcgen05.st bytes/clk, 2 MUFU ex2 results/clk,
 *   3 I2F results/clk, 4 FFMA2 lanes/clk, 5 legacy mma.sync m16n8k64 s4 ops/clk (the paper's Ada
 *   INT4 instruction, emulated on sm_100a), 6 legacy mma.sync m16n8k32 s8 ops/clk,
 *   7 F2FP e4m3x2 elements/clk, 8 FMNMX3 /clk, 9 the softmax instruction mix elements/clk,
 *   10 tcgen05.ld 16x64b bytes/clk, 11 tcgen05.st 16x64b bytes/clk. */
int sage2_microbench(int which, int iters, double* per_clk_per_sm);

#ifdef __cplusplus
}
#endif
#endif /* SAGE2_DEV_H_ */

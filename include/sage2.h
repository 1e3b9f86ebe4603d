/*
 * sage2.h -- C ABI of libsage2.so: the SageAttention2 (arXiv 2411.10958) quantized attention
 * forward pass, B200 (sm_100a) native.
 *
 * Citations: P:N = PAPER.md line N (the paper's LaTeX); DESIGN.md holds the readings (C-n).
 *
 * What it computes (Fig. 3; Alg. 1), per (batch b, query head h):
 *   1. smooth K:  gamma(K) = K - mean_tokens(K)
 *      smooth Q:  gamma(Q_i) = Q_i - mean(Q_i) per 128-token block i
 *      Delta S_i = q_bar_i gamma(K)^T
 *   2. per-thread INT4 quantization of gamma(Q), gamma(K) (groups of P:223),
 *      per-channel FP8 E4M3 quantization of V
 *   3. S = (psi^-1(Q^ K^T) + Delta S)/sqrt(d), exact INT32 QK^T on tcgen05 kind::i8 (INT4 values
 *      in int8 lanes: sm_100a has no dense INT4 tensor-core MMA), online softmax, P~ -> E4M3 with
 *      the static scale 448, R_j = P^ V^ on tcgen05 kind::f8f6f4 in a fresh
 *      accumulator, O = diag(exp(m_old - m_new)) O + R_j in FP32 (two-level accumulation,
 *      P:258), O = O / l / 448 * delta_V.
 *   softmax scale 1/sqrt(d); causal = key <= query; GQA: query head h uses KV head
 *   h / (H_q / H_kv).
 *
 * Layouts (all contiguous, row-major):
 *   q   [B, H_q,  N, d] fp16      k, v [B, H_kv, N, d] fp16      out [B, H_q, N, d] fp16
 * d in {64, 128}; 1 <= N <= 2^22 (ragged N allowed); H_q % H_kv == 0; B * H_q <= 65535.
 *
 * Ownership: every pointer is caller-owned.  Device pointers must be 16-byte aligned device
 * memory of the current CUDA device (workspaces 256-byte aligned).  The library never frees caller
 * memory; between calls it keeps only cached kernel attributes (per device) and its stream-ordered
 * memory pool (see sage2_attn, sage2_release_memory).
 *
 * Errors: functions return SAGE2_OK (0) or a negative code; nothing is printed and no C++
 * exception crosses the ABI.  Work is enqueued asynchronously on `stream` (a cudaStream_t, NULL =
 * legacy default stream); device-side faults surface at the caller's next synchronization.
 * There is no CPU fallback: on a device that is not sm_100 every entry point returns
 * SAGE2_EUNSUPPORTED.
 */
#ifndef SAGE2_H_
#define SAGE2_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAGE2_OK 0
#define SAGE2_EINVAL (-1)       /* bad shape / null or misaligned pointer / workspace too small */
#define SAGE2_EUNSUPPORTED (-2) /* current device is not sm_100 (B200)                          */
#define SAGE2_ENOMEM (-3)       /* stream-ordered workspace allocation failed                    */
#define SAGE2_ECUDA (-4)        /* a CUDA launch / API call failed (cudaGetLastError)            */

/* Variant flags (bitwise OR) for sage2_attn_ex / sage2_prepare / sage2_attention.  Flags that change
 * the preprocessed data (INT8, QK_E4M3, SMOOTH_V, GRAN_*, CAUSAL) must be passed identically to
 * sage2_prepare and sage2_attention.  Invalid combinations return SAGE2_EINVAL. */
#define SAGE2_F_CAUSAL 1          /* key <= query mask (C-18); causal workspaces store Delta S triangular */
#define SAGE2_F_INT8 2            /* SageAttn2-8b: INT8 per-thread Q/K codes (+-127), no Q smoothing     */
                                  /* (Table 3)                                     */
#define SAGE2_F_DS_SIMT 1024      /* sage2_prepare: Delta S with the SIMT fp32 kernel instead of the tf32 */
                                  /* tensor-core GEMM (the default for N <= 2048 anyway)                  */
#define SAGE2_F_QK_E4M3 2048      /* E4M3-carrier QK^T: the INT4 codes stored as E4M3 bytes and S on      */
                                  /* kind::f8f6f4 (fp32 accumulator, the same integer S; C-24). */
                                  /* Not with INT8 or KERNEL_V12.                                         */
#define SAGE2_F_KERNEL_V8 4096    /* force the v8 attention kernel (csrc/attn8.cuh)                        */
#define SAGE2_F_KERNEL_V12 131072 /* force the v12 kernel (csrc/attn12.cuh, d = 64 only: four Q tiles per  */
                                  /* CTA, b_kv = 64 -- the oracle's kv_tile is then 64, reading C-9).      */
                                  /* Not with QK_E4M3 / GRAN flags.                                       */
#define SAGE2_F_ONE_LEVEL 1048576 /* ablation of the two-level accumulation (Table): the  */
                                  /* PV MMA accumulates into O in TMEM (O rescaled in place where the row */
                                  /* max moved); kernel v8 only.  Not the SageAttn2 default.              */
#define SAGE2_F_SMOOTH_V 32768    /* optional smooth V (NEXT#2): V' = V - V_m before the       */
                                  /* per-channel FP8 quantization, O + V_m in the epilogue                */
#define SAGE2_F_GRAN_BLOCK 262144 /* NEXT#4 ablation: per-block Q/K quantization groups (Q: 128-token     */
                                  /* block, K: 64-token blocks) instead of per-thread      */
#define SAGE2_F_GRAN_TOKEN 524288 /* NEXT#4 ablation: per-token Q/K quantization groups.  GRAN flags:     */
                                  /* d = 128, kernel v8 only.                                             */
#define SAGE2_F_GRAN_TENSOR 2097152 /* NEXT#4 ablation: per-tensor Q/K scales (one per head,       */
                                  /* P:1099); not with SMOOTH_V                                          */

/* cudaGetErrorString of the last CUDA error an entry point of this thread returned SAGE2_ECUDA for. */
const char* sage2_last_cuda_error(void);

/* Library version (monotone integer). */
int sage2_version(void);

/* Human-readable name of an error code (static string). */
const char* sage2_strerror(int code);

/* Bytes of device workspace sage2_attn_ws needs for this problem: Q^/K^/V^ tile images, scales,
 * q_bar/k_bar, and Delta S (4 * B * H_q * (N_pad/128) * N_pad bytes, the dominant term;
 * N_pad = ceil(N/128)*128).  Returns 0 for invalid shapes. */
size_t sage2_workspace_bytes(int B, int H_q, int H_kv, int N, int d, int causal);

/* Full forward pass (preprocessing + attention kernel; Alg. 1, Fig. 3) -- the
 * north-star entry point: out = SageAttn2-4b(q, k, v), softmax scale 1/sqrt(d).  Allocates its
 * workspace stream-ordered from the library's per-device pool (cudaMallocFromPoolAsync /
 * cudaFreeAsync on `stream`); the pool keeps the peak footprint mapped for the next call until
 * sage2_release_memory().  causal: 0 or 1.  Errors: SAGE2_EINVAL (shape, null / misaligned pointer),
 * SAGE2_EUNSUPPORTED, SAGE2_ENOMEM, SAGE2_ECUDA. */
int sage2_attn(const void* q, const void* k, const void* v, void* out, int B, int H_q, int H_kv, int N,
               int d, int causal, void* stream);

/* Same, with a caller-provided device workspace of at least sage2_workspace_bytes(...) bytes
 * (256-byte aligned).  No allocation happens inside. */
int sage2_attn_ws(const void* q, const void* k, const void* v, void* out, int B, int H_q, int H_kv, int N,
                  int d, int causal, void* workspace, size_t ws_bytes, void* stream);

/* Same as sage2_attn_ws with variant flags (SAGE2_F_*). */
int sage2_attn_ex(const void* q, const void* k, const void* v, void* out, int B, int H_q, int H_kv, int N,
                  int d, int flags, void* workspace, size_t ws_bytes, void* stream);

/* End-to-end call on HOST buffers (the same computation as sage2_attn, Alg. 1; page-locked
 * memory required for copy/compute overlap; same
 * layouts as above).  Pipelined over up to 16 chunks of (b, h_kv) units on three internal streams:
 * each chunk's H2D copy, preprocessing, attention and D2H copy are stream-ordered, so one chunk's
 * copies overlap the others' kernels.  Device buffers (three chunk sets) are allocated and freed
 * stream-ordered on `stream`.  Asynchronous like every other entry point: the caller synchronizes
 * `stream` before reading out.  Errors: SAGE2_EINVAL, SAGE2_ENOMEM, SAGE2_ECUDA. */
int sage2_attn_host(const void* q_host, const void* k_host, const void* v_host, void* out_host, int B, int H_q,
                    int H_kv, int N, int d, int causal, void* stream);

/* ---- staged entry points (the same kernels, split so each stage can be timed / inspected) ---- */

/* Workspace layout: writes SAGE2_WS_NREGIONS byte offsets into offsets[] (regions in order:
 * ksum(int64 [B*H_kv*d]), vmax(u32 [B*H_kv*d]), vsum(int64 [B*H_kv*d], smooth V),
 * kbar(f32 [B*H_kv*d]), dv(f32 [B*H_kv*d]), vmean(f32 [B*H_kv*d], smooth V V_m),
 * qhat(int8 tile images [B*H_q][nT][128*d]), dq(f32 [B*H_q][nT][groups]: 32 per-thread groups per
 * block by default; sized for one per token), qbar(f32 [B*H_q][nT][d]),
 * khat(int8 tile images [B*H_kv][nT][128*d]), dk(f32 [B*H_kv][nT][groups]: 8 per 128 keys by
 * default; sized for one per token), vhat(E4M3 V^T tile images [B*H_kv][nT][d*128]), qbt(q_bar tf32
 * big/small split images [B*H_q][ceil(nT/256)][d/32][2][256*128 B], input of the tensor-core Delta S
 * GEMM), ds(f32, scaled by log2(e)/sqrt(d): [B*H_q][nT][N_pad] for non-causal calls; causal calls
 * (SAGE2_F_CAUSAL given to sage2_prepare) store row i of a head with only its 128(i+1) visible keys,
 * at 128*i*(i+1)/2 floats from the head's base 64*nT*(nT+1)*bhq -- half the bytes), end) -- the
 * offsets returned here are the non-causal ones (identical except end).  Tile images are K-major,
 * 128B (d=128) / 64B (d=64) swizzled, the exact shared-memory image the tensor cores read (DESIGN.md
 * "HBM layout").  Returns 0 or SAGE2_EINVAL. */
#define SAGE2_WS_NREGIONS 15
int sage2_workspace_layout(int B, int H_q, int H_kv, int N, int d, size_t* offsets);

/* Preprocessing only (Fig. 3 steps 1-3; Alg. 1 "Preprocessing" P:241 and the per-block Q line P:248):
 * k_bar and gamma(K), q_bar_i and gamma(Q_i), Delta S_i = q_bar_i gamma(K)^T
 * (P:193), per-thread INT4 groups of Q / K (INT8 with SAGE2_F_INT8), per-channel
 * E4M3 V; fills the workspace regions listed above.  Stream-ordered on `stream`: the Q
 * quantizer, the K half of the K/V quantizer and (for N <= 2048) Delta S run on library-owned side
 * streams of the device, forked from `stream` and joined back through events recorded per call, so the call behaves
 * as if it ran entirely on `stream` (also under CUDA graph capture of `stream`; tests/test_gpu_streams.py).
 * Errors: SAGE2_EINVAL (shape, flags, pointer / workspace size or alignment), SAGE2_EUNSUPPORTED,
 * SAGE2_ECUDA. */
int sage2_prepare(const void* q, const void* k, const void* v, int B, int H_q, int H_kv, int N, int d,
                  int flags, void* workspace, size_t ws_bytes, void* stream);

/* Which attention kernel sage2_attention runs for (N, d, flags): 12 or 8 (SAGE2_F_KERNEL_V12 / _V8; ONE_LEVEL implies 8; with no selector and no QK_E4M3 / GRAN flag: 12 for d = 64
 * non-causal, 8 otherwise -- v8 runs one Q tile per CTA, two CTAs per SM, for N <= 1024).  Host-only,
 * no CUDA call; never fails. */
int sage2_attention_kernel(int N, int d, int flags);

/* Attention kernel only (Fig. 3 step 4, Alg. 1 lines P:246-263: S = psi^-1(Q^K^T) + Delta S,
 * online softmax, P^ = e4m3(448 P~), R = P^V^ and O = alpha O + R,
 * O / l / 448 * delta_V), on a workspace filled by
 * sage2_prepare with the same shapes and data flags (256-byte aligned, at least
 * sage2_workspace_bytes).  The workspace is only read: several sage2_attention calls may share one
 * prepared workspace, also concurrently on different streams.  */
int sage2_attention(void* out, int B, int H_q, int H_kv, int N, int d, int flags, const void* workspace,
                    size_t ws_bytes, void* stream);

/* Debug (parity tests): runs the attention kernel sage2_attention would run for (N, d, flags)
 * non-causally (a KERNEL flag selects v8 or v12) and additionally writes the raw INT32 QK^T
 * accumulators read back from TMEM to s_int [B*H_q][N_pad][N_pad] (device, caller-owned,
 * 4*B*H_q*N_pad^2 bytes; intended for small N) and, if p_hat is not NULL, the E4M3 codes of
 * P^ = e4m3(448 P~) the kernel fed to the PV MMA, [B*H_q][N_pad][N_pad] bytes (the codes of KV tile j
 * are computed with the running max after tile j).  out receives the output.  GRAN flags: EINVAL. */
int sage2_debug_qk_int32(void* out, int32_t* s_int, uint8_t* p_hat, int B, int H_q, int H_kv, int N, int d,
                         int flags, const void* workspace, size_t ws_bytes, void* stream);

/* Returns the device memory the library's stream-ordered pool of the CURRENT device retains
 * (workspaces of sage2_attn, chunk buffers of sage2_attn_host, per-launch counters; kept mapped
 * between calls so repeated calls do not re-map gigabytes) to the driver.  Synchronizes the device
 * first (frees are stream-ordered).  Returns 0 or an error code. */
int sage2_release_memory(void);

#ifdef __cplusplus
}
#endif
#endif /* SAGE2_H_ */

/*
 * sage2_oracle.c -- CPU oracle for the SageAttention2 (arXiv 2411.10958) forward pass.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this code.  The product path
 * (paper_2411_10958_b200/, libsage2.so) never links, imports or executes it, and this
 * file shares no code, header, table or constant generator with the CUDA path.
 *
 * Plain, slow, obviously-correct loops.  Arithmetic is fp64 except where the paper (or a
 * DESIGN.md reading) fixes a narrower format:
 *   - inputs are FP16 (Alg. 1 "Input: Q(FP16), K(FP16), V(FP16)"),
 *   - Q/K codes are INT4 in [-7, 7] or INT8 [-127,127] for the 8-bit variant,
 *   - P~ and V are FP8 E4M3,
 *   - q_bar, k_bar, the smoothed K'/Q' and the scales delta are fp32, because they decide
 *     integer codes (readings C-1, C-2: the decision is taken in the kernel's precision).
 * Citations: P:N = /root/reference/PAPER.md line N;  C-n = DESIGN.md reading n (== SURVEY.md 8(c)).
 *
 * Pins (tests/test_oracle_*.py): exhaustive E4M3 table, fp16 decode/encode against numpy,
 * quantizer fixed points and endpoints, the paper's group examples, exact mode vs
 * an independent dense numpy softmax-attention, smoothing invariance, two-level ==
 * single-level in fp64, single tile == dense per-tile formula, brute force on tiny
 * inputs by a second naive Python implementation (per-thread, per-block and per-token groups), the
 * lossless special case, smooth V (constant V is reproduced exactly), and the paper's
 * directions (smoothing and granularity accuracy orderings, two-level under FP22).
 * Parity unpinned: the paper's accuracy NUMBERS (CosSim / Rel-L1 / RMSE on real CogVideoX tensors,
 * P:499-547) -- synthetic inputs can only pin their orderings.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_VERSION 1

/* ------------------------------------------------------------------------------------------ */
/* Configuration (mirrors SPEC AttentionConfig; defaults = SageAttn2-4b, Table 3)   */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int b_q;        /* Q block = smoothing block; 128                        */
    int kv_tile;    /* b_kv, the KV tile of the online softmax; C-9: = kernel's  */
    int causal;     /* key <= query (C-18)                                                      */
    int quant;      /* orc_attn_block_dbg: 1 = P~ quantized to E4M3 before the PV product
                       (Alg. 1 line P:256); 0 = quantization of P~ disabled (P^ = 448 P~ exactly),
                       so on inputs whose Q/K/V codes are lossless (Q' = dQ * codes, ...) the
                       block loop reduces to exact softmax attention -- the north-star pin
                       "quantization disabled => exact softmax attention" through the SAME
                       function that produces every parity reference (tests/test_oracle_lossless.py).
                       orc_attn_exact_tiled ignores it (it never quantizes).                    */
    int qk_max;     /* 7 = INT4, 127 = INT8 (SageAttn2-8b)                         */
    int smooth_q;   /* subtract per-block mean of Q and add Delta S             */
    int smooth_k;   /* subtract mean of K over all tokens                        */
    int pv_mode;    /* R accumulation: 0 fp64 (exact), 1 fp32 sequential, 2 FP22 truncate after
                       every 32-wide K step                            */
    int two_level;  /* 1: R fresh per tile then O = alpha O + R;  0: single level   */
    int smooth_v;   /* optional smooth V; NEXT#2                                    */
    int p_fp32;     /* 0 (default): everything in fp64, the paper's formulas verbatim;
                       1 (diagnostic only): the P^ code decision taken in fp32 in base 2 (scores
                       rounded to fp32, 2^(s - m + log2 448) rounded to fp32 before the E4M3 cast),
                       used to measure how many codes an fp32 implementation can flip (C-21)     */
    int qk_gran;    /* Q/K quantization granularity (NEXT#4 ablation):
                       0 per-thread (SageAttn2), 1 per-block (Q: 128-token block, K: 64-token
                       block), 2 per-token (every token its own group), 3 per-tensor (one
                       scale per head: max |gamma(Q)| over every block of the head / max |K'| over
                       every key, the per-tensor quantizer of P:99 / row "Per-tensor" of P:1099)  */
    double amb_eta; /* additive floor of the per-element ambiguity window (relative distance of
                       448 P~ to an E4M3 rounding midpoint under which an fp32 implementation may
                       round the other way, C-21); the window itself is the fp32 error
                       bound of the score derived element by element in orc_attn_block_dbg     */
    float q_delta;  /* qk_gran == 3: the head's per-tensor delta_Q (orc_q_head_delta); unused else */
} orc_cfg;

/* ------------------------------------------------------------------------------------------ */
/* Number formats                                                                              */
/* ------------------------------------------------------------------------------------------ */

/* IEEE binary16 -> value (exact in double).  Inputs are FP16 (Alg. 1). */
double orc_fp16_decode(uint16_t h) {
    int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0)       v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else              v = ldexp((double)(1024 + m), e - 25);
    return s ? -v : v;
}

/* FP16 value scaled by 2^24 as an exact integer (every finite fp16 is a multiple of 2^-24 with
 * |x| < 2^16, so |x * 2^24| < 2^40).  Used for exact means (C-1). */
static int64_t fp16_fixed24(uint16_t h) {
    int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
    int64_t v = (e == 0) ? (int64_t)m : ((int64_t)(1024 + m) << (e - 1));
    return s ? -v : v;
}

/* Round an exact real to the nearest binary16 value, ties to even, overflow to +-inf
 * (IEEE 754 default).  Used for the FP16 output O ("Write O_i"; C-17). */
double orc_fp16_round(double x) {
    if (x != x) return x;
    double a = fabs(x);
    if (a == 0.0) return x;
    int E;
    frexp(a, &E);                 /* a = f * 2^E, f in [0.5, 1)  => binade exponent E-1 */
    int qexp = (E - 1 > -14 ? E - 1 : -14) - 10;   /* quantum of the binade (subnormals: 2^-24) */
    double n = nearbyint(ldexp(a, -qexp));         /* default FE_TONEAREST = ties-to-even */
    double r = ldexp(n, qexp);
    if (r >= 65520.0) r = INFINITY;                /* 65504 + half-ulp(16) rounds to inf */
    else if (r > 65504.0) r = 65504.0;             /* cannot happen: kept for clarity */
    return x < 0 ? -r : r;
}

/* OCP FP8 E4M3 ("fn": no inf, 0x7f/0xff NaN, max 448).  Decode. ("range [-448,+448]") */
double orc_e4m3_decode(uint8_t c) {
    int s = c >> 7, e = (c >> 3) & 15, m = c & 7;
    double v;
    if (e == 15 && m == 7) v = NAN;
    else if (e == 0)       v = ldexp((double)m, -9);
    else                   v = ldexp((double)(8 + m), e - 10);
    return s ? -v : v;
}

/* Encode an exact real to E4M3: round to nearest, ties to even, saturate to +-448 (C-6).
 * Returns the code byte. */
uint8_t orc_e4m3_encode(double x) {
    uint8_t sign = signbit(x) ? 0x80 : 0x00;
    double a = fabs(x);
    if (a != a) return 0x7f;
    if (a >= 448.0) return sign | 0x7e;            /* satfinite */
    if (a == 0.0) return sign;
    int E;
    frexp(a, &E);                                  /* binade exponent E-1 */
    int be = E - 1;
    int qexp = (be < -6 ? -6 : be) - 3;            /* 3 mantissa bits; subnormal quantum 2^-9 */
    double n = nearbyint(ldexp(a, -qexp));          /* ties to even */
    double r = ldexp(n, qexp);
    if (r >= 448.0) return sign | 0x7e;
    if (r == 0.0) return sign;
    if (r < ldexp(1.0, -6)) return sign | (uint8_t)(int)ldexp(r, 9);   /* subnormal: m*2^-9 */
    int E2;
    double f = frexp(r, &E2);                      /* r = f*2^E2 = (1.mmm) * 2^(E2-1) */
    int ef = (E2 - 1) + 7;
    int m = (int)(ldexp(f, 4)) - 8;                /* f*16 in [8,16) */
    return sign | (uint8_t)((ef << 3) | m);
}

/* FP22 = 1 sign, 8 exponent, 13 mantissa bits: truncate the low 10 mantissa bits of an fp32
 * ("least significant 10 mantissa bits zeroed out (i.e., truncated)"). */
float orc_fp22_truncate(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if (((u >> 23) & 0xff) == 0xff) return x;      /* inf / nan pass through */
    u &= 0xfffffc00u;
    memcpy(&x, &u, 4);
    return x;
}

/* ------------------------------------------------------------------------------------------ */
/* Per-thread groups (readings C-7, C-8)                                    */
/* ------------------------------------------------------------------------------------------ */

/* Query token t -> group.  "Query tokens i, 8+i, 16+i, 24+i ... one quantization group",
 * 8 groups per 32-token warp tile, 32 per 128-token block. */
int orc_group_q(int t) { return 8 * (t / 32) + (t % 8); }

/* Key token t -> group.  "K_j[8k+2i] together with K_j[8k+2i+1] could share one quantization
 * scale"; 4 groups per 64-token block. */
int orc_group_k(int t) { return 4 * (t / 64) + (t % 8) / 2; }

/* Granularity-general group maps (NEXT#4).  Q: token t of a 128-token block -> group in the block;
 * K: key token t -> group in the head.  Per-block groups follow SageAttention's blocks (b_q = 128,
 * b_k = 64); per-token groups are single tokens. */
int orc_ngroups_q(int gran) { return gran == 1 || gran == 3 ? 1 : gran == 2 ? 128 : 32; }
/* per 128 keys; per-tensor (3): one group for the whole head, stored as group 0 */
int orc_ngroups_k128(int gran) { return gran == 1 ? 2 : gran == 2 ? 128 : gran == 3 ? 1 : 8; }
int orc_group_q_g(int t, int gran) { return gran == 1 || gran == 3 ? 0 : gran == 2 ? t : orc_group_q(t); }
int orc_group_k_g(int t, int gran) { return gran == 1 ? t / 64 : gran == 2 ? t : gran == 3 ? 0 : orc_group_k(t); }

/* ------------------------------------------------------------------------------------------ */
/* Quantizer psi: delta = max|A|/qmax, A_hat = round(A/delta), clamp.              */
/* ------------------------------------------------------------------------------------------ */

/* fp32 operations spelled out so that the compiler cannot contract or widen them. */
static float f32_sub(float a, float b) { volatile float r = a - b; return r; }
static float f32_div(float a, float b) { volatile float r = a / b; return r; }

/* Code for one fp32 element given its group's delta (C-2, C-3, C-4, C-5). */
static int quant_code(float x, float delta, int qmax) {
    if (delta == 0.0f) return 0;                  /* all-zero group (C-5) */
    float q = f32_div(x, delta);                  /* IEEE fp32 division (C-2) */
    double r = nearbyint((double)q);              /* round half to even (C-3) */
    if (r > qmax) r = qmax;
    if (r < -qmax) r = -qmax;
    return (int)r;
}

/* Exact fp16 mean of column c over rows [r0, r1) of an [*, d] fp16 matrix:
 * fp32( fp64(sum * 2^-24) / n )  (C-1: the sum is exact in int64). */
static float exact_mean_f32(const uint16_t* X, int d, int r0, int r1, int c) {
    int64_t s = 0;
    for (int r = r0; r < r1; ++r) s += fp16_fixed24(X[(size_t)r * d + c]);
    double m = ((double)s * 0x1p-24) / (double)(r1 - r0);
    return (float)m;
}
static double exact_mean_f64(const uint16_t* X, int d, int r0, int r1, int c) {
    int64_t s = 0;
    for (int r = r0; r < r1; ++r) s += fp16_fixed24(X[(size_t)r * d + c]);
    return ((double)s * 0x1p-24) / (double)(r1 - r0);
}

/* ------------------------------------------------------------------------------------------ */
/* Preprocessing of one KV head:  Alg. 1 line "Preprocessing: K = K - mean(K), (dV,V^)=psi_V(V)" */
/* ------------------------------------------------------------------------------------------ */
/* K, V: [N, d] fp16 bits.  Outputs (N_pad = ceil(N/128)*128 rows; rows >= N are zero codes):
 *   kbar[d]          fp32 k_bar (O-1)            (zero if !smooth_k)
 *   kprime[N*d]      fp32 gamma(K) = K - k_bar  (O-2)
 *   khat[N_pad*d]    int8 codes (O-3)
 *   dk[N_pad/128 * orc_ngroups_k128]  fp32 delta_K per group g_K (O-3; N_pad/16 per-thread
 *                    groups by default; groups with no token: 0)
 *   vhat[N_pad*d]    E4M3 codes (O-4)
 *   dv[d]            fp32 delta_V per channel   (O-4, reading C-15)
 *   vmean[d]         fp32 V_m (smooth_v only; else zero)
 * Returns 0. */
int orc_kv_head(const uint16_t* K, const uint16_t* V, int N, int d, const orc_cfg* cfg,
                float* kbar, float* kprime, int8_t* khat, float* dk,
                uint8_t* vhat, float* dv, float* vmean) {
    int Np = (N + 127) / 128 * 128;
    /* O-1: k_bar over all N tokens */
    for (int c = 0; c < d; ++c) kbar[c] = cfg->smooth_k ? exact_mean_f32(K, d, 0, N, c) : 0.0f;
    /* O-2: K' = fp32(K) - k_bar */
    for (int t = 0; t < N; ++t)
        for (int c = 0; c < d; ++c)
            kprime[(size_t)t * d + c] = f32_sub((float)orc_fp16_decode(K[(size_t)t * d + c]), kbar[c]);
    /* O-3: per-thread groups g_K, delta_K = max|K'|/qmax, codes */
    size_t ng = (size_t)(Np / 128) * (size_t)orc_ngroups_k128(cfg->qk_gran);
    for (size_t g = 0; g < ng; ++g) dk[g] = 0.0f;
    float* amax = (float*)calloc(ng, sizeof(float));
    for (int t = 0; t < N; ++t) {
        int g = orc_group_k_g(t, cfg->qk_gran);
        for (int c = 0; c < d; ++c) {
            float a = fabsf(kprime[(size_t)t * d + c]);
            if (a > amax[g]) amax[g] = a;
        }
    }
    for (size_t g = 0; g < ng; ++g) dk[g] = f32_div(amax[g], (float)cfg->qk_max);
    free(amax);
    memset(khat, 0, (size_t)Np * d);
    for (int t = 0; t < N; ++t) {
        float delta = dk[orc_group_k_g(t, cfg->qk_gran)];
        for (int c = 0; c < d; ++c)
            khat[(size_t)t * d + c] = (int8_t)quant_code(kprime[(size_t)t * d + c], delta, cfg->qk_max);
    }
    /* smooth V (optional): V_m = mean over tokens, V' = V - V_m (fp32) */
    for (int c = 0; c < d; ++c) vmean[c] = cfg->smooth_v ? exact_mean_f32(V, d, 0, N, c) : 0.0f;
    /* O-4: delta_V[c] = max_t |V[t,c]| / 448 ; V^ = E4M3(V / delta_V) */
    memset(vhat, 0, (size_t)Np * d);
    for (int c = 0; c < d; ++c) {
        float m = 0.0f;
        for (int t = 0; t < N; ++t) {
            float x = f32_sub((float)orc_fp16_decode(V[(size_t)t * d + c]), vmean[c]);
            float a = fabsf(x);
            if (a > m) m = a;
        }
        dv[c] = f32_div(m, 448.0f);
        for (int t = 0; t < N; ++t) {
            float x = f32_sub((float)orc_fp16_decode(V[(size_t)t * d + c]), vmean[c]);
            vhat[(size_t)t * d + c] = (dv[c] == 0.0f) ? 0 : orc_e4m3_encode((double)f32_div(x, dv[c]));
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Preprocessing of one Q block i:  Alg. 1 "q_bar_i = mean(Q_i), (dQ, Q^_i) = psi_Q(Q_i - q_bar_i)" */
/* ------------------------------------------------------------------------------------------ */
/* Qblk: rows [0, n) of the block (n = present tokens, <= 128), fp16 bits, row stride d.
 * Outputs: qbar[d] fp32 (O-5), qhat[128*d] int8 (rows >= n zero), dq[orc_ngroups_q] fp32 (O-6;
 * 32 per-thread groups by default). */
int orc_q_block(const uint16_t* Qblk, int n, int d, const orc_cfg* cfg,
                float* qbar, int8_t* qhat, float* dq) {
    for (int c = 0; c < d; ++c) qbar[c] = cfg->smooth_q ? exact_mean_f32(Qblk, d, 0, n, c) : 0.0f;
    const int ngq = orc_ngroups_q(cfg->qk_gran);
    float amax[128];
    for (int g = 0; g < ngq; ++g) amax[g] = 0.0f;
    float* qp = (float*)malloc(sizeof(float) * (size_t)n * d);
    for (int t = 0; t < n; ++t)
        for (int c = 0; c < d; ++c) {
            float x = f32_sub((float)orc_fp16_decode(Qblk[(size_t)t * d + c]), qbar[c]);
            qp[(size_t)t * d + c] = x;
            float a = fabsf(x);
            int g = orc_group_q_g(t, cfg->qk_gran);
            if (a > amax[g]) amax[g] = a;
        }
    for (int g = 0; g < ngq; ++g) dq[g] = f32_div(amax[g], (float)cfg->qk_max);
    if (cfg->qk_gran == 3) dq[0] = cfg->q_delta;        /* per-tensor: the head's delta */
    memset(qhat, 0, (size_t)128 * d);
    for (int t = 0; t < n; ++t) {
        float delta = dq[orc_group_q_g(t, cfg->qk_gran)];
        for (int c = 0; c < d; ++c)
            qhat[(size_t)t * d + c] = (int8_t)quant_code(qp[(size_t)t * d + c], delta, cfg->qk_max);
    }
    free(qp);
    return 0;
}

/* Per-tensor granularity (qk_gran == 3, NEXT#4, "per-tensor"): delta_Q of a whole
 * head = max over every Q block i and every element of |gamma(Q_i)| = |fp32(Q) - q_bar_i| (O-5),
 * divided by qmax (O-6).  Q: [N, d] fp16 bits. */
float orc_q_head_delta(const uint16_t* Q, int N, int d, const orc_cfg* cfg) {
    float amax = 0.0f;
    for (int r0 = 0; r0 < N; r0 += cfg->b_q) {
        const int n = (N - r0 < cfg->b_q) ? N - r0 : cfg->b_q;
        for (int c = 0; c < d; ++c) {
            const float qb = cfg->smooth_q ? exact_mean_f32(Q + (size_t)r0 * d, d, 0, n, c) : 0.0f;
            for (int t = 0; t < n; ++t) {
                const float a = fabsf(f32_sub((float)orc_fp16_decode(Q[(size_t)(r0 + t) * d + c]), qb));
                if (a > amax) amax = a;
            }
        }
    }
    return f32_div(amax, (float)cfg->qk_max);
}

/* O-7: Delta S_i[t] = q_bar_i . gamma(K)[t]   ("Delta S_ij = q_bar_i gamma(K_j)^T"),
 * fp64 accumulation of the fp32 operands.  ds has N entries.  ds_abs (optional, N entries):
 * sum_c |q_bar_c| |gamma(K)[t,c]|, the magnitude any fp32 evaluation of the dot product is
 * rounded against (used only for the ambiguity report, C-21). */
int orc_delta_s2(const float* qbar, const float* kprime, int N, int d, double* ds, double* ds_abs) {
    for (int t = 0; t < N; ++t) {
        double s = 0.0, a = 0.0;
        for (int c = 0; c < d; ++c) {
            s += (double)qbar[c] * (double)kprime[(size_t)t * d + c];
            a += fabs((double)qbar[c]) * fabs((double)kprime[(size_t)t * d + c]);
        }
        ds[t] = s;
        if (ds_abs) ds_abs[t] = a;
    }
    return 0;
}
int orc_delta_s(const float* qbar, const float* kprime, int N, int d, double* ds) {
    return orc_delta_s2(qbar, kprime, N, d, ds, NULL);
}

/* O-8a: integer Q^ K^T for one Q block against all keys: s_int[128 * Np] (int64, exact). */
int orc_s_int_block(const int8_t* qhat, const int8_t* khat, int Np, int d, int64_t* s_int) {
    for (int r = 0; r < 128; ++r)
        for (int t = 0; t < Np; ++t) {
            int64_t s = 0;
            for (int c = 0; c < d; ++c) s += (int64_t)qhat[(size_t)r * d + c] * (int64_t)khat[(size_t)t * d + c];
            s_int[(size_t)r * Np + t] = s;
        }
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Algorithm 1 inner loop for one Q block i (rows 128 i .. 128 i + 127), quantized path.      */
/* ------------------------------------------------------------------------------------------ */

/* Distance (relative) from v > 0 to the nearest E4M3 rounding midpoint around its code, and the
 * larger of the two neighbouring code gaps.  Used only for the ambiguity report. */
static double e4m3_midpoint_gap(double v, const double* e4m3, double* ulp_out) {
    uint8_t c = orc_e4m3_encode(v);
    double x = e4m3[c], best = INFINITY, ulp = 0.0;
    if (c > 0) {                                   /* lower neighbour (positive codes only) */
        double lo = e4m3[c - 1], mid = 0.5 * (lo + x);
        best = fabs(v - mid) / v;
        ulp = x - lo;
    }
    if (c < 0x7e) {
        double hi = e4m3[c + 1], mid = 0.5 * (x + hi);
        double g = fabs(v - mid) / v;
        if (g < best) best = g;
        if (hi - x > ulp) ulp = hi - x;
    }
    *ulp_out = ulp;
    return best;
}

/* Inputs: the block's qhat[128*d], dq[32], ds[N] (Delta S_i), the head's khat/dk/vhat/dv,
 * vmean (smooth_v).  Output: O[128*d] fp64 before fp16 rounding (rows >= N set to 0),
 * and optionally: l_out[128] final row sums (in units of P~), phat_out[128*Np] the P^ codes,
 * amb_out[128*Np] ambiguity flags, flip_out[128] = sum over ambiguous keys of
 * gap(P^) * max_c |V^ dV| / (448 l): how far O could move if every ambiguous decision flipped.
 *
 * Ambiguity (C-21): a P^ decision is ambiguous when 448 P~ lies within eta of an E4M3
 * rounding midpoint (relative), eta being the error bound of an fp32 evaluation of the score:
 * with u = 2^-24 and S = (s_int dQ dK + Delta S)/sqrt(d) (natural-log units),
 *   dS  = [4u |s_int dQ dK| + 2e-6 ds_abs + 1e-6 |Delta S|] / sqrt(d) + 2u (|S| + |m|)
 *         (three roundings in the scale product dQ dK log2e/sqrt(d); the Delta S bound of the
 *          product's Delta S kernels; fp32 rounding of the score, of S - m
 *          and of the running max),
 *   eta = dS + dS(argmax of the row so far) + amb_eta   (P~ = exp(S - m): relative error of P~ is
 *          the absolute error of S - m; amb_eta = 2^-21 covers ex2.approx and the 448 fold).
 * ds_abs (sum_c |q_bar_c||gamma(K)_tc|, orc_delta_s2) may be NULL: then only the roundings count. */
int orc_attn_block_dbg2(const int8_t* qhat, const float* dq, const double* ds, const double* ds_abs,
                        const int8_t* khat, const float* dk, const uint8_t* vhat, const float* dv,
                        const float* vmean, int N, int d, int i, const orc_cfg* cfg,
                        double* O, double* l_out, uint8_t* phat_out, uint8_t* amb_out, double* flip_out) {
    const double U = 0x1p-24;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);      /* P:77 scale 1/sqrt(d) (C-11) */
    const double LOG2E = 1.4426950408889634;
    const double LOG2_448 = log2(448.0);
    const int bkv = cfg->kv_tile;
    int Np = (N + 127) / 128 * 128;
    double e4m3[256];
    for (int c = 0; c < 256; ++c) e4m3[c] = orc_e4m3_decode((uint8_t)c);
    double* vmax_t = (double*)calloc((size_t)Np, sizeof(double));   /* max_c |V^ dV| per key */
    for (int t = 0; t < N; ++t)
        for (int c = 0; c < d; ++c) {
            double a = fabs(e4m3[vhat[(size_t)t * d + c]]) * (double)dv[c];
            if (a > vmax_t[t]) vmax_t[t] = a;
        }

#pragma omp parallel for schedule(dynamic, 4)
    for (int rr = 0; rr < 128; ++rr) {
        int r = 128 * i + rr;                       /* global query index */
        double* o = O + (size_t)rr * d;
        for (int c = 0; c < d; ++c) o[c] = 0.0;
        if (phat_out) memset(phat_out + (size_t)rr * Np, 0, (size_t)Np);
        if (amb_out) memset(amb_out + (size_t)rr * Np, 0, (size_t)Np);
        if (r >= N) { if (l_out) l_out[rr] = 0.0; if (flip_out) flip_out[rr] = 0.0; continue; }
        double* R = (double*)malloc(sizeof(double) * d);
        double* S = (double*)malloc(sizeof(double) * bkv);
        double* dS = (double*)malloc(sizeof(double) * bkv);   /* fp32 error bound of each score */
        double m = -INFINITY, l = 0.0, flip = 0.0, dm = 0.0;  /* dm: error bound of the running max */
        int kend = cfg->causal ? r + 1 : N;          /* keys visible to this row (C-18) */
        for (int j0 = 0; j0 < kend; j0 += bkv) {     /* KV tiles in ascending order (C-9) */
            int j1 = j0 + bkv;
            /* (a)+(b) S = (psi^-1(Q^ K^T) + Delta S) / sqrt(d); masked -> -inf.
             * p_fp32 (C-21): scores kept as fp32 values in base 2, S * log2(e). */
            double tmax = -INFINITY, dtmax = 0.0;
            for (int t = j0; t < j1; ++t) {
                double s, es = 0.0;
                if (t >= kend || t >= Np || t >= N) s = -INFINITY;
                else {
                    int64_t si = 0;
                    for (int c = 0; c < d; ++c)
                        si += (int64_t)qhat[(size_t)rr * d + c] * (int64_t)khat[(size_t)t * d + c];
                    const double sq = (double)si * (double)dq[orc_group_q_g(rr, cfg->qk_gran)] *
                                      (double)dk[orc_group_k_g(t, cfg->qk_gran)];
                    s = (sq + ds[t]) * inv_sqrt_d;
                    es = (4.0 * U * fabs(sq) + (ds_abs ? 2e-6 * ds_abs[t] : 0.0) + 1e-6 * fabs(ds[t])) * inv_sqrt_d +
                         2.0 * U * fabs(s);
                    if (cfg->p_fp32) s = (double)(float)(s * LOG2E);
                }
                S[t - j0] = s;
                dS[t - j0] = es;
                if (s > tmax) { tmax = s; dtmax = es; }
            }
            /* (c) online softmax: m_ij = max(m_i,j-1, rowmax S_ij) exactly (C-10) */
            double m_new = (tmax > m) ? tmax : m;
            if (tmax > m) dm = dtmax;
            double alpha = (m == -INFINITY) ? 0.0 : (cfg->p_fp32 ? exp2(m - m_new) : exp(m - m_new));
            double rowsum = 0.0;
            flip *= alpha;
            /* Level-1 accumulator.  two_level: R fresh per tile ("R_ij = P~_ij V_j").
             * single level (ablation): the running O itself is the MMA accumulator, rescaled
             * first (Eq. 1).  Precision per pv_mode: fp64, fp32, or FP22. */
            double* acc = cfg->two_level ? R : o;
            float accf[256];
            if (cfg->two_level) {
                for (int c = 0; c < d; ++c) { R[c] = 0.0; accf[c] = 0.0f; }
            } else {
                for (int c = 0; c < d; ++c) {
                    o[c] = alpha * o[c];
                    accf[c] = (float)o[c];
                    if (cfg->pv_mode == 2) accf[c] = orc_fp22_truncate(accf[c]);
                }
            }
            for (int t = j0; t < j1; ++t) {
                /* P~ = exp(S - m) ; the E4M3 operand is 448 * P~ */
                double p448;
                if (S[t - j0] == -INFINITY) p448 = 0.0;
                else if (cfg->p_fp32) p448 = (double)(float)exp2(S[t - j0] - m_new + LOG2_448);
                else p448 = 448.0 * exp(S[t - j0] - m_new);
                rowsum += p448 / 448.0;                                          /* C-13 */
                /* (d) P^ = E4M3(448 * P~); with quant == 0 the cast is skipped (P^ = 448 P~) */
                uint8_t code = orc_e4m3_encode(p448);
                double ph = cfg->quant ? e4m3[code] : p448;
                if (phat_out && t < Np) phat_out[(size_t)rr * Np + t] = code;
                if (p448 > 0.0 && (amb_out || flip_out)) {
                    double ulp;
                    double gap = e4m3_midpoint_gap(p448, e4m3, &ulp);
                    const double eta = dS[t - j0] + dm + 2.0 * U * fabs(m_new) + cfg->amb_eta;
                    if (gap <= eta) {
                        if (amb_out && t < Np) amb_out[(size_t)rr * Np + t] = 1;
                        flip += ulp * vmax_t[t];      /* divided by 448 l at the end */
                    }
                }
                if (ph != 0.0) {
                    /* (e) acc += P^ V^  ("Matmul((P~*448).to(FP8.e4m3), V_j)") */
                    for (int c = 0; c < d; ++c) {
                        double pv = ph * e4m3[vhat[(size_t)t * d + c]];   /* exact product */
                        if (cfg->pv_mode == 0) acc[c] += pv;
                        else accf[c] = (float)((double)accf[c] + pv);
                    }
                }
                if (cfg->pv_mode == 2 && ((t - j0) % 32) == 31)      /* one 32-deep MMA step */
                    for (int c = 0; c < d; ++c) accf[c] = orc_fp22_truncate(accf[c]);
            }
            if (cfg->pv_mode != 0)
                for (int c = 0; c < d; ++c) acc[c] = (double)accf[c];
            /* (f) level 2: O = diag(exp(m_old - m_new)) O + R */
            l = alpha * l + rowsum;
            if (cfg->two_level)
                for (int c = 0; c < d; ++c) o[c] = alpha * o[c] + R[c];
            m = m_new;
        }
        /* O-9: O_i = diag(l)^-1 O / 448 * delta_V (+ V_m if smooth V) */
        for (int c = 0; c < d; ++c) o[c] = o[c] / l / 448.0 * (double)dv[c] + (double)vmean[c];
        if (l_out) l_out[rr] = l;
        if (flip_out) flip_out[rr] = flip / (448.0 * l);
        free(R);
        free(S);
        free(dS);
    }
    free(vmax_t);
    return 0;
}

int orc_attn_block_dbg(const int8_t* qhat, const float* dq, const double* ds,
                       const int8_t* khat, const float* dk, const uint8_t* vhat, const float* dv,
                       const float* vmean, int N, int d, int i, const orc_cfg* cfg,
                       double* O, double* l_out, uint8_t* phat_out, uint8_t* amb_out, double* flip_out) {
    return orc_attn_block_dbg2(qhat, dq, ds, NULL, khat, dk, vhat, dv, vmean, N, d, i, cfg, O, l_out, phat_out,
                               amb_out, flip_out);
}

int orc_attn_block_q(const int8_t* qhat, const float* dq, const double* ds,
                     const int8_t* khat, const float* dk, const uint8_t* vhat, const float* dv,
                     const float* vmean, int N, int d, int i, const orc_cfg* cfg,
                     double* O, double* l_out) {
    return orc_attn_block_dbg(qhat, dq, ds, khat, dk, vhat, dv, vmean, N, d, i, cfg, O, l_out, NULL, NULL, NULL);
}

/* ------------------------------------------------------------------------------------------ */
/* Exact mode (quantization off) through the same tiled online softmax (Eq. 1),      */
/* smoothing applied in fp64 (P:193 decomposition); the pin is dense softmax attention P:77.   */
/* ------------------------------------------------------------------------------------------ */
/* Q, K, V: one head [N, d] fp16 bits (Q head and its KV head).  Rows [row0, row1) computed. */
int orc_attn_exact_tiled(const uint16_t* Q, const uint16_t* K, const uint16_t* V, int N, int d,
                         const orc_cfg* cfg, int row0, int row1, double* O) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int bq = cfg->b_q, bkv = cfg->kv_tile;
    double* kbar = (double*)calloc((size_t)d, sizeof(double));
    double* vm = (double*)calloc((size_t)d, sizeof(double));
    for (int c = 0; c < d; ++c) {
        if (cfg->smooth_k) kbar[c] = exact_mean_f64(K, d, 0, N, c);
        if (cfg->smooth_v) vm[c] = exact_mean_f64(V, d, 0, N, c);
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int r = row0; r < row1; ++r) {
        int blk = r / bq, b0 = blk * bq, b1 = (b0 + bq < N) ? b0 + bq : N;
        double* qbar = (double*)calloc((size_t)d, sizeof(double));
        double* qs = (double*)malloc(sizeof(double) * d);
        double* o = O + (size_t)(r - row0) * d;
        double* S = (double*)malloc(sizeof(double) * bkv);
        for (int c = 0; c < d; ++c) {
            if (cfg->smooth_q) qbar[c] = exact_mean_f64(Q, d, b0, b1, c);
            qs[c] = orc_fp16_decode(Q[(size_t)r * d + c]) - qbar[c];
            o[c] = 0.0;
        }
        double m = -INFINITY, l = 0.0;
        int kend = cfg->causal ? r + 1 : N;
        for (int j0 = 0; j0 < kend; j0 += bkv) {
            double tmax = -INFINITY;
            for (int t = j0; t < j0 + bkv; ++t) {
                double s = -INFINITY;
                if (t < kend) {
                    double qk = 0.0, dsv = 0.0;
                    for (int c = 0; c < d; ++c) {
                        double kp = orc_fp16_decode(K[(size_t)t * d + c]) - kbar[c];
                        qk += qs[c] * kp;          /* gamma(Q_i) gamma(K_j)^T */
                        dsv += qbar[c] * kp;       /* Delta S = q_bar gamma(K)^T */
                    }
                    s = (qk + dsv) * inv_sqrt_d;
                }
                S[t - j0] = s;
                if (s > tmax) tmax = s;
            }
            double m_new = tmax > m ? tmax : m;
            double alpha = (m == -INFINITY) ? 0.0 : exp(m - m_new);
            l *= alpha;
            for (int c = 0; c < d; ++c) o[c] *= alpha;
            for (int t = j0; t < j0 + bkv; ++t) {
                if (S[t - j0] == -INFINITY) continue;
                double p = exp(S[t - j0] - m_new);
                l += p;
                for (int c = 0; c < d; ++c)
                    o[c] += p * (orc_fp16_decode(V[(size_t)t * d + c]) - vm[c]);
            }
            m = m_new;
        }
        for (int c = 0; c < d; ++c) o[c] = o[c] / l + vm[c];
        free(qbar); free(qs); free(S);
    }
    free(kbar); free(vm);
    return 0;
}

int orc_version(void) { return ORC_VERSION; }

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Array helpers for the Python test harness (same scalar functions, looped). */
void orc_e4m3_encode_array(const double* x, long n, uint8_t* out) {
    for (long i = 0; i < n; ++i) out[i] = orc_e4m3_encode(x[i]);
}
void orc_e4m3_decode_array(const uint8_t* c, long n, double* out) {
    for (long i = 0; i < n; ++i) out[i] = orc_e4m3_decode(c[i]);
}
void orc_fp16_decode_array(const uint16_t* h, long n, double* out) {
    for (long i = 0; i < n; ++i) out[i] = orc_fp16_decode(h[i]);
}
void orc_fp16_round_array(const double* x, long n, double* out) {
    for (long i = 0; i < n; ++i) out[i] = orc_fp16_round(x[i]);
}
void orc_fp22_truncate_array(const float* x, long n, float* out) {
    for (long i = 0; i < n; ++i) out[i] = orc_fp22_truncate(x[i]);
}

// prep.cuh -- SageAttention2 preprocessing kernels (Fig. 3 steps 1-3; Alg. 1
// "Preprocessing", and the per-block Q lines):
//
//   k_kv_stats   : exact int64 fixed-point column sums of K (for k_bar = mean(K)) and the
//                  per-channel absmax of V (for delta_V).  HBM-bound, one read of K and V.
//   k_kv_quant   : gamma(K) = K - k_bar, per-thread INT4 groups of K (g_K), codes ->
//                  K^ tile images; per-channel E4M3 V^ -> transposed V^T tile images.
//   k_q_quant    : q_bar_i = mean(Q_i), gamma(Q_i), per-thread groups of Q (g_Q) -> Q^ tiles.
//   k_delta_s    : Delta S_i[t] = q_bar_i . gamma(K)[t], stored pre-scaled by log2(e)/sqrt(d).
//
// Bit-exactness contract with the oracle (readings C-1..C-6): means from exact integer
// sums, fp32 subtraction, IEEE fp32 division (__fdiv_rn), round-half-even, satfinite E4M3.  This
// file must never be compiled with --use_fast_math.
#pragma once
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdint>

#include "ptx.cuh"

namespace sage2 {

constexpr int kTile = 128;  // b_q = b_kv = 128 tokens
#ifndef SAGE2_STATS_U
#define SAGE2_STATS_U 8   // k_kv_stats row passes in flight (4: C2-4K prepare 373 us, 8: 356, 12: 396 -- registers)
#endif

// Quantization granularity of Q and K (NEXT#4 ablation, oracle qk_gran): 0 per-thread (P:223,
// SageAttn2), 1 per-block (Q: the 128-token block, K: 64-token blocks), 2 per-token, 3
// per-tensor (one scale per head; stored in the per-block layout with every entry equal, so
// the attention kernel runs its per-block instantiation).  4 (internal): the head-absmax pass of
// per-tensor preprocessing.  Groups per 128 tokens (stored layout): Q 32 / 1 / 128 / 1, K 8 / 4
// (2 used, padded for 16-byte bulk copies) / 128 / 4.
__host__ __device__ constexpr int gran_nq(int gran) { return gran == 1 || gran >= 3 ? 1 : gran == 2 ? 128 : 32; }
__host__ __device__ constexpr int gran_nk(int gran) { return gran == 1 || gran >= 3 ? 4 : gran == 2 ? 128 : 8; }


// FP16 bits -> exact integer value * 2^24 (every finite fp16 is a multiple of 2^-24).
__device__ __forceinline__ long long fp16_fixed24(uint16_t h) {
    int e = (h >> 10) & 31, m = h & 1023;
    long long v = (e == 0) ? (long long)m : ((long long)(1024 + m) << (e - 1));
    return (h & 0x8000) ? -v : v;
}

// fp16 -> fp64 (exact).  Sums of up to 2^29 / 65504 fp16 values in fp64 are exact in any order:
// every value is a multiple of 2^-24 below 2^16, so a partial sum of k values needs at most
// 40 + log2(k) bits (<= 53 for k <= 8192).  The kernels sum in fp64 within a CTA and convert the
// exact total to the int64 fixed point of reading C-1 for the cross-CTA atomics.
__device__ __forceinline__ double fp16_to_f64(uint16_t h) {
    double r;
    asm("{\n\t.reg .f16 t;\n\tmov.b16 t, %1;\n\tcvt.f64.f16 %0, t;\n\t}" : "=d"(r) : "h"(h));
    return r;
}

// mean = fp32( fp64(sum * 2^-24) / n )   (reading C-1; identical op sequence in the oracle)
__device__ __forceinline__ float fixed_mean(long long sum, int n) {
    double s = __dmul_rn((double)sum, 0x1p-24);
    return (float)__ddiv_rn(s, (double)n);
}

// fp32 -> nearest tf32 (10-bit mantissa) kept in an fp32 container; x - tf32_big(x) is exact.
__device__ __forceinline__ float tf32_big(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ int quant_code(float x, float delta, int qmax) {
    if (delta == 0.0f) return 0;                       // all-zero group (C-5)
    float q = rintf(__fdiv_rn(x, delta));              // IEEE division, ties-to-even (C-2, C-3)
    q = fminf(fmaxf(q, -(float)qmax), (float)qmax);    // clamp (C-4)
    return (int)q;
}

// 4 int codes -> 4 signed bytes (little endian)
__device__ __forceinline__ uint32_t pack4_s8(int a, int b, int c, int d) {
    // cvt.pack.sat.s8.s32.b32 d, x, y, z: d = { z[15:0], sat(x), sat(y) } (y in byte 0)
    uint32_t hi, r;
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(d), "r"(c));
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(a), "r"(hi));
    return r;
}

// 4 int codes in [-7, 7] -> 4 E4M3 bytes carrying the same integers (exact: |c| <= 16 fits the
// 3-bit mantissa).  The E4M3-carrier QK^T variant (SAGE2_F_QK_E4M3, SURVEY.md §8(a) note) feeds
// these to tcgen05.mma.kind::f8f6f4: same products, fp32 accumulator, identical integer S.
__device__ __forceinline__ uint32_t pack4_e4m3(int a, int b, int c, int d) {
    const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2((float)a, (float)b), __NV_SATFINITE, __NV_E4M3);
    const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2((float)c, (float)d), __NV_SATFINITE, __NV_E4M3);
    return lo | (hi << 16);
}
__device__ __forceinline__ uint2 pack8_codes(const int (&c)[8], bool e4m3) {
    return e4m3 ? make_uint2(pack4_e4m3(c[0], c[1], c[2], c[3]), pack4_e4m3(c[4], c[5], c[6], c[7]))
                : make_uint2(pack4_s8(c[0], c[1], c[2], c[3]), pack4_s8(c[4], c[5], c[6], c[7]));
}

// Eight codes straight to their packed tile bytes, bit-identical to quant_code() + pack8_codes():
// y = fma(x, rcp(delta), 1.5 * 2^23) rounds the exact product x * rcp(delta) to an integer n held in
// y's low mantissa bits (|n| <= 127 < 2^22), so n's two's-complement byte is y's low byte; the
// residual fma(x, rcp(delta), -n) is exact-then-rounded, and when it is more than 2^-12 away from
// +-1/2 the product, fl(x * rcp(delta)) and the IEEE quotient fl(x / delta) all round to n (they lie
// within 2^-16 of each other for |x / delta| <= 128).  |n| <= qmax needs no clamp: delta = absmax /
// qmax (C-2) bounds |x / delta| by qmax (1 + 2^-23).  Otherwise (rare) the group is redone with
// IEEE division.  Packed f32x2 arithmetic: about 3 issue slots per code instead of 7.
__device__ __forceinline__ uint2 quant_pack8(const float (&x)[8], float delta, int qmax, bool e4m3) {
    if (delta == 0.0f) return e4m3 ? make_uint2(0u, 0u) : make_uint2(0u, 0u);   // all-zero group (C-5)
    const float rd = __frcp_rn(delta);
    constexpr float M = 12582912.0f;                   // 1.5 * 2^23
    const float2 rd2 = make_float2(rd, rd), m2 = make_float2(M, M), nm2 = make_float2(-M, -M);
    float y[8];
    bool slow = false;
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
        const float2 xi = make_float2(x[i], x[i + 1]);
        const float2 yi = ffma2(xi, rd2, m2);          // M + RNE(x * rd)
        const float2 ni = fadd2(yi, nm2);              // n (exact)
        const float2 ri = ffma2(xi, rd2, make_float2(-ni.x, -ni.y));   // x * rd - n
        y[i] = yi.x;
        y[i + 1] = yi.y;
        slow |= (fabsf(ri.x) > 0.5f - 0x1p-12f) | (fabsf(ri.y) > 0.5f - 0x1p-12f);
    }
    if (slow) {
        int code[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) code[i] = quant_code(x[i], delta, qmax);
        return pack8_codes(code, e4m3);
    }
    if (e4m3) {                                        // the E4M3 carrier: the integers as E4M3 bytes
        int code[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) code[i] = (int)(__float_as_int(y[i]) - 0x4B400000);
        return pack8_codes(code, true);
    }
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = __float_as_uint(y[i]);
    // low bytes of y[0..3] / y[4..7] -> one word each (byte i = code i, little endian)
    const uint32_t a = __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410);
    const uint32_t b = __byte_perm(__byte_perm(w[4], w[5], 0x0040), __byte_perm(w[6], w[7], 0x0040), 0x5410);
    return make_uint2(a, b);
}

// Sum the int64 column partials of the lanes that hold the same 8 channels (lane % TPR).
template <int TPR>
__device__ __forceinline__ void warp_sum_cols(long long (&s)[8]) {
#pragma unroll
    for (int m = TPR; m < 32; m <<= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], m);
}

// ---------------------------------------------------------------------------------------------
// k_kv_stats: grid (row chunks, B*Hkv), 256 threads.  Each thread reads 8 consecutive channels
// (16 B) of a token row, four rows in flight.
// ---------------------------------------------------------------------------------------------
// SMV (optional smooth V, NEXT#2): V's column sums are accumulated instead of its absmax
// (the absmax of V - V_m needs V_m first: k_v_absmax_smooth).
template <int D, bool SMV = false>
__global__ void __launch_bounds__(256) k_kv_stats(const __half* __restrict__ K, const __half* __restrict__ V,
                                                  int N, int rows_per_cta, unsigned long long* __restrict__ ksum,
                                                  unsigned int* __restrict__ vmax,
                                                  unsigned long long* __restrict__ vsum) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    constexpr int TPR = D / 8;          // threads per row
    constexpr int RPP = 256 / TPR;      // rows per pass
    constexpr int U = SAGE2_STATS_U;    // passes in flight
    const int bh = blockIdx.y;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cg = threadIdx.x % TPR, rofs = threadIdx.x / TPR;
    const size_t base = (size_t)bh * N * D;
    const int r0 = blockIdx.x * rows_per_cta, r1 = min(N, r0 + rows_per_cta);
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};     // exact (<= 512 rows per CTA, see fp16_to_f64)
    double sv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t vm[4] = {0, 0, 0, 0};      // |V| as fp16 bits, two channels per word
    for (int rb = r0 + rofs; rb < r1; rb += U * RPP) {
        uint4 kk[U], vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = rb + u * RPP;
            kk[u] = vv[u] = make_uint4(0, 0, 0, 0);
            if (r < r1) {
                kk[u] = __ldg(reinterpret_cast<const uint4*>(K + base + (size_t)r * D + cg * 8));
                vv[u] = __ldg(reinterpret_cast<const uint4*>(V + base + (size_t)r * D + cg * 8));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint16_t* kh = reinterpret_cast<const uint16_t*>(&kk[u]);
#pragma unroll
            for (int i = 0; i < 8; ++i) s[i] += fp16_to_f64(kh[i]);
            if (SMV) {
                const uint16_t* vh = reinterpret_cast<const uint16_t*>(&vv[u]);
#pragma unroll
                for (int i = 0; i < 8; ++i) sv[i] += fp16_to_f64(vh[i]);
            } else {
                const uint32_t* vw = reinterpret_cast<const uint32_t*>(&vv[u]);
#pragma unroll
                for (int i = 0; i < 4; ++i) vm[i] = __vmaxu2(vm[i], vw[i] & 0x7FFF7FFFu);   // |fp16| orders as u16
            }
        }
    }
#pragma unroll
    for (int m = TPR; m < 32; m <<= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            s[i] += __shfl_xor_sync(0xffffffffu, s[i], m);
            if (SMV) sv[i] += __shfl_xor_sync(0xffffffffu, sv[i], m);
        }
#pragma unroll
    for (int m = TPR; m < 32; m <<= 1)
#pragma unroll
        for (int i = 0; i < 4; ++i) vm[i] = __vmaxu2(vm[i], __shfl_xor_sync(0xffffffffu, vm[i], m));
    __shared__ double ssum[8][D];
    __shared__ double svs[SMV ? 8 : 1][D];
    __shared__ uint32_t smax[8][D];
    if (lane < TPR) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            ssum[warp][cg * 8 + i] = s[i];
            if (SMV) svs[SMV ? warp : 0][cg * 8 + i] = sv[i];
            const uint32_t h = (vm[i / 2] >> (16 * (i % 2))) & 0xFFFFu;
            smax[warp][cg * 8 + i] = __float_as_uint(__half2float(__ushort_as_half((uint16_t)h)));
        }
    }
    __syncthreads();
    if (threadIdx.x < D) {
        const int c = threadIdx.x;
        double t = 0, tv = 0;
        uint32_t m = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            t += ssum[w][c];
            if (SMV) tv += svs[SMV ? w : 0][c];
            m = max(m, smax[w][c]);     // non-negative floats order as uints
        }
        // exact totals -> int64 fixed point (x 2^24, exact) -> order-independent atomics
        atomicAdd(ksum + (size_t)bh * D + c, (unsigned long long)__double2ll_rn(t * 0x1p24));
        if (SMV) atomicAdd(vsum + (size_t)bh * D + c, (unsigned long long)__double2ll_rn(tv * 0x1p24));
        else atomicMax(vmax + (size_t)bh * D + c, m);
    }
}

// ---------------------------------------------------------------------------------------------
// k_v_absmax_smooth (smooth V only): V_m = exact mean of V's columns (reading C-1, like
// k_bar), then vmax[c] = max_t |fp32(V[t,c]) - V_m[c]| (the absmax delta_V is taken over, O-4 on
// V' = V - V_m).  Same grid as k_kv_stats; block (0, bh) also writes vmean.
// ---------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_v_absmax_smooth(const __half* __restrict__ V, int N, int rows_per_cta,
                                                         const unsigned long long* __restrict__ vsum,
                                                         unsigned int* __restrict__ vmax, float* __restrict__ vmean_out) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    constexpr int TPR = D / 8, RPP = 256 / TPR, U = 4;
    const int bh = blockIdx.y;
    const int lane = threadIdx.x % 32;
    const int cg = threadIdx.x % TPR, rofs = threadIdx.x / TPR;
    const size_t base = (size_t)bh * N * D;
    __shared__ float vmean[D];
    if (threadIdx.x < D) {
        const float m = fixed_mean((long long)vsum[(size_t)bh * D + threadIdx.x], N);
        vmean[threadIdx.x] = m;
        if (blockIdx.x == 0) vmean_out[(size_t)bh * D + threadIdx.x] = m;
    }
    __syncthreads();
    float vm8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) vm8[i] = vmean[cg * 8 + i];
    float mx[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int r0 = blockIdx.x * rows_per_cta, r1 = min(N, r0 + rows_per_cta);
    for (int rb = r0 + rofs; rb < r1; rb += U * RPP) {
        uint4 vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = rb + u * RPP;
            vv[u] = make_uint4(0, 0, 0, 0);
            if (r < r1) vv[u] = __ldg(reinterpret_cast<const uint4*>(V + base + (size_t)r * D + cg * 8));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (rb + u * RPP < r1) {
                const __half* vh = reinterpret_cast<const __half*>(&vv[u]);
#pragma unroll
                for (int i = 0; i < 8; ++i) mx[i] = fmaxf(mx[i], fabsf(__fsub_rn(__half2float(vh[i]), vm8[i])));
            }
        }
    }
#pragma unroll
    for (int m = TPR; m < 32; m <<= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], m));
    if (lane < TPR) {
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicMax(vmax + (size_t)bh * D + cg * 8 + i, __float_as_uint(mx[i]));
    }
}

// ---------------------------------------------------------------------------------------------
// k_kv_quant: grid (N_pad/128, B*Hkv), 256 threads.  One 128-token tile of one KV head.
//   K^ tile image  : [128 tokens][D bytes], K-major swizzled (row = token), stored straight from
//                    registers (each warp writes whole 128-byte rows)
//   V^T tile image : [D channels][128 bytes], K-major swizzled (row = channel), E4M3; V is staged
//                    in padded shared memory and read back column-wise (thread = channel pair)
//   dk             : 8 groups per tile (g_K = 4*(t/64) + (t%8)/2)
// ---------------------------------------------------------------------------------------------
// PART: 3 = K and V (one launch), 1 = K only, 2 = V only (short sequences run the two halves as
// concurrent launches on two streams, sage2_api.cu launch_prepare).
template <int D, int GRAN = 0, int PART = 3>
__global__ void __launch_bounds__(256, 3) k_kv_quant(const __half* __restrict__ K, const __half* __restrict__ V,
                                                     int N, int qk_max, int e4m3_codes,
                                                     const unsigned long long* __restrict__ ksum,
                                                     const unsigned int* __restrict__ vmax, int8_t* __restrict__ khat,
                                                     float* __restrict__ dk, uint8_t* __restrict__ vhat,
                                                     float* __restrict__ kbar_out, float* __restrict__ dv_out,
                                                     const float* __restrict__ vmean, unsigned int* ktmax = nullptr) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    // ktmax (per-tensor granularity): GRAN 4 accumulates max|K'| of the head into ktmax[bh] and
    // stops; GRAN 3 then quantizes with delta_K = ktmax[bh] / qk_max for every group.
    constexpr int TPR = D / 8, RPP = 256 / TPR, NP = kTile / RPP;   // passes
    constexpr int VS = D + 8;                                       // padded V row (halves)
    const int tile = blockIdx.x, bh = blockIdx.y, nT = gridDim.x;
    const int lane = threadIdx.x % 32;
    const int cg = threadIdx.x % TPR, rofs = threadIdx.x / TPR;
    __shared__ float kbar[D], dvs[D];
    __shared__ __align__(16) __half vt[(PART & 2) ? kTile * VS : 8];
    const size_t base = (size_t)bh * N * D;
    // every K and V load in flight first; k_bar / delta_V (fp64 and IEEE divisions) computed under
    // their latency; then V is staged in shared memory (a store per load had each store wait out its
    // own load: the round-1 kernel's top stall)
    uint4 kraw[NP], vraw[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int t = tile * kTile + p * RPP + rofs;
        kraw[p] = vraw[p] = make_uint4(0, 0, 0, 0);
        if (t < N) {
            if (PART & 1) kraw[p] = __ldg(reinterpret_cast<const uint4*>(K + base + (size_t)t * D + cg * 8));
            if (PART & 2) vraw[p] = __ldg(reinterpret_cast<const uint4*>(V + base + (size_t)t * D + cg * 8));
        }
    }
    if (threadIdx.x < D) {
        const int c = threadIdx.x;
        if (PART & 1) kbar[c] = fixed_mean((long long)ksum[(size_t)bh * D + c], N);                 // O-1
        if (PART & 2) dvs[c] = __fdiv_rn(__uint_as_float(vmax[(size_t)bh * D + c]), 448.0f);      // O-4
        if (tile == 0) {
            if (PART & 1) kbar_out[(size_t)bh * D + c] = kbar[c];
            if (PART & 2) dv_out[(size_t)bh * D + c] = dvs[c];
        }
    }
    if constexpr ((PART & 2) != 0) {
#pragma unroll
        for (int p = 0; p < NP; ++p) *reinterpret_cast<uint4*>(&vt[(p * RPP + rofs) * VS + cg * 8]) = vraw[p];
    }
    __syncthreads();
    if constexpr ((PART & 1) != 0) {
    // K' = K - k_bar (O-2), kept in registers; absmax per key row -> rowmax, then the group
    // absmax of the granularity (per-thread group g = rows 64(g/4) + 8k + 2(g%4) + {0, 1},
    // "K[8k+2i] together with K[8k+2i+1]")
    __shared__ float rowmax[128];
    __shared__ float gdelta[128];
    float kx[NP][8];
    float kb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) kb[i] = kbar[cg * 8 + i];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs, t = tile * kTile + r;
        const __half2* kh2 = reinterpret_cast<const __half2*>(&kraw[p]);
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(kh2[i]);
            kx[p][2 * i] = (t < N) ? __fsub_rn(f.x, kb[2 * i]) : 0.0f;
            kx[p][2 * i + 1] = (t < N) ? __fsub_rn(f.y, kb[2 * i + 1]) : 0.0f;
            m = fmax3(m, fabsf(kx[p][2 * i]), fabsf(kx[p][2 * i + 1]));
        }
#pragma unroll
        for (int x = 1; x < TPR; x <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, x));
        if (cg == 0) rowmax[r] = m;
    }
    __syncthreads();
    constexpr int NGK = gran_nk(GRAN);
    if constexpr (GRAN == 4) {
        if (threadIdx.x < 32) {
            float m = fmaxf(fmaxf(rowmax[threadIdx.x], rowmax[threadIdx.x + 32]),
                            fmaxf(rowmax[threadIdx.x + 64], rowmax[threadIdx.x + 96]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (threadIdx.x == 0) atomicMax(ktmax + bh, __float_as_uint(m));   // |K'| >= 0: orders as uint
        }
        return;
    }
    if (threadIdx.x < NGK) {
        const int g = threadIdx.x;
        float amax = 0.f;
        if (GRAN == 3) {
            amax = __uint_as_float(__ldcg(ktmax + bh));
        } else if (GRAN == 2) {
            amax = rowmax[g];
        } else if (GRAN == 1) {
            if (g < 2)
                for (int r = 64 * g; r < 64 * g + 64; ++r) amax = fmaxf(amax, rowmax[r]);
        } else {
            const int r0 = 64 * (g / 4) + 2 * (g % 4);
            for (int k = 0; k < 8; ++k) amax = fmax3(amax, rowmax[r0 + 8 * k], rowmax[r0 + 8 * k + 1]);
        }
        const float delta = __fdiv_rn(amax, (float)qk_max);
        gdelta[g] = delta;
        dk[((size_t)bh * nT + tile) * NGK + g] = delta;
    }
    __syncthreads();
    // K codes (O-3) straight to the swizzled K^ tile image
    int8_t* kimg = khat + ((size_t)bh * nT + tile) * (size_t)kTile * D;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs;
        const float delta = gdelta[GRAN == 3 ? 0 : GRAN == 2 ? r : GRAN == 1 ? r / 64 : 4 * (r / 64) + (r % 8) / 2];
        *reinterpret_cast<uint2*>(kimg + swz_off<D>(r, cg * 8)) = quant_pack8(kx[p], delta, qk_max, e4m3_codes != 0);
    }
    }
    if constexpr ((PART & 2) != 0) {
    // V codes (O-4): thread = channel pair (c, c+1) x TOK consecutive tokens -> V^T rows c, c+1
    constexpr int NPAIR = D / 2, TOK = kTile / (256 / NPAIR);
    const int cp = threadIdx.x % NPAIR, t0 = (threadIdx.x / NPAIR) * TOK, c = 2 * cp;
    const float d0 = dvs[c], d1 = dvs[c + 1];
    const float d0s = d0 != 0.0f ? d0 : 1.0f, d1s = d1 != 0.0f ? d1 : 1.0f;    // all-zero channel: codes 0
    const float m0 = vmean ? vmean[(size_t)bh * D + c] : 0.0f, m1 = vmean ? vmean[(size_t)bh * D + c + 1] : 0.0f;
    uint8_t* vimg = vhat + ((size_t)bh * nT + tile) * (size_t)kTile * D;
#pragma unroll
    for (int tb = 0; tb < TOK; tb += 16) {
        uint32_t w0[4], w1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t pr[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const __half2 h = *reinterpret_cast<const __half2*>(&vt[(t0 + tb + 4 * q + e) * VS + c]);
                const float2 f = __half22float2(h);
                const bool pad = tile * kTile + t0 + tb + 4 * q + e >= N;   // padded token: code 0
                const float q0 = __fdiv_rn(__fsub_rn(f.x, m0), d0s);         // V' = V - V_m
                const float q1 = __fdiv_rn(__fsub_rn(f.y, m1), d1s);
                float2 qv;
                qv.x = (d0 != 0.0f && !pad) ? q0 : 0.0f;
                qv.y = (d1 != 0.0f && !pad) ? q1 : 0.0f;
                pr[e] = (uint32_t)__nv_cvt_float2_to_fp8x2(qv, __NV_SATFINITE, __NV_E4M3);   // lo = c, hi = c+1
            }
            const uint32_t x = pr[0] | (pr[1] << 16), y = pr[2] | (pr[3] << 16);
            w0[q] = __byte_perm(x, y, 0x6420);
            w1[q] = __byte_perm(x, y, 0x7531);
        }
        *reinterpret_cast<uint4*>(vimg + swz_off<128>(c, t0 + tb)) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
        *reinterpret_cast<uint4*>(vimg + swz_off<128>(c + 1, t0 + tb)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
    }
    }
}

// ---------------------------------------------------------------------------------------------
// k_q_quant: grid (N_pad/128, B*Hq), 256 threads.  One 128-token Q block (= smoothing block).
//   qbar [nT][D] fp32, Q^ tile image [128][D] swizzled, dq: 32 groups per block
//   (g_Q = 8*(t/32) + t%8, "tokens i, 8+i, 16+i, 24+i")
// Thread (cg, rofs) holds channels [8cg, 8cg+8) of rows rofs + RPP*p.  Instruction-lean form:
//  * exact means in fp64: 128 fp16 values are multiples of 2^-24 below 2^23 in magnitude, so every
//    partial sum fits 47 bits and the fp64 sum is exact in any order -- bit-identical to the int64
//    fixed-point sum of reading C-1 (and 8x fewer instructions than the fixed-point conversion);
//  * the group absmax without atomics: per-row maxima in shared memory, one thread per group;
//  * gamma(Q) is computed once and kept in registers for the quantizer.
// ---------------------------------------------------------------------------------------------

template <int D, int GRAN = 0>
__global__ void __launch_bounds__(256, 4) k_q_quant(const __half* __restrict__ Q, int N, int qk_max, int e4m3_codes, int smooth_q,
                                                    int8_t* __restrict__ qhat, float* __restrict__ dq,
                                                    float* __restrict__ qbar_out, uint8_t* __restrict__ qbt,
                                                    unsigned int* qtmax = nullptr) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    // qtmax (per-tensor granularity): GRAN 4 accumulates max|gamma(Q_i)| of the head into qtmax[bh]
    // and stops (q_bar and its images are written as usual); GRAN 3 quantizes with
    // delta_Q = qtmax[bh] / qk_max.
    constexpr int TPR = D / 8, RPP = 256 / TPR, NP = kTile / RPP;   // d=128: 16 / 16 / 8; d=64: 8 / 32 / 4
    const int tile = blockIdx.x, bh = blockIdx.y, nT = gridDim.x;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cg = threadIdx.x % TPR, rofs = threadIdx.x / TPR;
    const int n = min(kTile, N - tile * kTile);          // present tokens (C-18)
    __shared__ double part[8][D];
    __shared__ float qbar[D];
    const size_t base = (size_t)bh * N * D;
    uint4 raw[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs, t = tile * kTile + r;
        raw[p] = make_uint4(0, 0, 0, 0);
        if (r < n) raw[p] = __ldg(reinterpret_cast<const uint4*>(Q + base + (size_t)t * D + cg * 8));
    }
    if (smooth_q) {
        double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const uint16_t* h = reinterpret_cast<const uint16_t*>(&raw[p]);
#pragma unroll
            for (int i = 0; i < 8; ++i) s[i] += fp16_to_f64(h[i]);          // exact (see above)
        }
#pragma unroll
        for (int m = TPR; m < 32; m <<= 1)
#pragma unroll
            for (int i = 0; i < 8; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], m);
        if (lane < TPR) {
#pragma unroll
            for (int i = 0; i < 8; ++i) part[warp][cg * 8 + i] = s[i];
        }
    }
    __syncthreads();
    if (threadIdx.x < D) {
        const int c = threadIdx.x;
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += smooth_q ? part[w][c] : 0.0;
        const float qb = smooth_q ? (float)__ddiv_rn(t, (double)n) : 0.0f;   // O-5 (= fixed_mean of C-1)
        qbar[c] = qb;
        qbar_out[((size_t)bh * nT + tile) * D + c] = qb;
        // tf32 big/small split of q_bar for the tensor-core Delta S GEMM (dsg.cuh): image per
        // (bh, 256-block chunk, 32-channel atom) = [big 256 x 128 B][small 256 x 128 B], SW128.
        const int nch = (nT + 255) / 256, row = tile % 256;
        uint8_t* img = qbt + (((size_t)bh * nch + tile / 256) * (D / 32) + c / 32) * (2 * 256 * 128);
        const float big = tf32_big(qb);
        const uint32_t off = swz_off<128>(row, (c % 32) * 4);
        *reinterpret_cast<float*>(img + off) = big;
        *reinterpret_cast<float*>(img + 256 * 128 + off) = __fsub_rn(qb, big);
    }
    __syncthreads();
    // gamma(Q) (O-5), recomputed from the raw fp16 in both passes (cheaper than holding 8 x NP
    // floats: fewer registers, more CTAs in flight); absmax per row (over the TPR lanes of the row)
    // -> rowmax, then the group absmax of the granularity from rowmax (per-thread group g = rows
    // 32(g/8) + g%8 + 8k, k < 4, "tokens i, 8+i, 16+i, 24+i")
    __shared__ float rowmax[128];
    __shared__ float gdelta[128];
    float qv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) qv[i] = qbar[cg * 8 + i];
    auto gamma8 = [&](int p, float (&x)[8]) {
        const int r = p * RPP + rofs;
        const __half2* h2 = reinterpret_cast<const __half2*>(&raw[p]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h2[i]);
            x[2 * i] = (r < n) ? __fsub_rn(f.x, qv[2 * i]) : 0.0f;
            x[2 * i + 1] = (r < n) ? __fsub_rn(f.y, qv[2 * i + 1]) : 0.0f;
        }
    };
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs;
        float x[8];
        gamma8(p, x);
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) m = fmax3(m, fabsf(x[2 * i]), fabsf(x[2 * i + 1]));
#pragma unroll
        for (int o = 1; o < TPR; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (cg == 0) rowmax[r] = m;
    }
    __syncthreads();
    constexpr int NGQ = gran_nq(GRAN);
    if constexpr (GRAN == 4) {
        if (threadIdx.x < 32) {
            float m = fmaxf(fmaxf(rowmax[threadIdx.x], rowmax[threadIdx.x + 32]),
                            fmaxf(rowmax[threadIdx.x + 64], rowmax[threadIdx.x + 96]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (threadIdx.x == 0) atomicMax(qtmax + bh, __float_as_uint(m));
        }
        return;
    }
    if (threadIdx.x < NGQ) {
        const int g = threadIdx.x;
        float amax;
        if (GRAN == 3) {
            amax = __uint_as_float(__ldcg(qtmax + bh));
        } else if (GRAN == 2) {
            amax = rowmax[g];
        } else if (GRAN == 1) {
            amax = 0.f;
            for (int r = 0; r < 128; ++r) amax = fmaxf(amax, rowmax[r]);
        } else {
            const int r0 = 32 * (g / 8) + g % 8;
            amax = fmaxf(fmaxf(rowmax[r0], rowmax[r0 + 8]), fmaxf(rowmax[r0 + 16], rowmax[r0 + 24]));
        }
        const float delta = __fdiv_rn(amax, (float)qk_max);   // O-6
        gdelta[g] = delta;
        dq[((size_t)bh * nT + tile) * NGQ + g] = delta;
    }
    __syncthreads();
    int8_t* img = qhat + ((size_t)bh * nT + tile) * (size_t)kTile * D;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs;
        const float delta = gdelta[GRAN == 2 ? r : GRAN == 1 || GRAN == 3 ? 0 : 8 * (r / 32) + (r % 8)];
        float x[8];
        gamma8(p, x);
        *reinterpret_cast<uint2*>(img + swz_off<D>(r, cg * 8)) = quant_pack8(x, delta, qk_max, e4m3_codes != 0);
    }
}

// ---------------------------------------------------------------------------------------------
// k_delta_s: grid (N_pad/128 key tiles, B*Hq), 128 threads, thread = key.
//   ds[bh][i][t] = (log2(e)/sqrt(d)) * sum_c qbar_i[c] * (fp32(K[t,c]) - kbar[c])   (O-7)
// fp32 FMA chain over c ascending.  Keys t >= N get 0 (masked in the kernel anyway).
// ---------------------------------------------------------------------------------------------
template <int D, int NI = 16>
__global__ void __launch_bounds__(128) k_delta_s(const __half* __restrict__ K, const unsigned long long* __restrict__ ksum,
                                                 const float* __restrict__ qbar, int N, int Hq, int Hkv,
                                                 float scale_log2, float* __restrict__ ds, int tri) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    // Latency-lean form (the round-1 kernel held K' in 128 fp32 registers per thread -- 3 CTAs per SM --
    // and made 128 scalar k_bar loads per thread: C2-1K 28 us): the key tile is staged in padded shared
    // memory by coalesced loads (row stride D + 2 halves: thread t reads row t conflict-free), k_bar and
    // q_bar come from shared memory, and NI Q blocks (the launch picks 8 or 16 for nT) are accumulated
    // at once -- NI independent chains per thread.  Each output keeps its fp32 FMA chain over c ascending
    // with K'[t,c] = fp32(K[t,c]) - k_bar[c] (O-2).
    constexpr int KS = D + 2;                          // padded smem row (halves)
    const int kt = blockIdx.x, bhq = blockIdx.y, nT = gridDim.x, Np = nT * kTile;
    const int b = bhq / Hq, hq = bhq % Hq, hk = hq / (Hq / Hkv);
    const int bhk = b * Hkv + hk;
    const int t = kt * kTile + threadIdx.x;
    __shared__ __align__(16) float sq[NI][D];
    __shared__ __align__(16) float skb[D];
    __shared__ __align__(16) __half sk[kTile * KS];
    {
        const __half* kt0 = K + ((size_t)bhk * N + (size_t)kt * kTile) * D;
        constexpr int CPR = D / 8, NL = kTile * CPR / 128;   // 16-byte chunks per row / per thread
        uint4 u[NL];                                   // every load in flight before the first store
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            const int e = threadIdx.x + 128 * l, r = e / CPR, c8 = e % CPR;
            u[l] = make_uint4(0, 0, 0, 0);
            if (kt * kTile + r < N) u[l] = __ldg(reinterpret_cast<const uint4*>(kt0 + (size_t)r * D) + c8);
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            const int e = threadIdx.x + 128 * l, r = e / CPR, c8 = e % CPR;
            uint32_t* dst = reinterpret_cast<uint32_t*>(&sk[r * KS + c8 * 8]);   // 4-byte aligned (KS even)
            dst[0] = u[l].x;
            dst[1] = u[l].y;
            dst[2] = u[l].z;
            dst[3] = u[l].w;
        }
    }
    // k_bar from k_kv_stats' exact sums (the same fixed_mean as k_kv_quant, O-1): Delta S needs only
    // the statistics, so it runs concurrently with k_kv_quant (sage2_api.cu launch_prepare)
    if (threadIdx.x < D) skb[threadIdx.x] = fixed_mean((long long)ksum[(size_t)bhk * D + threadIdx.x], N);
    const float live = t < N ? 1.0f : 0.0f;            // keys t >= N: 0 (masked in the kernel anyway)
    const __half2* myk = reinterpret_cast<const __half2*>(&sk[threadIdx.x * KS]);
    const float* qb = qbar + (size_t)bhq * nT * D;
    // row offsets as ds_row() (common.cuh): full rows, or the causal triangular layout (i >= kt only)
    auto row = [&](int i) {
        return tri ? (size_t)bhq * 64 * (size_t)nT * (nT + 1) + 64 * (size_t)i * (i + 1) : ((size_t)bhq * nT + i) * Np;
    };
    for (int i0 = tri ? (kt / NI) * NI : 0; i0 < nT; i0 += NI) {
        const int ni = min(NI, nT - i0);
        __syncthreads();
        for (int e = threadIdx.x; e < ni * D / 4; e += 128)
            reinterpret_cast<float4*>(&sq[0][0])[e] = __ldg(reinterpret_cast<const float4*>(qb + (size_t)i0 * D) + e);
        __syncthreads();
        float acc[NI];
#pragma unroll
        for (int k = 0; k < NI; ++k) acc[k] = 0.f;
#pragma unroll 4
        for (int c = 0; c < D; c += 4) {
            const float4 kb4 = *reinterpret_cast<const float4*>(&skb[c]);
            const float2 f01 = __half22float2(myk[c / 2]);
            const float2 f23 = __half22float2(myk[c / 2 + 1]);
            const float k0 = __fsub_rn(f01.x, kb4.x) * live, k1 = __fsub_rn(f01.y, kb4.y) * live;
            const float k2 = __fsub_rn(f23.x, kb4.z) * live, k3 = __fsub_rn(f23.y, kb4.w) * live;
#pragma unroll
            for (int k = 0; k < NI; ++k) {                    // rows >= ni hold stale values, never stored
                const float4 qv = *reinterpret_cast<const float4*>(&sq[k][c]);
                acc[k] = fmaf(qv.x, k0, acc[k]);
                acc[k] = fmaf(qv.y, k1, acc[k]);
                acc[k] = fmaf(qv.z, k2, acc[k]);
                acc[k] = fmaf(qv.w, k3, acc[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < NI; ++k) {
            const int i = i0 + k;
            if (k < ni && (!tri || i >= kt)) ds[row(i) + t] = acc[k] * scale_log2;
        }
    }
}

}  // namespace sage2

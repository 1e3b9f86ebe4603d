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

// FP16 bits -> exact integer value * 2^24 (every finite fp16 is a multiple of 2^-24).
__device__ __forceinline__ long long fp16_fixed24(uint16_t h) {
    int e = (h >> 10) & 31, m = h & 1023;
    long long v = (e == 0) ? (long long)m : ((long long)(1024 + m) << (e - 1));
    return (h & 0x8000) ? -v : v;
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

// ---------------------------------------------------------------------------------------------
// k_kv_stats: grid (row chunks, B*Hkv), 256 threads.  Each thread reads 8 consecutive channels
// (16 B) of a token row.
// ---------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_kv_stats(const __half* __restrict__ K, const __half* __restrict__ V,
                                                  int N, int rows_per_cta, unsigned long long* __restrict__ ksum,
                                                  unsigned int* __restrict__ vmax) {
    constexpr int TPR = D / 8;          // threads per row
    constexpr int RPP = 256 / TPR;      // rows per pass
    const int bh = blockIdx.y;
    const int cg = threadIdx.x % TPR, rofs = threadIdx.x / TPR;
    const size_t base = (size_t)bh * N * D;
    const int r0 = blockIdx.x * rows_per_cta, r1 = min(N, r0 + rows_per_cta);
    long long s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t vm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int r = r0 + rofs; r < r1; r += RPP) {
        uint4 kk = __ldg(reinterpret_cast<const uint4*>(K + base + (size_t)r * D + cg * 8));
        uint4 vv = __ldg(reinterpret_cast<const uint4*>(V + base + (size_t)r * D + cg * 8));
        const uint16_t* kh = reinterpret_cast<const uint16_t*>(&kk);
        const uint16_t* vh = reinterpret_cast<const uint16_t*>(&vv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            s[i] += fp16_fixed24(kh[i]);
            float a = fabsf(__half2float(__ushort_as_half(vh[i])));
            vm[i] = max(vm[i], __float_as_uint(a));     // non-negative floats order as uints
        }
    }
    __shared__ long long ssum[256][8];
    __shared__ uint32_t smax[256][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        ssum[threadIdx.x][i] = s[i];
        smax[threadIdx.x][i] = vm[i];
    }
    __syncthreads();
    if (threadIdx.x < D) {
        const int c = threadIdx.x, g = c / 8, i = c % 8;
        long long t = 0;
        uint32_t m = 0;
        for (int k = 0; k < RPP; ++k) {
            t += ssum[k * TPR + g][i];
            m = max(m, smax[k * TPR + g][i]);
        }
        atomicAdd(ksum + (size_t)bh * D + c, (unsigned long long)t);   // two's-complement: exact
        atomicMax(vmax + (size_t)bh * D + c, m);
    }
}

// ---------------------------------------------------------------------------------------------
// k_kv_quant: grid (N_pad/128, B*Hkv), 256 threads.  One 128-token tile of one KV head.
//   K^ tile image  : [128 tokens][D bytes], K-major swizzled (row = token)
//   V^T tile image : [D channels][128 bytes], K-major swizzled (row = channel), E4M3
//   dk             : 8 groups per tile (g_K = 4*(t/64) + (t%8)/2)
// ---------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_kv_quant(const __half* __restrict__ K, const __half* __restrict__ V,
                                                  int N, int qk_max, const unsigned long long* __restrict__ ksum,
                                                  const unsigned int* __restrict__ vmax, int8_t* __restrict__ khat,
                                                  float* __restrict__ dk, uint8_t* __restrict__ vhat,
                                                  float* __restrict__ kbar_out, float* __restrict__ dv_out) {
    constexpr int TPR = D / 8, RPP = 256 / TPR, NP = kTile / RPP;   // passes
    const int tile = blockIdx.x, bh = blockIdx.y, nT = gridDim.x;
    const int cg = threadIdx.x % TPR, rofs = threadIdx.x / TPR;
    __shared__ float kbar[D], dvs[D];
    __shared__ uint32_t gmax[8];
    __shared__ __align__(1024) uint8_t simg[kTile * D];   // staging for the swizzled V^T tile
    __shared__ __align__(1024) uint8_t kimg[kTile * D];
    if (threadIdx.x < D) {
        const int c = threadIdx.x;
        kbar[c] = fixed_mean((long long)ksum[(size_t)bh * D + c], N);                 // O-1
        dvs[c] = __fdiv_rn(__uint_as_float(vmax[(size_t)bh * D + c]), 448.0f);      // O-4
        if (tile == 0) {
            kbar_out[(size_t)bh * D + c] = kbar[c];
            dv_out[(size_t)bh * D + c] = dvs[c];
        }
    }
    if (threadIdx.x < 8) gmax[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = (size_t)bh * N * D;
    float kp[NP][8];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs, t = tile * kTile + r;
        uint4 kk = make_uint4(0, 0, 0, 0);
        if (t < N) kk = __ldg(reinterpret_cast<const uint4*>(K + base + (size_t)t * D + cg * 8));
        const __half* kh = reinterpret_cast<const __half*>(&kk);
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            kp[p][i] = (t < N) ? __fsub_rn(__half2float(kh[i]), kbar[cg * 8 + i]) : 0.0f;  // O-2
            m = fmaxf(m, fabsf(kp[p][i]));
        }
        const int g = 4 * (r / 64) + (r % 8) / 2;                                      // g_K
        atomicMax(&gmax[g], __float_as_uint(m));
    }
    __syncthreads();
    // K codes (O-3)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs;
        const int g = 4 * (r / 64) + (r % 8) / 2;
        const float delta = __fdiv_rn(__uint_as_float(gmax[g]), (float)qk_max);
        uint32_t w[2] = {0, 0};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t code = (uint32_t)(uint8_t)(int8_t)quant_code(kp[p][i], delta, qk_max);
            w[i / 4] |= code << (8 * (i % 4));
        }
        *reinterpret_cast<uint2*>(kimg + swz_off<D>(r, cg * 8)) = make_uint2(w[0], w[1]);
    }
    if (threadIdx.x < 8)
        dk[(size_t)bh * (nT * 8) + tile * 8 + threadIdx.x] =
            __fdiv_rn(__uint_as_float(gmax[threadIdx.x]), (float)qk_max);
    // V codes (O-4), transposed into the V^T tile (row = channel, column byte = token)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs, t = tile * kTile + r;
        uint4 vv = make_uint4(0, 0, 0, 0);
        if (t < N) vv = __ldg(reinterpret_cast<const uint4*>(V + base + (size_t)t * D + cg * 8));
        const __half* vh = reinterpret_cast<const __half*>(&vv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int c = cg * 8 + i;
            const float dvc = dvs[c];
            uint8_t code = 0;
            if (dvc != 0.0f)
                code = (uint8_t)__nv_cvt_float_to_fp8(__fdiv_rn(__half2float(vh[i]), dvc), __NV_SATFINITE, __NV_E4M3);
            simg[swz_off<128>(c, r)] = code;
        }
    }
    __syncthreads();
    // coalesced 16-byte stores of both tile images
    const size_t tile_bytes = (size_t)kTile * D;
    uint4* kdst = reinterpret_cast<uint4*>(khat + ((size_t)bh * nT + tile) * tile_bytes);
    uint4* vdst = reinterpret_cast<uint4*>(vhat + ((size_t)bh * nT + tile) * tile_bytes);
    for (int i = threadIdx.x; i < (int)(tile_bytes / 16); i += 256) {
        kdst[i] = reinterpret_cast<const uint4*>(kimg)[i];
        vdst[i] = reinterpret_cast<const uint4*>(simg)[i];
    }
}

// ---------------------------------------------------------------------------------------------
// k_q_quant: grid (N_pad/128, B*Hq), 256 threads.  One 128-token Q block (= smoothing block).
//   qbar [nT][D] fp32, Q^ tile image [128][D] swizzled, dq: 32 groups per block
//   (g_Q = 8*(t/32) + t%8, "tokens i, 8+i, 16+i, 24+i")
// ---------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_q_quant(const __half* __restrict__ Q, int N, int qk_max, int smooth_q,
                                                 int8_t* __restrict__ qhat, float* __restrict__ dq,
                                                 float* __restrict__ qbar_out, uint8_t* __restrict__ qbt) {
    constexpr int TPR = D / 8, RPP = 256 / TPR, NP = kTile / RPP;
    const int tile = blockIdx.x, bh = blockIdx.y, nT = gridDim.x;
    const int cg = threadIdx.x % TPR, rofs = threadIdx.x / TPR;
    const int n = min(kTile, N - tile * kTile);          // present tokens (C-18)
    __shared__ unsigned long long csum[D];
    __shared__ float qbar[D];
    __shared__ uint32_t gmax[32];
    __shared__ __align__(1024) uint8_t qimg[kTile * D];
    if (threadIdx.x < D) csum[threadIdx.x] = 0;
    if (threadIdx.x < 32) gmax[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = (size_t)bh * N * D;
    uint4 raw[NP];
    long long s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs, t = tile * kTile + r;
        raw[p] = make_uint4(0, 0, 0, 0);
        if (r < n) raw[p] = __ldg(reinterpret_cast<const uint4*>(Q + base + (size_t)t * D + cg * 8));
        const uint16_t* h = reinterpret_cast<const uint16_t*>(&raw[p]);
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] += fp16_fixed24(h[i]);
    }
    if (smooth_q) {
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicAdd(&csum[cg * 8 + i], (unsigned long long)s[i]);
    }
    __syncthreads();
    if (threadIdx.x < D) {
        qbar[threadIdx.x] = smooth_q ? fixed_mean((long long)csum[threadIdx.x], n) : 0.0f;   // O-5
        qbar_out[((size_t)bh * nT + tile) * D + threadIdx.x] = qbar[threadIdx.x];
        // tf32 big/small split of q_bar for the tensor-core Delta S GEMM (dsg.cuh): image per
        // (bh, 256-block chunk, 32-channel atom) = [big 256 x 128 B][small 256 x 128 B], SW128.
        const int c = threadIdx.x, nch = (nT + 255) / 256, row = tile % 256;
        uint8_t* img = qbt + (((size_t)bh * nch + tile / 256) * (D / 32) + c / 32) * (2 * 256 * 128);
        const float big = tf32_big(qbar[c]);
        const uint32_t off = swz_off<128>(row, (c % 32) * 4);
        *reinterpret_cast<float*>(img + off) = big;
        *reinterpret_cast<float*>(img + 256 * 128 + off) = __fsub_rn(qbar[c], big);
    }
    __syncthreads();
    float qp[NP][8];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs;
        const __half* h = reinterpret_cast<const __half*>(&raw[p]);
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            qp[p][i] = (r < n) ? __fsub_rn(__half2float(h[i]), qbar[cg * 8 + i]) : 0.0f;
            m = fmaxf(m, fabsf(qp[p][i]));
        }
        atomicMax(&gmax[8 * (r / 32) + (r % 8)], __float_as_uint(m));
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int r = p * RPP + rofs;
        const float delta = __fdiv_rn(__uint_as_float(gmax[8 * (r / 32) + (r % 8)]), (float)qk_max);   // O-6
        uint32_t w[2] = {0, 0};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t code = (uint32_t)(uint8_t)(int8_t)quant_code(qp[p][i], delta, qk_max);
            w[i / 4] |= code << (8 * (i % 4));
        }
        *reinterpret_cast<uint2*>(qimg + swz_off<D>(r, cg * 8)) = make_uint2(w[0], w[1]);
    }
    if (threadIdx.x < 32)
        dq[((size_t)bh * nT + tile) * 32 + threadIdx.x] = __fdiv_rn(__uint_as_float(gmax[threadIdx.x]), (float)qk_max);
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(qhat + ((size_t)bh * nT + tile) * (size_t)kTile * D);
    for (int i = threadIdx.x; i < kTile * D / 16; i += 256) dst[i] = reinterpret_cast<const uint4*>(qimg)[i];
}

// ---------------------------------------------------------------------------------------------
// k_delta_s: grid (N_pad/128 key tiles, B*Hq), 128 threads, thread = key.
//   ds[bh][i][t] = (log2(e)/sqrt(d)) * sum_c qbar_i[c] * (fp32(K[t,c]) - kbar[c])   (O-7)
// fp32 FMA chain over c ascending.  Keys t >= N get 0 (masked in the kernel anyway).
// ---------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128) k_delta_s(const __half* __restrict__ K, const float* __restrict__ kbar,
                                                 const float* __restrict__ qbar, int N, int Hq, int Hkv,
                                                 float scale_log2, float* __restrict__ ds) {
    constexpr int ICH = 32;                            // Q blocks per smem chunk
    const int kt = blockIdx.x, bhq = blockIdx.y, nT = gridDim.x, Np = nT * kTile;
    const int b = bhq / Hq, hq = bhq % Hq, hk = hq / (Hq / Hkv);
    const int bhk = b * Hkv + hk;
    const int t = kt * kTile + threadIdx.x;
    __shared__ float sq[ICH][D];
    float kp[D];
    if (t < N) {
        const __half* krow = K + ((size_t)bhk * N + t) * D;
#pragma unroll
        for (int c = 0; c < D; c += 8) {
            uint4 u = __ldg(reinterpret_cast<const uint4*>(krow + c));
            const __half* h = reinterpret_cast<const __half*>(&u);
#pragma unroll
            for (int i = 0; i < 8; ++i) kp[c + i] = __fsub_rn(__half2float(h[i]), __ldg(kbar + (size_t)bhk * D + c + i));
        }
    } else {
#pragma unroll
        for (int c = 0; c < D; ++c) kp[c] = 0.0f;
    }
    const float* qb = qbar + (size_t)bhq * nT * D;
    float* out = ds + (size_t)bhq * nT * Np;
    for (int i0 = 0; i0 < nT; i0 += ICH) {
        const int ni = min(ICH, nT - i0);
        __syncthreads();
        for (int e = threadIdx.x; e < ni * D; e += 128) sq[e / D][e % D] = qb[(size_t)i0 * D + e];
        __syncthreads();
        for (int ii = 0; ii < ni; ++ii) {
            float acc = 0.0f;
#pragma unroll
            for (int c = 0; c < D; ++c) acc = fmaf(sq[ii][c], kp[c], acc);
            out[(size_t)(i0 + ii) * Np + t] = acc * scale_log2;
        }
    }
}

}  // namespace sage2

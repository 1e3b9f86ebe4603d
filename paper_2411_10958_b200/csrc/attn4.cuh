// attn4.cuh -- SageAttention2 attention kernel v4 for sm_100a (the default).
// Alg. 1 inner loop, same arithmetic as attn.cuh (v0), organised for overlap.
//
// CTA = one 128-row Q block i of one (b, h_q); KV tiles of 128 keys in ascending order (P:250,
// reading C-9).  TMEM: three S/R buffers X[0..2] (128 columns each) and O (D columns, fp32):
// QK(j+1), the softmax of S(j), PV(j) and the promotion of R(j-1) all overlap.
//
// 12 warps (384 threads):
//   warp 0       producer: bulk-async (TMA engine) copies of the pre-swizzled tile images
//   warp 1       MMA issuer (one thread):
//                  S(j) = Q^ K^_j^T   tcgen05.mma.kind::i8     -> X[j%3] (s32, exact)
//                  R(j) = P^(j) V^_j  tcgen05.mma.kind::f8f6f4 -> X[j%3] once S(j) was consumed
//                                     (a fresh fp32 accumulator per KV tile)
//                QK(j+1) goes into the next buffer while the softmax works on S(j).
//   warps 4-7    "half A": key columns 0..63 of every S row, O columns 0..D/2-1
//   warps 8-11   "half B": key columns 64..127,              O columns D/2..D-1
//                (warp w and warp w+4 own the same 32 query rows = TMEM lanes 32(w%4)..+31)
//                per KV tile j, one thread per (row, half):
//                  s = S*dQ*dK*log2e/sqrt(d) + Delta S', masks, half-row max;
//                  exact row max via a 64-thread named barrier with the partner warp (C-10);
//                  P^ = e4m3(2^(s - m + log2 448)) -> smem P^[j%2] (A operand of the PV MMA);
//                  then the two-level promotion of the previous tile, O = alpha(j-1) O + R(j-1)
//                  in fp32, freeing X[(j-1)%3] for QK(j+2).
//                epilogue O / l / 448 * delta_V -> fp16, l = l_A + l_B.
#pragma once
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdint>

#include "attn.cuh"
#include "ptx.cuh"

namespace sage2 {

constexpr int kStages4 = 4;

template <int D>
struct Attn4Smem {
    static constexpr uint32_t TILE = 128 * D;
    static constexpr uint32_t Q = 0;
    // stage: K^ | V^T | dS (512) | dK (32)
    static constexpr uint32_t ST_K = 0, ST_V = TILE, ST_DS = 2 * TILE, ST_DK = 2 * TILE + 512;
    static constexpr uint32_t STAGE = ((2 * TILE + 512 + 32) + 1023) / 1024 * 1024;
    static constexpr uint32_t ST0 = TILE;
    static constexpr uint32_t P = ST0 + kStages4 * STAGE;          // P^[2] 128 x 128 e4m3
    static constexpr uint32_t XCHG = P + 2 * 16384;                 // float [2 slots][2 halves][128]
    static constexpr uint32_t BAR = XCHG + 2 * 2 * 128 * 4;
    // q_full, kv_full[S], kv_empty[S], s_full[3], x_free[3], p_full[2], r_full[2]
    // (p_full / r_full alternate per KV tile: their producer can run one tile ahead of the waiter,
    //  and a parity wait must never be able to fall two phases behind)
    static constexpr uint32_t NBAR = 1 + 2 * kStages4 + 10;
    static constexpr uint32_t TMEMPTR = BAR + 8 * NBAR;
    static constexpr uint32_t BYTES = TMEMPTR + 16;
    static constexpr uint32_t ALLOC = BYTES + 1024;
};


template <int D, bool CAUSAL, bool DUMP, bool NULLSM = false, bool NULLMMA = false, bool TIMING = false>
__global__ void __launch_bounds__(384, 1) k_attn4(const AttnParams p) {
    using L = Attn4Smem<D>;
    constexpr int DH = D / 2;                      // O columns per half
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int wg = warp / 4;
    const int nT = p.nT, Np = nT * 128;
    const int i = CAUSAL ? (nT - 1 - (int)blockIdx.x) : (int)blockIdx.x;   // heavy causal tiles first
    const int hq = blockIdx.y, b = blockIdx.z;
    const int bhq = b * p.Hq + hq;
    const int bhk = b * p.Hkv + hq / (p.Hq / p.Hkv);
    const int nkv = CAUSAL ? i + 1 : nT;

    // TIMING builds: clock64 stamps of one thread per role in CTA (0,0,0) -> (uint64*)p.s_dump
    const bool tsel = TIMING && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
    auto ts = [&](int who, int j, int k) {
        if (TIMING && tsel && j < 64)
            reinterpret_cast<unsigned long long*>(p.s_dump)[(who * 64 + j) * 16 + k] = clock64();
    };
    const uint32_t bar0 = sbase + L::BAR;
    const uint32_t bar_q = bar0;
    auto bar_kv_full = [&](int s) { return bar0 + 8 * (1 + s); };
    auto bar_kv_empty = [&](int s) { return bar0 + 8 * (1 + kStages4 + s); };
    auto bar_s_full = [&](int bb) { return bar0 + 8 * (1 + 2 * kStages4 + bb); };
    auto bar_x_free = [&](int bb) { return bar0 + 8 * (4 + 2 * kStages4 + bb); };
    auto bar_p_full = [&](int j) { return bar0 + 8 * (7 + 2 * kStages4 + (j & 1)); };
    auto bar_r_full = [&](int j) { return bar0 + 8 * (9 + 2 * kStages4 + (j & 1)); };
    auto stage_addr = [&](int s) { return sbase + L::ST0 + s * L::STAGE; };

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < kStages4; ++s) {
            mbar_init(bar_kv_full(s), 1);
            mbar_init(bar_kv_empty(s), 1);
        }
        for (int bb = 0; bb < 3; ++bb) {
            mbar_init(bar_s_full(bb), 1);
            mbar_init(bar_x_free(bb), 256);
        }
        for (int jj = 0; jj < 2; ++jj) {
            mbar_init(bar_p_full(jj), 256);
            mbar_init(bar_r_full(jj), 1);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(sbase + L::TMEMPTR);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sgen + L::TMEMPTR);

    if (wg == 0) {
        setmaxnreg_dec<56>();
        if (warp == 0 && lane == 0) {
            // ===================== producer =====================
            const size_t tile_bytes = (size_t)128 * D;
            mbar_arrive_expect_tx(bar_q, L::TILE);
            bulk_g2s(sbase + L::Q, p.qhat + ((size_t)bhq * nT + i) * tile_bytes, L::TILE, bar_q);
            const uint64_t keep = policy_evict_last();
            for (int j = 0; j < nkv; ++j) {
                const int s = j % kStages4;
                if (j >= kStages4) mbar_wait(bar_kv_empty(s), ((j / kStages4) - 1) & 1);
                const uint32_t sa = stage_addr(s);
                mbar_arrive_expect_tx(bar_kv_full(s), 2 * L::TILE + 512 + 32);
                bulk_g2s_hint(sa + L::ST_K, p.khat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, bar_kv_full(s), keep);
                bulk_g2s_hint(sa + L::ST_V, p.vhat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, bar_kv_full(s), keep);
                bulk_g2s(sa + L::ST_DS, p.ds + ds_row(p.ds_tri, bhq, i, nT) + (size_t)j * 128, 512, bar_kv_full(s));
                bulk_g2s(sa + L::ST_DK, p.dk + (size_t)bhk * nT * 8 + (size_t)j * 8, 32, bar_kv_full(s));
            }
        } else if (warp == 1 && lane == 0) {
            // ===================== MMA issuer =====================
            constexpr uint32_t IDQK = idesc_i8(128, 128);
            constexpr uint32_t IDPV = idesc_e4m3(128, D);
            const uint64_t qdesc = smem_desc<D>(sbase + L::Q);
            auto issue_qk = [&](int j) {
                const int s = j % kStages4, bb = j % 3;
                mbar_wait(bar_kv_full(s), (j / kStages4) & 1);
                if (j >= 3) mbar_wait(bar_x_free(bb), ((j / 3) - 1) & 1);   // R(j-3) consumed
                tc_fence_after();
                const uint64_t kdesc = smem_desc<D>(stage_addr(s) + L::ST_K);
                if (!NULLMMA) {
#pragma unroll
                    for (int kk = 0; kk < D / 32; ++kk)
                        mma_i8(tmem + 128 * bb, qdesc + 2 * kk, kdesc + 2 * kk, IDQK, kk > 0);
                }
                mma_commit(bar_s_full(bb));
            };
            mbar_wait(bar_q, 0);
            issue_qk(0);
            for (int j = 0; j < nkv; ++j) {
                ts(2, j, 0);
                if (j + 1 < nkv) issue_qk(j + 1);
                ts(2, j, 1);
                const int s = j % kStages4, bb = j % 3;
                mbar_wait(bar_p_full(j), (j >> 1) & 1);           // both halves wrote P^(j)
                ts(2, j, 2);
                tc_fence_after();
                const uint64_t pdesc = smem_desc<128>(sbase + L::P + (j & 1) * 16384);
                const uint64_t vdesc = smem_desc<128>(stage_addr(s) + L::ST_V);
                if (!NULLMMA) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_f8f6f4(tmem + 128 * bb, pdesc + 2 * kk, vdesc + 2 * kk, IDPV, kk > 0);
                }
                mma_commit(bar_r_full(j));
                mma_commit(bar_kv_empty(s));
            }
        }
    } else {
        setmaxnreg_inc<224>();      // CTA register pool = 168 x 384: 56 + 2 x 224 <= 3 x 168
        // ===================== softmax / correction, one (row, half) per thread =====================
        const int h = wg - 1;                       // 0: key cols 0..63, O cols 0..DH-1 ; 1: the rest
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
        const uint32_t tX = tmem + lane_off + 64 * h;               // my S columns in X[0]
        const uint32_t tO = tmem + lane_off + 384 + DH * h;          // my O columns
        const uint32_t tR = tmem + lane_off + DH * h;                // my R columns in X[0]
        const int grow = i * 128 + row;
        const float dqr = p.dq[((size_t)bhq * nT + i) * 32 + 8 * (row / 32) + (row % 8)] * p.qk_scale_log2;
        float* xchg = reinterpret_cast<float*>(sgen + L::XCHG);
        float m = -INFINITY, l = 0.0f, alpha_prev = 0.0f;

        const int who = (TIMING && lane == 0 && wq == 0) ? h : -1;
        auto tss = [&](int j, int k) { if (who >= 0) ts(who, j, k); };
        // O = a * O + R(jr) on my DH columns
        auto correct = [&](int jr, float a, bool first) {
            mbar_wait(bar_r_full(jr), (jr >> 1) & 1);
            tc_fence_after();
            tss(jr + 1, 7);
            const float2 a2 = make_float2(a, a);
#pragma unroll
            for (int c0 = 0; c0 < DH; c0 += 64) {
                constexpr int NC = DH >= 64 ? 64 : DH;
                uint32_t r[64], o[64];
                tmem_ld32(tR + 128 * (jr % 3) + c0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
                if (NC == 64) tmem_ld32(tR + 128 * (jr % 3) + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
                if (!first) {
                    tmem_ld32(tO + c0, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
                    if (NC == 64) tmem_ld32(tO + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
                }
                tmem_wait_ld();
                reg_dep32(*reinterpret_cast<uint32_t(*)[32]>(&r[0]));
                if (NC == 64) reg_dep32(*reinterpret_cast<uint32_t(*)[32]>(&r[32]));
                if (!first) {
                    reg_dep32(*reinterpret_cast<uint32_t(*)[32]>(&o[0]));
                    if (NC == 64) reg_dep32(*reinterpret_cast<uint32_t(*)[32]>(&o[32]));
#pragma unroll
                    for (int c = 0; c < NC; c += 2) {
                        const float2 v = ffma2(a2, make_float2(__uint_as_float(o[c]), __uint_as_float(o[c + 1])),
                                               make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])));
                        o[c] = __float_as_uint(v.x);
                        o[c + 1] = __float_as_uint(v.y);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < NC; ++c) o[c] = r[c];
                }
                tmem_st32(tO + c0, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
                if (NC == 64) tmem_st32(tO + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(bar_x_free(jr % 3));
        };

        for (int j = 0; j < nkv; ++j) {
            const int s = j % kStages4, bb = j & 1, xb = j % 3;
            tss(j, 0);
            mbar_wait(bar_kv_full(s), (j / kStages4) & 1);          // Delta S / delta_K landed
            mbar_wait(bar_s_full(xb), (j / 3) & 1);
            tc_fence_after();
            tss(j, 1);
            if (NULLSM) {       // timing experiment only: the MMA/TMA pipeline without softmax work
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(bar_p_full(j));
                if (j >= 1) {
                    mbar_wait(bar_r_full(j - 1), ((j - 1) >> 1) & 1);
                    tc_fence_before();
                    mbar_arrive(bar_x_free((j - 1) % 3));
                }
                continue;
            }
            const uint32_t dss = stage_addr(s) + L::ST_DS + 256 * h;
            const float* dks = reinterpret_cast<const float*>(sgen + L::ST0 + s * L::STAGE + L::ST_DK) + 4 * h;
            float sc[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) sc[g] = dqr * dks[g];
            // ---- my 64 scores: dequant + Delta S ----
            float sv[64];
            {
                uint32_t r0[32], r1[32];
                tmem_ld32(tX + 128 * xb, r0);
                tmem_ld32(tX + 128 * xb + 32, r1);
                tmem_wait_ld();
                reg_dep32(r0);
                reg_dep32(r1);
                tss(j, 2);
                if (DUMP) {
                    int32_t* dst = p.s_dump + ((size_t)bhq * Np + grow) * (size_t)Np + j * 128 + 64 * h;
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        dst[c] = (int32_t)r0[c];
                        dst[32 + c] = (int32_t)r1[c];
                    }
                }
#pragma unroll
                for (int c = 0; c < 64; c += 4) {
                    const uint32_t* rr = c < 32 ? r0 : r1;
                    const float4 d4 = lds128(dss + 4 * c);
                    const float v0 = sc[(c % 8) / 2], v1 = sc[(c % 8) / 2 + 1];
                    const float2 a = ffma2(make_float2((float)(int32_t)rr[c % 32], (float)(int32_t)rr[c % 32 + 1]),
                                           make_float2(v0, v0), make_float2(d4.x, d4.y));
                    const float2 bq = ffma2(make_float2((float)(int32_t)rr[c % 32 + 2], (float)(int32_t)rr[c % 32 + 3]),
                                            make_float2(v1, v1), make_float2(d4.z, d4.w));
                    sv[c] = a.x;
                    sv[c + 1] = a.y;
                    sv[c + 2] = bq.x;
                    sv[c + 3] = bq.y;
                }
            }
            if ((CAUSAL && j == i) || (j * 128 + 128 > p.N)) {       // ragged end / causal diagonal (C-18)
#pragma unroll
                for (int c = 0; c < 64; ++c) {
                    const int key = j * 128 + 64 * h + c;
                    if (key >= p.N || (CAUSAL && key > grow)) sv[c] = -INFINITY;
                }
            }
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int c = 0; c < 64; c += 4) {
                mx0 = fmax3(mx0, sv[c], sv[c + 1]);
                mx1 = fmax3(mx1, sv[c + 2], sv[c + 3]);
            }
            // ---- exact row max across the two halves (64-thread named barrier) ----
            xchg[(bb * 2 + h) * 128 + row] = fmaxf(mx0, mx1);
            tss(j, 3);
            named_bar_sync(1 + wq, 64);
            tss(j, 4);
            const float m_new = fmax3(m, xchg[(bb * 2 + 0) * 128 + row], xchg[(bb * 2 + 1) * 128 + row]);
            const float alpha = (m == -INFINITY) ? 0.0f : ex2_approx(m - m_new);
            const float m_use = (m_new == -INFINITY) ? 0.0f : (m_new - kLog2_448);
            // ---- P^ = e4m3(448 P~) for my 64 keys, row sum ----
            uint8_t* sP = sgen + L::P + bb * 16384;
            const float2 negm = make_float2(-m_use, -m_use);
            float2 rs2 = make_float2(0.f, 0.f), rs2b = make_float2(0.f, 0.f);
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 16) {
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int c = c0 + 4 * q;
                    const float2 x01 = fadd2(make_float2(sv[c], sv[c + 1]), negm);
                    const float2 x23 = fadd2(make_float2(sv[c + 2], sv[c + 3]), negm);
                    const float2 p01 = make_float2(ex2_approx(x01.x), ex2_approx(x01.y));
                    const float2 p23 = make_float2(ex2_approx(x23.x), ex2_approx(x23.y));
                    rs2 = fadd2(rs2, p01);
                    rs2b = fadd2(rs2b, p23);
                    const uint32_t lo = __nv_cvt_float2_to_fp8x2(p01, __NV_SATFINITE, __NV_E4M3);
                    const uint32_t hi = __nv_cvt_float2_to_fp8x2(p23, __NV_SATFINITE, __NV_E4M3);
                    w[q] = lo | (hi << 16);
                }
                *reinterpret_cast<uint4*>(sP + swz_off<128>(row, 64 * h + c0)) = make_uint4(w[0], w[1], w[2], w[3]);
                if (DUMP && p.p_dump)
                    *reinterpret_cast<uint4*>(p.p_dump + ((size_t)bhq * Np + grow) * (size_t)Np + j * 128 + 64 * h + c0) =
                        make_uint4(w[0], w[1], w[2], w[3]);
            }
            tss(j, 5);
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(bar_p_full(j));
            tss(j, 6);
            // ---- two-level promotion of the previous KV tile (frees X[(j-1)%3]) ----
            if (j >= 1) correct(j - 1, alpha_prev, j == 1);
            tss(j, 8);
            l = alpha * l + ((rs2.x + rs2.y) + (rs2b.x + rs2b.y));
            m = m_new;
            alpha_prev = alpha;
        }
        if (NULLSM) {
            mbar_wait(bar_r_full(nkv - 1), ((nkv - 1) >> 1) & 1);
        } else {
            correct(nkv - 1, alpha_prev, nkv == 1);
        }
        // ---- epilogue: O / l / 448 * delta_V  (l = l_A + l_B carries the 448 factor) ----
        const int slot = nkv & 1;                 // an exchange slot no partner is still reading
        xchg[(slot * 2 + h) * 128 + row] = l;
        named_bar_sync(1 + wq, 64);
        const float lt = xchg[(slot * 2 + 0) * 128 + row] + xchg[(slot * 2 + 1) * 128 + row];
        const float inv_l = 1.0f / lt;
        tc_fence_after();
        const float* dvp = p.dv + (size_t)bhk * D + DH * h;
        __half* orow = p.out + (((size_t)b * p.Hq + hq) * p.N + grow) * D + DH * h;
#pragma unroll
        for (int c0 = 0; c0 < DH; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(tO + c0, o);
            tmem_wait_ld();
            reg_dep32(o);
            if (grow < p.N) {
#pragma unroll
                for (int c = 0; c < 32; c += 8) {
                    const float4 d0 = __ldg(reinterpret_cast<const float4*>(dvp + c0 + c));
                    const float4 d1 = __ldg(reinterpret_cast<const float4*>(dvp + c0 + c + 4));
                    __half2 h0 = __floats2half2_rn(__uint_as_float(o[c]) * inv_l * d0.x, __uint_as_float(o[c + 1]) * inv_l * d0.y);
                    __half2 h1 = __floats2half2_rn(__uint_as_float(o[c + 2]) * inv_l * d0.z, __uint_as_float(o[c + 3]) * inv_l * d0.w);
                    __half2 h2 = __floats2half2_rn(__uint_as_float(o[c + 4]) * inv_l * d1.x, __uint_as_float(o[c + 5]) * inv_l * d1.y);
                    __half2 h3 = __floats2half2_rn(__uint_as_float(o[c + 6]) * inv_l * d1.z, __uint_as_float(o[c + 7]) * inv_l * d1.w);
                    *reinterpret_cast<uint4*>(orow + c0 + c) =
                        make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                                   *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

}  // namespace sage2

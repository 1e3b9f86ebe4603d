// attn2.cuh -- SageAttention2 attention kernel v1 for sm_100a: two Q tiles per CTA in ping-pong
// (Alg. 1 inner loop; same arithmetic as attn.cuh v0, restructured for overlap).
//
// CTA = two 128-row Q blocks (i0 = 2*pair, i1 = i0 + 1) of one (b, h_q); KV tiles of 128 keys,
// ascending (reading C-9).  K^/V^ stages are shared by both Q tiles.
//
// 16 warps (512 threads), warp-specialised.  The single-thread roles sit in the HIGHEST warp ids:
// the issue arbiter favours high warp ids, so the producer / MMA threads are not starved by the
// softmax warps sharing their SM sub-partition (measured: 250-450 cycles of reaction latency
// when they were warps 0-2).
//   warp 12         producer: bulk-async copies (TMA engine) of pre-swizzled tile images
//   warp 13 / 14    MMA issuer for Q tile 0 / 1 (one elected thread each):
//                     S_k = Q^_k K^_j^T           tcgen05.mma.kind::i8      (exact s32, TMEM)
//                     R_k = P^_k V^_j             tcgen05.mma.kind::f8f6f4  (fresh fp32, TMEM,
//                                                  written over S_k once softmax consumed it)
//   warps 0-3       softmax for Q tile 0   } one thread per query row (TMEM lane = row):
//   warps 4-7       softmax for Q tile 1   } dequant + Delta S, exact running max, exp2,
//                                            P^ = e4m3(448 P~) -> smem, alpha -> smem
//   warps 8-11      correction for both tiles: O_k = alpha * O_k + R_k in fp32 (two-level
//                   accumulation; O_k lives in TMEM), then the epilogue
//                   O / l / 448 * delta_V -> fp16
// The two tiles' chains (QK -> softmax -> PV -> correction -> QK) interleave, so one tile's
// softmax overlaps the other tile's MMAs and correction.
// TMEM: S0/R0 [0,128), S1/R1 [128,256), O0 [256, 256+D), O1 [256+D, 256+2D).
#pragma once
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdint>

#include "attn.cuh"
#include "ptx.cuh"

namespace sage2 {

#ifndef SAGE2_KSTAGES
#define SAGE2_KSTAGES 3
#endif
constexpr int kStages2 = SAGE2_KSTAGES;   // K/V ring depth (A/B builds: -DSAGE2_KSTAGES=4)

template <int D>
struct Attn2Smem {
    static constexpr uint32_t TILE = 128 * D;
    static constexpr uint32_t Q0 = 0, Q1 = TILE;
    // stage: K^ | V^T | dS tile0 (512) | dS tile1 (512) | dK (32)
    static constexpr uint32_t ST_K = 0, ST_V = TILE, ST_DS0 = 2 * TILE, ST_DS1 = 2 * TILE + 512,
                              ST_DK = 2 * TILE + 1024;
    static constexpr uint32_t STAGE = ((2 * TILE + 1024 + 32) + 1023) / 1024 * 1024;
    static constexpr uint32_t ST0 = 2 * TILE;
    static constexpr uint32_t P0 = ST0 + kStages2 * STAGE;           // P^ tiles, 128 x 128 e4m3 each
    static constexpr uint32_t P1 = P0 + 16384;
    static constexpr uint32_t ALPHA = P1 + 16384;                     // float alpha[2][128]
    static constexpr uint32_t LSUM = ALPHA + 2 * 128 * 4;             // float l[2][128]
    static constexpr uint32_t BAR = LSUM + 2 * 128 * 4;
    // q_full, kv_full[S], kv_empty[S], s_full[2], p_full[2], r_full[2], s_free[2], l_ready[2]
    static constexpr uint32_t NBAR = 1 + 2 * kStages2 + 10;
    static constexpr uint32_t TMEMPTR = BAR + 8 * NBAR;
    static constexpr uint32_t BYTES = TMEMPTR + 16;
    static constexpr uint32_t ALLOC = BYTES + 1024;
};

template <int D, bool CAUSAL, bool DUMP, bool TIMING = false, bool NULLMMA = false, bool PINGPONG = true>
__global__ void __launch_bounds__(512, 1) k_attn2(const AttnParams p) {
    using L = Attn2Smem<D>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int wg = warp / 4;
    const int nT = p.nT, Np = nT * 128;
    const int npairs = (nT + 1) / 2;
    const int pair = CAUSAL ? (npairs - 1 - (int)blockIdx.x) : (int)blockIdx.x;   // heavy causal pairs first
    const int hq = blockIdx.y, b = blockIdx.z;
    const int bhq = b * p.Hq + hq;
    const int bhk = b * p.Hkv + hq / (p.Hq / p.Hkv);
    // per-tile scalars (no arrays: indexing them by a runtime tile id would go to local memory)
    const int it0 = 2 * pair, it1 = 2 * pair + 1;
    const int nkv0 = CAUSAL ? it0 + 1 : nT;
    const int nkv1 = (it1 < nT) ? (CAUSAL ? it1 + 1 : nT) : 0;
    const int nkv_max = nkv0 > nkv1 ? nkv0 : nkv1;
    const int ntiles = nkv1 > 0 ? 2 : 1;

    // TIMING builds: clock64 stamps of one thread per role in CTA (0,0,0) -> (uint64*)p.s_dump
    const bool tsel = TIMING && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
    auto ts = [&](int who, int j, int k) {
        if (TIMING && tsel && j < 64)
            reinterpret_cast<unsigned long long*>(p.s_dump)[(who * 64 + j) * 16 + k] = clock64();
    };
    const uint32_t bar0 = sbase + L::BAR;
    const uint32_t bar_q = bar0;
    auto bar_kv_full = [&](int s) { return bar0 + 8 * (1 + s); };
    auto bar_kv_empty = [&](int s) { return bar0 + 8 * (1 + kStages2 + s); };
    auto bar_s_full = [&](int k) { return bar0 + 8 * (1 + 2 * kStages2 + k); };
    auto bar_p_full = [&](int k) { return bar0 + 8 * (3 + 2 * kStages2 + k); };
    auto bar_r_full = [&](int k) { return bar0 + 8 * (5 + 2 * kStages2 + k); };
    auto bar_s_free = [&](int k) { return bar0 + 8 * (7 + 2 * kStages2 + k); };
    auto bar_l_ready = [&](int k) { return bar0 + 8 * (9 + 2 * kStages2 + k); };
    auto stage_addr = [&](int s) { return sbase + L::ST0 + s * L::STAGE; };

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(bar_kv_full(s), 1);
            mbar_init(bar_kv_empty(s), 2);      // one arrival per Q tile (MMA commit or bypass)
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(bar_s_full(k), 1);
            mbar_init(bar_p_full(k), 128);
            mbar_init(bar_r_full(k), 1);
            mbar_init(bar_s_free(k), 128);
            mbar_init(bar_l_ready(k), 128);
        }
        fence_mbar_init();
    }
    if (warp == 12) tmem_alloc<512>(sbase + L::TMEMPTR);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sgen + L::TMEMPTR);
    float* s_alpha = reinterpret_cast<float*>(sgen + L::ALPHA);
    float* s_lsum = reinterpret_cast<float*>(sgen + L::LSUM);

    if (wg == 3) {
        setmaxnreg_dec<56>();
        if (warp == 12 && lane == 0) {
            // ===================== producer =====================
            const size_t tile_bytes = (size_t)128 * D;
            mbar_arrive_expect_tx(bar_q, L::TILE * ntiles);
            bulk_g2s(sbase + L::Q0, p.qhat + ((size_t)bhq * nT + it0) * tile_bytes, L::TILE, bar_q);
            if (ntiles == 2)
                bulk_g2s(sbase + L::Q1, p.qhat + ((size_t)bhq * nT + it1) * tile_bytes, L::TILE, bar_q);
            const uint64_t keep = policy_evict_last();
            for (int j = 0; j < nkv_max; ++j) {
                const int s = j % kStages2;
                if (j >= kStages2) mbar_wait(bar_kv_empty(s), ((j / kStages2) - 1) & 1);
                const uint32_t sa = stage_addr(s);
                const bool d0 = j < nkv0, d1 = j < nkv1;
                mbar_arrive_expect_tx(bar_kv_full(s), 2 * L::TILE + 32 + 512 * (d0 + d1));
                bulk_g2s_hint(sa + L::ST_K, p.khat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, bar_kv_full(s), keep);
                bulk_g2s_hint(sa + L::ST_V, p.vhat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, bar_kv_full(s), keep);
                bulk_g2s(sa + L::ST_DK, p.dk + (size_t)bhk * nT * 8 + (size_t)j * 8, 32, bar_kv_full(s));
                if (d0)
                    bulk_g2s(sa + L::ST_DS0, p.ds + ds_row(p.ds_tri, bhq, it0, nT) + (size_t)j * 128, 512, bar_kv_full(s));
                if (d1)
                    bulk_g2s(sa + L::ST_DS1, p.ds + ds_row(p.ds_tri, bhq, it1, nT) + (size_t)j * 128, 512, bar_kv_full(s));
            }
        } else if ((warp == 13 || warp == 14) && lane == 0) {
            // ===================== MMA issuer for Q tile k =====================
            const int k = warp - 13;
            const int my_nkv = k ? nkv1 : nkv0;
            constexpr uint32_t IDQK = idesc_i8(128, 128);
            constexpr uint32_t IDPV = idesc_e4m3(128, D);
            const uint64_t qdesc = smem_desc<D>(sbase + (k ? L::Q1 : L::Q0));
            const uint64_t pdesc = smem_desc<128>(sbase + (k ? L::P1 : L::P0));
            const uint32_t tS = tmem + 128 * k;
            mbar_wait(bar_q, 0);
            for (int j = 0; j < nkv_max; ++j) {
                const int s = j % kStages2;
                mbar_wait(bar_kv_full(s), (j / kStages2) & 1);
                if (j >= my_nkv) {                 // this tile is done: release the stage for it
                    mbar_arrive(bar_kv_empty(s));
                    continue;
                }
                if (j >= 1) mbar_wait(bar_s_free(k), (j - 1) & 1);   // R_k(j-1) consumed
                tc_fence_after();
                const uint64_t kdesc = smem_desc<D>(stage_addr(s) + L::ST_K);
                if (!NULLMMA) {
#pragma unroll
                    for (int kk = 0; kk < D / 32; ++kk) mma_i8(tS, qdesc + 2 * kk, kdesc + 2 * kk, IDQK, kk > 0);
                }
                mma_commit(bar_s_full(k));
                ts(4 + k, j, 0);
                mbar_wait(bar_p_full(k), j & 1);                    // softmax_k(j) wrote P^_k
                ts(4 + k, j, 1);
                tc_fence_after();
                const uint64_t vdesc = smem_desc<128>(stage_addr(s) + L::ST_V);
                if (!NULLMMA) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) mma_f8f6f4(tS, pdesc + 2 * kk, vdesc + 2 * kk, IDPV, kk > 0);
                }
                mma_commit(bar_r_full(k));
                mma_commit(bar_kv_empty(s));
            }
        }
    } else if (wg == 0 || wg == 1) {
        setmaxnreg_inc<184>();
        // ===================== softmax for Q tile k =====================
        const int k = wg;
        const int my_nkv = k ? nkv1 : nkv0, my_it = k ? it1 : it0;
        // MUFU ping-pong: the exp2 phases of the two tiles alternate (named barriers 8 + k), so
        // one tile's ALU-bound dequant/max runs while the other saturates the MUFU pipe.
        auto turn_wait = [&]() { if (PINGPONG) named_bar_sync(8 + k, 256); };
        auto turn_pass = [&]() { if (PINGPONG) named_bar_arrive(8 + (1 - k), 256); };
        if (k == 1) turn_pass();                    // tile 0 takes the first turn
        if (my_nkv > 0) {
            const int wq = warp & 3;
            const int row = 32 * wq + lane;
            const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
            const uint32_t tS = tmem + 128 * k + lane_off;
            const int grow = my_it * 128 + row;
            const float dqr = p.dq[((size_t)bhq * nT + my_it) * 32 + 8 * (row / 32) + (row % 8)] * p.qk_scale_log2;
            uint8_t* sP = sgen + (k ? L::P1 : L::P0);
            float m = -INFINITY, l = 0.0f;
            const int who = (TIMING && lane == 0 && (warp & 3) == 0) ? k : -1;
            auto tss = [&](int j, int kk) { if (who >= 0) ts(who, j, kk); };
            for (int j = 0; j < my_nkv; ++j) {
                tss(j, 0);
                const int s = j % kStages2;
                mbar_wait(bar_kv_full(s), (j / kStages2) & 1);      // Delta S / delta_K landed
                mbar_wait(bar_s_full(k), j & 1);
                tc_fence_after();
                tss(j, 1);
                const uint8_t* st = sgen + L::ST0 + s * L::STAGE;
                const float4* dss = reinterpret_cast<const float4*>(st + (k ? L::ST_DS1 : L::ST_DS0));
                const float* dks = reinterpret_cast<const float*>(st + L::ST_DK);
                float2 sc2[8];
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const float v = dqr * dks[g];
                    sc2[g] = make_float2(v, v);
                }
                float sv[128];
                {
                    uint32_t r0[32], r1[32], r2[32], r3[32];
                    tmem_ld32(tS + 0, r0);
                    tmem_ld32(tS + 32, r1);
                    tmem_ld32(tS + 64, r2);
                    tmem_ld32(tS + 96, r3);
                    tmem_wait_ld();
                    reg_dep32(r0);
                    reg_dep32(r1);
                    reg_dep32(r2);
                    reg_dep32(r3);
                    tss(j, 2);
                    if (DUMP) {
                        int32_t* dst = p.s_dump + ((size_t)bhq * Np + grow) * (size_t)Np + j * 128;
#pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            dst[c] = (int32_t)r0[c];
                            dst[32 + c] = (int32_t)r1[c];
                            dst[64 + c] = (int32_t)r2[c];
                            dst[96 + c] = (int32_t)r3[c];
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 128; c += 4) {
                        const uint32_t* rr = c < 32 ? r0 : c < 64 ? r1 : c < 96 ? r2 : r3;
                        const float4 d4 = dss[c / 4];
                        const int g = (c / 64) * 4 + (c % 8) / 2;
                        const float2 a = ffma2(make_float2((float)(int32_t)rr[c % 32], (float)(int32_t)rr[c % 32 + 1]),
                                               sc2[g], make_float2(d4.x, d4.y));
                        const float2 bq = ffma2(make_float2((float)(int32_t)rr[c % 32 + 2], (float)(int32_t)rr[c % 32 + 3]),
                                                sc2[g + 1], make_float2(d4.z, d4.w));
                        sv[c] = a.x;
                        sv[c + 1] = a.y;
                        sv[c + 2] = bq.x;
                        sv[c + 3] = bq.y;
                    }
                }
                // masks: ragged end (keys >= N) and causal diagonal (key > query), C-18
                if ((CAUSAL && j == my_it) || (j * 128 + 128 > p.N)) {
#pragma unroll
                    for (int c = 0; c < 128; ++c) {
                        const int key = j * 128 + c;
                        if (key >= p.N || (CAUSAL && key > grow)) sv[c] = -INFINITY;
                    }
                }
                float mx[4] = {m, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c = 0; c < 128; c += 8) {
                    mx[0] = fmax3(mx[0], sv[c], sv[c + 1]);
                    mx[1] = fmax3(mx[1], sv[c + 2], sv[c + 3]);
                    mx[2] = fmax3(mx[2], sv[c + 4], sv[c + 5]);
                    mx[3] = fmax3(mx[3], sv[c + 6], sv[c + 7]);
                }
                const float m_new = fmax3(mx[0], mx[1], fmaxf(mx[2], mx[3]));
                tss(j, 3);
                const float alpha = (m == -INFINITY) ? 0.0f : ex2_approx(m - m_new);
                turn_wait();
                const float m_use = (m_new == -INFINITY) ? 0.0f : (m_new - kLog2_448);
                const float2 negm = make_float2(-m_use, -m_use);
                float2 rs2 = make_float2(0.f, 0.f), rs2b = make_float2(0.f, 0.f);
#pragma unroll
                for (int c0 = 0; c0 < 128; c0 += 16) {
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
                    *reinterpret_cast<uint4*>(sP + swz_off<128>(row, c0)) = make_uint4(w[0], w[1], w[2], w[3]);
                    if (DUMP && p.p_dump)
                        *reinterpret_cast<uint4*>(p.p_dump + ((size_t)bhq * Np + grow) * (size_t)Np + j * 128 + c0) =
                            make_uint4(w[0], w[1], w[2], w[3]);
                }
                s_alpha[k * 128 + row] = alpha;
                fence_proxy_async_smem();
                tc_fence_before();
                tss(j, 4);
                mbar_arrive(bar_p_full(k));
                turn_pass();
                const float rowsum = (rs2.x + rs2.y) + (rs2b.x + rs2b.y);
                l = alpha * l + rowsum;
                m = m_new;
            }
            s_lsum[k * 128 + row] = l;
            mbar_arrive(bar_l_ready(k));
        }
        for (int j = my_nkv; j < nkv_max; ++j) {    // keep the turn protocol balanced
            turn_wait();
            turn_pass();
        }
    } else {
        setmaxnreg_dec<88>();
        // ===================== correction + epilogue (both tiles) =====================
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
        const float* dvp = p.dv + (size_t)bhk * D;
        for (int j = 0; j < nkv_max; ++j) {
#pragma unroll 1
            for (int k = 0; k < 2; ++k) {
                if (j >= (k ? nkv1 : nkv0)) continue;
                if (TIMING && lane == 0 && (warp & 3) == 0) ts(2 + k, j, 0);
                mbar_wait(bar_p_full(k), j & 1);
                if (TIMING && lane == 0 && (warp & 3) == 0) ts(2 + k, j, 1);
                mbar_wait(bar_r_full(k), j & 1);
                if (TIMING && lane == 0 && (warp & 3) == 0) ts(2 + k, j, 2);
                tc_fence_after();
                if (NULLMMA) {
                    tc_fence_before();
                    mbar_arrive(bar_s_free(k));
                    continue;
                }
                const float alpha = s_alpha[k * 128 + row];
                const uint32_t tR = tmem + 128 * k + lane_off;
                const uint32_t tO = tmem + 256 + D * k + lane_off;
#pragma unroll
                for (int ch = 0; ch < D / 32; ++ch) {
                    uint32_t r[32];
                    tmem_ld32(tR + ch * 32, r);
                    if (j > 0) {
                        uint32_t o[32];
                        tmem_ld32(tO + ch * 32, o);
                        tmem_wait_ld();
                        reg_dep32(r);
                        reg_dep32(o);
                        const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
                        for (int c = 0; c < 32; c += 2) {
                            const float2 v = ffma2(a2, make_float2(__uint_as_float(o[c]), __uint_as_float(o[c + 1])),
                                                   make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])));
                            o[c] = __float_as_uint(v.x);
                            o[c + 1] = __float_as_uint(v.y);
                        }
                        tmem_st32(tO + ch * 32, o);
                    } else {
                        tmem_wait_ld();
                        reg_dep32(r);
                        tmem_st32(tO + ch * 32, r);
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(bar_s_free(k));
                if (TIMING && lane == 0 && (warp & 3) == 0) ts(2 + k, j, 3);
            }
        }
        // epilogue: O / l / 448 * delta_V  (l carries the 448 factor)
#pragma unroll 1
        for (int k = 0; k < 2; ++k) {
            if ((k ? nkv1 : nkv0) == 0) continue;
            mbar_wait(bar_l_ready(k), 0);
            tc_fence_after();
            const float inv_l = 1.0f / s_lsum[k * 128 + row];
            const int grow = (k ? it1 : it0) * 128 + row;
            const uint32_t tO = tmem + 256 + D * k + lane_off;
            __half* orow = p.out + (((size_t)b * p.Hq + hq) * p.N + grow) * D;
#pragma unroll
            for (int ch = 0; ch < D / 32; ++ch) {
                uint32_t o[32];
                tmem_ld32(tO + ch * 32, o);
                tmem_wait_ld();
                reg_dep32(o);
                if (grow < p.N) {
                    uint32_t h[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const int cc = ch * 32 + 2 * c;
                        const float a = __uint_as_float(o[2 * c]) * inv_l * __ldg(dvp + cc);
                        const float bb = __uint_as_float(o[2 * c + 1]) * inv_l * __ldg(dvp + cc + 1);
                        __half2 hv = __floats2half2_rn(a, bb);
                        h[c] = *reinterpret_cast<uint32_t*>(&hv);
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        reinterpret_cast<uint4*>(orow + ch * 32)[c] =
                            make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 12) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

}  // namespace sage2

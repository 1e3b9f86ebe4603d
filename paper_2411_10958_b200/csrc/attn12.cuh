// attn12.cuh -- SageAttention2 attention kernel v12 for sm_100a, head dim 64 (Alg. 1 inner loop,
// PAPER.md:246-263) with b_kv = 64 -- the paper's own KV block ("b_k = 64") -- and FOUR
// 128-row Q tiles per CTA.
//
// Why: at d = 64 a 128 x 128 score tile carries half the tensor work of d = 128 but the same exp
// count, so the MUFU is the roof and everything else must hide under it.  v8 keeps two Q tiles in
// flight: each tile's per-KV-step chain (PV -> R read -> QK -> S load -> dequant -> max) has to fit
// under ONE other tile's exp phase, and does not (v8 d=64: ~56% of the MUFU roof).  With b_kv = 64 a
// tile needs only 64 + 64 TMEM columns (S/R and O), so four tiles fit in TMEM and each tile's chain
// has three other tiles' exp phases to hide under; the MMAs of a step are half as long.
//
// CTA = Q blocks 4g .. 4g + 3 of one (b, h_q); the K^ / V^T / Delta S stages (one 128-key block each,
// serving two 64-key steps) are shared by the four tiles.  20 warps (640 threads):
//   warps 0-15   softmax of tile k = warp / 4, TMEM lane quarter warp % 4: one thread per query row
//                (32x32b loads), all 64 keys of a step in that thread, so the exact running max
//                (C-10) needs no exchange at all;
//   warp 16      producer (bulk-async copies of the pre-swizzled tile images);
//   warp 17      QK issuer for all tiles (whole warp, elect.sync): S = Q^ K^^T (kind::i8, M128 N64 K64)
//                as soon as the tile's previous R is out of TMEM;
//   warp 18      PV issuer for all tiles in the MUFU turn order: R = P^ V^ (kind::f8f6f4, M128 N64
//                K64) into a fresh accumulator.
// The tiles' exp phases overlap freely (SAGE2_V12_TURN below).  P^ is handed to the PV MMA in two
// halves (K steps of 32 keys).  Arithmetic per (row, key) is v8's: s = S_int dQ dK log2e/sqrt(d) +
// Delta S', masks (C-18), P^ = e4m3(2^(s - m + log2 448)), l from P~ (C-13),
// O = alpha O + R in fp32 in TMEM, O / l / 448 * delta_V (+ V_m) -> fp16.
// TMEM: S_k/R_k [64k, 64k + 64) (R written over S once S is in registers), O_k [256 + 64k, +64).
#pragma once
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdint>

#include "common.cuh"
#include "ptx.cuh"

namespace sage2 {

// MUFU scheduling between the four tiles.  Measured (C2-32K d=64, kernel only): free (0) 686 TOPS,
// round-robin turns (1) 616, turns + per-tile lockstep (2) 625, two tokens (3) 674, v8 665.  With one
// warp per SM sub-partition per tile a single exp phase cannot keep the MUFU busy (its MUFU ops issue
// in clusters: ~1000 cycles for 512 cycles of ex2), so the tiles are left to overlap freely.
#ifndef SAGE2_V12_TURN
#define SAGE2_V12_TURN 0
#endif

struct Attn12Smem {
    static constexpr uint32_t TILE = 128 * 64;                        // a 128 x 64 int8 / e4m3 tile image
    static constexpr uint32_t Q0 = 0;                                 // Q^ tiles 0-3
    // stage (one 128-key block): K^ | V^T | Delta S rows of the 4 tiles (512 B each) | delta_K (32 B)
    static constexpr uint32_t ST_K = 0, ST_V = TILE, ST_DS = 2 * TILE, ST_DK = 2 * TILE + 4 * 512;
    static constexpr uint32_t STAGE = ((2 * TILE + 4 * 512 + 32) + 1023) / 1024 * 1024;
    static constexpr uint32_t ST0 = 4 * TILE;
    static constexpr uint32_t P0 = ST0 + kStages2 * STAGE;           // P^ tiles, 128 x 64 e4m3 each (SW64)
    static constexpr uint32_t BAR = P0 + 4 * 8192;
    // q_full, kv_full[S], kv_empty[S], s_full[4], pa_full[4], pb_full[4], r_full[4], s_free[4]
    static constexpr uint32_t NBAR = 1 + 2 * kStages2 + 20;
    static constexpr uint32_t TMEMPTR = BAR + 8 * NBAR;
    static constexpr uint32_t BYTES = TMEMPTR + 16;
    static constexpr uint32_t ALLOC = BYTES + 1024;
};

template <bool CAUSAL, bool DUMP, bool TIMING = false>
__global__ void __launch_bounds__(640, 1) k_attn12(const AttnParams p) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    constexpr int D = 64;
    using L = Attn12Smem;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));

    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
    const int nT = p.nT, Np = nT * 128;
    const int nquads = (nT + 3) / 4;
    const int quad = CAUSAL ? (nquads - 1 - (int)blockIdx.x) : (int)blockIdx.x;   // heavy causal CTAs first
    const int hq = blockIdx.y, b = blockIdx.z;
    const int bhq = b * p.Hq + hq;
    const int bhk = b * p.Hkv + hq / (p.Hq / p.Hkv);
    const int it_base = 4 * quad;
    const int ntiles = min(4, nT - it_base);
    // 64-key steps of tile k: keys < min(N, 128 (it + 1)) when causal, < N otherwise
    auto nsteps = [&](int k) {
        if (k >= ntiles) return 0;
        const int kend = CAUSAL ? min(p.N, 128 * (it_base + k + 1)) : p.N;
        return (kend + 63) / 64;
    };
    const int nst_max = nsteps(ntiles - 1) > nsteps(0) ? nsteps(ntiles - 1) : nsteps(0);
    const int nblk = (nst_max + 1) / 2;                               // 128-key stages to load

    auto s_as_int = [](uint32_t u) { return (int32_t)u; };
    const bool tsel = TIMING && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
    auto ts = [&](int who, int j, int slot) {
        if (TIMING && tsel && j < 64)
            reinterpret_cast<unsigned long long*>(p.s_dump)[(who * 64 + j) * 16 + slot] = clock64();
    };
    const uint32_t bar0 = sbase + L::BAR;
    const uint32_t bar_q = bar0;
    auto bar_kv_full = [&](int s) { return bar0 + 8 * (1 + s); };
    auto bar_kv_empty = [&](int s) { return bar0 + 8 * (1 + kStages2 + s); };
    auto bar_s_full = [&](int k) { return bar0 + 8 * (1 + 2 * kStages2 + k); };
    auto bar_pa_full = [&](int k) { return bar0 + 8 * (5 + 2 * kStages2 + k); };
    auto bar_pb_full = [&](int k) { return bar0 + 8 * (9 + 2 * kStages2 + k); };
    auto bar_r_full = [&](int k) { return bar0 + 8 * (13 + 2 * kStages2 + k); };
    auto bar_s_free = [&](int k) { return bar0 + 8 * (17 + 2 * kStages2 + k); };
    auto stage_addr = [&](int s) { return sbase + L::ST0 + s * L::STAGE; };

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(bar_kv_full(s), 1);
            mbar_init(bar_kv_empty(s), 4);      // one arrival per Q tile (MMA commit or bypass)
        }
        for (int k = 0; k < 4; ++k) {
            mbar_init(bar_s_full(k), 1);
            mbar_init(bar_pa_full(k), 128);
            mbar_init(bar_pb_full(k), 128);
            mbar_init(bar_r_full(k), 1);
            mbar_init(bar_s_free(k), 128);
        }
        fence_mbar_init();
    }
    constexpr int PW = 16;                        // producer warp; QK issuer PW + 1, PV issuer PW + 2
    if (warp == PW) tmem_alloc<512>(sbase + L::TMEMPTR);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sgen + L::TMEMPTR);

    if (warp >= PW) {
        setmaxnreg_dec<32>();
        if (warp == PW && lane == 0) {
            // ===================== producer =====================
            const size_t tile_bytes = (size_t)128 * D;
            mbar_arrive_expect_tx(bar_q, L::TILE * ntiles);
            for (int k = 0; k < ntiles; ++k)
                bulk_g2s(sbase + L::Q0 + k * L::TILE, p.qhat + ((size_t)bhq * nT + it_base + k) * tile_bytes, L::TILE, bar_q);
            const uint64_t keep = policy_evict_last();
            for (int jb = 0; jb < nblk; ++jb) {
                const int s = jb % kStages2;
                if (jb >= kStages2) mbar_wait(bar_kv_empty(s), ((jb / kStages2) - 1) & 1);
                const uint32_t sa = stage_addr(s);
                int nds = 0;
                for (int k = 0; k < ntiles; ++k) nds += (2 * jb < nsteps(k));
                mbar_arrive_expect_tx(bar_kv_full(s), 2 * L::TILE + 32 + 512 * nds);
                bulk_g2s_hint(sa + L::ST_K, p.khat + ((size_t)bhk * nT + jb) * tile_bytes, L::TILE, bar_kv_full(s), keep);
                bulk_g2s_hint(sa + L::ST_V, p.vhat + ((size_t)bhk * nT + jb) * tile_bytes, L::TILE, bar_kv_full(s), keep);
                bulk_g2s(sa + L::ST_DK, p.dk + ((size_t)bhk * nT + jb) * 8, 32, bar_kv_full(s));
                for (int k = 0; k < ntiles; ++k)
                    if (2 * jb < nsteps(k))
                        bulk_g2s(sa + L::ST_DS + 512 * k, p.ds + ds_row(p.ds_tri, bhq, it_base + k, nT) + (size_t)jb * 128,
                                 512, bar_kv_full(s));
            }
        } else if (warp == PW + 1) {
            // ============ QK issuer (all four tiles; whole warp converged, one elected lane issues) ============
            constexpr uint32_t IDQK = idesc_i8(128, 64);
            if (ntiles > 0) mbar_wait(bar_q, 0);
            for (int j = 0; j < nst_max; ++j) {
                const int jb = j >> 1, h = j & 1, s = jb % kStages2;
                if (h == 0) mbar_wait(bar_kv_full(s), (jb / kStages2) & 1);
                // keys 64h .. 64h + 63 of the block: K^ rows 64h.. (64-byte rows, 4 KB per 64 rows)
                const uint64_t kdesc = smem_desc<64>(stage_addr(s) + L::ST_K + 4096 * h);
#pragma unroll 1
                for (int k = 0; k < 4; ++k) {
                    if (j >= nsteps(k)) continue;
                    if (j >= 1) mbar_wait(bar_s_free(k), (j - 1) & 1);   // R_k(j-1) read out of TMEM
                    if (lane == 0) ts(4 + k, j, 1);
                    tc_fence_after();
                    const uint64_t qdesc = smem_desc<64>(sbase + L::Q0 + k * L::TILE);
                    mma_i8_w(tmem + 64 * k, qdesc + 0, kdesc + 0, IDQK, 0);
                    mma_i8_w(tmem + 64 * k, qdesc + 2, kdesc + 2, IDQK, 1);
                    mma_commit_w(bar_s_full(k));
                    if (lane == 0) ts(4 + k, j, 2);
                }
            }
        } else if (warp == PW + 2) {
            // ============ PV issuer (all four tiles, in the MUFU turn order) ============
            constexpr uint32_t IDPV = idesc_e4m3(128, D);
            for (int j = 0; j < nst_max; ++j) {
                const int jb = j >> 1, h = j & 1, s = jb % kStages2;
                if (h == 0) mbar_wait(bar_kv_full(s), (jb / kStages2) & 1);
                // V^T columns (tokens) 64h .. 64h + 63 of the block, two K steps of 32
                const uint64_t vdesc = smem_desc<128>(stage_addr(s) + L::ST_V) + 4 * h;
#pragma unroll 1
                for (int k = 0; k < 4; ++k) {
                    const int ns = nsteps(k);
                    if (j < ns) {
                        const uint64_t pdesc = smem_desc<64>(sbase + L::P0 + k * 8192);
                        mbar_wait(bar_pa_full(k), j & 1);
                        if (lane == 0) ts(4 + k, j, 3);
                        tc_fence_after();
                        mma_f8f6f4_w(tmem + 64 * k, pdesc + 0, vdesc + 0, IDPV, 0);
                        mbar_wait(bar_pb_full(k), j & 1);
                        tc_fence_after();
                        mma_f8f6f4_w(tmem + 64 * k, pdesc + 2, vdesc + 2, IDPV, 1);
                        mma_commit_w(bar_r_full(k));
                        if (lane == 0) ts(4 + k, j, 4);
                        // this tile's last MMA on the stage (its QK finished before its softmax began)
                        if (h == 1 || j == ns - 1) mma_commit_w(bar_kv_empty(s));
                    } else if (h == 0 && lane == 0) {
                        mbar_arrive(bar_kv_empty(s));        // the tile does not use this stage
                    }
                }
            }
        }
    } else {
        setmaxnreg_inc<112>();      // pool = 96 x 640 (launch): 4 x 32 + 16 x 112 <= 20 x 96
        // ============ softmax (one thread per query row) + two-level promotion + epilogue ============
        const int k = warp >> 2, wq = warp & 3;
        const int my_ns = nsteps(k);
        auto turn_wait = [&]() {
            if (SAGE2_V12_TURN == 2) named_bar_sync(5 + k, 128);     // the tile's four warps in lockstep
            if (SAGE2_V12_TURN) named_bar_sync(1 + k, 256);
        };
        // TURN 3: two tokens -- tile k follows tile k - 2, so two tiles (one pair of warps per SMSP)
        // exponentiate at a time
        auto turn_pass = [&]() {
            if (SAGE2_V12_TURN == 3) named_bar_arrive(1 + ((k + 2) & 3), 256);
            else if (SAGE2_V12_TURN) named_bar_arrive(1 + ((k + 1) & 3), 256);
        };
        if (SAGE2_V12_TURN == 3 ? k >= 2 : k == 3) turn_pass();   // tile 0 (and 1) take the first turns
        if (my_ns > 0) {
            const int my_it = it_base + k;
            const int row = 32 * wq + lane;
            const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
            const uint32_t tS = tmem + 64 * k + lane_off;            // S_k / R_k
            const uint32_t tO = tmem + 256 + 64 * k + lane_off;      // O_k
            const int grow = my_it * 128 + row;
            const float dqr = p.dq[((size_t)bhq * nT + my_it) * 32 + 8 * wq + (lane & 7)] * p.qk_scale_log2;
            uint8_t* sP = sgen + L::P0 + k * 8192;
            float m = -INFINITY, l = 0.0f;
            const bool tme = TIMING && wq == 0 && lane == 0;
            auto tss = [&](int j, int slot) {
                if (tme) ts(k, j, slot);
                if (TIMING && lane == 0 && (slot == 4 || slot == 5)) ts(16 + warp, j, slot);   // every warp
            };
            for (int j = 0; j < my_ns; ++j) {
                const int jb = j >> 1, h = j & 1, s = jb % kStages2;
                tss(j, 0);
                mbar_wait(bar_kv_full(s), (jb / kStages2) & 1);     // Delta S / delta_K landed
                mbar_wait(bar_s_full(k), j & 1);
                tc_fence_after();
                tss(j, 1);
                const uint32_t dss = stage_addr(s) + L::ST_DS + 512 * k + 256 * h;
                // delta_K of keys 64h + c: group 4h + (c % 8) / 2 of the block (g_K)
                const float4 dk4 = lds128(stage_addr(s) + L::ST_DK + 16 * h);
                const float2 sc01 = make_float2(dqr * dk4.x, dqr * dk4.x), sc23 = make_float2(dqr * dk4.y, dqr * dk4.y);
                const float2 sc45 = make_float2(dqr * dk4.z, dqr * dk4.z), sc67 = make_float2(dqr * dk4.w, dqr * dk4.w);
                float sv[64];
                {
                    uint32_t r0[32], r1[32];
                    tmem_ld32(tS + 0, r0);
                    tmem_ld32(tS + 32, r1);
                    tmem_wait_ld();
                    reg_dep32(r0);
                    reg_dep32(r1);
                    tss(j, 9);
                    if (DUMP) {
                        int32_t* dst = p.s_dump + ((size_t)bhq * Np + grow) * (size_t)Np + j * 64;
#pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            dst[c] = s_as_int(r0[c]);
                            dst[32 + c] = s_as_int(r1[c]);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 64; c += 8) {
                        const uint32_t* rr = c < 32 ? r0 : r1;
#ifdef SAGE2_ABL_NODS
                        const float4 d0 = make_float4(0.f, 0.f, 0.f, 0.f), d1 = d0;   // ablation build only
#else
                        const float4 d0 = lds128(dss + 4 * c), d1 = lds128(dss + 4 * c + 16);
#endif
                        const float2 a = ffma2(make_float2((float)(int32_t)rr[c % 32], (float)(int32_t)rr[c % 32 + 1]), sc01,
                                               make_float2(d0.x, d0.y));
                        const float2 bq = ffma2(make_float2((float)(int32_t)rr[c % 32 + 2], (float)(int32_t)rr[c % 32 + 3]), sc23,
                                                make_float2(d0.z, d0.w));
                        const float2 cq = ffma2(make_float2((float)(int32_t)rr[c % 32 + 4], (float)(int32_t)rr[c % 32 + 5]), sc45,
                                                make_float2(d1.x, d1.y));
                        const float2 dq = ffma2(make_float2((float)(int32_t)rr[c % 32 + 6], (float)(int32_t)rr[c % 32 + 7]), sc67,
                                                make_float2(d1.z, d1.w));
                        sv[c] = a.x;
                        sv[c + 1] = a.y;
                        sv[c + 2] = bq.x;
                        sv[c + 3] = bq.y;
                        sv[c + 4] = cq.x;
                        sv[c + 5] = cq.y;
                        sv[c + 6] = dq.x;
                        sv[c + 7] = dq.y;
                    }
                }
                tss(j, 2);
                if ((CAUSAL && 64 * j + 63 > 128 * my_it) || (64 * j + 64 > p.N)) {   // C-18
#pragma unroll
                    for (int c = 0; c < 64; ++c) {
                        const int key = 64 * j + c;
                        if (key >= p.N || (CAUSAL && key > grow)) sv[c] = -INFINITY;
                    }
                }
                float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c = 0; c < 64; c += 8) {
                    mx[0] = fmax3(mx[0], sv[c], sv[c + 1]);
                    mx[1] = fmax3(mx[1], sv[c + 2], sv[c + 3]);
                    mx[2] = fmax3(mx[2], sv[c + 4], sv[c + 5]);
                    mx[3] = fmax3(mx[3], sv[c + 6], sv[c + 7]);
                }
                // the whole row is in this thread: the exact running max (C-10) is local
                const float m_new = fmax3(m, fmax3(mx[0], mx[1], mx[2]), mx[3]);
                const float alpha = (m == -INFINITY) ? 0.0f : ex2_approx(m - m_new);
                const float m_use = (m_new == -INFINITY) ? 0.0f : (m_new - kLog2_448);
                tss(j, 3);
                turn_wait();
                tss(j, 4);
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
                    *reinterpret_cast<uint4*>(sP + swz_off<64>(row, c0)) = make_uint4(w[0], w[1], w[2], w[3]);
                    if (DUMP && p.p_dump)
                        *reinterpret_cast<uint4*>(p.p_dump + ((size_t)bhq * Np + grow) * (size_t)Np + j * 64 + c0) =
                            make_uint4(w[0], w[1], w[2], w[3]);
                    if (c0 == 16 || c0 == 48) {              // a 32-key half of the row's codes is in smem
                        fence_proxy_async_smem();
                        tc_fence_before();
                        mbar_arrive(c0 == 16 ? bar_pa_full(k) : bar_pb_full(k));
                    }
                }
                tss(j, 5);
                turn_pass();
                l = alpha * l + ((rs2.x + rs2.y) + (rs2b.x + rs2b.y));
                m = m_new;
                // ---- two-level promotion O = alpha * O + R(j) ----
                mbar_wait(bar_r_full(k), j & 1);
                tc_fence_after();
                tss(j, 6);
                uint32_t r[64];
                tmem_ld32(tS + 0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
                tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
                tmem_wait_ld();
                reg_dep32(*reinterpret_cast<uint32_t(*)[32]>(&r[0]));
                reg_dep32(*reinterpret_cast<uint32_t(*)[32]>(&r[32]));
                tc_fence_before();
                mbar_arrive(bar_s_free(k));                // R in registers: QK(j+1) may overwrite S/R
                tss(j, 7);
                const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
#ifdef SAGE2_ABL_NOPROMO
                if (j == 0)                                                 // ablation build only
#endif
                for (int c0 = 0; c0 < 64; c0 += 32) {
                    uint32_t o[32];
                    if (j > 0) {
                        tmem_ld32(tO + c0, o);
                        tmem_wait_ld();
                        reg_dep32(o);
#pragma unroll
                        for (int c = 0; c < 32; c += 2) {
                            const float2 v = ffma2(a2, make_float2(__uint_as_float(o[c]), __uint_as_float(o[c + 1])),
                                                   make_float2(__uint_as_float(r[c0 + c]), __uint_as_float(r[c0 + c + 1])));
                            o[c] = __float_as_uint(v.x);
                            o[c + 1] = __float_as_uint(v.y);
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] = r[c0 + c];
                    }
                    tmem_st32(tO + c0, o);
                }
                tmem_wait_st();
                tss(j, 8);
            }
            // ---- epilogue: O / l / 448 * delta_V (+ V_m), l carries the 448 factor ----
            const float inv_l = 1.0f / l;
            const float* dvp = p.dv + (size_t)bhk * D;
            const float* vmp = p.vmean ? p.vmean + (size_t)bhk * D : nullptr;   // smooth V: O + V_m
            __half* orow = p.out + (((size_t)b * p.Hq + hq) * p.N + grow) * D;
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) {
                uint32_t o[32];
                tmem_ld32(tO + c0, o);
                tmem_wait_ld();
                reg_dep32(o);
                if (grow < p.N) {
#pragma unroll
                    for (int c = 0; c < 32; c += 8) {
                        const float4 d0 = __ldg(reinterpret_cast<const float4*>(dvp + c0 + c));
                        const float4 d1 = __ldg(reinterpret_cast<const float4*>(dvp + c0 + c + 4));
                        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                        const float4 m0 = vmp ? __ldg(reinterpret_cast<const float4*>(vmp + c0 + c)) : z;
                        const float4 m1 = vmp ? __ldg(reinterpret_cast<const float4*>(vmp + c0 + c + 4)) : z;
                        __half2 h0 = __floats2half2_rn(fmaf(__uint_as_float(o[c]) * inv_l, d0.x, m0.x),
                                                       fmaf(__uint_as_float(o[c + 1]) * inv_l, d0.y, m0.y));
                        __half2 h1 = __floats2half2_rn(fmaf(__uint_as_float(o[c + 2]) * inv_l, d0.z, m0.z),
                                                       fmaf(__uint_as_float(o[c + 3]) * inv_l, d0.w, m0.w));
                        __half2 h2 = __floats2half2_rn(fmaf(__uint_as_float(o[c + 4]) * inv_l, d1.x, m1.x),
                                                       fmaf(__uint_as_float(o[c + 5]) * inv_l, d1.y, m1.y));
                        __half2 h3 = __floats2half2_rn(fmaf(__uint_as_float(o[c + 6]) * inv_l, d1.z, m1.z),
                                                       fmaf(__uint_as_float(o[c + 7]) * inv_l, d1.w, m1.w));
                        *reinterpret_cast<uint4*>(orow + c0 + c) =
                            make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                                       *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
                    }
                }
            }
        }
        for (int j = my_ns; j < nst_max; ++j) {     // keep the MUFU turn rotation balanced
            turn_wait();
            turn_pass();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == PW) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

}  // namespace sage2

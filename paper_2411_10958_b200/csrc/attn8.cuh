// attn8.cuh -- SageAttention2 attention kernel v8 for sm_100a (Alg. 1 inner loop, PAPER.md:246-263;
// b_kv = 128).
//
// Each Q tile's softmax is split over TWO warpgroups by key columns: 16 softmax warps, four per SM
// sub-partition.  (Measured against one warpgroup per tile, the former v6: with one softmax warp per
// tile per sub-partition the MUFU idled ~40% of a tile's exp phase and the dequant + max phase was
// latency-bound; two warps per tile per sub-partition give both phases twice the independent work.)
//
// CTA = two 128-row Q blocks (i0 = 2*pair, i1 = i0 + 1) of one (b, h_q); K^/V^ stages shared.
// 20 warps (640 threads):
//   warp 0       producer: bulk-async (TMA engine) copies of the pre-swizzled tile images
//   warps 1/2    MMA issuer of tile 0 / 1 (whole warp, elect.sync): S = Q^ K^^T kind::i8 (exact
//                s32), R = P^ V^ kind::f8f6f4 (E4M3, fresh fp32 accumulator)
//   warps 4 + 8k + 4h + {0..3}   Q tile k, key half h (columns [64h, 64h + 64) of each 128-key
//                            tile), one thread per (query row, half) (TMEM lane = row):
//     s = S*dQ*dK*log2e/sqrt(d) + Delta S', masks (C-18); the exact row max (C-10) of the
//       two halves is exchanged through shared memory; P^ = e4m3(2^(s-m+log2 448)) -> smem
//       (P:254-256); partial row sums l_h (summed in the epilogue);
//     two-level promotion O = alpha O + R for output channels [hD/2, hD/2 + D/2) in fp32 against
//       O in TMEM; epilogue O / l / 448 * delta_V -> fp16.
//     The exp2 phases of the two Q tiles alternate (named barriers 1/2).
// TMEM: S_k/R_k [128k, 128k + 128) (R written over S once both halves have read S), O_k
// [128 NT + D k, +D) (NT = Q tiles per CTA: 2, or 1 for short sequences -- two CTAs per SM).
#pragma once
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdint>

#include "common.cuh"
#include "prep.cuh"
#include "ptx.cuh"

namespace sage2 {

#ifndef SAGE2_KSTAGES1
#define SAGE2_KSTAGES1 2   // K/V ring depth of the one-tile form (two CTAs per SM must fit the 228 KB)
#endif

// NT = Q tiles per CTA: 2 (the default form) or 1 (short sequences: 256 TMEM columns and ~110 KB of
// shared memory, so two CTAs share an SM and one's prologue / epilogue overlaps the other's loop).
template <int D, int NT = 2>
struct Attn8Smem {
    using B2 = PairSmem<D>;
    static constexpr int KS = NT == 2 ? kStages2 : SAGE2_KSTAGES1;
    static constexpr uint32_t TILE = B2::TILE;
    static constexpr uint32_t Q0 = 0, Q1 = NT == 2 ? TILE : 0;
    static constexpr uint32_t ST_K = B2::ST_K, ST_V = B2::ST_V, ST_DS0 = B2::ST_DS0, ST_DS1 = B2::ST_DS1,
                              ST_DK = B2::ST_DK, STAGE = B2::STAGE, ST0 = NT * TILE;
    static constexpr uint32_t P0 = ST0 + KS * STAGE, P1 = NT == 2 ? P0 + 16384 : P0;
    static constexpr uint32_t XM = P0 + NT * 16384;          // float xm[NT tiles][2 buf][2 halves][128]
    static constexpr uint32_t XL = XM + NT * 2 * 2 * 128 * 4;  // float xl[NT tiles][2 halves][128]
    static constexpr uint32_t BAR = XL + NT * 2 * 128 * 4;
    static constexpr uint32_t NBAR = 1 + 2 * KS + 10;
    static constexpr uint32_t TMEMPTR = BAR + 8 * NBAR;
    static constexpr uint32_t BYTES = TMEMPTR + 16;
    static constexpr uint32_t ALLOC = BYTES + 1024;
};

// GRAN: Q/K quantization granularity of the NEXT#4 ablation (0 per-thread = SageAttn2, 1 per-block,
// 2 per-token; prep.cuh gran_nq / gran_nk give the stored scales per 128 tokens).
// ONE: single-level accumulation ablation (P:1082 row "+ Two-level accumulation"; oracle two_level =
// false): the PV MMA accumulates straight into O in TMEM (enable-input-D after the first key tile),
// O is rescaled in place only in rows whose running max moved (alpha = 1 exactly otherwise), and S_k
// no longer shares its TMEM columns with R_k, so QK(j+1) is issued as soon as S(j) is in registers.
template <int D, bool CAUSAL, bool DUMP, bool QKF8 = false, bool TIMING = false, int GRAN = 0, bool ONE = false,
          int NT = 2>
__global__ void __launch_bounds__(NT == 2 ? 640 : 384, NT == 2 ? 1 : 2) k_attn8(const AttnParams p) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    using L = Attn8Smem<D, NT>;
    constexpr int KST = L::KS;                     // K/V ring depth
    constexpr int DH = D / 2;                      // output channels per half
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));

    // warp index through a shuffle: provably warp-uniform, so everything derived from it (role,
    // tile, half, TMEM / shared addresses) can live in uniform registers instead of being
    // rematerialised from threadIdx every iteration under the softmax warps' register pressure
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
    const int wg = warp / 4;
    const int nT = p.nT, Np = nT * 128;
    const int npairs = NT == 2 ? (nT + 1) / 2 : nT;   // CTAs per head
    // causal: heavy Q-block pairs first, within each head (long sequences: a head's K/V stays in L2
    // while its CTAs run) or over all heads (p.lpt, short sequences: the tail wave holds only light
    // pairs -- C2-1K 456 -> 482, C2-4K 907 -> 932 TOPS in round 1)
    int pair = CAUSAL ? (npairs - 1 - (int)blockIdx.x) : (int)blockIdx.x;
    int hq = blockIdx.y, b = blockIdx.z;
    if (CAUSAL && p.lpt) {
        const int nh = gridDim.y * gridDim.z;
        const int lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        pair = npairs - 1 - lin / nh;
        hq = (lin % nh) % p.Hq;
        b = (lin % nh) / p.Hq;
    }
    const int bhq = b * p.Hq + hq;
    const int bhk = b * p.Hkv + hq / (p.Hq / p.Hkv);
    const int it0 = NT * pair, it1 = NT == 2 ? it0 + 1 : nT;
    const int nkv0 = CAUSAL ? it0 + 1 : nT;
    const int nkv1 = (it1 < nT) ? (CAUSAL ? it1 + 1 : nT) : 0;
    const int nkv_max = nkv0 > nkv1 ? nkv0 : nkv1;
    const int ntiles = nkv1 > 0 ? 2 : 1;

    auto s_as_float = [](uint32_t u) { return QKF8 ? __uint_as_float(u) : (float)(int32_t)u; };
    auto s_as_int = [](uint32_t u) { return QKF8 ? (int32_t)__uint_as_float(u) : (int32_t)u; };
    // TIMING builds: clock64 stamps (CTA (0,0,0); thread 0 of the half-0 warpgroup of each tile) ->
    // (uint64*)p.s_dump [tile][j][slot]
    const bool tsel = TIMING && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
    auto ts = [&](int who, int j, int slot) {
        if (TIMING && tsel && j < 64)
            reinterpret_cast<unsigned long long*>(p.s_dump)[(who * 64 + j) * 16 + slot] = clock64();
    };
    const uint32_t bar0 = sbase + L::BAR;
    const uint32_t bar_q = bar0;
    auto bar_kv_full = [&](int s) { return bar0 + 8 * (1 + s); };
    auto bar_kv_empty = [&](int s) { return bar0 + 8 * (1 + KST + s); };
    auto bar_s_full = [&](int k) { return bar0 + 8 * (1 + 2 * KST + k); };
    auto bar_p_full = [&](int k) { return bar0 + 8 * (3 + 2 * KST + k); };
    auto bar_r_full = [&](int k) { return bar0 + 8 * (5 + 2 * KST + k); };
    auto bar_s_free = [&](int k) { return bar0 + 8 * (7 + 2 * KST + k); };
    auto bar_pa_full = [&](int k) { return bar0 + 8 * (9 + 2 * KST + k); };   // first halves of P^
    auto stage_addr = [&](int s) { return sbase + L::ST0 + s * L::STAGE; };
    const size_t tile_bytes = (size_t)128 * D;
    // producer: one K/V ring stage (K^, V^T, delta_K, the two tiles' Delta S rows)
    auto load_stage = [&](int j, uint64_t keep) {
        const int s = j % KST;
        const uint32_t sa = stage_addr(s);
        const bool d0 = j < nkv0, d1 = j < nkv1;
        constexpr int NGK = gran_nk(GRAN);
        mbar_arrive_expect_tx(bar_kv_full(s), 2 * L::TILE + 4 * NGK + 512 * (d0 + d1));
        bulk_g2s_hint(sa + L::ST_K, p.khat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, bar_kv_full(s), keep);
        bulk_g2s_hint(sa + L::ST_V, p.vhat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, bar_kv_full(s), keep);
        bulk_g2s(sa + L::ST_DK, p.dk + ((size_t)bhk * nT + j) * NGK, 4 * NGK, bar_kv_full(s));
        if (d0) bulk_g2s(sa + L::ST_DS0, p.ds + ds_row(p.ds_tri, bhq, it0, nT) + (size_t)j * 128, 512, bar_kv_full(s));
        if (d1) bulk_g2s(sa + L::ST_DS1, p.ds + ds_row(p.ds_tri, bhq, it1, nT) + (size_t)j * 128, 512, bar_kv_full(s));
    };
    const int jpre = nkv_max < KST ? nkv_max : KST;   // stages issued before the CTA-wide sync

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < KST; ++s) {
            mbar_init(bar_kv_full(s), 1);
            mbar_init(bar_kv_empty(s), NT);     // one arrival per Q tile (MMA commit or bypass)
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(bar_s_full(k), 1);
            mbar_init(bar_p_full(k), 256);
            mbar_init(bar_pa_full(k), 256);
            mbar_init(bar_r_full(k), 1);
            mbar_init(bar_s_free(k), 256);
        }
        fence_mbar_init();
        // the producer thread starts the Q and first K/V loads right away: their latency overlaps the
        // TMEM allocation and the CTA-wide barrier (short sequences pay it once per few KV steps)
        mbar_arrive_expect_tx(bar_q, L::TILE * ntiles);
        bulk_g2s(sbase + L::Q0, p.qhat + ((size_t)bhq * nT + it0) * tile_bytes, L::TILE, bar_q);
        if (ntiles == 2) bulk_g2s(sbase + L::Q1, p.qhat + ((size_t)bhq * nT + it1) * tile_bytes, L::TILE, bar_q);
        const uint64_t keep = policy_evict_last();
        for (int j = 0; j < jpre; ++j) load_stage(j, keep);
    }
    // control warpgroup first (warps 0-3: producer, MMA issuers), softmax warpgroups 1-4 (measured
    // +1.5% against the control warps at the highest ids: the issuer hand-offs wake up sooner)
    constexpr int CW = 0, SW0 = 1;
    if (warp == 4 * CW) tmem_alloc<NT == 2 ? 512 : 256>(sbase + L::TMEMPTR);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sgen + L::TMEMPTR);

    if (wg == CW) {
        setmaxnreg_dec<32>();
        if (warp == 4 * CW && lane == 0) {
            // ===================== producer (the first jpre stages were issued before the sync) =====================
            const uint64_t keep = policy_evict_last();
            for (int j = jpre; j < nkv_max; ++j) {
                const int s = j % KST;
                mbar_wait(bar_kv_empty(s), ((j / KST) - 1) & 1);
                load_stage(j, keep);
            }
        } else if (warp == 4 * CW + 1 || (NT == 2 && warp == 4 * CW + 2)) {
            // ============ MMA issuer for Q tile k (whole warp converged, one elected lane issues) ============
            const int k = warp - (4 * CW + 1);
            const int my_nkv = k ? nkv1 : nkv0;
            constexpr uint32_t IDQK = QKF8 ? idesc_e4m3(128, 128) : idesc_i8(128, 128);
            constexpr uint32_t IDPV = idesc_e4m3(128, D);
            const uint64_t qdesc = smem_desc<D>(sbase + (k ? L::Q1 : L::Q0));
            const uint64_t pdesc = smem_desc<128>(sbase + (k ? L::P1 : L::P0));
            const uint32_t tS = tmem + 128 * k;
            const uint32_t tPV = ONE ? tmem + 128 * NT + D * k : tS;   // R over S (two-level) or O itself (ONE)
            mbar_wait(bar_q, 0);
            for (int j = 0; j < nkv_max; ++j) {
                const int s = j % KST;
                mbar_wait(bar_kv_full(s), (j / KST) & 1);
                if (lane == 0) ts(2 + k, j, 0);
                if (j >= my_nkv) {                 // this tile is done: release the stage for it
                    if (lane == 0) mbar_arrive(bar_kv_empty(s));
                    continue;
                }
                if (j >= 1) mbar_wait(bar_s_free(k), (j - 1) & 1);   // R_k(j-1) read out of TMEM
                if (lane == 0) ts(2 + k, j, 1);
                tc_fence_after();
                const uint64_t kdesc = smem_desc<D>(stage_addr(s) + L::ST_K);
#pragma unroll
                for (int kk = 0; kk < D / 32; ++kk) {
                    if (QKF8) mma_f8f6f4_w(tS, qdesc + 2 * kk, kdesc + 2 * kk, IDQK, kk > 0);
                    else mma_i8_w(tS, qdesc + 2 * kk, kdesc + 2 * kk, IDQK, kk > 0);
                }
                mma_commit_w(bar_s_full(k));
                if (lane == 0) ts(2 + k, j, 2);
                const uint64_t vdesc = smem_desc<128>(stage_addr(s) + L::ST_V);
                if (SAGE2_PSPLIT) {
                    // each key half's first 32 codes (P^ columns 0-31 and 64-95: K steps 0 and 2) are
                    // multiplied while the softmax still exponentiates the second 32
                    mbar_wait(bar_pa_full(k), j & 1);
                    if (lane == 0) ts(2 + k, j, 3);
                    tc_fence_after();
                    mma_f8f6f4_w(tPV, pdesc + 0, vdesc + 0, IDPV, ONE && j > 0);
                    mma_f8f6f4_w(tPV, pdesc + 4, vdesc + 4, IDPV, 1);
                    mbar_wait(bar_p_full(k), j & 1);                // softmax_k(j) wrote all of P^_k
                    tc_fence_after();
                    mma_f8f6f4_w(tPV, pdesc + 2, vdesc + 2, IDPV, 1);
                    mma_f8f6f4_w(tPV, pdesc + 6, vdesc + 6, IDPV, 1);
                } else {
                    mbar_wait(bar_p_full(k), j & 1);                // softmax_k(j) wrote P^_k
                    if (lane == 0) ts(2 + k, j, 3);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) mma_f8f6f4_w(tPV, pdesc + 2 * kk, vdesc + 2 * kk, IDPV, kk > 0 || (ONE && j > 0));
                }
                mma_commit_w(bar_r_full(k));
                mma_commit_w(bar_kv_empty(s));
                if (lane == 0) ts(2 + k, j, 4);
            }
        }
    } else {
        // pool = 96 x 640 (launch): 32 + 4 x 112 = 5 x 96 (inc blocks otherwise); one-tile form: 80 x 384
        if constexpr (NT == 2) setmaxnreg_inc<112>();
        else setmaxnreg_inc<104>();
        // ============ softmax (key half h) + two-level promotion + epilogue for Q tile k ============
        const int k = (wg - SW0) >> 1, h = (wg - SW0) & 1;
        const int my_nkv = k ? nkv1 : nkv0, my_it = k ? it1 : it0;
        // the MUFU turns alternate between the two tiles of a CTA (no partner in the one-tile form)
        auto turn_wait = [&]() { if (NT == 2) named_bar_sync(1 + k, 512); };
        auto turn_pass = [&]() { if (NT == 2) named_bar_arrive(1 + (1 - k), 512); };
        auto pair_sync = [&]() { named_bar_sync(3 + k, 256); };   // the two halves of tile k
        if (k == 1) turn_pass();                    // tile 0 takes the first MUFU turn
        if (my_nkv > 0) {
            const int wq = warp & 3;
            const int row = 32 * wq + lane;
            const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
            const uint32_t tS = tmem + 128 * k + lane_off + 64 * h;      // this half's S columns
            const uint32_t tR = tmem + 128 * k + lane_off + DH * h;      // this half's R channels
            const uint32_t tO = tmem + 128 * NT + D * k + lane_off + DH * h;  // this half's O channels
            const int grow = my_it * 128 + row;
            const float dqr = p.dq[((size_t)bhq * nT + my_it) * gran_nq(GRAN) +
                                   (GRAN == 2 ? row : GRAN == 1 ? 0 : 8 * (row / 32) + (row % 8))] * p.qk_scale_log2;
            uint8_t* sP = sgen + (k ? L::P1 : L::P0);
            float* xm = reinterpret_cast<float*>(sgen + L::XM) + k * 512;    // [buf][half][128]
            float m = -INFINITY, l = 0.0f;
            const bool tme = TIMING && h == 0 && row == 0;
            auto tss = [&](int j, int slot) { if (tme) ts(k, j, slot); };
            for (int j = 0; j < my_nkv; ++j) {
                const int s = j % KST;
                tss(j, 0);
                mbar_wait(bar_kv_full(s), (j / KST) & 1);      // Delta S / delta_K landed
                mbar_wait(bar_s_full(k), j & 1);
                tc_fence_after();
                tss(j, 1);
                const uint32_t dss = stage_addr(s) + (k ? L::ST_DS1 : L::ST_DS0) + 256 * h;
                const float* dks = reinterpret_cast<const float*>(sgen + L::ST0 + s * L::STAGE + L::ST_DK) +
                                   (GRAN == 1 ? h : 4 * h);
                const uint32_t dkv = stage_addr(s) + L::ST_DK + 256 * h;   // per-token delta_K of this half
                float2 sc2[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const float v = dqr * dks[GRAN == 1 ? 0 : g];
                    sc2[g] = make_float2(v, v);
                }
                const float2 dq2 = make_float2(dqr, dqr);
                float sv[64];
                {
                    uint32_t r0[32], r1[32];
                    tmem_ld32(tS + 0, r0);
                    tmem_ld32(tS + 32, r1);
                    tmem_wait_ld();
                    reg_dep32(r0);
                    reg_dep32(r1);
                    if (ONE) {                                  // S in registers: QK(j+1) may overwrite it
                        tc_fence_before();
                        mbar_arrive(bar_s_free(k));
                    }
                    tss(j, 9);
                    if (DUMP) {
                        int32_t* dst = p.s_dump + ((size_t)bhq * Np + grow) * (size_t)Np + j * 128 + 64 * h;
#pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            dst[c] = s_as_int(r0[c]);
                            dst[32 + c] = s_as_int(r1[c]);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 64; c += 4) {
                        const uint32_t* rr = c < 32 ? r0 : r1;
#ifdef SAGE2_ABL_NODS
                        const float4 d4 = make_float4(0.f, 0.f, 0.f, 0.f);   // ablation build only
#else
                        const float4 d4 = lds128(dss + 4 * c);
#endif
                        const int g = (c % 8) / 2;
                        float2 sa2 = sc2[g], sb2 = sc2[g + 1];
                        if (GRAN == 2) {                     // one delta_K per key column
                            const float4 k4 = lds128(dkv + 4 * c);
                            sa2 = fmul2(make_float2(k4.x, k4.y), dq2);
                            sb2 = fmul2(make_float2(k4.z, k4.w), dq2);
                        }
                        const float2 a = ffma2(make_float2(s_as_float(rr[c % 32]), s_as_float(rr[c % 32 + 1])),
                                               sa2, make_float2(d4.x, d4.y));
                        const float2 bq = ffma2(make_float2(s_as_float(rr[c % 32 + 2]), s_as_float(rr[c % 32 + 3])),
                                                sb2, make_float2(d4.z, d4.w));
                        sv[c] = a.x;
                        sv[c + 1] = a.y;
                        sv[c + 2] = bq.x;
                        sv[c + 3] = bq.y;
                    }
                }
                tss(j, 2);
                if ((CAUSAL && j == my_it) || (j * 128 + 128 > p.N)) {   // C-18
#pragma unroll
                    for (int c = 0; c < 64; ++c) {
                        const int key = j * 128 + 64 * h + c;
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
                // exact row max over both halves (C-10): exchange through shared memory
                const float mh = fmax3(mx[0], mx[1], fmaxf(mx[2], mx[3]));
                float* xmb = xm + (j & 1) * 256;
                xmb[h * 128 + row] = mh;
#ifdef SAGE2_ABL_NOXCHG
                const float m_new = fmaxf(m, mh);                          // ablation build only
#else
                pair_sync();
                const float m_new = fmax3(m, mh, xmb[(1 - h) * 128 + row]);
#endif
                const float alpha = (m == -INFINITY) ? 0.0f : ex2_approx(m - m_new);
                const float m_use = (m_new == -INFINITY) ? 0.0f : (m_new - kLog2_448);
                tss(j, 3);
                if (ONE && j > 0) {
                    // PV(j-1) has finished reading P^ and accumulating into O; rows whose max moved
                    // get O *= alpha before PV(j) accumulates (alpha is exactly 1 in the others)
                    mbar_wait(bar_r_full(k), (j - 1) & 1);
                    tc_fence_after();
                    if (__any_sync(0xffffffffu, m_new != m)) {
                        const float f = (m_new != m) ? alpha : 1.0f;
                        const float2 f2 = make_float2(f, f);
#pragma unroll
                        for (int c0 = 0; c0 < DH; c0 += 8) {     // S(j) stays live: 8 columns at a time
                            uint32_t o[8];
                            tmem_ld8(tO + c0, o);
                            tmem_wait_ld();
                            reg_dep8(o);
#pragma unroll
                            for (int c = 0; c < 8; c += 2) {
                                const float2 v = fmul2(f2, make_float2(__uint_as_float(o[c]), __uint_as_float(o[c + 1])));
                                o[c] = __float_as_uint(v.x);
                                o[c + 1] = __float_as_uint(v.y);
                            }
                            tmem_st8(tO + c0, o);
                        }
                        tmem_wait_st();
                    }
                }
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
                    *reinterpret_cast<uint4*>(sP + swz_off<128>(row, 64 * h + c0)) = make_uint4(w[0], w[1], w[2], w[3]);
                    if (DUMP && p.p_dump)
                        *reinterpret_cast<uint4*>(p.p_dump + ((size_t)bhq * Np + grow) * (size_t)Np + j * 128 + 64 * h + c0) =
                            make_uint4(w[0], w[1], w[2], w[3]);
                    if (SAGE2_PSPLIT && c0 == 16) {                  // this half's first 32 codes are in smem
                        fence_proxy_async_smem();
                        tc_fence_before();
                        mbar_arrive(bar_pa_full(k));
                    }
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(bar_p_full(k));
                tss(j, 5);
                turn_pass();
                l = alpha * l + ((rs2.x + rs2.y) + (rs2b.x + rs2b.y));
                m = m_new;
                if (ONE) continue;
                // ---- two-level promotion O = alpha * O + R(j) ----
                mbar_wait(bar_r_full(k), j & 1);
                tc_fence_after();
                tss(j, 6);
                uint32_t r[DH];
#pragma unroll
                for (int c = 0; c < DH; c += 32) tmem_ld32(tR + c, *reinterpret_cast<uint32_t(*)[32]>(&r[c]));
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < DH; c += 32) reg_dep32(*reinterpret_cast<uint32_t(*)[32]>(&r[c]));
                tc_fence_before();
                mbar_arrive(bar_s_free(k));                // R in registers: QK(j+1) may overwrite S/R
                tss(j, 7);
                if (TIMING && k == 0 && lane == 0) ts(4 + wq + 4 * h, j, 7);   // every warp's R read
                const float2 a2 = make_float2(alpha, alpha);
#ifdef SAGE2_ABL_NOPROMO
                if (j == 0)                                                 // ablation build only
#endif
#pragma unroll
                for (int c0 = 0; c0 < DH; c0 += 32) {
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
            if (ONE) {                                      // the last PV has accumulated into O
                mbar_wait(bar_r_full(k), (my_nkv - 1) & 1);
                tc_fence_after();
            }
            // ---- epilogue: O / (l_0 + l_1) / 448 * delta_V  (l carries the 448 factor) ----
            float* xl = reinterpret_cast<float*>(sgen + L::XL) + k * 256;
            xl[h * 128 + row] = l;
            pair_sync();
            const float inv_l = 1.0f / (xl[row] + xl[128 + row]);
            const float* dvp = p.dv + (size_t)bhk * D + DH * h;
            const float* vmp = p.vmean ? p.vmean + (size_t)bhk * D + DH * h : nullptr;   // smooth V: O + V_m
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
        for (int j = my_nkv; j < nkv_max; ++j) {    // keep the MUFU turn protocol balanced
            turn_wait();
            turn_pass();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4 * CW) {
        tc_fence_after();
        tmem_dealloc<NT == 2 ? 512 : 256>(tmem);
    }
}

}  // namespace sage2

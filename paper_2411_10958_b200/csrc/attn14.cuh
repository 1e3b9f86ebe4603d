// attn14.cuh -- SageAttention2 attention kernel v14 for sm_100a (Alg. 1 inner loop, PAPER.md:246-263;
// b_kv = 128): ONE 128-row Q block per CTA, its KV tiles split over two softmax warpgroup PAIRS
// (pair A: even tiles, pair B: odd tiles), S double-buffered in TMEM.  Experimental (not the default).
//
// Why: in v8 the TMEM budget (two Q tiles x [S/R 128 + O 128 columns]) forces
// R = P^V^ to be written over S, so QK(j+1) can only start once the softmax has read R(j) back; each
// tile's critical chain is exp -> PV -> R read -> QK -> S read -> dequant -> max exchange -> exp
// (~2000 cycles per 128 x 128 tile against the 1024-cycle MUFU floor).  v14 spends the same 512
// columns as S0 | S1 | R | O for one Q tile: QK(j+2) is issued as soon as S(j) is in registers (two
// tiles ahead), and the two pairs alternate the MUFU: while pair B exponentiates tile j+1, pair A
// promotes R(j) into O and dequantizes tile j+2.  The running max stays exact (C-10):
// M_j = max(M_{j-1}, rowmax S_j) is handed from pair to pair through shared memory (M_{j-1} is known
// before tile j-1 is exponentiated, so the hand-off is off the MUFU path); the promotions
// O = alpha_j O + R_j stay in tile order through a named-barrier hand-off.
//
// Two forms (template CORR; the library builds CORR = 1, SAGE2_V14_CORR in sage2_api.cu):
//   CORR = 0, 640 threads (20 warps): the pair that exponentiated tile j also promotes R(j) and, for
//             the last tile, runs the epilogue (warps 4-19 softmax);
//   CORR = 1, 768 threads (24 warps): a correction warpgroup (warps 4-7, thread = query row, 16-column
//             TMEM round trips) does every promotion and the epilogue; softmax warps 8-23.
//   warp 0        producer: bulk-async copies of the pre-swizzled K^ / V^T tiles, Delta S row, delta_K
//                 (NST-deep mbarrier ring, L2 evict-last)
//   warps 1, 2    MMA issuers (whole warp converged, elect.sync): S_{j%2} = Q^ K^_j^T (kind::i8, exact
//                 s32) / R = P^_j V^_j (kind::f8f6f4, fresh fp32 accumulator; tile 0 straight into O)
//   softmax       pair P = tiles j = P (mod 2), key half h (columns [64h, 64h + 64)), thread = (row,
//                 half): s = S dQ dK log2e/sqrt(d) + Delta S', exact row max through shared
//                 memory, P^ = e4m3(2^(s - M_j + log2 448)) -> smem, partial row sums
//   promotion     O = alpha_j O + R_j in tile order; epilogue O / l / 448 * delta_V
//                 -> fp16
// Measured slower than v8 in both forms; kept as the experimental selector
// SAGE2_F_KERNEL_V14.
// TMEM columns: S_0 [0,128) | S_1 [128,256) | R [256,256+D) | O [256+D,256+2D).
#pragma once
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdint>

#include "common.cuh"
#include "prep.cuh"
#include "ptx.cuh"

#ifndef SAGE2_V14_CC
#define SAGE2_V14_CC 16   // correction warpgroup chunk: 32 spills its 64 live values at 72 registers
#endif
#ifndef SAGE2_K14STAGES
#define SAGE2_K14STAGES 4
#endif

namespace sage2 {

template <int D>
struct Attn14Smem {
    static constexpr int NST = SAGE2_K14STAGES;              // K/V ring: tiles j, j+1, j+2 live + 1 prefetch
    static constexpr int NM = 4;                            // running-max ring M_j -> pair of j+1 (8 with CORR)
    static constexpr uint32_t TILE = 128 * D;
    static constexpr uint32_t Q = 0;
    // stage: K^ | V^T | Delta S row (512 B) | delta_K (32 B)
    static constexpr uint32_t ST_K = 0, ST_V = TILE, ST_DS = 2 * TILE, ST_DK = 2 * TILE + 512;
    static constexpr uint32_t STAGE = ((2 * TILE + 1024) + 1023) / 1024 * 1024;
    static constexpr uint32_t ST0 = TILE;
    static constexpr uint32_t P0 = ST0 + NST * STAGE;      // P^ of pair 0 / 1: 128 x 128 e4m3 (SW128)
    static constexpr uint32_t MR = P0 + 2 * 16384;         // float M[8][128]
    static constexpr uint32_t XM = MR + 8 * 128 * 4;      // float xm[2 pairs][2 buf][2 halves][128]
    static constexpr uint32_t XL = XM + 2 * 2 * 2 * 128 * 4;   // float l[2 pairs][2 halves][128], m[2][128]
    static constexpr uint32_t BAR = XL + (2 * 2 * 128 + 2 * 128) * 4;
    static constexpr uint32_t NBAR = 1 + 2 * NST + 2 + 2 + 2 + 2 + 1 + 1 + 2 + 8 + 1;
    static constexpr uint32_t TMEMPTR = BAR + 8 * NBAR;
    static constexpr uint32_t BYTES = TMEMPTR + 16;
    static constexpr uint32_t ALLOC = BYTES + 1024;
};

// Epilogue of one query row: NC output channels from TMEM (tO, consecutive columns) starting at channel
// c_base: O / l (inv_l; l carries the 448 factor) * delta_V (+ V_m with smooth V) -> fp16.
template <int D, int NC>
__device__ __forceinline__ void epilogue14(const AttnParams& p, uint32_t tO, float inv_l, int b, int hq, int bhk, int grow,
                                           int c_base) {
    const float* dvp = p.dv + (size_t)bhk * D + c_base;
    const float* vmp = p.vmean ? p.vmean + (size_t)bhk * D + c_base : nullptr;
    __half* orow = p.out + (((size_t)b * p.Hq + hq) * p.N + grow) * D + c_base;
#pragma unroll
    for (int c0 = 0; c0 < NC; c0 += 32) {
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

// TIMING builds (dev library): clock64 stamps of CTA (0,0,0) -> (uint64*)p.s_dump [who][j][slot]; who = pair
// (its row-0 thread of half 0) or 2 (MMA issuer lane 0).
// CORR: the promotion and the epilogue run in a separate correction warpgroup (warps 4-7, thread = query
// row, 768 threads: registers 24 / 72 / 96 for control / correction / softmax) instead of in the pair that
// exponentiated the tile.
template <int D, bool QKF8 = false, bool TIMING = false, bool CORR = false>
__global__ void __launch_bounds__(CORR ? 768 : 640, 1) k_attn14(const AttnParams p) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    using L = Attn14Smem<D>;
    constexpr int NST = L::NST, NM = CORR ? 8 : L::NM;
    constexpr int SW0 = CORR ? 2 : 1;           // first softmax warpgroup
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));

    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
    const int wg = warp / 4;
    const int nT = p.nT, nkv = nT;
    const int it = blockIdx.x, hq = blockIdx.y, b = blockIdx.z;
    const int bhq = b * p.Hq + hq;
    const int bhk = b * p.Hkv + hq / (p.Hq / p.Hkv);

    const bool tsel = TIMING && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
    auto ts = [&](int who, int j, int slot) {
        if (TIMING && tsel && j < 64)
            reinterpret_cast<unsigned long long*>(p.s_dump)[(who * 64 + j) * 16 + slot] = clock64();
    };
    const uint32_t bar0 = sbase + L::BAR;
    const uint32_t bar_q = bar0;
    auto kv_full = [&](int s) { return bar0 + 8 * (1 + s); };
    auto kv_empty = [&](int s) { return bar0 + 8 * (1 + NST + s); };
    auto s_full = [&](int k) { return bar0 + 8 * (1 + 2 * NST + k); };
    auto s_free = [&](int k) { return bar0 + 8 * (3 + 2 * NST + k); };
    auto pa_full = [&](int k) { return bar0 + 8 * (5 + 2 * NST + k); };   // first 32 codes of each half
    auto p_full = [&](int k) { return bar0 + 8 * (7 + 2 * NST + k); };
    const uint32_t r_full = bar0 + 8 * (9 + 2 * NST);                    // PV(j >= 1) done
    const uint32_t r_free = bar0 + 8 * (10 + 2 * NST);                   // R(j) read by its pair
    auto pv_done = [&](int k) { return bar0 + 8 * (11 + 2 * NST + k); };  // P^ buffer k read by PV
    auto m_full = [&](int k) { return bar0 + 8 * (13 + 2 * NST + k); };   // M_j in the ring
    const uint32_t o_full = bar0 + 8 * (13 + 2 * NST + NM);              // last PV done
    auto stage_addr = [&](int s) { return sbase + L::ST0 + s * L::STAGE; };
    const size_t tile_bytes = (size_t)128 * D;

    auto load_stage = [&](int j, uint64_t keep) {
        const int s = j % NST;
        const uint32_t sa = stage_addr(s);
        mbar_arrive_expect_tx(kv_full(s), 2 * L::TILE + 32 + 512);
        bulk_g2s_hint(sa + L::ST_K, p.khat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, kv_full(s), keep);
        bulk_g2s_hint(sa + L::ST_V, p.vhat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, kv_full(s), keep);
        bulk_g2s(sa + L::ST_DK, p.dk + ((size_t)bhk * nT + j) * 8, 32, kv_full(s));
        bulk_g2s(sa + L::ST_DS, p.ds + ds_row(0, bhq, it, nT) + (size_t)j * 128, 512, kv_full(s));
    };
    const int jpre = nkv < NST ? nkv : NST;

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < NST; ++s) {
            mbar_init(kv_full(s), 1);
            mbar_init(kv_empty(s), 2);          // commits after QK(j) and after PV(j)
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(s_full(k), 1);
            mbar_init(s_free(k), 256);
            mbar_init(pa_full(k), 256);
            mbar_init(p_full(k), 256);
            mbar_init(pv_done(k), 1);
        }
        mbar_init(r_full, 1);
        mbar_init(r_free, CORR ? 128 : 256);
        for (int k = 0; k < NM; ++k) mbar_init(m_full(k), 128);   // the half-0 threads of a pair
        mbar_init(o_full, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar_q, L::TILE);
        bulk_g2s(sbase + L::Q, p.qhat + ((size_t)bhq * nT + it) * tile_bytes, L::TILE, bar_q);
        const uint64_t keep = policy_evict_last();
        for (int j = 0; j < jpre; ++j) load_stage(j, keep);
    }
    if (warp == 0) tmem_alloc<512>(sbase + L::TMEMPTR);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sgen + L::TMEMPTR);
    float* mring = reinterpret_cast<float*>(sgen + L::MR);

    if (wg == 0) {
        if constexpr (CORR) setmaxnreg_dec<24>();
        else setmaxnreg_dec<32>();
        if (warp == 0 && lane == 0) {
            // ===================== producer =====================
            const uint64_t keep = policy_evict_last();
            for (int j = jpre; j < nkv; ++j) {
                const int s = j % NST;
                mbar_wait(kv_empty(s), ((j / NST) - 1) & 1);
                load_stage(j, keep);
            }
        } else if (warp == 1 || warp == 2) {
            // ============ MMA issuers: warp 1 QK^T, warp 2 PV (issue blocks ~70-100 cycles per MMA, so one
            // warp for both serialises them: PV(j) committed ~1500 cycles after P^(j), measured) ============
            constexpr uint32_t IDQK = QKF8 ? idesc_e4m3(128, 128) : idesc_i8(128, 128);
            constexpr uint32_t IDPV = idesc_e4m3(128, D);
            if (warp == 1) {
                const uint64_t qdesc = smem_desc<D>(sbase + L::Q);
                mbar_wait(bar_q, 0);
                for (int j = 0; j < nkv; ++j) {
                    const int s = j % NST;
                    if (j >= 2) mbar_wait(s_free(j & 1), ((j - 2) >> 1) & 1);   // S(j-2) in the pair's registers
                    mbar_wait(kv_full(s), (j / NST) & 1);
                    if (lane == 0) ts(2, j, 1);
                    tc_fence_after();
                    const uint64_t kdesc = smem_desc<D>(stage_addr(s) + L::ST_K);
                    const uint32_t tS = tmem + 128 * (j & 1);
#pragma unroll
                    for (int kk = 0; kk < D / 32; ++kk) {
                        if (QKF8) mma_f8f6f4_w(tS, qdesc + 2 * kk, kdesc + 2 * kk, IDQK, kk > 0);
                        else mma_i8_w(tS, qdesc + 2 * kk, kdesc + 2 * kk, IDQK, kk > 0);
                    }
                    mma_commit_w(s_full(j & 1));
                    mma_commit_w(kv_empty(s));                // K^_j consumed
                    if (lane == 0) ts(2, j, 2);
                }
            } else {
                const uint32_t tR = tmem + 256, tO = tmem + 256 + D;
                for (int j = 0; j < nkv; ++j) {
                    const int bb = j & 1, u = j >> 1, s = j % NST;
                    if (lane == 0) ts(2, j, 0);
                    const uint64_t vdesc = smem_desc<128>(stage_addr(s) + L::ST_V);
                    const uint64_t pdesc = smem_desc<128>(sbase + L::P0 + bb * 16384);
                    const uint32_t tD = j == 0 ? tO : tR;     // tile 0's R is O itself
                    // each key half's first 32 codes (K steps 0 and 2) go while the second 32 are exponentiated
                    mbar_wait(pa_full(bb), u & 1);
                    if (lane == 0) ts(2, j, 3);
                    if (j >= 2) mbar_wait(r_free, (j - 2) & 1);   // R(j-1) drained
                    if (lane == 0) ts(2, j, 4);
                    tc_fence_after();
                    mma_f8f6f4_w(tD, pdesc + 0, vdesc + 0, IDPV, 0);
                    mma_f8f6f4_w(tD, pdesc + 4, vdesc + 4, IDPV, 1);
                    mbar_wait(p_full(bb), u & 1);
                    if (lane == 0) ts(2, j, 5);
                    tc_fence_after();
                    mma_f8f6f4_w(tD, pdesc + 2, vdesc + 2, IDPV, 1);
                    mma_f8f6f4_w(tD, pdesc + 6, vdesc + 6, IDPV, 1);
                    if (j >= 1) mma_commit_w(r_full);
                    mma_commit_w(kv_empty(s));                // V^_j consumed (and Delta S / delta_K: read before P^)
                    mma_commit_w(pv_done(bb));
                    if (lane == 0) ts(2, j, 6);
                }
                mma_commit_w(o_full);
            }
        }
    } else if (CORR && wg == 1) {
        setmaxnreg_dec<72>();
        constexpr int CC = SAGE2_V14_CC;                  // promotion chunk (columns per TMEM round trip)
        // ============ correction: O = alpha_j O + R_j, then the epilogue ============
        // M ring protocol: M_{j+1} is read BEFORE R(j) is released (r_free), and its slot is rewritten only
        // with M_{j+9}, which needs PV(j+5) to have run, which needs R(j+3) drained -- so the read can never
        // see a newer value and the m_full phase can never be ambiguous.
        const int wq = warp & 3, row = 32 * wq + lane;
        const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
        const uint32_t tR = tmem + 256 + lane_off, tO = tmem + 256 + D + lane_off;
        mbar_wait(m_full(0), 0);
        float m_prev = mring[row], m_cur = m_prev;
        if (nkv > 1) {
            mbar_wait(m_full(1), 0);
            m_cur = mring[128 + row];
        }
        for (int j = 1; j < nkv; ++j) {
            const float alpha = (m_prev == -INFINITY) ? 0.0f : ex2_approx(m_prev - m_cur);
            const float2 a2 = make_float2(alpha, alpha);
            mbar_wait(r_full, (j - 1) & 1);
            tc_fence_after();
            float m_next = m_cur;
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += CC) {
                if (c0 == D - CC && j + 1 < nkv) {         // M_{j+1} before R(j) is released (see above)
                    mbar_wait(m_full((j + 1) % NM), ((j + 1) / NM) & 1);
                    m_next = mring[((j + 1) % NM) * 128 + row];
                }
                uint32_t r[CC], o[CC];
#if SAGE2_V14_CC == 32
                tmem_ld32(tR + c0, r);
                tmem_ld32(tO + c0, o);
                tmem_wait_ld();
                reg_dep32(r);
                reg_dep32(o);
#else
                tmem_ld16(tR + c0, r);
                tmem_ld16(tO + c0, o);
                tmem_wait_ld();
                reg_dep16(r);
                reg_dep16(o);
#endif
                if (c0 == D - CC) {                        // all of R(j) has been read
                    tc_fence_before();
                    mbar_arrive(r_free);
                }
#pragma unroll
                for (int c = 0; c < CC; c += 2) {
                    const float2 v = ffma2(a2, make_float2(__uint_as_float(o[c]), __uint_as_float(o[c + 1])),
                                           make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])));
                    o[c] = __float_as_uint(v.x);
                    o[c + 1] = __float_as_uint(v.y);
                }
#if SAGE2_V14_CC == 32
                tmem_st32(tO + c0, o);
#else
                tmem_st16(tO + c0, o);
#endif
            }
            tmem_wait_st();
            m_prev = m_cur;
            m_cur = m_next;
        }
        mbar_wait(o_full, 0);                              // the last PV has landed
        tc_fence_after();
        named_bar_sync(7, 640);                            // the four softmax partial sums are in smem
        const float* xl = reinterpret_cast<const float*>(sgen + L::XL);
        const float mf = m_cur;
        float lsum = 0.0f;
#pragma unroll
        for (int PP = 0; PP < 2; ++PP) {
            const float mp = xl[512 + PP * 128 + row];
            const float f = (mp == -INFINITY) ? 0.0f : ex2_approx(mp - mf);
            lsum += (xl[(2 * PP) * 128 + row] + xl[(2 * PP + 1) * 128 + row]) * f;
        }
        epilogue14<D, D>(p, tO, 1.0f / lsum, b, hq, bhk, it * 128 + row, 0);
    } else {
        if constexpr (CORR) setmaxnreg_inc<96>();   // pool = 80 x 768: 128 x 24 + 128 x 72 + 512 x 96
        else setmaxnreg_inc<112>();                 // pool = 96 x 640 (launch): 128 x 32 + 512 x 112
        // ============ softmax: pair P (tiles j = P mod 2), key half h ============
        const int P = (wg - SW0) >> 1, h = (wg - SW0) & 1;
        constexpr int DH = D / 2;
        auto turn_wait = [&]() { named_bar_sync(1 + P, 512); };
        auto turn_pass = [&]() { named_bar_arrive(1 + (1 - P), 512); };
        auto pair_sync = [&]() { named_bar_sync(3 + P, 256); };
        auto promo_wait = [&]() { named_bar_sync(5 + P, 512); };          // promotion j-1 is in O
        auto promo_pass = [&]() { named_bar_arrive(5 + (1 - P), 512); };
        if (P == 1) turn_pass();                    // pair 0 takes the first MUFU turn
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
        const uint32_t tS = tmem + 128 * P + lane_off + 64 * h;
        const uint32_t tR = tmem + 256 + lane_off + DH * h;          // this half's R channels
        const uint32_t tO = tmem + 256 + D + lane_off + DH * h;      // this half's O channels
        const int grow = it * 128 + row;
        const float dqr = p.dq[((size_t)bhq * nT + it) * 32 + 8 * (row / 32) + (row % 8)] * p.qk_scale_log2;
        uint8_t* sP = sgen + L::P0 + P * 16384;
        float* xm = reinterpret_cast<float*>(sgen + L::XM) + P * 512;    // [buf][half][128]
        float m_run = -INFINITY, l = 0.0f;
        auto s_as_float = [](uint32_t u) { return QKF8 ? __uint_as_float(u) : (float)(int32_t)u; };
        const bool tme = TIMING && h == 0 && row == 0;
        auto tss = [&](int j, int slot) { if (tme) ts(P, j, slot); };
        for (int j = P; j < nkv; j += 2) {
            const int s = j % NST, u = j >> 1;
            tss(j, 0);
            mbar_wait(kv_full(s), (j / NST) & 1);      // Delta S / delta_K landed
            mbar_wait(s_full(P), u & 1);
            tss(j, 1);
            tc_fence_after();
            const uint32_t dss = stage_addr(s) + L::ST_DS + 256 * h;
            const float* dks = reinterpret_cast<const float*>(sgen + L::ST0 + s * L::STAGE + L::ST_DK) + 4 * h;
            float2 sc2[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const float v = dqr * dks[g];
                sc2[g] = make_float2(v, v);
            }
            float sv[64];
            {
                uint32_t r0[32], r1[32];
                tmem_ld32(tS + 0, r0);
                tmem_ld32(tS + 32, r1);
                tmem_wait_ld();
                reg_dep32(r0);
                reg_dep32(r1);
                tc_fence_before();
                mbar_arrive(s_free(P));                 // S(j) in registers: QK(j+2) may overwrite it
                tss(j, 2);
#pragma unroll
                for (int c = 0; c < 64; c += 4) {
                    const uint32_t* rr = c < 32 ? r0 : r1;
                    const float4 d4 = lds128(dss + 4 * c);
                    const int g = (c % 8) / 2;
                    const float2 a = ffma2(make_float2(s_as_float(rr[c % 32]), s_as_float(rr[c % 32 + 1])),
                                           sc2[g], make_float2(d4.x, d4.y));
                    const float2 bq = ffma2(make_float2(s_as_float(rr[c % 32 + 2]), s_as_float(rr[c % 32 + 3])),
                                            sc2[g + 1], make_float2(d4.z, d4.w));
                    sv[c] = a.x;
                    sv[c + 1] = a.y;
                    sv[c + 2] = bq.x;
                    sv[c + 3] = bq.y;
                }
            }
            if (j * 128 + 128 > p.N) {                 // ragged last tile: padded keys -> -inf (C-18)
#pragma unroll
                for (int c = 0; c < 64; ++c)
                    if (j * 128 + 64 * h + c >= p.N) sv[c] = -INFINITY;
            }
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int c = 0; c < 64; c += 8) {
                mx[0] = fmax3(mx[0], sv[c], sv[c + 1]);
                mx[1] = fmax3(mx[1], sv[c + 2], sv[c + 3]);
                mx[2] = fmax3(mx[2], sv[c + 4], sv[c + 5]);
                mx[3] = fmax3(mx[3], sv[c + 6], sv[c + 7]);
            }
            // exact row max (C-10): the two halves through shared memory, M_{j-1} from the other pair
            const float mh = fmax3(mx[0], mx[1], fmaxf(mx[2], mx[3]));
            float* xmb = xm + (u & 1) * 256;
            xmb[h * 128 + row] = mh;
            tss(j, 3);
            float m_prev = -INFINITY;
            if (j > 0) {
                mbar_wait(m_full((j - 1) % NM), ((j - 1) / NM) & 1);
                m_prev = mring[((j - 1) % NM) * 128 + row];
            }
            pair_sync();
            tss(j, 4);
            const float m_new = fmax3(m_prev, mh, xmb[(1 - h) * 128 + row]);
            if (h == 0) {
                mring[(j % NM) * 128 + row] = m_new;
                mbar_arrive(m_full(j % NM));
            }
            const float alpha = (m_run == -INFINITY) ? 0.0f : ex2_approx(m_run - m_new);      // l of this pair
            const float alpha_o = (m_prev == -INFINITY) ? 0.0f : ex2_approx(m_prev - m_new);  // O (tile order)
            const float m_use = (m_new == -INFINITY) ? 0.0f : (m_new - kLog2_448);
            if (j >= 2) mbar_wait(pv_done(P), (u - 1) & 1);   // PV(j-2) has read this pair's P^ buffer
            turn_wait();
            tss(j, 5);
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
                if (c0 == 16) {                          // this half's first 32 codes are in smem
                    fence_proxy_async_smem();
                    tc_fence_before();
                    mbar_arrive(pa_full(P));
                }
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(p_full(P));
            tss(j, 6);
            if (j + 1 < nkv) turn_pass();               // the last tile keeps the turn (balanced protocol)
            l = alpha * l + ((rs2.x + rs2.y) + (rs2b.x + rs2b.y));
            m_run = m_new;
            if (CORR || j == 0) continue;                // PV(0) wrote O itself
            // ---- two-level promotion O = alpha_j O + R(j), in tile order ----
            mbar_wait(r_full, (j - 1) & 1);
            tss(j, 7);
            if (j >= 2) promo_wait();                    // the other pair's promotion of tile j-1 is in O
            tss(j, 8);
            tc_fence_after();
            const float2 a2 = make_float2(alpha_o, alpha_o);
#pragma unroll
            for (int c0 = 0; c0 < DH; c0 += 32) {
                uint32_t r[32], o[32];
                tmem_ld32(tR + c0, r);
                tmem_ld32(tO + c0, o);
                tmem_wait_ld();
                reg_dep32(r);
                reg_dep32(o);
                if (c0 + 32 == DH) {                     // R(j) in registers: PV(j+1) may overwrite it
                    tc_fence_before();
                    mbar_arrive(r_free);
                }
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                    const float2 v = ffma2(a2, make_float2(__uint_as_float(o[c]), __uint_as_float(o[c + 1])),
                                           make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])));
                    o[c] = __float_as_uint(v.x);
                    o[c + 1] = __float_as_uint(v.y);
                }
                tmem_st32(tO + c0, o);
            }
            tmem_wait_st();
            tss(j, 9);
            if (j + 1 < nkv) {
                tc_fence_before();
                promo_pass();
            }
        }
        // ---- epilogue (the pair holding the last tile, or the correction warpgroup): O / l / 448 * delta_V ----
        float* xl = reinterpret_cast<float*>(sgen + L::XL);
        xl[(2 * P + h) * 128 + row] = l;
        if (h == 0) xl[512 + P * 128 + row] = m_run;
        if constexpr (CORR) {
            named_bar_arrive(7, 640);
        } else {
            named_bar_sync(7, 512);
            if (P == ((nkv - 1) & 1)) {
                if (nkv == 1) mbar_wait(o_full, 0);      // PV(0) wrote O
                tc_fence_after();
                const float mf = m_run;                  // M of the last tile = the final row max
                float lsum = 0.0f;
#pragma unroll
                for (int PP = 0; PP < 2; ++PP) {
                    const float mp = xl[512 + PP * 128 + row];
                    const float f = (mp == -INFINITY) ? 0.0f : ex2_approx(mp - mf);
                    lsum += (xl[(2 * PP) * 128 + row] + xl[(2 * PP + 1) * 128 + row]) * f;
                }
                epilogue14<D, DH>(p, tO, 1.0f / lsum, b, hq, bhk, grow, DH * h);
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

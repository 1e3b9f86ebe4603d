// attn.cuh -- SageAttention2 attention kernel for sm_100a (Alg. 1 inner loop).
//
// One CTA = one 128-row Q block i of one (b, h_q) (b_q = 128 = smoothing block = per-thread group
// block), KV tiles of b_kv = 128 keys in ascending order (reading C-9).
//
// Warp roles (192 threads):
//   warp 0      producer: bulk-async (TMA engine) copies of the pre-swizzled tile images
//               Q^_i once; per stage K^_j, V^T_j, Delta S'_i[j], delta_K[j]  (mbarrier ring)
//   warp 1      MMA issuer (one thread):
//                 S_j  = Q^_i K^_j^T   tcgen05.mma.kind::i8, s32 accumulator in TMEM (exact)
//                 R_j  = P^_j V^_j     tcgen05.mma.kind::f8f6f4 E4M3 x E4M3, fresh fp32 accumulator
//   warps 2..5  softmax + correction, one thread per query row (TMEM lane = row):
//                 s = S_int * dQ*dK*log2e/sqrt(d) + Delta S'     (dequant + Delta S)
//                 online softmax in base 2 with an exact running max (C-10)
//                 P^ = e4m3(448 * P~) -> shared memory (SW128, A operand of the PV MMA)
//                 two-level accumulation: O(fp32, TMEM) = alpha * O + R_j
//                 epilogue O / l / 448 * delta_V -> fp16
// TMEM columns: S double buffer [0,256), R [256, 256+D), O [256+D, 256+2D).
#pragma once
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdint>

#include "ptx.cuh"

namespace sage2 {

struct AttnParams {
    const int8_t* qhat;     // [B*Hq][nT] tile images 128 x D
    const float* dq;        // [B*Hq][nT*32]
    const int8_t* khat;     // [B*Hkv][nT] tile images 128 x D
    const float* dk;        // [B*Hkv][nT*8]
    const uint8_t* vhat;    // [B*Hkv][nT] V^T tile images D x 128 (E4M3)
    const float* dv;        // [B*Hkv][D]
    const float* vmean;     // [B*Hkv][D] V_m of the optional smooth V, or null
    const float* ds;        // Delta S * log2(e)/sqrt(d): [B*Hq][nT][N_pad], or triangular (ds_tri)
    int ds_tri;             // causal workspaces: row i of a head holds only keys < 128 (i + 1)
    unsigned int* sched;    // v10 work-item counters [0] next item - grid, [1] finished CTAs (self-resetting)
    __half* out;            // [B][Hq][N][D]
    int32_t* s_dump;        // debug: [B*Hq][N_pad][N_pad] raw S_int (DUMP builds only)
    uint8_t* p_dump;        // debug: [B*Hq][N_pad][N_pad] P^ codes (DUMP builds only; may be null)
    int Hq, Hkv, N, nT;
    float qk_scale_log2;    // log2(e)/sqrt(d)
};

// Offset of Delta S row (query block) i of head bhq: full [nT][N_pad] rows, or the causal compact
// layout where row i keeps only the 128 (i + 1) keys a causal query block can see (NEXT#3).
__host__ __device__ __forceinline__ size_t ds_row(int tri, int bhq, int i, int nT) {
    const size_t Np = (size_t)nT * 128;
    return tri ? (size_t)bhq * 64 * (size_t)nT * (nT + 1) + 64 * (size_t)i * (i + 1)
               : ((size_t)bhq * nT + i) * Np;
}

constexpr int kStages = 3;
constexpr float kLog2_448 = 8.807354922057604f;   // log2(448): folds the static P scale

template <int D>
struct AttnSmem {
    static constexpr uint32_t Q = 0;
    static constexpr uint32_t TILE = 128 * D;                         // bytes of one 128 x D int8 tile
    static constexpr uint32_t STAGE = ((2 * TILE + 512 + 32) + 1023) / 1024 * 1024;
    static constexpr uint32_t ST0 = TILE;                             // stage 0
    static constexpr uint32_t P = ST0 + kStages * STAGE;              // P^ tile, 128 x 128 e4m3
    static constexpr uint32_t BAR = P + 128 * 128;
    static constexpr uint32_t NBAR = 1 + 2 * kStages + 2 + 2 + 1 + 1;
    static constexpr uint32_t TMEMPTR = BAR + 8 * NBAR;
    static constexpr uint32_t BYTES = TMEMPTR + 16;
    static constexpr uint32_t ALLOC = BYTES + 1024;                   // + alignment slack
};

template <int D, bool CAUSAL, bool DUMP>
__global__ void __launch_bounds__(192, 1) k_attn(const AttnParams p) {
    using L = AttnSmem<D>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nT = p.nT;
    const int i = CAUSAL ? (nT - 1 - (int)blockIdx.x) : (int)blockIdx.x;   // heavy causal tiles first
    const int hq = blockIdx.y, b = blockIdx.z;
    const int bhq = b * p.Hq + hq;
    const int bhk = b * p.Hkv + hq / (p.Hq / p.Hkv);
    const int nkv = CAUSAL ? (i + 1) : nT;

    // barriers
    const uint32_t bar_q = sbase + L::BAR;
    auto bar_kv_full = [&](int s) { return sbase + L::BAR + 8 * (1 + s); };
    auto bar_kv_empty = [&](int s) { return sbase + L::BAR + 8 * (1 + kStages + s); };
    auto bar_s_full = [&](int s) { return sbase + L::BAR + 8 * (1 + 2 * kStages + s); };
    auto bar_s_empty = [&](int s) { return sbase + L::BAR + 8 * (3 + 2 * kStages + s); };
    const uint32_t bar_p_full = sbase + L::BAR + 8 * (5 + 2 * kStages);
    const uint32_t bar_r_full = sbase + L::BAR + 8 * (6 + 2 * kStages);
    auto stage_addr = [&](int s) { return sbase + L::ST0 + s * L::STAGE; };

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar_kv_full(s), 1);
            mbar_init(bar_kv_empty(s), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(bar_s_full(s), 1);
            mbar_init(bar_s_empty(s), 128);
        }
        mbar_init(bar_p_full, 128);
        mbar_init(bar_r_full, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(sbase + L::TMEMPTR);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sgen + L::TMEMPTR);
    const uint32_t tS = tmem, tR = tmem + 256, tO = tmem + 256 + D;

    if (warp == 0) {
        // ===================== producer =====================
        if (lane == 0) {
            const size_t tile_bytes = (size_t)128 * D;
            mbar_arrive_expect_tx(bar_q, L::TILE);
            bulk_g2s(sbase + L::Q, p.qhat + ((size_t)bhq * nT + i) * tile_bytes, L::TILE, bar_q);
            const int Np = nT * 128;
            for (int j = 0; j < nkv; ++j) {
                const int s = j % kStages;
                if (j >= kStages) mbar_wait(bar_kv_empty(s), ((j / kStages) - 1) & 1);
                const uint32_t sa = stage_addr(s);
                mbar_arrive_expect_tx(bar_kv_full(s), 2 * L::TILE + 512 + 32);
                bulk_g2s(sa, p.khat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, bar_kv_full(s));
                bulk_g2s(sa + L::TILE, p.vhat + ((size_t)bhk * nT + j) * tile_bytes, L::TILE, bar_kv_full(s));
                bulk_g2s(sa + 2 * L::TILE, p.ds + ds_row(p.ds_tri, bhq, i, nT) + (size_t)j * 128, 512,
                         bar_kv_full(s));
                bulk_g2s(sa + 2 * L::TILE + 512, p.dk + (size_t)bhk * nT * 8 + (size_t)j * 8, 32, bar_kv_full(s));
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t IDQK = idesc_i8(128, 128);
            constexpr uint32_t IDPV = idesc_e4m3(128, D);
            const uint64_t qdesc = smem_desc<D>(sbase + L::Q);
            const uint64_t pdesc = smem_desc<128>(sbase + L::P);
            auto issue_pv = [&](int jj) {
                mbar_wait(bar_p_full, jj & 1);
                tc_fence_after();
                const uint64_t vdesc = smem_desc<128>(stage_addr(jj % kStages) + L::TILE);
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_f8f6f4(tR, pdesc + 2 * k, vdesc + 2 * k, IDPV, k > 0);
                mma_commit(bar_r_full);
                mma_commit(bar_kv_empty(jj % kStages));
            };
            mbar_wait(bar_q, 0);
            for (int j = 0; j < nkv; ++j) {
                const int s = j % kStages, sb = j & 1;
                mbar_wait(bar_kv_full(s), (j / kStages) & 1);
                if (j >= 2) mbar_wait(bar_s_empty(sb), ((j >> 1) - 1) & 1);
                tc_fence_after();
                const uint64_t kdesc = smem_desc<D>(stage_addr(s));
#pragma unroll
                for (int k = 0; k < D / 32; ++k) mma_i8(tS + sb * 128, qdesc + 2 * k, kdesc + 2 * k, IDQK, k > 0);
                mma_commit(bar_s_full(sb));
                if (j >= 1) issue_pv(j - 1);
            }
            issue_pv(nkv - 1);
        }
    } else {
        // ===================== softmax + correction (warps 2..5) =====================
        const int wq = warp & 3;                   // TMEM lane quarter this warp may access
        const int row = 32 * wq + lane;            // query row in the tile == TMEM lane
        const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
        const int grow = i * 128 + row;
        const float dqr = p.dq[((size_t)bhq * nT + i) * 32 + 8 * (row / 32) + (row % 8)] * p.qk_scale_log2;
        uint8_t* sP = sgen + L::P;
        float m = -INFINITY, l = 0.0f;
        for (int j = 0; j < nkv; ++j) {
            const int s = j % kStages, sb = j & 1;
            mbar_wait(bar_kv_full(s), (j / kStages) & 1);     // Delta S / delta_K landed
            mbar_wait(bar_s_full(sb), (j >> 1) & 1);
            tc_fence_after();
            const uint8_t* st = sgen + L::ST0 + s * L::STAGE;
            const float* dss = reinterpret_cast<const float*>(st + 2 * L::TILE);
            const float* dks = reinterpret_cast<const float*>(st + 2 * L::TILE + 512);
            float sc[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) sc[g] = dqr * dks[g];
            float sv[128];
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t raw[32];
                tmem_ld32(tS + sb * 128 + lane_off + ch * 32, raw);
                tmem_wait_ld();
                reg_dep32(raw);
                if (DUMP) {
                    int32_t* dst = p.s_dump + ((size_t)bhq * (nT * 128) + grow) * (size_t)(nT * 128) + j * 128 + ch * 32;
#pragma unroll
                    for (int k = 0; k < 32; ++k) dst[k] = (int32_t)raw[k];
                }
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const int c = ch * 32 + k;
                    sv[c] = fmaf((float)(int32_t)raw[k], sc[(c / 64) * 4 + (c % 8) / 2], dss[c]);
                }
            }
            tc_fence_before();
            mbar_arrive(bar_s_empty(sb));
            // masks: ragged end (keys >= N) and causal diagonal (key > query), C-18
            if ((CAUSAL && j == i) || (j * 128 + 128 > p.N)) {
#pragma unroll
                for (int c = 0; c < 128; ++c) {
                    const int key = j * 128 + c;
                    if (key >= p.N || (CAUSAL && key > grow)) sv[c] = -INFINITY;
                }
            }
            float tmax = -INFINITY;
#pragma unroll
            for (int c = 0; c < 128; ++c) tmax = fmaxf(tmax, sv[c]);
            const float m_new = fmaxf(m, tmax);
            const float alpha = (m == -INFINITY) ? 0.0f : ex2_approx(m - m_new);
            const float m_use = (m_new == -INFINITY) ? 0.0f : (m_new - kLog2_448);
            float rowsum = 0.0f;
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 16) {
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float p0 = ex2_approx(sv[c0 + 4 * q + 0] - m_use);
                    const float p1 = ex2_approx(sv[c0 + 4 * q + 1] - m_use);
                    const float p2 = ex2_approx(sv[c0 + 4 * q + 2] - m_use);
                    const float p3 = ex2_approx(sv[c0 + 4 * q + 3] - m_use);
                    rowsum += (p0 + p1) + (p2 + p3);
                    const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(p0, p1), __NV_SATFINITE, __NV_E4M3);
                    const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(p2, p3), __NV_SATFINITE, __NV_E4M3);
                    w[q] = lo | (hi << 16);
                }
                *reinterpret_cast<uint4*>(sP + swz_off<128>(row, c0)) = make_uint4(w[0], w[1], w[2], w[3]);
                if (DUMP && p.p_dump)
                    *reinterpret_cast<uint4*>(p.p_dump + ((size_t)bhq * (nT * 128) + grow) * (size_t)(nT * 128) +
                                              j * 128 + c0) = make_uint4(w[0], w[1], w[2], w[3]);
            }
            fence_proxy_async_smem();
            mbar_arrive(bar_p_full);
            l = alpha * l + rowsum;
            m = m_new;
            // two-level accumulation: O = alpha * O + R_j
            mbar_wait(bar_r_full, j & 1);
            tc_fence_after();
#pragma unroll
            for (int ch = 0; ch < D / 32; ++ch) {
                uint32_t r[32], o[32];
                tmem_ld32(tR + lane_off + ch * 32, r);
                if (j > 0) tmem_ld32(tO + lane_off + ch * 32, o);
                tmem_wait_ld();
                reg_dep32(r);
                if (j > 0) {
                    reg_dep32(o);
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        o[k] = __float_as_uint(fmaf(alpha, __uint_as_float(o[k]), __uint_as_float(r[k])));
                    tmem_st32(tO + lane_off + ch * 32, o);
                } else {
                    tmem_st32(tO + lane_off + ch * 32, r);
                }
            }
            tmem_wait_st();
            tc_fence_before();
        }
        // epilogue: O / l / 448 * delta_V (l carries the 448 factor: l = sum 448 P~)
        const float inv_l = 1.0f / l;
        const float* dvp = p.dv + (size_t)bhk * D;
        __half* orow = p.out + (((size_t)b * p.Hq + hq) * p.N + grow) * D;
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
            uint32_t o[32];
            tmem_ld32(tO + lane_off + ch * 32, o);
            tmem_wait_ld();
            reg_dep32(o);
            if (grow < p.N) {
                uint32_t h[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int c = ch * 32 + 2 * k;
                    const float a = __uint_as_float(o[2 * k]) * inv_l * __ldg(dvp + c);
                    const float bb = __uint_as_float(o[2 * k + 1]) * inv_l * __ldg(dvp + c + 1);
                    __half2 hv = __floats2half2_rn(a, bb);
                    h[k] = *reinterpret_cast<uint32_t*>(&hv);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    reinterpret_cast<uint4*>(orow + ch * 32)[k] = make_uint4(h[4 * k], h[4 * k + 1], h[4 * k + 2], h[4 * k + 3]);
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

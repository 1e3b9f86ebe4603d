// dsg.cuh -- Delta S = q_bar_i . gamma(K)[t]  ("Delta S = q_bar_m gamma(K)^T") on the
// 5th-generation tensor cores.
//
// Per (b, h_q) head Delta S is a GEMM: [nT query blocks] x [N_pad keys] x [d channels], with
// q_bar fp32 (exact means, C-1) and K' = fp32(K - k_bar) (O-2).  fp32 operands on a tf32 tensor
// core use the 3-pass split x = big + small (big = x rounded to tf32, small = x - big exactly):
//     q_bar . K'  ~  big_K.big_Q + big_K.small_Q + small_K.big_Q
// (dropped small.small <= 2^-22, hardware truncation of `small` <= 2^-21 relative per product),
// fp32 accumulation in TMEM.  Error <= ~2^-20 * sum_c |q_bar_c||K'_tc| -- inside the parity bound
// of DESIGN.md §5 (2e-6 * the same sum) and far inside the C-21 ambiguity margin.
//
// Roles (448 threads, one CTA per SM, persistent over work items (head, key tile, 256-block chunk)):
//   warps 0-3, 10-13  A producers (two groups, alternate atoms): thread = key row; K' = fp32(K - k_bar)
//               split into big/small and written as K-major SW128 tf32 slices (32 channels = one
//               128-byte atom per stage)
//   warps 4-7   epilogue: TMEM -> fp32 * log2(e)/sqrt(d) -> ds[bhq][i][t] (coalesced along t)
//   warp 8      TMEM allocation + MMA issuer (tcgen05.mma.kind::tf32, M = 128 keys, N <= 256)
//   warp 9      B loader: bulk-async copy of the pre-split q_bar slices written by k_q_quant
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

#include "common.cuh"
#include "prep.cuh"
#include "ptx.cuh"

namespace sage2 {

constexpr int kDsgChunk = 256;             // query blocks per MMA (N)

template <int D>
struct DsgSmem {
    static constexpr int NA = D / 32;                  // 128-byte tf32 atoms along d
    static constexpr int A_SLICE = 128 * 128;          // 128 keys x 32 fp32
    static constexpr int B_SLICE = kDsgChunk * 128;    // 256 query blocks x 32 fp32
    static constexpr int A_BIG = 0, A_SMALL = A_SLICE, B_BIG = 2 * A_SLICE, B_SMALL = 2 * A_SLICE + B_SLICE;
    static constexpr int STAGE = 2 * A_SLICE + 2 * B_SLICE;   // 96 KB
    static constexpr int NST = 2;
    static constexpr int BAR = NST * STAGE;
    static constexpr int TMEMPTR = BAR + 128;
    static constexpr int ALLOC = TMEMPTR + 16 + 1024;  // + alignment slack
    // q_bar split image per (bhq, chunk, atom): [big: 256 rows x 128 B][small: 256 rows x 128 B]
    static constexpr int QIMG = 2 * B_SLICE;
};

template <int D>
__global__ void __launch_bounds__(448, 1) k_delta_s_tc(const __half* __restrict__ K, const float* __restrict__ kbar,
                                                       const uint8_t* __restrict__ qbt, int N, int Hq, int Hkv,
                                                       int BHq, float scale_log2, float* __restrict__ ds, int tri) {
    griddep_wait_and_release();   // PDL (ptx.cuh)

    // tri (causal workspaces): only query blocks i >= kt see key tile kt; rows are stored in the
    // compact triangular layout of ds_row() and items whose whole chunk lies above the diagonal are
    // skipped by every role alike (the same `live` predicate).
    using L = DsgSmem<D>;
    constexpr int NA = L::NA;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nT = (N + 127) / 128, Np = nT * 128, nch = (nT + kDsgChunk - 1) / kDsgChunk;
    const int items = BHq * nT * nch;

    const uint32_t bar0 = sbase + L::BAR;
    auto a_full = [&](int s) { return bar0 + 8 * s; };
    auto b_full = [&](int s) { return bar0 + 8 * (2 + s); };
    auto st_empty = [&](int s) { return bar0 + 8 * (4 + s); };
    auto acc_full = [&](int s) { return bar0 + 8 * (6 + s); };
    auto acc_empty = [&](int s) { return bar0 + 8 * (8 + s); };
    auto stage = [&](int s) { return sbase + s * L::STAGE; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(a_full(s), 128);
            mbar_init(b_full(s), 1);
            mbar_init(st_empty(s), 1);
            mbar_init(acc_full(s), 1);
            mbar_init(acc_empty(s), 128);
        }
        fence_mbar_init();
    }
    if (warp == 8) tmem_alloc<512>(sbase + L::TMEMPTR);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sgen + L::TMEMPTR);

    // work item w -> (bhq, key tile kt, query-block chunk c); heads outermost so a head's q_bar
    // images stay in L2 while its key tiles stream.
    auto decode = [&](int w, int& bhq, int& kt, int& c) {
        bhq = w / (nT * nch);
        const int r = w % (nT * nch);
        kt = r / nch;
        c = r % nch;
    };
    auto chunk_rows = [&](int c) { return min(kDsgChunk, nT - c * kDsgChunk); };
    auto live = [&](int w) {
        int bhq, kt, c;
        decode(w, bhq, kt, c);
        return !tri || c * kDsgChunk + chunk_rows(c) - 1 >= kt;
    };

    if (warp < 4 || warp >= 10) {
        // ===================== A producers: K' = fp32(K - k_bar) -> tf32 big/small =====================
        // two groups of 128 threads (warps 0-3 and 10-13), thread = key row: group pg writes the atoms
        // a = pg, pg + 2, .. and therefore always stage pg (NA is even, so the global atom counter has
        // the parity of a).  One group alone was latency-bound (one dependent chain per SM
        // sub-partition): C2-4K 142 us, C2-32K 1.59 ms for this kernel.
        const int pg = warp >= 10 ? 1 : 0;
        const int t = threadIdx.x - (pg ? 320 : 0);
        constexpr int NAG = NA / 2;                        // atoms per group
        uint32_t it = 0;                                   // live items done by this CTA
        for (int w = blockIdx.x; w < items; w += gridDim.x) {
            if (!live(w)) continue;
            int bhq, kt, c;
            decode(w, bhq, kt, c);
            const int b = bhq / Hq, hk = (bhq % Hq) / (Hq / Hkv), bhk = b * Hkv + hk;
            const int key = kt * 128 + t;
            const float* kb = kbar + (size_t)bhk * D;
            uint4 raw[NAG * 4];                            // this group's channels of the key row
#pragma unroll
            for (int ai = 0; ai < NAG; ++ai)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    raw[ai * 4 + jj] =
                        key < N ? __ldg(reinterpret_cast<const uint4*>(K + ((size_t)bhk * N + key) * D) +
                                        (2 * ai + pg) * 4 + jj)
                                : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int ai = 0; ai < NAG; ++ai) {
                const int a = 2 * ai + pg;
                const uint32_t g = it * NA + a;            // the MMA issuer's atom counter
                const int s = pg;
                if (g >= 2) mbar_wait(st_empty(s), ((g >> 1) - 1) & 1);
                const uint32_t sa = stage(s);
                // this atom's 32 k_bar channels up front (vector loads): the shared stores below are
                // asm with a memory clobber, so per-channel loads would each wait out their latency
                float4 kb4[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) kb4[q] = __ldg(reinterpret_cast<const float4*>(kb + a * 32) + q);
#pragma unroll
                for (int q = 0; q < 8; ++q) {              // 16-byte chunk = 4 channels
                    const __half* h = reinterpret_cast<const __half*>(&raw[ai * 4 + q / 2]) + (q % 2) * 4;
                    const float kbq[4] = {kb4[q].x, kb4[q].y, kb4[q].z, kb4[q].w};
                    float big[4], sml[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float kp = key < N ? __fsub_rn(__half2float(h[e]), kbq[e]) : 0.0f;   // O-2
                        big[e] = tf32_big(kp);
                        sml[e] = __fsub_rn(kp, big[e]);
                    }
                    const uint32_t off = swz_off<128>(t, q * 16);
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sa + L::A_BIG + off), "f"(big[0]),
                                 "f"(big[1]), "f"(big[2]), "f"(big[3]) : "memory");
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sa + L::A_SMALL + off), "f"(sml[0]),
                                 "f"(sml[1]), "f"(sml[2]), "f"(sml[3]) : "memory");
                }
                fence_proxy_async_smem();                  // generic-proxy stores -> tcgen05.mma reads
                mbar_arrive(a_full(s));
            }
            ++it;
        }
    } else if (warp < 8) {
        // ===================== epilogue =====================
        const int t = threadIdx.x - 128;
        const uint32_t lane_off = (uint32_t)(32 * (warp - 4)) << 16;
        uint32_t m = 0;
        for (int w = blockIdx.x; w < items; w += gridDim.x) {
            if (!live(w)) continue;
            int bhq, kt, c;
            decode(w, bhq, kt, c);
            const int buf = m & 1, ni = chunk_rows(c);
            mbar_wait(acc_full(buf), (m >> 1) & 1);
            ++m;
            tc_fence_after();
            const int i0 = c * kDsgChunk;
            // row pointer advanced incrementally (row i -> i+1: N_pad floats, or 128 (i+1) in the
            // triangular layout): the epilogue warps are the throughput limit of this kernel
            float* rp = ds + ds_row(tri, bhq, i0, nT) + (size_t)kt * 128 + t;
            size_t stride = tri ? (size_t)128 * (i0 + 1) : (size_t)Np;
            for (int col0 = 0; col0 < ni; col0 += 32) {
                uint32_t r[32];
                tmem_ld32(tmem + buf * 256 + col0 + lane_off, r);
                tmem_wait_ld();
                reg_dep32(r);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (col0 + j < ni && (!tri || i0 + col0 + j >= kt)) __stcs(rp, __uint_as_float(r[j]) * scale_log2);
                    rp += stride;
                    if (tri) stride += 128;
                }
            }
            tc_fence_before();
            mbar_arrive(acc_empty(buf));
        }
    } else if (warp == 8) {
        if (lane == 0) {
            // ===================== MMA issuer =====================
            uint32_t g = 0, m = 0;
            for (int w = blockIdx.x; w < items; w += gridDim.x) {
                if (!live(w)) continue;
                int bhq, kt, c;
                decode(w, bhq, kt, c);
                const int ni = chunk_rows(c), nmma = (ni + 15) & ~15;
                const uint32_t idesc = idesc_tf32(128, nmma);
                const int buf = m & 1;
                if (m >= 2) mbar_wait(acc_empty(buf), ((m >> 1) - 1) & 1);
                ++m;
                tc_fence_after();
                const uint32_t d = tmem + buf * 256;
                for (int a = 0; a < NA; ++a, ++g) {
                    const int s = g & 1;
                    mbar_wait(a_full(s), (g >> 1) & 1);
                    mbar_wait(b_full(s), (g >> 1) & 1);
                    tc_fence_after();
                    const uint32_t sa = stage(s);
                    const uint64_t ab = smem_desc<128>(sa + L::A_BIG), as = smem_desc<128>(sa + L::A_SMALL);
                    const uint64_t bb = smem_desc<128>(sa + L::B_BIG), bs = smem_desc<128>(sa + L::B_SMALL);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {       // 8 tf32 = 32 bytes per MMA K step
                        mma_tf32(d, as + 2 * kk, bb + 2 * kk, idesc, (a | kk) != 0);
                        mma_tf32(d, ab + 2 * kk, bs + 2 * kk, idesc, 1);
                        mma_tf32(d, ab + 2 * kk, bb + 2 * kk, idesc, 1);
                    }
                    mma_commit(st_empty(s));
                }
                mma_commit(acc_full(buf));
            }
        }
    } else {
        if (lane == 0) {
            // ===================== B loader (pre-split q_bar slices) =====================
            uint32_t g = 0;
            for (int w = blockIdx.x; w < items; w += gridDim.x) {
                if (!live(w)) continue;
                int bhq, kt, c;
                decode(w, bhq, kt, c);
                const int nmma = (chunk_rows(c) + 15) & ~15;
                const uint32_t bytes = nmma * 128;
                for (int a = 0; a < NA; ++a, ++g) {
                    const int s = g & 1;
                    if (g >= 2) mbar_wait(st_empty(s), ((g >> 1) - 1) & 1);
                    const uint8_t* src = qbt + (((size_t)bhq * nch + c) * NA + a) * L::QIMG;
                    mbar_arrive_expect_tx(b_full(s), 2 * bytes);
                    bulk_g2s(stage(s) + L::B_BIG, src, bytes, b_full(s));
                    bulk_g2s(stage(s) + L::B_SMALL, src + L::B_SLICE, bytes, b_full(s));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) tmem_dealloc<512>(tmem);
}

}  // namespace sage2

// common.cuh -- what the attention kernels share: their parameter block, the Delta S row layout,
// the K/V ring depth and the shared-memory plan of a two-Q-tile CTA.  Product code (libsage2.so).
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

#ifndef SAGE2_PSPLIT
#define SAGE2_PSPLIT 1   // v8: hand P^ to the PV MMA in two halves (A/B builds: 0 = one hand-off per tile)
#endif

namespace sage2 {

struct AttnParams {
    const int8_t* qhat;     // [B*Hq][nT] tile images 128 x D
    const float* dq;        // [B*Hq][nT * groups] (32 per-thread groups per block by default)
    const int8_t* khat;     // [B*Hkv][nT] tile images 128 x D
    const float* dk;        // [B*Hkv][nT * groups] (8 per-thread groups per 128 keys by default)
    const uint8_t* vhat;    // [B*Hkv][nT] V^T tile images D x 128 (E4M3)
    const float* dv;        // [B*Hkv][D]
    const float* vmean;     // [B*Hkv][D] V_m of the optional smooth V, or null
    const float* ds;        // Delta S * log2(e)/sqrt(d): [B*Hq][nT][N_pad], or triangular (ds_tri)
    int ds_tri;             // causal workspaces: row i of a head holds only keys < 128 (i + 1)
    unsigned int* sched;    // persistent kernels: per-launch work counters [0] next item, [1] CTAs done
    __half* out;            // [B][Hq][N][D]
    int32_t* s_dump;        // debug: [B*Hq][N_pad][N_pad] raw S_int (DUMP builds only)
    uint8_t* p_dump;        // debug: [B*Hq][N_pad][N_pad] P^ codes (DUMP builds only; may be null)
    int Hq, Hkv, N, nT;
    int lpt;                // causal v8: CTAs in longest-first order over ALL heads (short sequences)
    float qk_scale_log2;    // log2(e)/sqrt(d)
};

// Offset of Delta S row (query block) i of head bhq: full [nT][N_pad] rows, or the causal compact
// layout where row i keeps only the 128 (i + 1) keys a causal query block can see (NEXT#3).
__host__ __device__ __forceinline__ size_t ds_row(int tri, int bhq, int i, int nT) {
    const size_t Np = (size_t)nT * 128;
    return tri ? (size_t)bhq * 64 * (size_t)nT * (nT + 1) + 64 * (size_t)i * (i + 1)
               : ((size_t)bhq * nT + i) * Np;
}

constexpr float kLog2_448 = 8.807354922057604f;   // log2(448): folds the static P scale

#ifndef SAGE2_KSTAGES
#define SAGE2_KSTAGES 3
#endif
constexpr int kStages2 = SAGE2_KSTAGES;   // K/V ring depth (A/B builds: -DSAGE2_KSTAGES=4)

// Shared memory of a CTA that owns two 128-row Q tiles and shares the K/V stages between them.
template <int D>
struct PairSmem {
    static constexpr uint32_t TILE = 128 * D;
    static constexpr uint32_t Q0 = 0, Q1 = TILE;
    // stage: K^ | V^T | dS tile0 (512) | dS tile1 (512) | dK (per-token granularity: up to 512)
    static constexpr uint32_t ST_K = 0, ST_V = TILE, ST_DS0 = 2 * TILE, ST_DS1 = 2 * TILE + 512,
                              ST_DK = 2 * TILE + 1024;
    static constexpr uint32_t STAGE = ((2 * TILE + 1024 + 512) + 1023) / 1024 * 1024;
    static constexpr uint32_t ST0 = 2 * TILE;
    static constexpr uint32_t P0 = ST0 + kStages2 * STAGE;           // P^ tiles, 128 x 128 e4m3 each
    static constexpr uint32_t P1 = P0 + 16384;
};

}  // namespace sage2

// probe.cuh -- hardware probes for sm_100a tensor cores:
//  * run_probe_accumulator: the paper's FP22 experiment on tcgen05.mma.kind::f8f6f4 --
//    initialise the TMEM accumulator D with chosen fp32 bit patterns, issue C = A*B + D with A = B = 0
//    (and with a single non-zero product), read C back.  Tells whether the FP8 MMA accumulator keeps
//    all 23 mantissa bits on B200 (the paper found 13 on Ada/Hopper), i.e. how much the two-level
//    accumulation of P:289-292 buys here.
//  * run_bench_mma: dense tcgen05 kind::i8 / kind::f8f6f4 throughput (M=128, N=256, K=32), all SMs.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "ptx.cuh"

namespace sage2 {

__global__ void __launch_bounds__(128, 1) k_probe_acc(const uint32_t* d_bits, const uint8_t* prod, int n,
                                                      int with_prod, uint32_t* c_out) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];
    __shared__ __align__(1024) uint8_t sB[32 * 128];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tptr;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    for (int e = t; e < 128 * 128; e += 128) sA[e] = 0;
    for (int e = t; e < 32 * 128; e += 128) sB[e] = 0;
    __syncthreads();
    const int idx = blockIdx.x * 128 + t;
    if (with_prod) {
        sA[swz_off<128>(t, 0)] = idx < n ? prod[idx] : 0;
        if (t < 32) sB[swz_off<128>(t, 0)] = 0x38;   // E4M3 1.0
    }
    if (t == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<32>(smem_u32(&tptr));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tptr;
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    uint32_t v[32];
    const uint32_t dval = idx < n ? d_bits[idx] : 0u;
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = dval;
    tmem_st32(tmem + lane_off, v);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    if (t == 0) {
        tc_fence_after();
        mma_f8f6f4(tmem, smem_desc<128>(smem_u32(sA)), smem_desc<128>(smem_u32(sB)), idesc_e4m3(128, 32), 1);
        mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    tmem_ld32(tmem + lane_off, v);
    tmem_wait_ld();
    reg_dep32(v);
    if (idx < n) c_out[idx] = v[0];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<32>(tmem);
    }
}

inline int run_probe_accumulator(const uint32_t* d_bits, const uint8_t* prod_vals, int n, uint32_t* c_zero,
                                 uint32_t* c_prod) {
    if (n == 0) return 0;
    uint32_t *dd = nullptr, *dc = nullptr;
    uint8_t* dp = nullptr;
    int rc = -4;
    if (cudaMalloc(&dd, n * 4) == cudaSuccess && cudaMalloc(&dc, n * 4) == cudaSuccess &&
        cudaMalloc(&dp, n) == cudaSuccess && cudaMemcpy(dd, d_bits, n * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
        cudaMemcpy(dp, prod_vals, n, cudaMemcpyHostToDevice) == cudaSuccess) {
        const int grid = (n + 127) / 128;
        k_probe_acc<<<grid, 128>>>(dd, dp, n, 0, dc);
        bool ok = cudaMemcpy(c_zero, dc, n * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
        k_probe_acc<<<grid, 128>>>(dd, dp, n, 1, dc);
        ok = ok && cudaMemcpy(c_prod, dc, n * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
        rc = ok ? 0 : -4;
    }
    cudaFree(dd);
    cudaFree(dc);
    cudaFree(dp);
    return rc;
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_bench_mma(int iters, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tptr;
    const int t = threadIdx.x, warp = t / 32;
    for (int e = t; e < (128 + 256) * 128 / 16; e += 128) reinterpret_cast<uint4*>(sgen)[e] = make_uint4(0, 0, 0, 0);
    if (t == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<256>(smem_u32(&tptr));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tptr;
    if (t == 0) {
        const uint64_t a = smem_desc<128>(sbase), b = smem_desc<128>(sbase + 128 * 128);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t k = it & 3;
            if (KIND == 0) mma_i8(tmem, a + 2 * k, b + 2 * k, idesc_i8(128, 256), it > 0);
            else mma_f8f6f4(tmem, a + 2 * k, b + 2 * k, idesc_e4m3(128, 256), it > 0);
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        const long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

inline int run_bench_mma(int kind, int iters, double* ops_per_s) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = (128 + 256) * 128 + 1024;
    unsigned long long* cyc = nullptr;
    if (cudaMalloc(&cyc, 8) != cudaSuccess) return -4;
    auto kern = kind == 0 ? k_bench_mma<0> : k_bench_mma<1>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -4;
    kern<<<sms, 128, smem>>>(16, cyc);   // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) return -4;
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(cyc);
    const double ops = 2.0 * 128 * 256 * 32 * (double)iters * sms;
    *ops_per_s = ops / (ms * 1e-3);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace sage2

namespace sage2 {

// ---------------------------------------------------------------------------------------------
// Unit microbenchmarks: per-SM throughputs that bound the softmax side of the kernel.
//   which 0: tcgen05.ld 32x32b.x32  (bytes / clk / SM), 8 warps, 4 loads in flight per wait
//   which 1: tcgen05.st 32x32b.x32  (bytes / clk / SM)
//   which 2: MUFU ex2.approx.f32    (results / clk / SM)
//   which 3: I2FP cvt.rn.f32.s32    (results / clk / SM)
//   which 4: FFMA2 fma.rn.f32x2     (fp32 lanes / clk / SM)
//   which 5: legacy mma.sync m16n8k64 s4.s4.s32   (ops / clk / SM)  -- the paper's Ada INT4 MMA
//   which 6: legacy mma.sync m16n8k32 s8.s8.s32   (ops / clk / SM)
// ---------------------------------------------------------------------------------------------
template <int WHICH>
__global__ void __launch_bounds__(256, 1) k_micro(int iters, unsigned long long* cyc, float* sink) {
    __shared__ uint32_t tptr;
    const int warp = threadIdx.x / 32;
    constexpr bool TM = WHICH <= 1 || WHICH == 10 || WHICH == 11;
    if (TM) {
        if (warp == 0) tmem_alloc<512>(smem_u32(&tptr));
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t col0 = (warp >> 2) * 256;
    // 16x64b: the two warps of a lane quarter take its lanes 0-15 / 16-31 (as attn11.cuh)
    const uint32_t lane16 = (uint32_t)(32 * (warp & 3) + 16 * ((warp >> 2) & 1)) << 16;
    uint32_t acc = threadIdx.x;
    float f[8];
    for (int i = 0; i < 8; ++i) f[i] = 0.001f * (threadIdx.x + i);
    int ia[8];
    for (int i = 0; i < 8; ++i) ia[i] = threadIdx.x * 3 + i;
    unsigned long long x2[4];
    for (int i = 0; i < 4; ++i) x2[i] = 0x3f8000003f800000ull + i;
    uint32_t a4[4] = {threadIdx.x, 2u, 3u, 4u}, b2[2] = {5u, threadIdx.x}, c4[4] = {0, 0, 0, 0};
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (WHICH == 0) {
            uint32_t r0[32], r1[32], r2[32], r3[32];
            tmem_ld32(tptr + lane_off + col0 + 0, r0);
            tmem_ld32(tptr + lane_off + col0 + 32, r1);
            tmem_ld32(tptr + lane_off + col0 + 64, r2);
            tmem_ld32(tptr + lane_off + col0 + 96, r3);
            tmem_wait_ld();
            reg_dep32(r0); reg_dep32(r1); reg_dep32(r2); reg_dep32(r3);
            acc ^= r0[3] ^ r1[7] ^ r2[11] ^ r3[29];
        } else if (WHICH == 1) {
            uint32_t r0[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) r0[k] = acc + k;
            tmem_st32(tptr + lane_off + col0 + 0, r0);
            tmem_st32(tptr + lane_off + col0 + 32, r0);
            tmem_st32(tptr + lane_off + col0 + 64, r0);
            tmem_st32(tptr + lane_off + col0 + 96, r0);
            tmem_wait_st();
            acc += 1;
        } else if (WHICH == 10) {
            uint32_t r0[32], r1[32], r2[32], r3[32];
            tmem_ld16x64(tptr + lane16 + 0, r0);
            tmem_ld16x64(tptr + lane16 + 64, r1);
            tmem_ld16x64(tptr + lane16 + 128, r2);
            tmem_ld16x64(tptr + lane16 + 192, r3);
            tmem_wait_ld();
            reg_dep32(r0); reg_dep32(r1); reg_dep32(r2); reg_dep32(r3);
            acc ^= r0[3] ^ r1[7] ^ r2[11] ^ r3[29];
        } else if (WHICH == 11) {
            uint32_t r0[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) r0[k] = acc + k;
            tmem_st16x64(tptr + lane16 + 0, r0);
            tmem_st16x64(tptr + lane16 + 64, r0);
            tmem_st16x64(tptr + lane16 + 128, r0);
            tmem_st16x64(tptr + lane16 + 192, r0);
            tmem_wait_st();
            acc += 1;
        } else if (WHICH == 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = ex2_approx(f[i]);
        } else if (WHICH == 3) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                f[i] += (float)ia[i];
                ia[i] += 1;
            }
        } else if (WHICH == 4) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(x2[i]));
        } else if (WHICH == 5) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                asm volatile(
                    "mma.sync.aligned.m16n8k64.row.col.s32.s4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+r"(c4[0]), "+r"(c4[1]), "+r"(c4[2]), "+r"(c4[3])
                    : "r"(a4[0]), "r"(a4[1]), "r"(a4[2]), "r"(a4[3]), "r"(b2[0]), "r"(b2[1]));
        } else if (WHICH == 7) {   // F2FP e4m3x2 pack
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                uint32_t v = __nv_cvt_float2_to_fp8x2(make_float2(f[i], f[i + 1]), __NV_SATFINITE, __NV_E4M3);
                f[i] += __uint_as_float(v & 0x3f3f);
            }
        } else if (WHICH == 8) {   // 3-input max
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float r;
                asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(f[i]), "f"(f[(i + 1) & 7]), "f"(f[(i + 2) & 7]));
                f[i] = r;
            }
        } else if (WHICH == 9) {   // the softmax element mix: I2F, FFMA2, FMNMX3, FADD2, MUFU, FADD2, F2FP
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                float2 s2 = make_float2((float)ia[i], (float)ia[i + 1]);
                unsigned long long a = *reinterpret_cast<unsigned long long*>(&s2), r;
                asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(a));
                float2 t = *reinterpret_cast<float2*>(&r);
                float mm;
                asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(mm) : "f"(t.x), "f"(t.y), "f"(f[i]));
                const float e0 = ex2_approx(t.x - mm), e1 = ex2_approx(t.y - mm);
                uint32_t v = __nv_cvt_float2_to_fp8x2(make_float2(e0, e1), __NV_SATFINITE, __NV_E4M3);
                f[i] += e0 + __uint_as_float(v & 0x3f00);
                f[i + 1] += e1;
                ia[i] += 1;
                ia[i + 1] += 3;
            }
        } else if (WHICH == 6) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                asm volatile(
                    "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+r"(c4[0]), "+r"(c4[1]), "+r"(c4[2]), "+r"(c4[3])
                    : "r"(a4[0]), "r"(a4[1]), "r"(a4[2]), "r"(a4[3]), "r"(b2[0]), "r"(b2[1]));
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
    float s = (float)acc + (float)(c4[0] ^ c4[1] ^ c4[2] ^ c4[3]);
    for (int i = 0; i < 8; ++i) s += f[i] + (float)ia[i];
    for (int i = 0; i < 4; ++i) s += (float)(x2[i] & 0xff);
    if (s == 1234.5f) sink[threadIdx.x] = s;
    if (TM) {
        tc_fence_before();
        __syncthreads();
        if (warp == 0) {
            tc_fence_after();
            tmem_dealloc<512>(tptr);
        }
    }
}

inline int run_micro(int which, int iters, double* per_clk_per_sm) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    unsigned long long* cyc = nullptr;
    float* sink = nullptr;
    if (cudaMalloc(&cyc, 8) != cudaSuccess || cudaMalloc(&sink, 1024) != cudaSuccess) return -4;
    void (*kern)(int, unsigned long long*, float*) = nullptr;
    switch (which) {
        case 7: kern = k_micro<7>; break;
        case 8: kern = k_micro<8>; break;
        case 9: kern = k_micro<9>; break;
        case 0: kern = k_micro<0>; break;
        case 1: kern = k_micro<1>; break;
        case 2: kern = k_micro<2>; break;
        case 3: kern = k_micro<3>; break;
        case 4: kern = k_micro<4>; break;
        case 5: kern = k_micro<5>; break;
        case 6: kern = k_micro<6>; break;
        case 10: kern = k_micro<10>; break;
        case 11: kern = k_micro<11>; break;
        default: return -1;
    }
    kern<<<sms, 256>>>(16, cyc, sink);
    kern<<<sms, 256>>>(iters, cyc, sink);
    unsigned long long c = 0;
    if (cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -4;
    cudaFree(cyc);
    cudaFree(sink);
    const double per_iter_per_sm =
        which >= 10 ? 8.0 * 32 * 128 * 4            // bytes, as 0 / 1
      : which >= 7 ? 256.0 * 8                      // 8 elements per thread per iteration
      : which == 0 ? 8.0 * 32 * 128 * 4            // bytes: 8 warps x 32 lanes x 128 cols x 4 B
      : which == 1 ? 8.0 * 32 * 128 * 4
      : which == 2 ? 256.0 * 8
      : which == 3 ? 256.0 * 8
      : which == 4 ? 256.0 * 8                      // 4 FFMA2 x 2 lanes
      : which == 5 ? 8.0 * 4 * 2 * 16 * 8 * 64      // 8 warps x 4 mma x ops
                   : 8.0 * 4 * 2 * 16 * 8 * 32;
    *per_clk_per_sm = per_iter_per_sm * iters / (double)c;
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace sage2

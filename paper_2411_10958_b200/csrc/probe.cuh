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

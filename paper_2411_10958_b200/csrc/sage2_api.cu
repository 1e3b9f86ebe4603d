// sage2_api.cu -- the C ABI of libsage2.so (include/sage2.h): validation, workspace layout,
// stream-ordered launches of the preprocessing kernels (prep.cuh, dsg.cuh) and the tcgen05
// attention kernels (attn8.cuh, attn12.cuh).
//
// Built twice from this one source (paper_2411_10958_b200/build.py):
//   libsage2.so      the product: only the entry points of include/sage2.h;
//   libsage2_dev.so  -DSAGE2_DEV: additionally the measurement entry points of include/sage2_dev.h
//                    (clock64 phase-trace kernel builds, the FP22 accumulator probe, tensor-core and
//                    unit microbenchmarks).  Never loaded by the product path.
#include <cuda_runtime.h>
#include <cstdlib>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/sage2.h"
#include "attn12.cuh"
#ifdef SAGE2_DEV
#include "attn14.cuh"   // experimental kernel: dev library only
#endif
#include "attn8.cuh"
#include "dsg.cuh"
#include "prep.cuh"
#ifdef SAGE2_DEV
#include "../../include/sage2_dev.h"
#include "probe.cuh"
#else
#define SAGE2_F_DEBUG_TIMING 0   // phase-trace builds exist in libsage2_dev.so only
#endif

using namespace sage2;

namespace {

constexpr int kVersion = 2;
thread_local cudaError_t g_last_cuda_error = cudaSuccess;

int cuda_rc() {   // map the launch status to a return code, remembering the CUDA error
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) g_last_cuda_error = e;
    return e == cudaSuccess ? SAGE2_OK : SAGE2_ECUDA;
}

int current_device(int* dev) {
    if (cudaGetDevice(dev) != cudaSuccess) return cuda_rc();
    return (*dev >= 0 && *dev < 64) ? SAGE2_OK : SAGE2_EUNSUPPORTED;
}

// sm_100 check, cached per device ordinal (a process may drive several GPUs).
int check_device() {
    static std::atomic<int> state[64];   // 0 unknown, 1 ok, -1 unsupported
    int dev = 0;
    int rc = current_device(&dev);
    if (rc) return rc;
    int s = state[dev].load(std::memory_order_relaxed);
    if (s == 0) {
        int major = 0, minor = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
            return cuda_rc();
        s = (major == 10 && minor == 0) ? 1 : -1;
        state[dev].store(s, std::memory_order_relaxed);
    }
    return s == 1 ? SAGE2_OK : SAGE2_EUNSUPPORTED;
}

int sm_count(int* nsm) {
    int dev = 0;
    int rc = current_device(&dev);
    if (rc) return rc;
    if (cudaDeviceGetAttribute(nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return cuda_rc();
    return SAGE2_OK;
}

// Opt a kernel into > 48 KB of dynamic shared memory.  cudaFuncSetAttribute is per device (context),
// so the "done" set is a per-kernel bitmask of device ordinals; concurrent first calls may both set
// the attribute, which is idempotent.
template <auto Kernel>
int configure_smem(uint32_t bytes) {
    static std::atomic<unsigned long long> done{0};
    int dev = 0;
    int rc = current_device(&dev);
    if (rc) return rc;
    const unsigned long long bit = 1ull << dev;
    if (done.load(std::memory_order_acquire) & bit) return SAGE2_OK;
    if (cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
        return cuda_rc();
    done.fetch_or(bit, std::memory_order_acq_rel);
    return SAGE2_OK;
}

// Shapes every kernel supports.  B*H_q and B*H_kv sit on gridDim.y of the preprocessing kernels
// (limit 65535); N <= 2^22 keeps the exact int64 means (C-1) and the Delta S offsets in range.
bool shapes_ok(int B, int Hq, int Hkv, int N, int d) {
    return B >= 1 && Hq >= 1 && Hkv >= 1 && N >= 1 && (d == 64 || d == 128) && Hq % Hkv == 0 &&
           N <= (1 << 22) && Hq <= 65535 && B <= 65535 && (long long)B * Hq <= 65535;
}

struct Layout {
    size_t off[SAGE2_WS_NREGIONS];
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

Layout make_layout(int B, int Hq, int Hkv, int N, int d, bool causal = false) {
    const size_t nT = (size_t)(N + 127) / 128, Np = nT * 128;
    const size_t BHk = (size_t)B * Hkv, BHq = (size_t)B * Hq;
    const size_t sizes[SAGE2_WS_NREGIONS - 1] = {
        BHk * d * 8,          // ksum
        BHk * d * 4,          // vmax
        BHk * d * 8,          // vsum (smooth V)
        BHk * d * 4,          // kbar
        BHk * d * 4,          // dv
        BHk * d * 4,          // vmean (smooth V)
        BHq * Np * d,         // qhat
        BHq * Np * 4,         // dq (up to one scale per token: per-token granularity)
        BHq * nT * d * 4,     // qbar
        BHk * Np * d,         // khat
        BHk * Np * 4,         // dk (up to one scale per token)
        BHk * Np * d,         // vhat
        BHq * ((nT + 255) / 256) * (size_t)(d / 32) * 65536,   // qbt (q_bar tf32 split images)
        // ds last (its size is the only one that depends on causal): full [nT][N_pad] rows, or the
        // triangular causal layout of ds_row() (common.cuh), half the bytes
        causal ? BHq * 64 * nT * (nT + 1) * 4 : BHq * nT * Np * 4,
    };
    Layout L;
    size_t o = 0;
    for (int r = 0; r < SAGE2_WS_NREGIONS - 1; ++r) {
        L.off[r] = o;
        o = align_up(o + sizes[r], 1024);
    }
    L.off[SAGE2_WS_NREGIONS - 1] = o;
    return L;
}

enum { R_KSUM, R_VMAX, R_VSUM, R_KBAR, R_DV, R_VMEAN, R_QHAT, R_DQ, R_QBAR, R_KHAT, R_DK, R_VHAT, R_QBT, R_DS, R_END };

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
bool aligned256(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 255) == 0; }

// Library-owned stream-ordered memory pool per device for the internal allocations of sage2_attn /
// sage2_attn_host (workspace, host-path device buffers) and the persistent kernels' per-launch work
// counters.  Its release threshold is unlimited, so freed blocks stay mapped for the next call instead
// of being unmapped and re-mapped (gigabytes per call): the pool retains the peak footprint of the
// calls made so far (about sage2_workspace_bytes of the largest call, plus 3 chunk buffer sets for
// sage2_attn_host) until sage2_release_memory() trims it.  torch's allocator and the process's default
// pool are not touched.
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};

cudaMemPool_t lib_pool() {
    int dev = 0;
    if (current_device(&dev)) return nullptr;
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (!g_pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        g_pools[dev] = pool;
    }
    return g_pools[dev];
}

// Library-owned side stream per device: sage2_prepare runs the Q quantizer on it, concurrently with the
// K/V statistics and quantizer on the caller's stream (fork / join through events recorded per call,
// so concurrent calls on other streams stay ordered by their own events).  Null if creation failed:
// the kernels then run in sequence on the caller's stream.
std::mutex g_side_mu;
cudaStream_t g_side[64][2] = {};

cudaStream_t side_stream(int i = 0) {
    int dev = 0;
    if (current_device(&dev)) return nullptr;
    std::lock_guard<std::mutex> g(g_side_mu);
    if (!g_side[dev][i] && cudaStreamCreateWithFlags(&g_side[dev][i], cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        g_side[dev][i] = nullptr;
    }
    return g_side[dev][i];
}

cudaError_t lib_malloc_async(void** ptr, size_t bytes, cudaStream_t st) {
    cudaMemPool_t pool = lib_pool();
    return pool ? cudaMallocFromPoolAsync(ptr, bytes, pool, st) : cudaMallocAsync(ptr, bytes, st);
}

constexpr int kKernelFlags = SAGE2_F_KERNEL_V8 | SAGE2_F_KERNEL_V12
#ifdef SAGE2_DEV
                             | SAGE2_F_KERNEL_V14
#endif
    ;

// Kernel launch with programmatic dependent launch (PDL): the kernel may start launching while the
// previous kernel on the stream drains; every kernel of the library waits for its predecessor grid
// at entry (griddep_wait_and_release, ptx.cuh), so the stream order of the data is unchanged.
#ifndef SAGE2_NO_PDL
#define SAGE2_PDL 1
#else
#define SAGE2_PDL 0
#endif
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = SAGE2_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

constexpr int kGranFlags = SAGE2_F_GRAN_BLOCK | SAGE2_F_GRAN_TOKEN | SAGE2_F_GRAN_TENSOR;
constexpr int kKnownFlags = SAGE2_F_CAUSAL | SAGE2_F_INT8 | SAGE2_F_DS_SIMT | SAGE2_F_QK_E4M3 | SAGE2_F_SMOOTH_V | SAGE2_F_ONE_LEVEL |
                            kGranFlags | kKernelFlags
#ifdef SAGE2_DEV
                            | SAGE2_F_DEBUG_TIMING
#endif
    ;

bool flags_ok(int flags) {
    if (flags & ~kKnownFlags) return false;
    const int kf = flags & kKernelFlags;
    if (kf & (kf - 1)) return false;                       // at most one kernel selector
    // granularity ablation: v8 only; v12: kind::i8 codes only
    if ((flags & kGranFlags) && (flags & SAGE2_F_KERNEL_V12)) return false;
    if ((flags & SAGE2_F_QK_E4M3) && (flags & SAGE2_F_KERNEL_V12)) return false;
    // v14: non-causal, two-level, per-thread granularity
#ifdef SAGE2_DEV
    if ((flags & SAGE2_F_KERNEL_V14) && (flags & (kGranFlags | SAGE2_F_ONE_LEVEL | SAGE2_F_CAUSAL))) return false;
#endif
    const int granf = kGranFlags;
    if ((flags & granf) & ((flags & granf) - 1)) return false;     // at most one granularity
    if ((flags & SAGE2_F_GRAN_TENSOR) && (flags & SAGE2_F_SMOOTH_V)) return false;   // shares vsum
    // single-level ablation: v8 only, per-thread granularity
    if ((flags & SAGE2_F_ONE_LEVEL) && (flags & (granf | SAGE2_F_KERNEL_V12))) return false;
    // granularity ablation (NEXT#4): v8 at d = 128 only, no carrier
    if ((flags & granf) && (flags & SAGE2_F_QK_E4M3)) return false;
    // the E4M3 carrier holds the INT4 codes only (|c| <= 7); v8 and v11 only
    if ((flags & SAGE2_F_QK_E4M3) && (flags & SAGE2_F_INT8)) return false;
    return true;
}

// Which kernel a call runs (shared by launch_prepare, launch_attention and sage2_attention_kernel: the
// kernel fixes the order of the keys inside the V^T tile images and Delta S rows).
int kernel_of(int N, int d, int flags) {
    if (flags & SAGE2_F_KERNEL_V12) return 12;
#ifdef SAGE2_DEV
    if (flags & SAGE2_F_KERNEL_V14) return 14;
#endif
    if (flags & (SAGE2_F_KERNEL_V8 | SAGE2_F_ONE_LEVEL)) return 8;
    // no selector: d = 64 non-causal -> v12 (four Q tiles per CTA, b_kv = 64: C2-32K 686 vs 665 TOPS,
    // C2-4K 643 vs 610, C2-1K 457 vs 434); v8 elsewhere.  (The persistent v10 of round 1 lost
    // everywhere once v8 handed P^ to the PV MMA in two halves -- C2-1K d=128 706 vs 735, causal 438
    // vs 502, C2-4K 1096 vs 1118 TOPS -- and was removed.)
    const bool plain = !(flags & (SAGE2_F_CAUSAL | SAGE2_F_QK_E4M3 | kGranFlags));
    if (plain && d == 64) return 12;
    return 8;
}

#ifndef SAGE2_KV_SPLIT_MAX_N
#define SAGE2_KV_SPLIT_MAX_N (1 << 30)   // k_kv_quant as concurrent K / V launches (every N: DESIGN.md section 9)
#endif

template <int D>
int launch_prepare(const __half* q, const __half* k, const __half* v, int B, int Hq, int Hkv, int N, int flags,
                   uint8_t* ws, const Layout& L, cudaStream_t st) {
    const int nT = (N + 127) / 128;
    const bool causal = (flags & SAGE2_F_CAUSAL) != 0;     // Delta S in the triangular layout
    const int qk_max = (flags & SAGE2_F_INT8) ? 127 : 7;
    const int smooth_q = (flags & SAGE2_F_INT8) ? 0 : 1;   // SageAttn2-8b: no Q smoothing
    const size_t BHk = (size_t)B * Hkv, BHq = (size_t)B * Hq;
    if (cudaMemsetAsync(ws + L.off[R_KSUM], 0, L.off[R_KBAR] - L.off[R_KSUM], st) != cudaSuccess) return cuda_rc();
    auto* ksum = reinterpret_cast<unsigned long long*>(ws + L.off[R_KSUM]);
    auto* vmax = reinterpret_cast<unsigned int*>(ws + L.off[R_VMAX]);
    const bool smv = (flags & SAGE2_F_SMOOTH_V) != 0;
    auto* vsum = reinterpret_cast<unsigned long long*>(ws + L.off[R_VSUM]);
    auto* vmean = reinterpret_cast<float*>(ws + L.off[R_VMEAN]);
    const int gran = (flags & SAGE2_F_GRAN_TENSOR) ? 3 : (flags & SAGE2_F_GRAN_TOKEN) ? 2 : (flags & SAGE2_F_GRAN_BLOCK) ? 1 : 0;
    auto kvq = gran == 3 ? k_kv_quant<D, 3> : gran == 2 ? k_kv_quant<D, 2> : gran == 1 ? k_kv_quant<D, 1> : k_kv_quant<D, 0>;
    auto qq = gran == 3 ? k_q_quant<D, 3> : gran == 2 ? k_q_quant<D, 2> : gran == 1 ? k_q_quant<D, 1> : k_q_quant<D, 0>;
    // per-tensor granularity: the heads' max |K'| / max |gamma(Q_i)| first (GRAN 4 passes, atomics
    // into the zeroed vsum region, unused without smooth V)
    auto* ktmax = reinterpret_cast<unsigned int*>(vsum);
    auto* qtmax = ktmax + BHk;
    const int e4 = (flags & SAGE2_F_QK_E4M3) ? 1 : 0;
    auto* khat_p = reinterpret_cast<int8_t*>(ws + L.off[R_KHAT]);
    auto* dk_p = reinterpret_cast<float*>(ws + L.off[R_DK]);
    auto* kbar_p = reinterpret_cast<float*>(ws + L.off[R_KBAR]);
    auto* dv_p = reinterpret_cast<float*>(ws + L.off[R_DV]);
    auto* qhat_p = reinterpret_cast<int8_t*>(ws + L.off[R_QHAT]);
    auto* dq_p = reinterpret_cast<float*>(ws + L.off[R_DQ]);
    auto* qbar_p = reinterpret_cast<float*>(ws + L.off[R_QBAR]);
    // library side stream for the Q quantizer and Delta S (below); none for per-tensor granularity
    cudaStream_t side = gran == 3 ? nullptr : side_stream();
    // Delta S (needs q_bar and the K column sums, not k_kv_quant's outputs): the persistent tf32
    // tensor-core GEMM, except for short sequences (N <= 2048) where its per-item pipeline overhead
    // loses to the SIMT kernel (1K: 40 vs 28 us).  Both are pinned to the oracle by the same bound
    // (DESIGN.md section 5); the SIMT kernel takes k_bar from the exact sums itself (it may run before
    // k_kv_quant), the GEMM the k_bar k_kv_quant wrote.
    const float scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
    auto launch_ds = [&](cudaStream_t s) -> int {
        if ((flags & SAGE2_F_DS_SIMT) || N <= 2048) {
            // Q blocks per pass sized to nT (8 / 16 accumulators per thread; more passes beyond 16 blocks)
            auto kds = nT <= 8 ? k_delta_s<D, 8> : k_delta_s<D, 16>;
            launch_k(kds, dim3(nT, BHq), dim3(128), 0, s, k, ksum, reinterpret_cast<const float*>(ws + L.off[R_QBAR]), N, Hq,
                     Hkv, scale_log2, reinterpret_cast<float*>(ws + L.off[R_DS]), causal ? 1 : 0);
            return SAGE2_OK;
        }
        int nsm = 0, rc2 = sm_count(&nsm);
        if (rc2) return rc2;
        if ((rc2 = configure_smem<k_delta_s_tc<D>>(DsgSmem<D>::ALLOC))) return rc2;
        const long long items = (long long)BHq * nT * ((nT + 255) / 256);
        const int grid = (int)std::min<long long>(items, nsm);
        // (after k_kv_quant: it reads the k_bar k_kv_quant wrote)
        launch_k(k_delta_s_tc<D>, dim3(grid), dim3(448), DsgSmem<D>::ALLOC, s, k, reinterpret_cast<const float*>(kbar_p),
                 ws + L.off[R_QBT], N, Hq, Hkv, (int)BHq, scale_log2, reinterpret_cast<float*>(ws + L.off[R_DS]),
                 causal ? 1 : 0);
        return SAGE2_OK;
    };
    // Side stream (short sequences gain most: every kernel here is latency-bound at 1K-2K): the Q
    // quantizer forked after the memset, then -- once k_kv_stats has the column sums, and for N <= 2048
    // -- Delta S, concurrent with k_kv_stats / k_kv_quant on `st`; joined before Delta S otherwise.
    cudaEvent_t ev_fork = nullptr, ev_stats = nullptr, ev_join = nullptr;
    if (side && (cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                 cudaEventCreateWithFlags(&ev_stats, cudaEventDisableTiming) != cudaSuccess ||
                 cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess ||
                 cudaEventRecord(ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(side, ev_fork, 0) != cudaSuccess)) {
        cudaGetLastError();
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_stats) cudaEventDestroy(ev_stats);
        if (ev_join) cudaEventDestroy(ev_join);
        ev_fork = ev_stats = ev_join = nullptr;
        side = nullptr;
    }
    if (side) launch_k(qq, dim3(nT, BHq), dim3(256), 0, side, q, N, qk_max, e4, smooth_q, qhat_p, dq_p, qbar_p, ws + L.off[R_QBT], qtmax);
    // rows per k_kv_stats CTA: 512 for long sequences; fewer for short ones so the grid still has
    // ~4 CTAs per SM (1K tokens: 22 -> ~10 us).  fp64 in-CTA sums stay exact up to 8192 rows.
    int rows_per_cta = 512;
    while (rows_per_cta > 64 && (long long)((N + rows_per_cta - 1) / rows_per_cta) * (long long)BHk < 4LL * 148)
        rows_per_cta /= 2;
    const dim3 sgrid((N + rows_per_cta - 1) / rows_per_cta, BHk);
    if (smv) {
        launch_k(k_kv_stats<D, true>, sgrid, dim3(256), 0, st, k, v, N, rows_per_cta, ksum, vmax, vsum);
        launch_k(k_v_absmax_smooth<D>, sgrid, dim3(256), 0, st, v, N, rows_per_cta, vsum, vmax, vmean);
    } else {
        launch_k(k_kv_stats<D, false>, sgrid, dim3(256), 0, st, k, v, N, rows_per_cta, ksum, vmax, vsum);
    }
    // Delta S joins the side stream only in its SIMT form (N <= 2048: C2-1K prepare 92 -> 83 us); the
    // persistent tensor-core GEMM (one 197 KB CTA per SM) loses its SMs to k_kv_quant when the two run
    // together (4K 343 -> 352 us, 32K 3.24 -> 3.44 ms), so it runs after the join
    const bool ds_side = side && ((flags & SAGE2_F_DS_SIMT) || N <= 2048);
    // k_kv_quant split into its K and V halves on two streams (a second side stream takes the K half):
    // each CTA's serial load / reduce / quantize phases halved (C2-1K 83 -> 81 us, 4K 343 -> 329,
    // 32K 3.20 -> 3.08 ms)
    cudaStream_t side2 = side && N <= SAGE2_KV_SPLIT_MAX_N ? side_stream(1) : nullptr;
    cudaEvent_t ev_join2 = nullptr;
    if (side2 && cudaEventCreateWithFlags(&ev_join2, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        ev_join2 = nullptr;
        side2 = nullptr;
    }
    // the K column sums are complete here: both side launches below wait for this event
    if ((ds_side || side2) && cudaEventRecord(ev_stats, st) != cudaSuccess) return cuda_rc();
    if (side) {
        if (ds_side) {
            if (cudaStreamWaitEvent(side, ev_stats, 0) != cudaSuccess) return cuda_rc();
            int rc2 = launch_ds(side);
            if (rc2) return rc2;
        }
        if (cudaEventRecord(ev_join, side) != cudaSuccess) return cuda_rc();
    }
    if (side2) {
        if (cudaStreamWaitEvent(side2, ev_stats, 0) != cudaSuccess) return cuda_rc();
        auto kq = gran == 2 ? k_kv_quant<D, 2, 1> : gran == 1 ? k_kv_quant<D, 1, 1> : k_kv_quant<D, 0, 1>;
        launch_k(kq, dim3(nT, BHk), dim3(256), 0, side2, k, v, N, qk_max, e4, ksum, vmax, khat_p, dk_p, ws + L.off[R_VHAT],
                 kbar_p, dv_p, smv ? vmean : nullptr, ktmax);
        if (cudaEventRecord(ev_join2, side2) != cudaSuccess) return cuda_rc();
        auto vq = gran == 2 ? k_kv_quant<D, 2, 2> : gran == 1 ? k_kv_quant<D, 1, 2> : k_kv_quant<D, 0, 2>;
        launch_k(vq, dim3(nT, BHk), dim3(256), 0, st, k, v, N, qk_max, e4, ksum, vmax, khat_p, dk_p, ws + L.off[R_VHAT],
                 kbar_p, dv_p, smv ? vmean : nullptr, ktmax);
        const bool ok = cudaStreamWaitEvent(st, ev_join2, 0) == cudaSuccess;
        cudaEventDestroy(ev_join2);
        if (!ok) return cuda_rc();
    }
    if (gran == 3) {
        launch_k(k_kv_quant<D, 4>, dim3(nT, BHk), dim3(256), 0, st, k, v, N, qk_max, e4, ksum, vmax, khat_p, dk_p, ws + L.off[R_VHAT],
                                                        kbar_p, dv_p, nullptr, ktmax);
        launch_k(k_q_quant<D, 4>, dim3(nT, BHq), dim3(256), 0, st, q, N, qk_max, e4, smooth_q, qhat_p, dq_p, qbar_p, ws + L.off[R_QBT],
                                                       qtmax);
    }
    if (!side2)
        launch_k(kvq, dim3(nT, BHk), dim3(256), 0, st, k, v, N, qk_max, e4, ksum, vmax, khat_p, dk_p, ws + L.off[R_VHAT], kbar_p,
                 dv_p, smv ? vmean : nullptr, ktmax);
    if (side) {
        const bool ok = cudaStreamWaitEvent(st, ev_join, 0) == cudaSuccess;
        cudaEventDestroy(ev_fork);
        cudaEventDestroy(ev_stats);
        cudaEventDestroy(ev_join);
        if (!ok) return cuda_rc();
        if (!ds_side) {
            int rc2 = launch_ds(st);
            if (rc2) return rc2;
        }
        return cuda_rc();
    }
    launch_k(qq, dim3(nT, BHq), dim3(256), 0, st, q, N, qk_max, e4, smooth_q, qhat_p, dq_p, qbar_p, ws + L.off[R_QBT], qtmax);
    int rc3 = launch_ds(st);
    if (rc3) return rc3;
    return cuda_rc();
}

template <int D, bool CAUSAL, bool DUMP, bool QKF8 = false, bool TIMING = false, int GRAN = 0, bool ONE = false, int NT = 2>
int launch_attn8_t(const AttnParams& p, int B, cudaStream_t st) {
    constexpr uint32_t smem = Attn8Smem<D, NT>::ALLOC;
    int rc = configure_smem<k_attn8<D, CAUSAL, DUMP, QKF8, TIMING, GRAN, ONE, NT>>(smem);
    if (rc) return rc;
    launch_k(k_attn8<D, CAUSAL, DUMP, QKF8, TIMING, GRAN, ONE, NT>, dim3(NT == 2 ? (p.nT + 1) / 2 : p.nT, p.Hq, B),
             dim3(NT == 2 ? 640 : 384), smem, st, p);
    return cuda_rc();
}

#ifndef SAGE2_NT1_MAX_TILES
#define SAGE2_NT1_MAX_TILES 8   // v8 in its one-Q-tile form (two CTAs per SM) up to N = 1K
#endif

template <bool CAUSAL, bool DUMP, bool TIMING = false>
int launch_attn12_t(const AttnParams& p, int B, cudaStream_t st) {
    constexpr uint32_t smem = Attn12Smem::ALLOC;
    int rc = configure_smem<k_attn12<CAUSAL, DUMP, TIMING>>(smem);
    if (rc) return rc;
    launch_k(k_attn12<CAUSAL, DUMP, TIMING>, dim3((p.nT + 3) / 4, p.Hq, B), dim3(640), smem, st, p);
    return cuda_rc();
}

#ifdef SAGE2_DEV
#ifndef SAGE2_V14_CORR
#define SAGE2_V14_CORR 1   // correction warpgroup (16-column chunks): 1132 vs 1086 TOPS in-pair
#endif
template <int D, bool QKF8, bool TIMING = false>
int launch_attn14_t(const AttnParams& p, int B, cudaStream_t st) {
    constexpr bool CORR = SAGE2_V14_CORR != 0;
    constexpr uint32_t smem = Attn14Smem<D>::ALLOC;
    int rc = configure_smem<k_attn14<D, QKF8, TIMING, CORR>>(smem);
    if (rc) return rc;
    launch_k(k_attn14<D, QKF8, TIMING, CORR>, dim3(p.nT, p.Hq, B), dim3(CORR ? 768 : 640), smem, st, p);
    return cuda_rc();
}
#endif

template <int D>
int launch_attention_d(const AttnParams& p, int B, int flags, bool dump, cudaStream_t st) {
    const bool causal = (flags & SAGE2_F_CAUSAL) != 0;
    const bool f8 = (flags & SAGE2_F_QK_E4M3) != 0;
    const int kern = kernel_of(p.N, D, flags);
#ifdef SAGE2_DEV
    if (flags & SAGE2_F_DEBUG_TIMING) {   // clock64 phase stamps (non-causal) into s_dump
        if constexpr (D == 64) {
            if (kern == 12) return launch_attn12_t<false, false, true>(p, B, st);
        }
        if (kern == 14) return launch_attn14_t<D, false, true>(p, B, st);   // (inside #ifdef SAGE2_DEV)
        return launch_attn8_t<D, false, false, false, true>(p, B, st);
    }
#endif
#ifdef SAGE2_DEV
    if (kern == 14 && !dump) {   // one Q tile per CTA, S double-buffered (DUMP builds: v8)
        return f8 ? launch_attn14_t<D, true>(p, B, st) : launch_attn14_t<D, false>(p, B, st);
    }
#endif
    if (kern == 12) {     // four Q tiles per CTA, b_kv = 64: head dim 64 only
        if constexpr (D != 64) {
            return SAGE2_EINVAL;
        } else {
            if (dump) return launch_attn12_t<false, true>(p, B, st);
            return causal ? launch_attn12_t<true, false>(p, B, st) : launch_attn12_t<false, false>(p, B, st);
        }
    }
    if (flags & SAGE2_F_ONE_LEVEL) {   // single-level accumulation ablation (v8 only)
        if (dump) return f8 ? launch_attn8_t<D, false, true, true, false, 0, true>(p, B, st)
                            : launch_attn8_t<D, false, true, false, false, 0, true>(p, B, st);
        if (f8) return causal ? launch_attn8_t<D, true, false, true, false, 0, true>(p, B, st)
                              : launch_attn8_t<D, false, false, true, false, 0, true>(p, B, st);
        return causal ? launch_attn8_t<D, true, false, false, false, 0, true>(p, B, st)
                      : launch_attn8_t<D, false, false, false, false, 0, true>(p, B, st);
    }
    if (flags & kGranFlags) {   // NEXT#4 granularity ablation (d = 128); per-tensor runs the per-block kernel
        if constexpr (D != 128) {
            return SAGE2_EINVAL;
        } else {
            if (dump) return SAGE2_EINVAL;
            if (flags & SAGE2_F_GRAN_TOKEN)
                return causal ? launch_attn8_t<D, true, false, false, false, 2>(p, B, st)
                              : launch_attn8_t<D, false, false, false, false, 2>(p, B, st);
            return causal ? launch_attn8_t<D, true, false, false, false, 1>(p, B, st)
                          : launch_attn8_t<D, false, false, false, false, 1>(p, B, st);
        }
    }
    if (dump) return f8 ? launch_attn8_t<D, false, true, true>(p, B, st) : launch_attn8_t<D, false, true>(p, B, st);
    if (f8) return causal ? launch_attn8_t<D, true, false, true>(p, B, st) : launch_attn8_t<D, false, false, true>(p, B, st);
    if (p.nT <= SAGE2_NT1_MAX_TILES)   // short sequences: one Q tile per CTA, two CTAs per SM
        return causal ? launch_attn8_t<D, true, false, false, false, 0, false, 1>(p, B, st)
                      : launch_attn8_t<D, false, false, false, false, 0, false, 1>(p, B, st);
    return causal ? launch_attn8_t<D, true, false>(p, B, st) : launch_attn8_t<D, false, false>(p, B, st);
}

int launch_attention(void* out, int32_t* s_dump, uint8_t* p_dump, int B, int Hq, int Hkv, int N, int d, int flags,
                     const uint8_t* ws, const Layout& L, cudaStream_t st) {
    AttnParams p;
    p.qhat = reinterpret_cast<const int8_t*>(ws + L.off[R_QHAT]);
    p.dq = reinterpret_cast<const float*>(ws + L.off[R_DQ]);
    p.khat = reinterpret_cast<const int8_t*>(ws + L.off[R_KHAT]);
    p.dk = reinterpret_cast<const float*>(ws + L.off[R_DK]);
    p.vhat = ws + L.off[R_VHAT];
    p.dv = reinterpret_cast<const float*>(ws + L.off[R_DV]);
    p.vmean = (flags & SAGE2_F_SMOOTH_V) ? reinterpret_cast<const float*>(ws + L.off[R_VMEAN]) : nullptr;
    p.ds = reinterpret_cast<const float*>(ws + L.off[R_DS]);
    p.sched = nullptr;
    p.ds_tri = (flags & SAGE2_F_CAUSAL) ? 1 : 0;
    p.out = reinterpret_cast<__half*>(out);
    p.s_dump = s_dump;
    p.p_dump = p_dump;
    p.Hq = Hq;
    p.Hkv = Hkv;
    p.N = N;
    p.nT = (N + 127) / 128;
    // causal CTAs longest-first over all heads up to N = 8K (C2-1K d=128 459 -> 504, 4K 890 -> 939, 8K
    // 1040 -> 1068 TOPS); head-major beyond (16K-100K d=128 lose 3-8% to L2 misses otherwise)
    p.lpt = p.nT <= 64;
    p.qk_scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
    const bool dump = s_dump != nullptr && !(flags & SAGE2_F_DEBUG_TIMING);
    return d == 64 ? launch_attention_d<64>(p, B, flags, dump, st) : launch_attention_d<128>(p, B, flags, dump, st);
}

int validate(const void* q, const void* k, const void* v, const void* out, int B, int Hq, int Hkv, int N, int d) {
    if (!shapes_ok(B, Hq, Hkv, N, d)) return SAGE2_EINVAL;
    if (!q || !k || !v || !out) return SAGE2_EINVAL;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out)) return SAGE2_EINVAL;
    return SAGE2_OK;
}

}  // namespace

extern "C" {

int sage2_version(void) { return kVersion; }

const char* sage2_last_cuda_error(void) { return cudaGetErrorString(g_last_cuda_error); }

const char* sage2_strerror(int code) {
    switch (code) {
        case SAGE2_OK: return "ok";
        case SAGE2_EINVAL: return "invalid argument (shape, flags, pointer, alignment or workspace size)";
        case SAGE2_EUNSUPPORTED: return "unsupported device: libsage2 requires sm_100 (B200)";
        case SAGE2_ENOMEM: return "workspace allocation failed";
        case SAGE2_ECUDA: return "CUDA error";
        default: return "unknown error";
    }
}

size_t sage2_workspace_bytes(int B, int H_q, int H_kv, int N, int d, int causal) {
    if (!shapes_ok(B, H_q, H_kv, N, d)) return 0;
    return make_layout(B, H_q, H_kv, N, d, causal != 0).off[R_END];
}

int sage2_workspace_layout(int B, int H_q, int H_kv, int N, int d, size_t* offsets) {
    if (!shapes_ok(B, H_q, H_kv, N, d) || !offsets) return SAGE2_EINVAL;
    Layout L = make_layout(B, H_q, H_kv, N, d);
    std::memcpy(offsets, L.off, sizeof(L.off));
    return SAGE2_OK;
}

int sage2_prepare(const void* q, const void* k, const void* v, int B, int H_q, int H_kv, int N, int d, int flags,
                  void* workspace, size_t ws_bytes, void* stream) {
    int rc = check_device();
    if (rc) return rc;
    if (!shapes_ok(B, H_q, H_kv, N, d) || !q || !k || !v || !workspace || !flags_ok(flags)) return SAGE2_EINVAL;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned256(workspace)) return SAGE2_EINVAL;
    Layout L = make_layout(B, H_q, H_kv, N, d, (flags & SAGE2_F_CAUSAL) != 0);
    if (ws_bytes < L.off[R_END]) return SAGE2_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    auto* ws = reinterpret_cast<uint8_t*>(workspace);
    auto* hq = reinterpret_cast<const __half*>(q);
    auto* hk = reinterpret_cast<const __half*>(k);
    auto* hv = reinterpret_cast<const __half*>(v);
    return d == 64 ? launch_prepare<64>(hq, hk, hv, B, H_q, H_kv, N, flags, ws, L, st)
                   : launch_prepare<128>(hq, hk, hv, B, H_q, H_kv, N, flags, ws, L, st);
}

int sage2_attention_kernel(int N, int d, int flags) { return kernel_of(N, d, flags); }

int sage2_attention(void* out, int B, int H_q, int H_kv, int N, int d, int flags, const void* workspace,
                    size_t ws_bytes, void* stream) {
    int rc = check_device();
    if (rc) return rc;
    if (!shapes_ok(B, H_q, H_kv, N, d) || !out || !workspace || !aligned16(out) || !aligned256(workspace) ||
        !flags_ok(flags))
        return SAGE2_EINVAL;
    Layout L = make_layout(B, H_q, H_kv, N, d, (flags & SAGE2_F_CAUSAL) != 0);
    if (ws_bytes < L.off[R_END]) return SAGE2_EINVAL;
    return launch_attention(out, nullptr, nullptr, B, H_q, H_kv, N, d, flags, reinterpret_cast<const uint8_t*>(workspace), L,
                            reinterpret_cast<cudaStream_t>(stream));
}

int sage2_debug_qk_int32(void* out, int32_t* s_int, uint8_t* p_hat, int B, int H_q, int H_kv, int N, int d,
                         int flags, const void* workspace, size_t ws_bytes, void* stream) {
    int rc = check_device();
    if (rc) return rc;
    if (!shapes_ok(B, H_q, H_kv, N, d) || !out || !s_int || !workspace || !aligned16(out) || !aligned256(workspace) ||
        !flags_ok(flags) || (flags & kGranFlags))
        return SAGE2_EINVAL;
    Layout L = make_layout(B, H_q, H_kv, N, d);
    if (ws_bytes < L.off[R_END]) return SAGE2_EINVAL;
    return launch_attention(out, s_int, p_hat, B, H_q, H_kv, N, d, flags & ~SAGE2_F_CAUSAL,
                            reinterpret_cast<const uint8_t*>(workspace), L, reinterpret_cast<cudaStream_t>(stream));
}

int sage2_attn_ex(const void* q, const void* k, const void* v, void* out, int B, int H_q, int H_kv, int N, int d,
                  int flags, void* workspace, size_t ws_bytes, void* stream) {
    int rc = check_device();
    if (rc) return rc;
    rc = validate(q, k, v, out, B, H_q, H_kv, N, d);
    if (rc) return rc;
    rc = sage2_prepare(q, k, v, B, H_q, H_kv, N, d, flags, workspace, ws_bytes, stream);
    if (rc) return rc;
    return sage2_attention(out, B, H_q, H_kv, N, d, flags, workspace, ws_bytes, stream);
}

int sage2_attn_ws(const void* q, const void* k, const void* v, void* out, int B, int H_q, int H_kv, int N, int d,
                  int causal, void* workspace, size_t ws_bytes, void* stream) {
    return sage2_attn_ex(q, k, v, out, B, H_q, H_kv, N, d, causal ? SAGE2_F_CAUSAL : 0, workspace, ws_bytes, stream);
}

int sage2_attn(const void* q, const void* k, const void* v, void* out, int B, int H_q, int H_kv, int N, int d,
               int causal, void* stream) {
    int rc = check_device();
    if (rc) return rc;
    rc = validate(q, k, v, out, B, H_q, H_kv, N, d);
    if (rc) return rc;
    const size_t bytes = sage2_workspace_bytes(B, H_q, H_kv, N, d, causal);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    void* ws = nullptr;
    if (lib_malloc_async(&ws, bytes, st) != cudaSuccess) {
        cudaGetLastError();
        return SAGE2_ENOMEM;
    }
    rc = sage2_attn_ws(q, k, v, out, B, H_q, H_kv, N, d, causal, ws, bytes, stream);
    if (cudaFreeAsync(ws, st) != cudaSuccess && rc == SAGE2_OK) rc = cuda_rc();
    return rc;
}

int sage2_attn_host(const void* q_host, const void* k_host, const void* v_host, void* out_host, int B, int H_q,
                    int H_kv, int N, int d, int causal, void* stream) {
    // Pipelined over chunks of (b, h_kv) units (one KV head + its H_q/H_kv query heads; contiguous
    // in every [B, H, N, d] tensor and independent): chunk c runs H2D ->
    // prepare -> attention -> D2H on internal stream c % 3, so the copy engines of one chunk overlap
    // the kernels of the others.  Three device buffer sets (inputs, output, workspace) are reused.
    int rc = check_device();
    if (rc) return rc;
    if (!shapes_ok(B, H_q, H_kv, N, d) || !q_host || !k_host || !v_host || !out_host) return SAGE2_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int grp = H_q / H_kv, units = B * H_kv;
    const int nch0 = units < 16 ? units : 16;
    const int U = (units + nch0 - 1) / nch0;               // units per full chunk
    // chunk sizes: 1, 2, 4, ... < U, then full chunks, then ... 4, 2, 1 -- the first H2D and the
    // last kernels + D2H are the parts the pipeline cannot overlap, so they are kept small
    std::vector<int> ramp, csz;
    int ramp_sum = 0;
    for (int s = 1; s < U; s *= 2) {
        ramp.push_back(s);
        ramp_sum += s;
    }
    if (units >= 2 * ramp_sum + U) {
        csz = ramp;
        const int mid = units - 2 * ramp_sum;
        for (int k = 0; k < mid / U; ++k) csz.push_back(U);
        if (mid % U) csz.push_back(mid % U);
        csz.insert(csz.end(), ramp.rbegin(), ramp.rend());
    } else {
        for (int u = 0; u < units; u += U) csz.push_back(units - u < U ? units - u : U);
    }
    const int nch = (int)csz.size();
    const size_t qu = (size_t)grp * N * d * 2, ku = (size_t)N * d * 2;   // bytes per unit
    const size_t wsb = sage2_workspace_bytes(1, U * grp, U, N, d, causal);
    // three streams / buffer sets in flight: chunk c's kernels, chunk c+1's H2D and chunk c-1's D2H
    // overlap (measured e2e at C2-32K: 2 sets 75.4 ms, 3 sets 66.3 ms, 4 sets 66.3 ms)
    constexpr int NB = 3;
    const int nbuf = nch < NB ? nch : NB;
    void* buf[NB][5] = {{nullptr}};
    cudaStream_t ss[NB] = {};
    cudaEvent_t ev_start = nullptr, ev_done[NB] = {};
    auto bad = [&]() { if (rc == SAGE2_OK) rc = cuda_rc(); };
    for (int i = 0; i < nbuf && rc == SAGE2_OK; ++i) {
        if (cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming) != cudaSuccess)
            bad();
        const size_t sz[5] = {U * qu, U * ku, U * ku, U * qu, wsb};
        for (int r = 0; r < 5 && rc == SAGE2_OK; ++r)
            if (lib_malloc_async(&buf[i][r], sz[r], st) != cudaSuccess) {
                cudaGetLastError();
                rc = SAGE2_ENOMEM;
            }
    }
    if (rc == SAGE2_OK && (cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) != cudaSuccess ||
                           cudaEventRecord(ev_start, st) != cudaSuccess))
        bad();
    for (int i = 0; i < nbuf && rc == SAGE2_OK; ++i)
        if (cudaStreamWaitEvent(ss[i], ev_start, 0) != cudaSuccess) bad();   // allocations are ready
    const int flags = causal ? SAGE2_F_CAUSAL : 0;
    for (int c = 0, u0 = 0; c < nch && rc == SAGE2_OK; u0 += csz[c], ++c) {
        const int i = c % NB, nu = csz[c];
        cudaStream_t s = ss[i];
        const char* qh = static_cast<const char*>(q_host) + (size_t)u0 * qu;
        const char* kh = static_cast<const char*>(k_host) + (size_t)u0 * ku;
        const char* vh = static_cast<const char*>(v_host) + (size_t)u0 * ku;
        char* oh = static_cast<char*>(out_host) + (size_t)u0 * qu;
        if (cudaMemcpyAsync(buf[i][0], qh, nu * qu, cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(buf[i][1], kh, nu * ku, cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(buf[i][2], vh, nu * ku, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            bad();
            break;
        }
        rc = sage2_attn_ex(buf[i][0], buf[i][1], buf[i][2], buf[i][3], 1, nu * grp, nu, N, d, flags, buf[i][4],
                           wsb, s);
        if (rc == SAGE2_OK && cudaMemcpyAsync(oh, buf[i][3], nu * qu, cudaMemcpyDeviceToHost, s) != cudaSuccess) bad();
    }
    for (int i = 0; i < nbuf; ++i) {
        if (ss[i] && ev_done[i]) {
            cudaEventRecord(ev_done[i], ss[i]);
            cudaStreamWaitEvent(st, ev_done[i], 0);        // the caller's stream sees every chunk done
        }
        for (int r = 0; r < 5; ++r)
            if (buf[i][r]) cudaFreeAsync(buf[i][r], st);
    }
    for (int i = 0; i < nbuf; ++i) {
        if (ev_done[i]) cudaEventDestroy(ev_done[i]);
        if (ss[i]) cudaStreamDestroy(ss[i]);               // released once its work completes
    }
    if (ev_start) cudaEventDestroy(ev_start);
    return rc;
}

int sage2_release_memory(void) {
    int rc = check_device();
    if (rc) return rc;
    int dev = 0;
    if ((rc = current_device(&dev))) return rc;
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (!g_pools[dev]) return SAGE2_OK;
    if (cudaDeviceSynchronize() != cudaSuccess) return cuda_rc();
    if (cudaMemPoolTrimTo(g_pools[dev], 0) != cudaSuccess) return cuda_rc();
    return SAGE2_OK;
}

#ifdef SAGE2_DEV
int sage2_dev_trace(void* out, uint64_t* stamps, int B, int H_q, int H_kv, int N, int d, int flags,
                    const void* workspace, size_t ws_bytes, void* stream) {
    int rc = check_device();
    if (rc) return rc;
    if (!shapes_ok(B, H_q, H_kv, N, d) || !out || !stamps || !workspace || !flags_ok(flags)) return SAGE2_EINVAL;
    Layout L = make_layout(B, H_q, H_kv, N, d);
    if (ws_bytes < L.off[R_END]) return SAGE2_EINVAL;
    return launch_attention(out, reinterpret_cast<int32_t*>(stamps), nullptr, B, H_q, H_kv, N, d,
                            (flags & ~SAGE2_F_CAUSAL) | SAGE2_F_DEBUG_TIMING, reinterpret_cast<const uint8_t*>(workspace),
                            L, reinterpret_cast<cudaStream_t>(stream));
}

int sage2_probe_accumulator(const uint32_t* d_bits, const uint8_t* prod_vals, int n, uint32_t* c_zero,
                            uint32_t* c_prod) {
    int rc = check_device();
    if (rc) return rc;
    if (n < 0 || (n > 0 && (!d_bits || !prod_vals || !c_zero || !c_prod))) return SAGE2_EINVAL;
    return run_probe_accumulator(d_bits, prod_vals, n, c_zero, c_prod);
}

int sage2_bench_mma(int kind, int iters, double* ops_per_s) {
    int rc = check_device();
    if (rc) return rc;
    if ((kind != 0 && kind != 1) || iters < 1 || !ops_per_s) return SAGE2_EINVAL;
    return run_bench_mma(kind, iters, ops_per_s);
}

int sage2_microbench(int which, int iters, double* per_clk_per_sm) {
    int rc = check_device();
    if (rc) return rc;
    if (which < 0 || which > 11 || iters < 1 || !per_clk_per_sm) return SAGE2_EINVAL;
    return run_micro(which, iters, per_clk_per_sm);
}
#endif

}  // extern "C"

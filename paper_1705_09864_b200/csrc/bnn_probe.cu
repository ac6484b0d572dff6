// Pipe-peak probes: measure the roofline denominators the bench reports
// against (the POPC pipe has no vendor figure for sm_100a; SURVEY 0 asks
// for a microbenchmark before the 16/clk/SM figure is used).
#include "bnn_common.cuh"

namespace bnn {

// 8 independent LOP3+POPC chains per thread: one ALU op per POPC, so the
// loop is POPC-bound unless POPC runs at the full ALU rate.
__global__ void probe_popc_kernel(uint32_t seed, int64_t iters, uint32_t *sink) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
    const uint32_t k0 = seed ^ 0x5bd1e995u, k1 = seed ^ 0x1b873593u;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __popc(v[i] ^ ((i & 1) ? k1 : k0));
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= v[i];
    if (acc == 0x12345678u) sink[0] = acc;  // keep the loop alive
}

// Dense tcgen05 MMA issue rate: one CTA per SM issues `reps` back-to-back
// 128 x 256 MMAs from fixed SMEM operands (kind::i8, K = 32, or kind::mxf4 with
// UE8M0 scales = 1, K = 64) and waits for their completion.  The MAC rate is the
// tensor-pipe roofline of the engine that uses that kind.
__device__ __forceinline__ uint32_t probe_smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t probe_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <int kKind, int kN = 256, bool kTS = false>
__global__ void __launch_bounds__(512) probe_mma_kernel(int reps, uint32_t *sink) {
    extern __shared__ __align__(1024) uint8_t psm[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bar2;
    const int tid = threadIdx.x, warp = tid >> 5;
    uint8_t *ops = psm + ((1024 - (probe_smem_u32(psm) & 1023)) & 1023);
    for (int i = tid; i < (kKind >= 8 ? 3 * 16384 + 3 * 8192 : (128 + 256) * 128) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(ops)[i] = 0x11111111u * (i & 3);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            probe_smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(probe_smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(probe_smem_u32(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    // UE8M0 scale factors = 1.0 in columns 384.. (kind::mxf4)
    for (int c = 0; c < 128; c += 8) {
        const uint32_t one = 0x7F7F7F7Fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};\n" ::"r"(
                         tmem + ((uint32_t)(warp * 32) << 16) + 384 + c),
                     "r"(one));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    __shared__ int probe_done;
    if (tid == 0) probe_done = 0;
    __syncthreads();
    if (kKind >= 10 && tid >= 128) {
        // other warps poll a shared flag while warp 0 issues (kKind 10: tight spin,
        // 11: with nanosleep backoff) -- the interference of waiting warps
        while (*(volatile int *)&probe_done == 0) {
            if (kKind == 11) __nanosleep(64);
        }
    }
    if (kKind >= 6 && tid == 0) {
        // kind::mxf4 SS 128 x kN, 9 MMAs per group with varying descriptors (the small-
        // channel conv's tile), one commit per group; kKind 7 also waits for each group's
        // commit before issuing the next (a serialised pipeline)
        const uint32_t a = probe_smem_u32(ops), b = a + (kKind >= 8 ? 3 * 16384 : 128 * 128);  // (kinds 8-11)
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) | (1u << 23) | (8u << 24);
        uint32_t phase = 0;
        for (int i = 0; i < reps / 9; ++i) {
            for (int s = 0; s < 9; ++s) {
                // the small-channel conv's pattern: A over 16 KB blocks, B over 8 KB blocks
                const uint64_t ad = probe_sw128(a + (kKind >= 8 ? (s >> 2) * 16384 : 0) + (s & 3) * 32);
                const uint64_t bd = probe_sw128(b + (kKind >= 8 ? (s >> 2) * 8192 : 0) + (s & 3) * 32);
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(
                        tmem + (kKind >= 8 ? (i & 3) * 64 : (i & 1) * 128)),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(s ? 1u : 0u), "r"(tmem + (kKind >= 8 ? 256 : 384)),
                    "r"(tmem + (kKind >= 8 ? 256 : 384)));
            }
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    probe_smem_u32(&bar))
                : "memory");
            if (kKind == 7 || kKind >= 9) {
                uint32_t done = 0;
                do {
                    asm volatile(
                        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                        "selp.u32 %0, 1, 0, p;\n}\n"
                        : "=r"(done)
                        : "r"(probe_smem_u32(&bar)), "r"(phase)
                        : "memory");
                } while (!done);
                phase ^= 1;
            }
        }
        uint32_t done = 0;  // drain: one more commit, wait for everything
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                probe_smem_u32(&bar2))
            : "memory");
        do {
            asm volatile(
                "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                "selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(probe_smem_u32(&bar2))
                : "memory");
        } while (!done);
        *(volatile int *)&probe_done = 1;
    }
    if (kKind < 6 && tid == 0) {
        const uint32_t a = probe_smem_u32(ops), b = a + 128 * 128;
        for (int i = 0; i < reps; ++i) {
            const int kk = i & 3;
            const uint64_t ad = probe_sw128(a + kk * 32), bd = probe_sw128(b + kk * 32);
            if (kKind == 1) {
                const uint32_t idesc = (2u << 4) | (32u << 17) | (8u << 24);
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
            } else if (kTS) {  // A from TMEM (columns 256.., 8 per K = 64 step)
                const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) |
                                       (1u << 23) | (8u << 24);
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(
                        tmem),
                    "r"(tmem + 256 + kk * 8), "l"(bd), "r"(idesc), "r"(1u), "r"(tmem + 384),
                    "r"(tmem + 384));
            } else {
                const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) |
                                       (1u << 23) | (8u << 24);
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(
                        tmem),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(1u), "r"(tmem + 384), "r"(tmem + 384));
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                probe_smem_u32(&bar))
            : "memory");
        uint32_t done = 0;
        do {
            asm volatile(
                "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                "selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(probe_smem_u32(&bar))
                : "memory");
        } while (!done);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
    if (tid == 0 && reps < 0) sink[0] = 1;
}

}  // namespace bnn

using namespace bnn;

extern "C" int bnn_probe_pipe_peak(int pipe, int64_t iters, uint32_t *sink,
                                   double *ops_per_sec, bnn_stream_t stream) {
    if (pipe < 0 || pipe > 11 || iters < 1 || !ops_per_sec || !sink)
        return set_error(BNN_EINVAL,
                         "probe: pipe must be 0 (POPC), 1 (tcgen05 i8) or 2 (tcgen05 mxf4), "
                         "iters >= 1, sink non-null");
    int sms = bnn_device_sm_count();
    if (sms <= 0) return set_error(BNN_ECUDA, "probe: no CUDA device");
    cudaStream_t s = as_stream(stream);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double work = 0;
    int rc = BNN_OK;
    if (pipe == 0) {
        const int threads = 256, blocks = sms * 8;
        probe_popc_kernel<<<blocks, threads, 0, s>>>(1u, iters / 8 + 1, sink);  // warm-up
        cudaEventRecord(e0, s);
        probe_popc_kernel<<<blocks, threads, 0, s>>>(7u, iters, sink);
        cudaEventRecord(e1, s);
        rc = check_launch("probe_popc_kernel");
        work = (double)blocks * threads * (double)iters * 8.0;  // 32-bit popcounts
    } else {
        const int smem = (pipe >= 8 ? 3 * 16384 + 3 * 8192 : (128 + 256) * 128) + 1024;
        const int reps = (int)(iters < (1 << 20) ? iters : (1 << 20));
        // 3: kind::mxf4 with A in TMEM, N = 64; 4: kind::mxf4 SS, N = 64; 5: TS, N = 256
        auto kern = pipe == 1 ? probe_mma_kernel<1>
                    : pipe == 2 ? probe_mma_kernel<2>
                    : pipe == 3 ? probe_mma_kernel<2, 64, true>
                    : pipe == 4 ? probe_mma_kernel<2, 64, false>
                    : pipe == 5 ? probe_mma_kernel<2, 256, true>
                    : pipe == 6 ? probe_mma_kernel<6, 64, false>
                    : pipe == 7 ? probe_mma_kernel<7, 64, false>
                    : pipe == 8 ? probe_mma_kernel<8, 64, false>
                    : pipe == 9 ? probe_mma_kernel<9, 64, false>
                    : pipe == 10 ? probe_mma_kernel<10, 64, false>
                                 : probe_mma_kernel<11, 64, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int nthr = pipe >= 10 ? 448 : 128;
        kern<<<sms, nthr, smem, s>>>(reps / 8 + 1, sink);  // warm-up
        cudaEventRecord(e0, s);
        kern<<<sms, nthr, smem, s>>>(reps, sink);
        cudaEventRecord(e1, s);
        rc = check_launch("probe_mma_kernel");
        const double n = (pipe == 3 || pipe == 4 || pipe >= 6) ? 64.0 : 256.0;
        const double nmma = pipe >= 6 ? (double)(reps / 9) * 9.0 : (double)reps;
        work = (double)sms * nmma * 128.0 * n * (pipe == 1 ? 32.0 : 64.0);  // MACs
    }
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc) return rc;
    *ops_per_sec = work / (ms * 1e-3);
    return BNN_OK;
}

// debug: dst[0] = %globaltimer when this one-thread kernel runs (timeline probes)
static __global__ void stamp_kernel(uint64_t *dst) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *dst = t;
}

extern "C" int bnn_debug_stamp(uint64_t *dst, bnn_stream_t stream) {
    stamp_kernel<<<1, 1, 0, as_stream(stream)>>>(dst);
    return check_launch("stamp_kernel");
}

// Exhaustive monotonicity check of tanhf (the CUDA math library's, which
// torch.tanh uses for f32): count adjacent finite floats a < b with
// tanhf(a) > tanhf(b).  Zero violations make maxpool(tanh(x)) == tanh(maxpool(x))
// exact, so the fused LeNet stem can pool before the tanh (4x fewer tanh).
static __global__ void tanh_monotone_kernel(unsigned long long *violations) {
    unsigned long long bad = 0;
    const uint32_t n = 0x7F800000u;  // positive finite magnitudes: [0, +inf)
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += gridDim.x * blockDim.x) {
        const float a = __uint_as_float(i), b = __uint_as_float(i + 1);
        if (tanhf(a) > tanhf(b)) ++bad;  // (b may be +inf: tanhf(inf) = 1)
        if (tanhf(-b) > tanhf(-a)) ++bad;
    }
    if (bad) atomicAdd(violations, bad);
}

extern "C" int bnn_probe_tanh_monotone(unsigned long long *violations_dev, bnn_stream_t stream) {
    if (!violations_dev) return bnn::set_error(BNN_EINVAL, "null pointer");
    tanh_monotone_kernel<<<148 * 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(violations_dev);
    return bnn::check_launch("tanh_monotone_kernel");
}

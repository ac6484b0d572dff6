// MMA issue-rate probe: one CTA per SM issues R back-to-back tcgen05.mma on fixed
// SMEM operands; reports MAC/clk/SM for kind::i8 (K=32) and kind::mxf4 (K=64).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61;
    return d;
}
template <int KIND, int N>
__global__ void rate(int reps, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x11111111u * (i & 3);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;\n"); }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    if (warp < 4) {
        for (int c = 0; c < 64; c += 8) {
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + 384 + c;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};\n" ::"r"(taddr), "r"(0x7F7F7F7Fu));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (tid == 0) {
        const uint32_t a = smem_u32(smem), b = a + 128 * 128;
        long long t0 = clock64();
        for (int i = 0; i < reps; ++i) {
            const int kk = i & 3;
            const uint64_t ad = sw128_desc(a + kk * 32), bd = sw128_desc(b + kk * 32);
            if (KIND == 0) {
                const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
            } else {
                const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1u), "r"(tmem + 384), "r"(tmem + 416));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t done = 0;
        do { asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(smem_u32(&bar)) : "memory"); } while (!done);
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
template <int KIND, int N>
void run(const char *name) {
    long long *d; cudaMalloc(&d, 148 * 8);
    const int smem = (128 + 256) * 128 + 1024, reps = 4096;
    cudaFuncSetAttribute(rate<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    rate<KIND, N><<<148, 128, smem>>>(reps, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rate<KIND, N><<<148, 128, smem>>>(reps, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double kdim = KIND == 0 ? 32 : 64;
    const double macs = 128.0 * N * kdim * reps;
    printf("%s N=%d: %.1f cyc/MMA, %.0f MAC/clk/SM, %.1f TOPS (2 x MAC, wall %.3f ms) err=%s\n", name, N,
           (double)h[0] / reps, macs / h[0], 2 * macs * 148 / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<0, 128>("i8  "); run<0, 176>("i8  "); run<0, 256>("i8  ");
    run<1, 128>("mxf4"); run<1, 176>("mxf4"); run<1, 256>("mxf4");
    return 0;
}

// tcgen05.mma kind::mxf4 (M = 128, K = 64) issue rate with the A operand read from SMEM
// through a NO-SWIZZLE K-major descriptor (16-byte entries, SBO = 128 B, LBO = plane
// stride) at aligned / misaligned start addresses, against the SWIZZLE_128B layout.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61;
    return d;
}
__device__ __forceinline__ uint64_t nosw_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46;
    return d;
}
// MODE 0: A SW128; 1: A no-swizzle aligned; 2: A no-swizzle, start + 16 * (i % 8) (misaligned); 3: mode 2 and
// accumulators alternating (independent MMAs)
template <int MODE, int N>
__global__ void rate(int reps, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x11111111u * (i & 3);
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
        const uint32_t a = smem_u32(smem), b = a + 64 * 1024;
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
        long long t0 = clock64();
        for (int i = 0; i < reps; ++i) {
            const int kk = i & 3;
            uint64_t ad;
            if (MODE == 0) ad = sw128_desc(a + kk * 32);
            else if (MODE == 1) ad = nosw_desc(a + (i & 7) * 128, 32768, 128);
            else ad = nosw_desc(a + (i & 7) * 16 + (i & 3) * 928, 32768, 128);
            const uint64_t bd = sw128_desc(b + kk * 32);
            const uint32_t d = tmem + ((MODE == 3) ? (i & 1) * 128 : 0);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
                         ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(1u), "r"(tmem + 384), "r"(tmem + 416));
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
template <int MODE, int N>
void run(const char *name) {
    long long *d; cudaMalloc(&d, 148 * 8);
    const int smem = 100 * 1024, reps = 4096;
    cudaFuncSetAttribute(rate<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    rate<MODE, N><<<148, 128, smem>>>(reps, d);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-44s N=%3d: %6.1f cyc/MMA  (ideal %d)  err=%s\n", name, N, (double)h[0] / reps, 128 * N * 64 / 16384, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<0, 64>("A SW128, B SW128"); run<1, 64>("A no-swizzle aligned"); run<2, 64>("A no-swizzle misaligned"); run<3, 64>("A no-swizzle misaligned, alternating D");
    run<0, 128>("A SW128, B SW128"); run<1, 128>("A no-swizzle aligned"); run<2, 128>("A no-swizzle misaligned"); run<3, 128>("A no-swizzle misaligned, alternating D");
    run<0, 256>("A SW128, B SW128"); run<2, 256>("A no-swizzle misaligned");
    return 0;
}

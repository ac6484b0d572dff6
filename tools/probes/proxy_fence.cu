// Cost of the generic -> async proxy hand-off that every SMEM-staged tcgen05 operand
// pays: per iteration each thread does NST st.shared.v4, then (variant) a
// fence.proxy.async, then a warp-elected mbarrier arrive.  Reports cycles / iteration
// for 1..8 warps so the per-fence latency and its scaling with writers are visible.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int VARIANT, int NST>
__global__ void k(int iters, long long *out) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"((1u << 20) - 1));
    __syncthreads();
    const uint32_t dst = smem_u32(smem) + tid * 16;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < NST; ++j)
            asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};\n" ::"r"(dst + j * blockDim.x * 16), "r"(i + j) : "memory");
        if (VARIANT == 1) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (VARIANT == 2) asm volatile("fence.proxy.async;\n" ::: "memory");
        if (VARIANT == 3) asm volatile("membar.cta;\n" ::: "memory");
        __syncwarp();
        if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    }
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
}
template <int VARIANT, int NST>
void run(const char *name) {
    long long *d; cudaMalloc(&d, 8);
    for (int warps = 1; warps <= 16; warps *= 2) {
        const int iters = 2000, smem = NST * warps * 32 * 16;
        cudaFuncSetAttribute(k<VARIANT, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<VARIANT, NST><<<1, warps * 32, smem>>>(iters, d);
        cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-28s NST=%2d warps=%2d: %7.1f cycles/iter  (%s)\n", name, NST, warps, (double)h / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
int main() {
    run<0, 12>("no fence");
    run<1, 12>("fence.proxy.async.shared::cta");
    run<2, 12>("fence.proxy.async");
    run<3, 12>("membar.cta");
    run<1, 2>("fence.proxy.async.shared::cta");
    run<1, 0>("fence.proxy.async.shared::cta");
    return 0;
}

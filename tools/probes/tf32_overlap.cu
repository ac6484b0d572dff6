// Probe for the stride-2 stem: tcgen05.mma kind::tf32 with A (weights) in TMEM and
// B (pixels) read from SMEM through a NO-SWIZZLE K-major descriptor whose two
// 16-byte K chunks OVERLAP rows (LBO = 32 B, SBO = 128 B over a 16-byte-per-pixel
// array): B[n][k] = x[2n - 4 + k], k = 0..7, straight from a duplicated input row
// D[q] = x[2q-4 .. 2q-1] -- no im2col gather.  Checks the numbers and the rate.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t nosw_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
constexpr int N = 112, NQ = 116;
__global__ void probe(const float *a, const float *x, float *out, int reps, long long *cyc) {
    __shared__ __align__(128) float drow[NQ * 4];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < NQ * 4; i += blockDim.x) {
        const int q = i >> 2, j = i & 3, xi = 2 * q - 4 + j;
        drow[i] = (xi >= 0 && xi < 224) ? x[xi] : 0.0f;
    }
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
    {   // A[m][0..7] -> TMEM columns 256..263, lane m
        uint32_t v[8];
        for (int k = 0; k < 8; ++k) v[k] = __float_as_uint(a[tid * 8 + k]);
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + 256;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (tid == 0) {
        const uint64_t bd = nosw_desc(smem_u32(drow), 32, 128);
        long long t0 = clock64();
        for (int i = 0; i < reps; ++i)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(tmem + (i & 1) * 128), "r"(tmem + 256), "l"(bd), "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t done = 0;
        do { asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(smem_u32(&bar)) : "memory"); } while (!done);
        long long t1 = clock64();
        if (cyc) cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (blockIdx.x == 0) {
        for (int c = 0; c < N; c += 8) {
            uint32_t v[8];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
            for (int k = 0; k < 8; ++k) out[tid * N + c + k] = __uint_as_float(v[k]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
int main() {
    std::vector<float> a(128 * 8), x(224), out(128 * N);
    srand(1);
    for (auto &v : a) v = (float)(rand() % 17 - 8);
    for (auto &v : x) v = (float)(rand() % 17 - 8);
    float *da, *dx, *dout; long long *dc;
    cudaMalloc(&da, a.size() * 4); cudaMalloc(&dx, x.size() * 4); cudaMalloc(&dout, out.size() * 4); cudaMalloc(&dc, 148 * 8);
    cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(da, dx, dout, 1, nullptr);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    printf("launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            float ref = 0;
            for (int k = 0; k < 8; ++k) { const int xi = 2 * n - 4 + k; ref += a[m * 8 + k] * ((xi >= 0 && xi < 224) ? x[xi] : 0.0f); }
            if (ref != out[m * N + n]) { if (bad < 5) printf("mismatch m=%d n=%d got %g want %g\n", m, n, out[m * N + n], ref); ++bad; }
        }
    printf("overlap descriptor (LBO=32, SBO=128): %d mismatches of %d\n", bad, 128 * N);
    const int reps = 8192;
    probe<<<148, 128>>>(da, dx, dout, reps, dc);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("tf32 128x%dx8 A(TMEM) B(SMEM no-swizzle): %.1f cyc/MMA, %.0f MAC/clk/SM  err=%s\n", N, (double)h[0] / reps,
           128.0 * N * 8 * reps / h[0], cudaGetErrorString(cudaGetLastError()));
    return 0;
}

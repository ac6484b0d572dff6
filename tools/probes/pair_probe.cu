// Standalone probe: 2-CTA (cta_group::2) kind::mxf4 MMA with the e2m1 bit expansion.
// Cluster of 2 CTAs computes D[256 x 256] = popc(A[256,K] & B[256,K]) for K = 256 bits:
// CTA r holds A rows [128 r, 128 r + 128) and B rows [128 r, 128 r + 128) in SMEM (same
// offsets), the leader (rank 0) issues the MMAs, a multicast commit signals both CTAs,
// each CTA reads its 128 accumulator rows from its own TMEM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o pair_probe pair_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cooperative_groups.h>

constexpr int M = 256, N = 256, KB = 256, ROWB = KB / 2;
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void expand_b(uint32_t w, uint32_t (&r)[4]) {
    r[0] = w & 0x11111111u; r[1] = w & 0x22222222u; r[2] = w & 0x44444444u; r[3] = (w >> 1) & 0x44444444u;
}
__device__ __forceinline__ void expand_a(uint32_t w, uint32_t (&r)[4]) {
    r[0] = (w << 2) & 0x44444444u; r[1] = w & 0x22222222u; r[2] = (w >> 2) & 0x11111111u; r[3] = (w >> 3) & 0x11111111u;
}
__device__ __forceinline__ uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

__global__ void __cluster_dims__(2, 1, 1) probe(const uint32_t *A, const uint32_t *B, float *D, uint32_t idesc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sa = smem;                    // 128 rows x 128 B (this CTA's A half)
    uint8_t *sb = smem + 128 * ROWB;       // 128 rows x 128 B (this CTA's B half)
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar_done;   // MMA complete (multicast commit)
    __shared__ __align__(8) uint64_t bar_ready;  // leader: both CTAs' operands written
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar_done)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;\n" ::"r"(smem_u32(&bar_ready)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    // expand this CTA's halves
    for (int r = tid; r < 256; r += blockDim.x) {
        const bool is_a = r < 128;
        const int row = r & 127;
        const int grow = rank * 128 + row;
        const uint32_t *src = is_a ? A + grow * (KB / 32) : B + grow * (KB / 32);
        uint8_t *base = is_a ? sa : sb;
        for (int q = 0; q < KB / 32; ++q) {
            uint32_t v[4];
            if (is_a) expand_a(src[q], v); else expand_b(src[q], v);
            *reinterpret_cast<uint4 *>(base + row * ROWB + ((q ^ (row & 7)) << 4)) = make_uint4(v[0], v[1], v[2], v[3]);
        }
    }
    // scale factors 1.0 in columns 256..511 of every lane (this CTA's TMEM)
    if (warp < 4) {
        for (int c = 256; c < 512; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};\n" ::"r"(
                tmem + ((uint32_t)(warp * 32) << 16) + c), "r"(0x7F7F7F7Fu));
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    // both CTAs signal the leader's bar_ready (remote arrive for rank 1)
    if (tid == 0) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(remote) : "r"(smem_u32(&bar_ready)));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
    }
    if (rank == 0 && tid == 0) {
        uint32_t done = 0;
        do {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(smem_u32(&bar_ready)) : "memory");
        } while (!done);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        for (int kk = 0; kk < KB / 64; ++kk) {
            const uint64_t ad = sw128_desc(smem_u32(sa) + kk * 32);
            const uint64_t bd = sw128_desc(smem_u32(sb) + kk * 32);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
                ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(kk ? 1u : 0u), "r"(tmem + 256), "r"(tmem + 256));
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                     ::"r"(smem_u32(&bar_done)), "h"((uint16_t)3) : "memory");
    }
    {
        uint32_t done = 0;
        do {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(smem_u32(&bar_done)) : "memory");
        } while (!done);
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp < 4) {
        for (int c = 0; c < N; c += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
            for (int j = 0; j < 8; ++j) D[(rank * 128 + warp * 32 + lane) * N + c + j] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
    const int W = KB / 32;
    std::vector<uint32_t> A(M * W), B(N * W);
    srand(3);
    for (auto &x : A) x = (uint32_t)rand() * 2654435761u ^ (uint32_t)rand();
    for (auto &x : B) x = (uint32_t)rand() * 2246822519u ^ (uint32_t)rand();
    std::vector<float> expect(M * N);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int c = 0;
            for (int w = 0; w < W; ++w) c += __builtin_popcount(A[m * W + w] & B[n * W + w]);
            expect[m * N + n] = (float)c;
        }
    uint32_t *dA, *dB; float *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xFF, M * N * 4);
    const int smem = 256 * ROWB + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // idesc: E2M1 x E2M1, UE8M0 scales, N = 256, M = 256 (bits 24..28 = M >> 4)
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
    probe<<<2, 256, smem>>>(dA, dB, dD, idesc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> D(M * N);
    cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0, bad0 = 0, bad1 = 0;
    for (int i = 0; i < M * N; ++i) if (D[i] != expect[i]) { ++bad; if (i < 128 * N) ++bad0; else ++bad1; }
    printf("pair mxf4: bad %d/%d (rows 0-127: %d, rows 128-255: %d); sample got %.0f %.0f %.0f %.0f expect %.0f %.0f %.0f %.0f\n",
           bad, M * N, bad0, bad1, D[0], D[200], D[130 * N + 7], D[255 * N + 255], expect[0], expect[200], expect[130 * N + 7], expect[255 * N + 255]);
    return 0;
}

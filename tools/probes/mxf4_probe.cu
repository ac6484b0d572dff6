// Standalone probe: does tcgen05.mma kind::mxf4 (e2m1 x e2m1, UE8M0 scales = 1.0)
// compute popc(a & b) exactly with the nibble expansion planned for the binary
// engine?  One CTA, M=128, N=NT, K=256 bits (4 MMAs of K=64).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mxf4_probe mxf4_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

constexpr int BM = 128, NT = 128, KB = 256;  // K in bits
constexpr int ROWB = KB / 2;                 // fp4 bytes per row = 128

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// B side: register r of word w -> nibble n holds bit 4n + r; values 0.5 / 1 / 2 / 2
__device__ __forceinline__ void expand_b(uint32_t w, uint32_t (&r)[4]) {
    r[0] = w & 0x11111111u;          // code 1 = 0.5
    r[1] = w & 0x22222222u;          // code 2 = 1.0
    r[2] = w & 0x44444444u;          // code 4 = 2.0
    r[3] = (w >> 1) & 0x44444444u;   // bit 4n+3 -> code 4 = 2.0
}
// A side: complementary values so every product of set bits is 1
__device__ __forceinline__ void expand_a(uint32_t w, uint32_t (&r)[4]) {
    r[0] = (w << 2) & 0x44444444u;   // bit 4n   -> 2.0
    r[1] = w & 0x22222222u;          // bit 4n+1 -> 1.0
    r[2] = (w >> 2) & 0x11111111u;   // bit 4n+2 -> 0.5
    r[3] = (w >> 3) & 0x11111111u;   // bit 4n+3 -> 0.5
}

__global__ void probe(const uint32_t *A, const uint32_t *B, float *D, uint32_t idesc, int sfcol,
                      int variant) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sa = smem;                 // 128 rows x 128 B
    uint8_t *sb = smem + BM * ROWB;     // NT rows x 128 B
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    // expand: thread t < 128 -> A row t; t < 128 + NT -> B row
    for (int row = tid; row < BM + NT; row += blockDim.x) {
        const bool is_a = row < BM;
        const int r = is_a ? row : row - BM;
        const uint32_t *src = is_a ? A + r * (KB / 32) : B + r * (KB / 32);
        uint8_t *base = is_a ? sa : sb;
        for (int q = 0; q < KB / 32; ++q) {  // 8 words -> 8 x 16 B
            uint32_t v[4];
            if (is_a) expand_a(src[q], v); else expand_b(src[q], v);
            const int chunk = q ^ (r & 7);
            uint4 *dst = reinterpret_cast<uint4 *>(base + r * ROWB + chunk * 16);
            *dst = make_uint4(v[0], v[1], v[2], v[3]);
        }
    }
    // scale factors: all bytes 0x7F (UE8M0 2^0) in columns sfcol .. sfcol+63, all lanes
    if (warp < 4) {
        const uint32_t ones = variant == 1 ? 0x80808080u : 0x7F7F7F7Fu;
        for (int c = 0; c < 64; c += 8) {
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + sfcol + c;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};\n" ::"r"(taddr), "r"(ones));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (tid == 0) {
        for (int kk = 0; kk < KB / 64; ++kk) {
            const uint64_t ad = sw128_desc(smem_u32(sa) + kk * 32);
            const uint64_t bd = sw128_desc(smem_u32(sb) + kk * 32);
            const uint32_t acc = kk ? 1u : 0u;
            const uint32_t sfa = tmem + sfcol, sfb = tmem + sfcol + 32;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
                ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    }
    // wait
    {
        uint32_t done = 0;
        do {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        } while (!done);
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp < 4) {
        for (int c = 0; c < NT; c += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
            for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * NT + c + j] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
    const int W = KB / 32;
    std::vector<uint32_t> A(BM * W), B(NT * W);
    srand(1);
    for (auto &x : A) x = (uint32_t)rand() * 2654435761u ^ (uint32_t)rand();
    for (auto &x : B) x = (uint32_t)rand() * 2246822519u ^ (uint32_t)rand();
    std::vector<float> expect(BM * NT);
    for (int m = 0; m < BM; ++m)
        for (int n = 0; n < NT; ++n) {
            int c = 0;
            for (int w = 0; w < W; ++w) c += __builtin_popcount(A[m * W + w] & B[n * W + w]);
            expect[m * NT + n] = (float)c;
        }
    uint32_t *dA, *dB; float *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, BM * NT * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const int smem = BM * ROWB + NT * ROWB + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // idesc candidates for kind::mxf4 (CUTLASS InstrDescriptorBlockScaled layout)
    struct Cand { const char *name; uint32_t idesc; int variant; };
    auto mk = [](uint32_t af, uint32_t bf, uint32_t mfield) {
        return (af << 7) | (bf << 10) | ((uint32_t)(NT >> 3) << 17) | (1u << 23) | mfield;
    };
    Cand cands[] = {
        {"fmt1 m>>4@24", mk(1, 1, (uint32_t)(BM >> 4) << 24), 0},
        {"fmt1 m>>7@27", mk(1, 1, (uint32_t)(BM >> 7) << 27), 0},
        {"fmt5 m>>4@24", mk(5, 5, (uint32_t)(BM >> 4) << 24), 0},
        {"fmt1 m>>4@24 scale 0x80", mk(1, 1, (uint32_t)(BM >> 4) << 24), 1},
    };
    std::vector<float> D(BM * NT);
    for (auto &c : cands) {
        cudaMemset(dD, 0xFF, BM * NT * 4);
        probe<<<1, 256, smem>>>(dA, dB, dD, c.idesc, 384, c.variant);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%-28s idesc=%08x: CUDA error %s\n", c.name, c.idesc, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D.data(), dD, BM * NT * 4, cudaMemcpyDeviceToHost);
        int bad = 0; double ratio = 0; int nr = 0;
        for (int i = 0; i < BM * NT; ++i) {
            if (D[i] != expect[i]) ++bad;
            if (expect[i] > 0) { ratio += D[i] / expect[i]; ++nr; }
        }
        printf("%-28s idesc=%08x: bad %d/%d  mean ratio %.4f  sample got %.3f %.3f %.3f expect %.0f %.0f %.0f\n", c.name, c.idesc, bad, BM * NT,
               ratio / nr, D[0], D[1], D[NT + 5], expect[0], expect[1], expect[NT + 5]);
    }
    return 0;
}

// xnor-popcount GEMM / implicit-im2col binary conv on the 5th-gen tensor
// cores (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM), the BNN_ALGO_UMMA
// engine.  Replaces the same reference functions as bnn_gemm_popc.cu
// (gemm.py:80-159, layers.py:225-245); results are bit-identical.
//
// B200 has no binary tensor-core MMA (b1 mma.sync is emulated on sm_100a,
// SURVEY 0), so each CTA expands its packed operands to bytes in shared
// memory right before the MMA consumes them.  The expansion is one LOP3 per
// 4 bytes.  For u32 word w, register r in 0..7 and byte j in 0..3, byte j of
// register r stands for bit 8j + r of w:
//     B (activations):  w & (0x01010101 << r)        -> bit * 2^r
//     A (weights):      w' & (0x80808080 >> r)       -> bit * 2^(7-r)
// where w' = w with the bits of every byte reversed (BREV + PRMT, 2 ops per
// A word).  Every product is therefore 2^7 * [a_k = 1 and b_k = 1] and the
// s32 accumulator holds 128 * C with C = popc(a & b) (exact for K < 2^24).
// Both operands use the same K permutation (byte 4r + j of a word's 32
// expanded bytes <- bit 8j + r), and a sum over K is permutation invariant.
// The xnor count is then recovered as in the north star's .and.popc form:
//     X = popc(a) + popc(b) - 2C,   P = k_eff - X
// with popc(a), popc(b) counted by the producer threads as they expand.
//
// CTA tile 128 (M) x 256 (N); K streamed in 128-bit slices (128 expanded
// bytes per row = one SWIZZLE_128B K-major atom row).  Warp roles:
//   warps 0..11  producers: one operand row each (128 A rows + 256 B rows);
//                cp.async packed words into a private 4-deep ring, expand,
//                st.shared into the 4-stage expanded ring, fence.proxy.async,
//                arrive on full[s]
//   warp 12      TMEM allocator + single-thread tcgen05.mma issuer; each
//                stage = 4 MMAs of K=32; tcgen05.commit -> empty[s]
//   warps 0..3   epilogue after the K loop: tcgen05.ld 32x32b.x16 (thread t
//                owns TMEM lane t = tile row t), decode, store f32.
#include "bnn_loaders.cuh"

namespace bnn {
namespace umma {

constexpr int BM = 128, BN = 256;
constexpr int kWordsPerStage = 4;                // u32 words of K per row per stage
constexpr int kRowBytes = 128;                   // expanded bytes per row per stage
constexpr int ES = 4;                            // expanded stages
constexpr int PD = 4;                            // packed prefetch depth (per thread)
constexpr int kProducers = BM + BN;              // 384
constexpr int kThreads = kProducers + 32;        // + MMA warp
constexpr int kMmaWarp = kProducers / 32;        // 12
constexpr int kStageA = BM * kRowBytes;          // 16 KB
constexpr int kStageB = BN * kRowBytes;          // 32 KB
constexpr int kStageBytes = kStageA + kStageB;   // 48 KB
constexpr int kTmemCols = 256;

struct Smem {  // offsets from the 1024-aligned dynamic smem base
    static constexpr int expanded = 0;
    static constexpr int packed = ES * kStageBytes;                       // 192 KB
    static constexpr int popc_b = packed + PD * kProducers * 16;          // +24 KB
    static constexpr int bars = popc_b + BN * 4;
    static constexpr int tmem_slot = bars + (2 * ES + 1) * 8;
    static constexpr int total = tmem_slot + 16;
};
constexpr int kSmemBytes = Smem::total + 1024;  // alignment slack

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
    } while (!done);
}

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (8-row atoms of 1024 B)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
    d |= (uint64_t)1 << 16;                         // LBO (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;               // SBO: 8-row group stride
    d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                         // SWIZZLE_128B
    return d;
}

// instruction descriptor: kind::i8, D s32, A u8, B u8, both K-major, M=128, N=256
constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     bar)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// expand one packed u32 word into 32 bytes (two 16-byte chunks) of a row
template <bool kIsA>
__device__ __forceinline__ void expand_store(uint32_t w, uint32_t row_base, int row, int q) {
    uint32_t r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = kIsA ? (w & (0x80808080u >> i)) : (w & (0x01010101u << i));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int chunk = (2 * q + h) ^ (row & 7);
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(row_base + chunk * 16),
                     "r"(r[4 * h]), "r"(r[4 * h + 1]), "r"(r[4 * h + 2]), "r"(r[4 * h + 3]));
    }
}

template <int kVec, class ALoad, class BLoad, class Store>
__global__ void __launch_bounds__(kThreads, 1)
    xnor_umma_kernel(ALoad aload, BLoad bload, Store store, Epilogue ep, int64_t kw32) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase_raw = smem_u32(smem_raw);
    const uint32_t sbase = (sbase_raw + 1023u) & ~1023u;
    uint8_t *sgen = smem_raw + (sbase - sbase_raw);
    const uint32_t s_exp = sbase + Smem::expanded;
    const uint32_t s_pk = sbase + Smem::packed;
    int32_t *s_popc_b = reinterpret_cast<int32_t *>(sgen + Smem::popc_b);
    const uint32_t bar_full = sbase + Smem::bars;            // ES barriers
    const uint32_t bar_empty = bar_full + ES * 8;           // ES barriers
    const uint32_t bar_done = bar_empty + ES * 8;           // 1 barrier
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sgen + Smem::tmem_slot);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const int64_t ktiles = ceil_div(kw32, kWordsPerStage);

    if (tid == 0) {
        for (int s = 0; s < ES; ++s) {
            mbar_init(bar_full + 8 * s, kProducers);
            mbar_init(bar_empty + 8 * s, 1);
        }
        mbar_init(bar_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(s_tmem)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *s_tmem;

    int32_t my_popc = 0;
    if (warp < kMmaWarp) {
        // ------------------------------------------------------------ producer
        const bool is_a = tid < BM;
        const int row = is_a ? tid : tid - BM;
        // private packed ring, slot-major so a warp's 16-byte slots are contiguous
        const uint32_t ring = s_pk + tid * 16;
        typename ALoad::Cursor ca{};
        typename BLoad::Cursor cb{};
        if (is_a) ca = aload.row(m0 + row);
        else cb = bload.row(n0 + row);
        auto fetch = [&](int64_t kt) {
            const uint32_t dst = ring + (uint32_t)(kt % PD) * (kProducers * 16);
#pragma unroll
            for (int p = 0; p < kWordsPerStage / kVec; ++p) {
                const int64_t w = kt * kWordsPerStage + p * kVec;
                if (is_a) aload.template load<kVec>(ca, w, dst + p * kVec * 4);
                else bload.template load<kVec>(cb, w, dst + p * kVec * 4);
            }
        };
#pragma unroll
        for (int p = 0; p < PD - 1; ++p) {
            if (p < ktiles) fetch(p);
            cp_async_commit();
        }
        for (int64_t kt = 0; kt < ktiles; ++kt) {
            if (kt + PD - 1 < ktiles) fetch(kt + PD - 1);
            cp_async_commit();
            cp_async_wait<PD - 1>();
            uint32_t wv[4];
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                         : "=r"(wv[0]), "=r"(wv[1]), "=r"(wv[2]), "=r"(wv[3])
                         : "r"(ring + (uint32_t)(kt % PD) * (kProducers * 16)));
            const int s = (int)(kt % ES);
            if (kt >= ES) mbar_wait(bar_empty + 8 * s, (uint32_t)((kt / ES) - 1) & 1u);
            const uint32_t row_base = s_exp + s * kStageBytes + (is_a ? 0 : kStageA) + row * kRowBytes;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                my_popc += __popc(wv[q]);
                if (is_a) expand_store<true>(__byte_perm(__brev(wv[q]), 0, 0x0123), row_base, row, q);
                else expand_store<false>(wv[q], row_base, row, q);
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_arrive(bar_full + 8 * s);
        }
        cp_async_wait<0>();
        if (!is_a) s_popc_b[row] = my_popc;
        asm volatile("bar.sync 1, %0;\n" ::"n"(kProducers) : "memory");  // s_popc_b visible
    } else if (lane == 0) {
        // ------------------------------------------------------------ MMA issuer
        for (int64_t kt = 0; kt < ktiles; ++kt) {
            const int s = (int)(kt % ES);
            mbar_wait(bar_full + 8 * s, (uint32_t)(kt / ES) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t a_addr = s_exp + s * kStageBytes;
            const uint32_t b_addr = a_addr + kStageA;
#pragma unroll
            for (int kk = 0; kk < kRowBytes / 32; ++kk)
                mma_i8(tmem, sw128_desc(a_addr + kk * 32), sw128_desc(b_addr + kk * 32),
                       (kt | kk) != 0 ? 1u : 0u);
            umma_commit(bar_empty + 8 * s);
        }
        umma_commit(bar_done);
    }

    // ---------------------------------------------------------------- epilogue
    if (warp < 4) {
        mbar_wait(bar_done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int64_t m = m0 + tid;  // TMEM lane tid == tile row tid
        const bool mrow_ok = store.ok(m, n0);
        const int32_t pa = my_popc;
        const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
        for (int c = 0; c < BN / 16; ++c) {
            uint32_t v[16];
            tmem_ld16(lane_addr + c * 16, v);
            if (!mrow_ok) continue;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                float o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int nn = c * 16 + g * 4 + i;
                    const int32_t cnt = (int32_t)(v[g * 4 + i] >> 7);
                    const int32_t x = pa + s_popc_b[nn] - 2 * cnt;
                    o[i] = ep.apply(x, (int)m);
                }
                const int64_t n = n0 + c * 16 + g * 4;
                if (store.ok(m, n)) store.put4(m, n, o);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                     "n"(kTmemCols));
    }
}

}  // namespace umma

template <int kVec, class ALoad, class BLoad, class Store>
static int launch_umma(const ALoad &a, const BLoad &b, const Store &st, const Epilogue &ep,
                       int64_t M, int64_t N, int64_t kw32, cudaStream_t s) {
    auto kern = umma::xnor_umma_kernel<kVec, ALoad, BLoad, Store>;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, umma::kSmemBytes);
        configured = true;
    }
    dim3 grid((unsigned)ceil_div(N, umma::BN), (unsigned)ceil_div(M, umma::BM));
    if (grid.y > 65535) return set_error(BNN_EUNSUP, "M too large");
    kern<<<grid, umma::kThreads, umma::kSmemBytes, s>>>(a, b, st, ep, kw32);
    return check_launch("xnor_umma_kernel");
}

int launch_xnor_gemm_umma(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                          int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n,
                          const Epilogue &ep, cudaStream_t s) {
    const int64_t kw32 = 2 * ceil_div(K, 64);
    DenseRows a{reinterpret_cast<const uint32_t *>(A), 2 * lda, M, kw32};
    DenseRows b{reinterpret_cast<const uint32_t *>(B), 2 * ldb, N, kw32};
    GemmStore st{C, ldc_m, ldc_n, M, N};
    const bool vec4 = (lda % 2 == 0) && (ldb % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
    return vec4 ? launch_umma<4>(a, b, st, ep, M, N, kw32, s)
                : launch_umma<2>(a, b, st, ep, M, N, kw32, s);
}

int launch_bconv2d_umma(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
                        const uint64_t *w, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                        int64_t sw, int64_t ph, int64_t pw, int64_t oh, int64_t ow, float *y,
                        const Epilogue &ep, cudaStream_t s) {
    const int64_t cw64 = ceil_div(C, 64);
    const int64_t cs32 = 2 * cw64;
    const int64_t kw32 = kh * kw * cs32;
    const int64_t npix = B * oh * ow;
    DenseRows a{reinterpret_cast<const uint32_t *>(w), kw32, F, kw32};
    ConvRows b{reinterpret_cast<const uint32_t *>(x), npix, (int)H, (int)W, (int)cs32, (int)C,
               (int)kw, (int)sh, (int)sw, (int)ph, (int)pw, (int)oh, (int)ow, kw32};
    ConvStore st{y, F, oh * ow, npix};
    const bool vec4 = (cw64 % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) == 0;
    return vec4 ? launch_umma<4>(a, b, st, ep, F, npix, kw32, s)
                : launch_umma<2>(a, b, st, ep, F, npix, kw32, s);
}

}  // namespace bnn

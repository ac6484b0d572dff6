// xnor-popcount GEMM / implicit-im2col conv on warp-level binary MMA
// (mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc), the
// BNN_ALGO_BMMA engine -- the north star's second contestant.
//
// On sm_100a ptxas lowers the b1 MMA to an out-of-line IMMA-u8 emulation
// (SURVEY 0), so this engine exists to be measured against the CUDA-core
// (bnn_gemm_popc.cu) and tcgen05 (bnn_gemm_umma.cu) engines.  The .and.popc
// form gives C = popc(a & b); the xnor count is recovered as
//     X = popc(a) + popc(b) - 2C,  P = k_eff - X
// with the row / column popcounts accumulated from the same register
// fragments the MMAs consume (each 256-bit k-step of a row is spread over the
// 4 threads of a quad, reduced with two shuffles at the end).
//
// CTA 128 x 128, 8 warps as 2 (M) x 4 (N), warp tile 64 x 32 = 4 x 4 MMAs of
// 16 x 8; K streamed in 1024-bit slices through the same swizzled cp.async
// ring as the CUDA-core engine.
#include "bnn_loaders.cuh"

namespace bnn {
namespace bmma {

constexpr int BM = 128, BN = 128, kWarpsM = 2, kWarpsN = 4, kThreads = 256;
constexpr int kStages = 3;
constexpr int kBKWords = 32;
constexpr int MT = 4, NT = 4;  // 16x8 MMA tiles per warp

__device__ __forceinline__ uint32_t lds32(const uint8_t *tile, int r, int word) {
    const int c16 = word >> 2;
    return *reinterpret_cast<const uint32_t *>(tile + r * 128 + ((c16 ^ (r & 7)) << 4) +
                                               ((word & 3) << 2));
}

template <int kVec, class ALoad, class BLoad, class Store>
__global__ void __launch_bounds__(kThreads)
    xnor_bmma_kernel(ALoad aload, BLoad bload, Store store, Epilogue ep, int64_t kw32) {
    constexpr int kPieces = kBKWords / kVec;
    constexpr int kRowsPerPass = kThreads / kPieces;
    constexpr int kPassA = BM / kRowsPerPass, kPassB = BN / kRowsPerPass;
    constexpr int kTileBytes = 128 * 128;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *sA = smem;
    uint8_t *sB = smem + kStages * kTileBytes;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % kWarpsM, wn = warp / kWarpsM;
    const int g = lane >> 2, t = lane & 3;  // quad id / thread in quad
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;

    const int lp = tid % kPieces, lr = tid / kPieces;
    typename ALoad::Cursor ca[kPassA];
    typename BLoad::Cursor cb[kPassB];
#pragma unroll
    for (int q = 0; q < kPassA; ++q) ca[q] = aload.row(m0 + lr + q * kRowsPerPass);
#pragma unroll
    for (int q = 0; q < kPassB; ++q) cb[q] = bload.row(n0 + lr + q * kRowsPerPass);
    const int64_t ktiles = ceil_div(kw32, kBKWords);
    auto issue = [&](int64_t kt, int stage) {
        const int w = (int)(kt * kBKWords + lp * kVec);
        const uint32_t a_base = smem_u32(sA + stage * kTileBytes);
        const uint32_t b_base = smem_u32(sB + stage * kTileBytes);
#pragma unroll
        for (int q = 0; q < kPassA; ++q)
            aload.template load<kVec>(ca[q], w, a_base + tile_off<kVec>(lr + q * kRowsPerPass, lp));
#pragma unroll
        for (int q = 0; q < kPassB; ++q)
            bload.template load<kVec>(cb[q], w, b_base + tile_off<kVec>(lr + q * kRowsPerPass, lp));
    };

    int32_t acc[MT][NT][4];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[i][j][r] = 0;
    int32_t popa[MT][2] = {}, popb[NT] = {};

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < ktiles) issue(s, s);
        cp_async_commit();
    }
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + kStages - 1;
            if (nk < ktiles) issue(nk, (int)(nk % kStages));
            cp_async_commit();
        }
        const uint8_t *tA = sA + (kt % kStages) * kTileBytes;
        const uint8_t *tB = sB + (kt % kStages) * kTileBytes;
#pragma unroll
        for (int ks = 0; ks < kBKWords / 8; ++ks) {  // 256-bit k-steps
            uint32_t af[MT][4], bf[NT][2];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const int r = wm * 64 + i * 16 + g;
                af[i][0] = lds32(tA, r, 8 * ks + t);
                af[i][1] = lds32(tA, r + 8, 8 * ks + t);
                af[i][2] = lds32(tA, r, 8 * ks + 4 + t);
                af[i][3] = lds32(tA, r + 8, 8 * ks + 4 + t);
                popa[i][0] += __popc(af[i][0]) + __popc(af[i][2]);
                popa[i][1] += __popc(af[i][1]) + __popc(af[i][3]);
            }
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int r = wn * 32 + j * 8 + g;
                bf[j][0] = lds32(tB, r, 8 * ks + t);
                bf[j][1] = lds32(tB, r, 8 * ks + 4 + t);
                popb[j] += __popc(bf[j][0]) + __popc(bf[j][1]);
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    asm volatile(
                        "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
                        "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};\n"
                        : "+r"(acc[i][j][0]), "+r"(acc[i][j][1]), "+r"(acc[i][j][2]),
                          "+r"(acc[i][j][3])
                        : "r"(af[i][0]), "r"(af[i][1]), "r"(af[i][2]), "r"(af[i][3]),
                          "r"(bf[j][0]), "r"(bf[j][1]));
        }
    }
    cp_async_wait<0>();

    // full-row popcounts: sum over the 4 threads of each quad
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            popa[i][h] += __shfl_xor_sync(0xffffffffu, popa[i][h], 1);
            popa[i][h] += __shfl_xor_sync(0xffffffffu, popa[i][h], 2);
        }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        popb[j] += __shfl_xor_sync(0xffffffffu, popb[j], 1);
        popb[j] += __shfl_xor_sync(0xffffffffu, popb[j], 2);
    }
    // D fragment: d0,d1 -> row g, cols 2t, 2t+1; d2,d3 -> row g+8.  The column
    // popcount for col 2t+c lives in the quad of lane 4*(2t+c).
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const int pb0 = __shfl_sync(0xffffffffu, popb[j], 4 * (2 * t));
        const int pb1 = __shfl_sync(0xffffffffu, popb[j], 4 * (2 * t + 1));
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t m = m0 + wm * 64 + i * 16 + g + (r >= 2 ? 8 : 0);
                const int64_t n = n0 + wn * 32 + j * 8 + 2 * t + (r & 1);
                if (store.ok(m, n)) {
                    const int32_t x = popa[i][r >> 1] + ((r & 1) ? pb1 : pb0) - 2 * acc[i][j][r];
                    store.put(m, n, ep.apply(x, (int)m));
                }
            }
    }
}

}  // namespace bmma

template <int kVec, class ALoad, class BLoad, class Store>
static int launch_bmma(const ALoad &a, const BLoad &b, const Store &st, const Epilogue &ep,
                       int64_t M, int64_t N, int64_t kw32, cudaStream_t s) {
    constexpr int kSmem = bmma::kStages * 2 * 128 * 128;
    auto kern = bmma::xnor_bmma_kernel<kVec, ALoad, BLoad, Store>;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        configured = true;
    }
    dim3 grid((unsigned)ceil_div(N, bmma::BN), (unsigned)ceil_div(M, bmma::BM));
    if (grid.y > 65535) return set_error(BNN_EUNSUP, "M too large");
    kern<<<grid, bmma::kThreads, kSmem, s>>>(a, b, st, ep, kw32);
    return check_launch("xnor_bmma_kernel");
}

int launch_xnor_gemm_bmma(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                          int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n,
                          const Epilogue &ep, cudaStream_t s, const float *res) {
    const int64_t kw32 = 2 * ceil_div(K, 64);
    DenseRows a{reinterpret_cast<const uint32_t *>(A), 2 * lda, M, kw32};
    DenseRows b{reinterpret_cast<const uint32_t *>(B), 2 * ldb, N, kw32};
    GemmStore st{C, ldc_m, ldc_n, M, N, res};
    const bool vec4 = (lda % 2 == 0) && (ldb % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
    return vec4 ? launch_bmma<4>(a, b, st, ep, M, N, kw32, s)
                : launch_bmma<2>(a, b, st, ep, M, N, kw32, s);
}

int launch_bconv2d_bmma(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
                        const uint64_t *w, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                        int64_t sw, int64_t ph, int64_t pw, int64_t oh, int64_t ow, float *y,
                        const Epilogue &ep, cudaStream_t s, const float *res) {
    const int64_t cw64 = ceil_div(C, 64);
    const int64_t cs32 = 2 * cw64;
    const int64_t kw32 = kh * kw * cs32;
    const int64_t npix = B * oh * ow;
    DenseRows a{reinterpret_cast<const uint32_t *>(w), kw32, F, kw32};
    ConvRows b{reinterpret_cast<const uint32_t *>(x), npix, (int)H, (int)W, (int)cs32, (int)C,
               (int)kw, (int)sh, (int)sw, (int)ph, (int)pw, (int)oh, (int)ow, kw32};
    ConvStore st{y, F, oh * ow, npix, res};
    const bool vec4 = (cw64 % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) == 0;
    return vec4 ? launch_bmma<4>(a, b, st, ep, F, npix, kw32, s)
                : launch_bmma<2>(a, b, st, ep, F, npix, kw32, s);
}

}  // namespace bnn

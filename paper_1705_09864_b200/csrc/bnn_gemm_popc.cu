// xnor-popcount GEMM and implicit-im2col binary convolution on the CUDA
// cores (LOP3 xor + POPC), the BNN_ALGO_POPC engine.
//
// Replaces the reference xnor kernel family (gemm.py:80-159; hot loop
// gemm.py:128-139) and QConv2d's im2col + pack_matrix_b + GEMM chain
// (layers.py:230-236, tensor.py:60-78).
//
// Both operands are K-contiguous packed rows (u32 view of the u64 words).
// A CTA computes a BM x BN tile of X[m, n] = sum_w popc(A[m, w] ^ B[n, w]);
// the K loop streams 32-word (1024-bit) slices of both operands through a
// STAGES-deep cp.async ring in shared memory.  Rows are 128 B in shared
// memory with the 16-byte chunk index XOR-swizzled by (row & 7), so the
// 8 distinct rows a warp touches per LDS.128 land in 8 distinct bank quads.
// Each thread owns a TM x TN register tile; lane (lm, ln) = (lane & 7,
// lane >> 3) takes rows lm + 8i and columns ln + 4j of its warp tile.
#include "bnn_loaders.cuh"

namespace bnn {

constexpr int kBKWords = 32;  // u32 words per K slice (1024 bits = 128 B per row)

// ------------------------------------------------------------------ kernel
template <int TM, int TN, int WARPS_M, int WARPS_N, int STAGES, int kVec, class ALoad,
          class BLoad, class Store>
__global__ void __launch_bounds__(WARPS_M *WARPS_N * 32)
    xnor_popc_kernel(ALoad aload, BLoad bload, Store store, Epilogue ep, int64_t kw32) {
    constexpr int kThreads = WARPS_M * WARPS_N * 32;
    constexpr int WM = 8 * TM, WN = 4 * TN;
    constexpr int BM = WM * WARPS_M, BN = WN * WARPS_N;
    constexpr int kPieces = kBKWords / kVec;  // pieces per row per slice
    constexpr int kTileBytesA = BM * 128, kTileBytesB = BN * 128;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *sA = smem;
    uint8_t *sB = smem + STAGES * kTileBytesA;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;
    const int lm = lane & 7, ln = lane >> 3;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;

    // loader assignment: thread -> (row, piece), rows strided by kThreads/kPieces
    constexpr int kRowsPerPass = kThreads / kPieces;
    constexpr int kPassA = BM / kRowsPerPass, kPassB = BN / kRowsPerPass;
    static_assert(BM % kRowsPerPass == 0 && BN % kRowsPerPass == 0, "loader tiling");
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
        const uint32_t a_base = smem_u32(sA + stage * kTileBytesA);
        const uint32_t b_base = smem_u32(sB + stage * kTileBytesB);
#pragma unroll
        for (int q = 0; q < kPassA; ++q)
            aload.template load<kVec>(ca[q], w, a_base + tile_off<kVec>(lr + q * kRowsPerPass, lp));
#pragma unroll
        for (int q = 0; q < kPassB; ++q)
            bload.template load<kVec>(cb[q], w, b_base + tile_off<kVec>(lr + q * kRowsPerPass, lp));
    };

    int32_t acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) issue(s, s);
        cp_async_commit();
    }

    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + STAGES - 1;
            if (nk < ktiles) issue(nk, (int)(nk % STAGES));
            cp_async_commit();
        }
        const int stage = (int)(kt % STAGES);
        const uint8_t *tA = sA + stage * kTileBytesA;
        const uint8_t *tB = sB + stage * kTileBytesB;
#pragma unroll 2
        for (int c16 = 0; c16 < 8; ++c16) {
            uint4 a[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const int r = wm * WM + lm + 8 * i;
                a[i] = *reinterpret_cast<const uint4 *>(tA + r * 128 + ((c16 ^ (r & 7)) << 4));
            }
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int r = wn * WN + ln + 4 * j;
                const uint4 b = *reinterpret_cast<const uint4 *>(tB + r * 128 + ((c16 ^ (r & 7)) << 4));
#pragma unroll
                for (int i = 0; i < TM; ++i)
                    acc[i][j] += __popc(a[i].x ^ b.x) + __popc(a[i].y ^ b.y) +
                                 __popc(a[i].z ^ b.z) + __popc(a[i].w ^ b.w);
            }
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t m = m0 + wm * WM + lm + 8 * i;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int64_t n = n0 + wn * WN + ln + 4 * j;
            if (store.ok(m, n)) store.put(m, n, ep.apply(acc[i][j], (int)m));
        }
    }
}

// ------------------------------------------------------------------ launch
template <int TM, int TN, int WARPS_M, int WARPS_N, int STAGES, int kVec, class ALoad,
          class BLoad, class Store>
static int launch_cfg(const ALoad &a, const BLoad &b, const Store &st, const Epilogue &ep,
                      int64_t M, int64_t N, int64_t kw32, cudaStream_t s) {
    constexpr int BM = 8 * TM * WARPS_M, BN = 4 * TN * WARPS_N;
    constexpr int kSmem = STAGES * (BM + BN) * 128;
    auto kern = xnor_popc_kernel<TM, TN, WARPS_M, WARPS_N, STAGES, kVec, ALoad, BLoad, Store>;
    static bool configured = false;  // attribute set once per instantiation
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        configured = true;
    }
    dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM));
    if (grid.y > 65535) return set_error(BNN_EUNSUP, "M=%lld too large", (long long)M);
    kern<<<grid, WARPS_M * WARPS_N * 32, kSmem, s>>>(a, b, st, ep, kw32);
    return check_launch("xnor_popc_kernel");
}

// tile selection: big tiles when there are enough of them to fill 148 SMs
template <int kVec, class ALoad, class BLoad, class Store>
static int dispatch(const ALoad &a, const BLoad &b, const Store &st, const Epilogue &ep,
                    int64_t M, int64_t N, int64_t kw32, cudaStream_t s) {
    const int64_t big_tiles = ceil_div(M, 128) * ceil_div(N, 128);
    if (big_tiles >= 2 * 148)
        return launch_cfg<8, 8, 2, 4, 3, kVec>(a, b, st, ep, M, N, kw32, s);
    return launch_cfg<4, 4, 2, 4, 4, kVec>(a, b, st, ep, M, N, kw32, s);
}

int launch_xnor_gemm_popc(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                          int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n,
                          const Epilogue &ep, cudaStream_t s, const float *res) {
    const int64_t kw32 = 2 * ceil_div(K, 64);
    DenseRows a{reinterpret_cast<const uint32_t *>(A), 2 * lda, M, kw32};
    DenseRows b{reinterpret_cast<const uint32_t *>(B), 2 * ldb, N, kw32};
    GemmStore st{C, ldc_m, ldc_n, M, N, res};
    const bool vec4 = (lda % 2 == 0) && (ldb % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
    return vec4 ? dispatch<4>(a, b, st, ep, M, N, kw32, s) : dispatch<2>(a, b, st, ep, M, N, kw32, s);
}

int launch_bconv2d_popc(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
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
    return vec4 ? dispatch<4>(a, b, st, ep, F, npix, kw32, s)
                : dispatch<2>(a, b, st, ep, F, npix, kw32, s);
}

}  // namespace bnn

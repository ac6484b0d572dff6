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
#include "bnn_common.cuh"

namespace bnn {

constexpr int kBKWords = 32;  // u32 words per K slice (1024 bits = 128 B per row)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kBytes>
__device__ __forceinline__ void cp_async(uint32_t dst, const void *src, int src_bytes) {
    if constexpr (kBytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                     "r"(src_bytes));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(dst), "l"(src),
                     "n"(kBytes), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// byte offset of piece p (of kVec words) of row r inside a [rows][32-word] tile
template <int kVec>
__device__ __forceinline__ uint32_t tile_off(int r, int p) {
    const int byte = p * kVec * 4;  // logical byte within the 128-B row
    const int c16 = byte >> 4;
    return (uint32_t)(r * 128 + ((c16 ^ (r & 7)) << 4) + (byte & 15));
}

// ------------------------------------------------------------------ loaders
// Dense operand: row r of a [rows, ld32] u32 matrix, kw32 valid words.
struct DenseRows {
    const uint32_t *base;
    int64_t ld32;
    int64_t rows;
    int64_t kw32;
    struct Cursor { const uint32_t *p; bool ok; };
    __device__ Cursor row(int64_t r) const { return {base + r * ld32, r < rows}; }
    // load kVec words at word w of this row into smem address dst
    template <int kVec>
    __device__ void load(const Cursor &c, int64_t w, uint32_t dst) const {
        int64_t left = kw32 - w;
        int bytes = (!c.ok || left <= 0) ? 0 : (int)(left >= kVec ? kVec * 4 : left * 4);
        const uint32_t *src = bytes ? c.p + w : base;
        cp_async<kVec * 4>(dst, src, bytes);
    }
};

// Implicit im2col rows: row n = output pixel (b, oy, ox); word w = tap-major
// (i, j, channel word).  Out-of-image taps read the constant "+1" word
// (valid channel bits set, channel tail 0), the reference's zero-pad-then-
// binarize composition (tensor.py:73-74 + bitpack.py:39).
struct ConvRows {
    const uint32_t *x;  // NHWC words, pixel stride cs32
    int64_t npix;       // B * oh * ow
    int H, W, cs32, C, kw, sh, sw, ph, pw, oh, ow;
    int64_t kw32;       // kh * kw * cs32
    struct Cursor { const uint32_t *img; int iy0, ix0; bool ok; };
    __device__ Cursor row(int64_t n) const {
        Cursor c;
        c.ok = n < npix;
        int64_t nn = c.ok ? n : 0;
        int64_t ohw = (int64_t)oh * ow;
        int64_t b = nn / ohw;
        int pix = (int)(nn - b * ohw);
        int oy = pix / ow, ox = pix - (pix / ow) * ow;
        c.img = x + b * (int64_t)H * W * cs32;
        c.iy0 = oy * sh - ph;
        c.ix0 = ox * sw - pw;
        return c;
    }
    template <int kVec>
    __device__ void load(const Cursor &c, int64_t w, uint32_t dst) const {
        if (!c.ok || w >= kw32) {
            cp_async<kVec * 4>(dst, x, 0);
            return;
        }
        int tap = (int)(w / cs32);
        int cw = (int)(w - (int64_t)tap * cs32);
        int i = tap / kw, j = tap - (tap / kw) * kw;
        int iy = c.iy0 + i, ix = c.ix0 + j;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
            cp_async<kVec * 4>(dst, c.img + ((int64_t)iy * W + ix) * cs32 + cw, kVec * 4);
        } else {
            uint32_t v[kVec];
#pragma unroll
            for (int q = 0; q < kVec; ++q) {
                int valid = C - 32 * (cw + q);
                v[q] = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
            }
            if constexpr (kVec == 4)
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(dst), "r"(v[0]),
                             "r"(v[1]), "r"(v[2]), "r"(v[3]));
            else
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(dst), "r"(v[0]),
                             "r"(v[1]));
        }
    }
};

// ------------------------------------------------------------------ stores
struct GemmStore {
    float *C;
    int64_t ldc_m, ldc_n, M, N;
    __device__ bool ok(int64_t m, int64_t n) const { return m < M && n < N; }
    __device__ void put(int64_t m, int64_t n, float v) const { C[m * ldc_m + n * ldc_n] = v; }
};

struct ConvStore {  // y NCHW [B, F, oh*ow]; m = filter, n = b*ohw + pixel
    float *y;
    int64_t F, ohw, npix;
    __device__ bool ok(int64_t m, int64_t n) const { return m < F && n < npix; }
    __device__ void put(int64_t m, int64_t n, float v) const {
        int64_t b = n / ohw, p = n - b * ohw;
        y[(b * F + m) * ohw + p] = v;
    }
};

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
        const int64_t w = kt * kBKWords + lp * kVec;
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
                          const Epilogue &ep, cudaStream_t s) {
    const int64_t kw32 = 2 * ceil_div(K, 64);
    DenseRows a{reinterpret_cast<const uint32_t *>(A), 2 * lda, M, kw32};
    DenseRows b{reinterpret_cast<const uint32_t *>(B), 2 * ldb, N, kw32};
    GemmStore st{C, ldc_m, ldc_n, M, N};
    const bool vec4 = (lda % 2 == 0) && (ldb % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
    return vec4 ? dispatch<4>(a, b, st, ep, M, N, kw32, s) : dispatch<2>(a, b, st, ep, M, N, kw32, s);
}

int launch_bconv2d_popc(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
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
    return vec4 ? dispatch<4>(a, b, st, ep, F, npix, kw32, s)
                : dispatch<2>(a, b, st, ep, F, npix, kw32, s);
}

}  // namespace bnn

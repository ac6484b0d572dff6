// Full-precision (f32) convolution on the 5th-gen tensor cores for the float
// stem layers of the network runners: ResNet-18's conv7x7/2 (3 -> 64) and
// LeNet's conv5x5 (1 -> 64) (BASELINE configs[2..3]: "first conv ... full
// precision"; reference Conv2d, layers.py:81-141, an f32 im2col GEMM).
//
// f32 accuracy from TF32 MMAs by a three-term split ("3xTF32"): every operand
// is split into hi = round_tf32(v) and lo = v - hi (exact in f32), and
//     x . w  ~  x_hi w_hi + x_hi w_lo + x_lo w_hi
// accumulated in f32 by tcgen05.mma kind::tf32 (the dropped x_lo w_lo term and
// the TF32 truncation of lo are ~2^-22 relative per product).  The result
// differs from an f32 CUDA-core convolution only by summation-order rounding.
//
// Implicit GEMM: D[pixel, filter] = sum_k A[pixel, k] W[filter, k], k = (c, ky,
// kx) in the reference's weight flattening order.  Persistent CTA per SM,
// 128-pixel tiles (TMEM lanes), N = 64 filters:
//   warps 0-7   gather: one output pixel per thread, 32 K values per chunk
//               (two groups of 4 warps on alternate chunks), split hi/lo and
//               tcgen05.st both halves into a TMEM A stage (ring of 6 stages)
//   warp 8      TMEM allocator + one thread issuing 3 x 4 MMAs (128x64x8, A
//               from TMEM, W hi/lo resident in SMEM, SWIZZLE_128B K-major)
//               per chunk; commit frees the stage, per tile commit -> epilogue
//   warps 9-12  epilogue: tcgen05.ld of the 64 accumulators of a pixel (double
//               buffered in TMEM), + bias, coalesced NCHW stores (32 consecutive
//               pixels of one channel per warp store)
#include "bnn_umma_impl.cuh"

namespace bnn {
namespace stem {

using namespace umma;

constexpr int BM = 128;  // pixels per tile (TMEM lanes)
constexpr int NF = 64;   // filters (MMA N)
constexpr int KC = 32;   // K per chunk: one 128-byte SWIZZLE_128B atom of f32
constexpr int kMaxChunks = 10;
constexpr int S = 6;     // TMEM A stages (32 hi + 32 lo columns each)
constexpr int kProdWarps = 8, kMmaWarp = 8, kEpiWarp0 = 9, kEpiWarps = 4;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kAStage0 = 2 * NF;  // TMEM columns [0, 128): two accumulator buffers
static_assert(kAStage0 + S * 2 * KC <= 512, "TMEM budget");
// kind::tf32: D f32 (bit 4), A / B TF32 (format 2), K-major, N >> 3, M >> 4
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NF >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

struct Geom {
    const float *x, *w, *bias;
    float *y;
    int C, H, W, kh, kw, sh, sw, ph, pw, ow, ohw;
    int K, nch;
    int64_t npix;
    int ntiles;
};

__device__ __forceinline__ uint32_t tf32_hi(float v) {
    return (__float_as_uint(v) + 0x1000u) & 0xFFFFE000u;  // round to 10 mantissa bits
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31, %32};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
        "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
        "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

// shared memory: W hi / W lo [chunk][64 rows][128 B] (SWIZZLE_128B K-major),
// K table, barriers, TMEM base
struct Smem {
    static constexpr int kB = kMaxChunks * NF * 128;
    static constexpr int off_bhi = 0, off_blo = kB, off_ktab = 2 * kB;
    static constexpr int off_bars = off_ktab + kMaxChunks * KC * 16;
    static constexpr int kNumBars = 2 * S + 4;
    static constexpr int off_tmem = off_bars + kNumBars * 8;
    static constexpr int kBytes = off_tmem + 16 + 1024;  // + alignment slack
};

__global__ void __launch_bounds__(kThreads, 1) conv_tf32x3_kernel(const __grid_constant__ Geom g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *smem = smem_raw + (base - raw);
    const uint32_t s_bhi = base + Smem::off_bhi, s_blo = base + Smem::off_blo;
    int4 *ktab = reinterpret_cast<int4 *>(smem + Smem::off_ktab);
    const uint32_t bar_full = base + Smem::off_bars, bar_empty = bar_full + 8 * S;
    const uint32_t bar_tfull = bar_empty + 8 * S, bar_tempty = bar_tfull + 16;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + Smem::off_tmem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int kpad = g.nch * KC;

    // weights -> SMEM as hi / lo TF32 operands (zero past K); gather table
    for (int i = tid; i < NF * kpad; i += kThreads) {
        const int r = i / kpad, k = i - r * kpad;
        const float v = k < g.K ? __ldg(g.w + (int64_t)r * g.K + k) : 0.0f;
        const uint32_t hi = tf32_hi(v);
        const float lo = v - __uint_as_float(hi);
        const int kb = (k & 31) * 4;
        const uint32_t off = (uint32_t)((k >> 5) * (NF * 128) + (r >> 3) * 1024 + (r & 7) * 128 +
                                        ((((kb >> 4) ^ (r & 7)) << 4) | (kb & 15)));
        asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(s_bhi + off), "r"(hi));
        asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(s_blo + off), "f"(lo));
    }
    for (int k = tid; k < kpad; k += kThreads) {
        int4 t = make_int4(0, -(1 << 20), -(1 << 20), 0);  // padding: fails the bounds test
        if (k < g.K) {
            const int taps = g.kh * g.kw, ci = k / taps, r = k - ci * taps;
            const int ky = r / g.kw, kx = r - ky * g.kw;
            t = make_int4((ci * g.H + ky) * g.W + kx, ky, kx, 0);
        }
        ktab[k] = t;
    }
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(bar_full + 8 * s, 4);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    // the MMA (async proxy) reads the weights written above by the generic proxy
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp < kProdWarps) {
        // ------------------------------------------------------------ gather
        const int grp = warp >> 2, q = warp & 3, row = q * 32 + lane;
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + kAStage0;
        int gch = 0;
        for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
            const int64_t p = (int64_t)tile * BM + row;
            const bool pv = p < g.npix;
            const int64_t b = pv ? p / g.ohw : 0;
            const int rem = pv ? (int)(p - b * g.ohw) : 0;
            const int oy = rem / g.ow, ox = rem - oy * g.ow;
            const int iy0 = oy * g.sh - g.ph, ix0 = ox * g.sw - g.pw;
            const float *xb = g.x + b * g.C * g.H * g.W + (int64_t)iy0 * g.W + ix0;
            for (int c = 0; c < g.nch; ++c, ++gch) {
                if ((gch & 1) != grp) continue;
                const int st = gch % S;
                mbar_wait(bar_empty + 8 * st, ((gch / S) & 1) ^ 1);
                fence_after();
                uint32_t hi[32], lo[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int4 t = ktab[c * KC + j];
                    const int iy = iy0 + t.y, ix = ix0 + t.z;
                    float v = 0.0f;
                    if (pv && (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W)
                        v = __ldg(xb + t.x);
                    hi[j] = tf32_hi(v);
                    lo[j] = __float_as_uint(v - __uint_as_float(hi[j]));
                }
                tmem_st32(tq + st * 2 * KC, hi);
                tmem_st32(tq + st * 2 * KC + KC, lo);
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_full + 8 * st);
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issue
        if (lane == 0) {
            int gch = 0, it = 0;
            for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++it) {
                const int buf = it & 1;
                mbar_wait(bar_tempty + 8 * buf, ((it >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t d = tmem + buf * NF;
                for (int c = 0; c < g.nch; ++c, ++gch) {
                    const int st = gch % S;
                    mbar_wait(bar_full + 8 * st, (gch / S) & 1);
                    fence_after();
                    const uint32_t a = tmem + kAStage0 + st * 2 * KC;
#pragma unroll
                    for (int kk = 0; kk < KC / 8; ++kk) {
                        const uint32_t boff = (uint32_t)(c * NF * 128 + kk * 32);
                        const uint64_t bh = sw128_desc(s_bhi + boff), bl = sw128_desc(s_blo + boff);
                        mma_tf32_ts(d, a + kk * 8, bh, (c | kk) != 0);  // hi x hi
                        mma_tf32_ts(d, a + kk * 8, bl, 1u);              // hi x lo
                        mma_tf32_ts(d, a + KC + kk * 8, bh, 1u);         // lo x hi
                    }
                    umma_commit(bar_empty + 8 * st);
                }
                umma_commit(bar_tfull + 8 * buf);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;
        int it = 0;
        for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++it) {
            const int buf = it & 1;
            mbar_wait_sleep(bar_tfull + 8 * buf, (it >> 1) & 1);
            fence_after();
            uint32_t v0[32], v1[32];
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + buf * NF;
            tmem_ld32(ta, v0);
            tmem_ld32(ta + 32, v1);
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_tempty + 8 * buf);
            const int64_t p = (int64_t)tile * BM + q * 32 + lane;
            if (p < g.npix) {
                const int64_t b = p / g.ohw;
                float *yo = g.y + b * NF * g.ohw + (p - b * g.ohw);
#pragma unroll
                for (int f = 0; f < 32; ++f) {
                    float a0 = __uint_as_float(v0[f]), a1 = __uint_as_float(v1[f]);
                    if (g.bias) {
                        a0 = __fadd_rn(a0, __ldg(g.bias + f));
                        a1 = __fadd_rn(a1, __ldg(g.bias + 32 + f));
                    }
                    __stcs(yo + (int64_t)f * g.ohw, a0);
                    __stcs(yo + (int64_t)(32 + f) * g.ohw, a1);
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

}  // namespace stem

int launch_conv2d_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                         const float *w, const float *bias, int64_t F, int64_t kh, int64_t kw,
                         int64_t sh, int64_t sw, int64_t ph, int64_t pw, int64_t oh, int64_t ow,
                         float *y, cudaStream_t s) {
    using namespace stem;
    const int64_t K = C * kh * kw;
    if (F != NF) return set_error(BNN_EUNSUP, "tensor-core f32 conv: F must be %d, got %lld", NF, (long long)F);
    if (K > kMaxChunks * KC)
        return set_error(BNN_EUNSUP, "tensor-core f32 conv: C*kh*kw=%lld exceeds %d", (long long)K,
                         kMaxChunks * KC);
    const int64_t npix = B * oh * ow;
    if (npix == 0) return BNN_OK;
    if (C * H * W >= (1ll << 31) || npix / stem::BM >= (1ll << 31))
        return set_error(BNN_EUNSUP, "tensor-core f32 conv: tensor too large");
    Geom g{};
    g.x = x, g.w = w, g.bias = bias, g.y = y;
    g.C = (int)C, g.H = (int)H, g.W = (int)W, g.kh = (int)kh, g.kw = (int)kw;
    g.sh = (int)sh, g.sw = (int)sw, g.ph = (int)ph, g.pw = (int)pw, g.ow = (int)ow;
    g.ohw = (int)(oh * ow), g.K = (int)K, g.nch = (int)ceil_div(K, KC), g.npix = npix;
    g.ntiles = (int)ceil_div(npix, stem::BM);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(conv_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Smem::kBytes);
        configured = true;
    }
    const int grid = g.ntiles < sm_count() ? g.ntiles : sm_count();
    conv_tf32x3_kernel<<<grid, kThreads, Smem::kBytes, s>>>(g);
    return check_launch("conv_tf32x3_kernel");
}

}  // namespace bnn

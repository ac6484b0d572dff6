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

// wait with a short sleep between probes: the gather / loader warps wait often and
// would otherwise spin on the issue slots the epilogue needs
__device__ __forceinline__ void mbar_wait_backoff(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    while (true) {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
        if (done) return;
        __nanosleep(64);
    }
}

__device__ __forceinline__ uint32_t tf32_hi(float v) {
    // truncate to 10 mantissa bits: lo = v - hi (exact) has |lo| < 2^-10 |v| and
    // loses only its own bits below TF32 in the MMA (~2^-21 relative)
    return __float_as_uint(v) & 0xFFFFE000u;
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

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15])
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

// ---------------------------------------------------------------------------
// Fused stem: conv (3xTF32, as above) -> BatchNorm -> ReLU -> maxpool 3x3/2/1
// (ResNet-18's stem, nets.StemPost; reference BN op order layers.py:598-602).
// The pool runs before the BatchNorm on sign-adjusted values: with s_c = +1
// (gamma >= 0) or -1 (gamma < 0), f(v) = relu?(bn(v)) is monotone in s_c v, so
//     maxpool(f(v)) = f(s_c * maxpool(s_c * v))
// exactly (negation is exact; the rounded BN ops are monotone), and the conv
// output never leaves the SM: only the pooled tensor is written.
//
// Work item = (image, band of pooled rows); tile = one conv output row (OW <= 128
// pixels = TMEM lanes), processed top to bottom so that the pooled rows are
// completed in registers:
//   warps 0-7   gather from the SMEM-staged input rows (zero-padded; for stride 2
//               the columns are stored de-interleaved by parity, so the 32 lanes
//               of a warp read 32 consecutive words), split hi/lo, tcgen05.st
//   warps 8-9   loader: the C x kh input rows of the next conv row -> SMEM
//               (double buffered)
//   warp 10     TMEM allocator + MMA issuer (3 x 4 MMAs per 32-wide K chunk)
//   warps 11-14 epilogue: TMEM -> s_c * v into a row buffer, horizontal 3-max,
//               vertical running max in registers, BN + ReLU, pooled NCHW stores
namespace stem {

constexpr int kPLoadWarp0 = 8, kPLoadWarps = 4, kPMmaWarp = 12, kPEpiWarp0 = 13;
constexpr int kPX = 4;    // staged input buffers (tiles in flight between loader and gather)
constexpr int kPAcc = 3;  // TMEM accumulator buffers (tiles in flight between MMA and epilogue)
constexpr int kPS = 5;    // TMEM A stages (chunks)
constexpr int kPAStage0 = kPAcc * NF;
static_assert(kPAStage0 + kPS * 2 * KC <= 512, "TMEM budget (fused stem)");
constexpr int kPLoadBatch = 12;  // float4 loads in flight per loader thread (C*kh <= 24 rows)
// epilogue warps kEW (a template parameter): kEW / 4 per TMEM lane quadrant, each
// with NF / (kEW / 4) accumulator columns; the pooling phase spreads (channel group,
// pooled column) over the kEW * 32 threads.  8 for the ResNet stem, 16 for LeNet's
// (tanh per element, measured)
template <int kEW>
struct PEpi {
    static constexpr int kCG = kEW * 32 / 64;         // channel groups of the pooling phase
    static constexpr int kCPer = NF / kCG;            // channels per pooling thread
    static constexpr int kThreads = (kPEpiWarp0 + kEW) * 32;
};
constexpr int kRowPitchR = 132;  // epilogue row buffer pitch (floats)

struct PoolGeom {
    const float *x, *w, *mean, *inv, *gamma, *beta;
    float *y;
    int relu;
    int C, H, W, kh, kw, sh, sw, ph, pw, OH, OW, PH, PW;
    int K, nch;
    int par;        // stride-2 parity layout of the staged rows
    int rpitch;     // staged row pitch (floats)
    int xs_floats;  // one staging buffer: C * kh * rpitch
    int pyb, nbands, items;
    int mode;  // 0: BN + ReLU? + maxpool 3x3/2/1; 1: + bias, tanh, maxpool 2x2/2/0 (LeNet)
    int R;     // conv rows per tile (mode 1: an even number of narrow rows fills the lanes)
    int pool_first;  // mode 1: tanhf is monotone (probed): max-pool, then one tanh per output
    uint16_t *pack16;    // mode 0, optional: sign-packed NHWC words of y as 16-bit pieces
    uint8_t *pack8;      // mode 1, optional: the same as 8-bit pieces (16 epilogue warps); y may then be null
    int32_t *pack_flags;
    int NR;    // staged input rows per channel: (R - 1) * sh + kh
    int rbufs; // epilogue row buffers: 2 = double-buffered (one CTA-wide barrier per tile instead of two)
    int dbg;  // debug (BNN_STEM_DEBUG, wrong results): 1 no gather loads, 2 no MMAs,
              // 4 no epilogue work, 8 no loader loads
};

struct PoolSmem {
    int off_bhi, off_blo, off_ktab, off_xs, off_r, off_bn, off_bars, off_tmem, bytes;
    __host__ __device__ PoolSmem(int nch, int xs_floats, int rbufs = 1) {
        off_bhi = 0;
        off_blo = nch * NF * 128;
        off_ktab = 2 * nch * NF * 128;
        off_xs = off_ktab + nch * KC * 4;
        off_r = off_xs + kPX * xs_floats * 4;
        off_bn = off_r + rbufs * NF * kRowPitchR * 4;
        off_bars = off_bn + 5 * NF * 4;
        off_tmem = off_bars + (2 * kPS + 2 * kPAcc + 2 * kPX) * 8;
        bytes = off_tmem + 16 + 1024;
    }
};

template <int kEW>
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(kEW * 32) : "memory"); }

// compile-time stem geometry (gather offsets become immediates); kStatic = false:
// the runtime table
struct GeoDyn {
    static constexpr bool kStatic = false;
};
template <int kC, int kKH, int kKW, int kPitch>
struct GeoStride2 {  // stride 2, parity layout, pitch kPitch
    static constexpr bool kStatic = true;
    static constexpr int K = kC * kKH * kKW;
    __device__ static constexpr int off(int k) {
        return k >= K ? 0
                      : ((k / (kKH * kKW)) * kKH + (k % (kKH * kKW)) / kKW) * kPitch +
                            ((k % kKW) & 1) * (kPitch / 2) + ((k % kKW) >> 1);
    }
};

template <class Geo, int kChunk>
__device__ __forceinline__ void gather_static(const float *src, uint32_t ta) {
    if constexpr (kChunk * KC < Geo::K) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float v = src[Geo::off(kChunk * KC + 16 * h + j)];
                hi[j] = tf32_hi(v);
                lo[j] = __float_as_uint(v - __uint_as_float(hi[j]));
            }
            tmem_st16(ta + 16 * h, hi);
            tmem_st16(ta + KC + 16 * h, lo);
        }
    }
}

template <class Geo, int kEW>
__global__ void __launch_bounds__(PEpi<kEW>::kThreads, 1) conv_pool_kernel(const __grid_constant__ PoolGeom g) {
    constexpr int kPEpiW = kEW, kPCG = PEpi<kEW>::kCG, kPCPer = PEpi<kEW>::kCPer;
    constexpr int kPThreads = PEpi<kEW>::kThreads;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *smem = smem_raw + (base - raw);
    const PoolSmem L(g.nch, g.xs_floats, g.rbufs);
    const uint32_t s_bhi = base + L.off_bhi, s_blo = base + L.off_blo;
    int *ktab = reinterpret_cast<int *>(smem + L.off_ktab);
    float *xs = reinterpret_cast<float *>(smem + L.off_xs);
    float *rbuf0 = reinterpret_cast<float *>(smem + L.off_r);
    float *bnt = reinterpret_cast<float *>(smem + L.off_bn);  // sign, mean, inv, gamma, beta
    const uint32_t bar_full = base + L.off_bars, bar_empty = bar_full + 8 * kPS;
    const uint32_t bar_tfull = bar_empty + 8 * kPS, bar_tempty = bar_tfull + 8 * kPAcc;
    const uint32_t bar_xfull = bar_tempty + 8 * kPAcc, bar_xempty = bar_xfull + 8 * kPX;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + L.off_tmem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int kpad = g.nch * KC;

    for (int i = tid; i < NF * kpad; i += kPThreads) {
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
    // gather offsets relative to the pixel's base word; K padding reads the pixel's
    // first tap (finite; its weights are zero)
    for (int k = tid; k < kpad; k += kPThreads) {
        int off = 0;
        if (k < g.K) {
            const int taps = g.kh * g.kw, ci = k / taps, r = k - ci * taps;
            const int ky = r / g.kw, kx = r - ky * g.kw;
            off = (ci * g.NR + ky) * g.rpitch + (g.par ? (kx & 1) * (g.rpitch >> 1) + (kx >> 1) : kx);
        }
        ktab[k] = off;
    }
    for (int i = tid; i < kPX * g.xs_floats; i += kPThreads) xs[i] = 0.0f;  // zero borders
    for (int c = tid; c < NF && g.mode == 1; c += kPThreads) {  // bias, no sign flip
        bnt[c] = 1.0f;
        bnt[NF + c] = g.mean ? __ldg(g.mean + c) : 0.0f;
    }
    for (int c = tid; c < NF && g.mode == 0; c += kPThreads) {
        const float gm = __ldg(g.gamma + c);
        bnt[c] = gm < 0.0f ? -1.0f : 1.0f;
        bnt[NF + c] = __ldg(g.mean + c);
        bnt[2 * NF + c] = __ldg(g.inv + c);
        bnt[3 * NF + c] = gm;
        bnt[4 * NF + c] = __ldg(g.beta + c);
    }
    if (tid == 0) {
        for (int s = 0; s < kPS; ++s) {
            mbar_init(bar_full + 8 * s, 4);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < kPAcc; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, kPEpiW);
        }
        for (int b = 0; b < kPX; ++b) {
            mbar_init(bar_xfull + 8 * b, kPLoadWarps);
            mbar_init(bar_xempty + 8 * b, kProdWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == kPMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *s_tmem;

    // the tile sequence every role walks: items (image, band) -> conv rows oy
#define POOL_ITEMS_BEGIN                                                              \
    for (int item = blockIdx.x; item < g.items; item += gridDim.x) {                  \
        const int b = item / g.nbands, band = item - b * g.nbands;                    \
        const int py0 = band * g.pyb, py1 = min(g.PH, py0 + g.pyb);                   \
        const int oy_s = g.mode ? 2 * py0 : max(0, 2 * py0 - 1), oy_e = min(g.OH - 1, 2 * py1 - 1);
#define POOL_ITEMS_END }

    if (warp < kProdWarps) {
        // ------------------------------------------------------------ gather
        const int grp = warp >> 2, q = warp & 3, ox = q * 32 + lane;
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + kPAStage0;
        const int prow = ox / g.OW, pcol = ox - prow * g.OW;  // conv row within the tile
        const int pb = prow < g.R ? prow * g.sh * g.rpitch + (g.par ? pcol : pcol * g.sw) : 0;
        int gch = 0, it = 0;
        POOL_ITEMS_BEGIN
        for (int oy = oy_s; oy <= oy_e; oy += g.R, ++it) {
            const int xb = it % kPX;
            mbar_wait_backoff(bar_xfull + 8 * xb, (it / kPX) & 1);
            const float *src = xs + xb * g.xs_floats + pb;
            for (int c = 0; c < g.nch; ++c, ++gch) {
                if ((gch & 1) != grp) continue;
                const int st = gch % kPS;
                mbar_wait_backoff(bar_empty + 8 * st, ((gch / kPS) & 1) ^ 1);
                fence_after();
                const uint32_t ta = tq + st * 2 * KC;
                if (g.dbg & 1) {
                } else if constexpr (Geo::kStatic) {
                    switch (c) {  // compile-time gather offsets: LDS [base + imm]
                        case 0: gather_static<Geo, 0>(src, ta); break;
                        case 1: gather_static<Geo, 1>(src, ta); break;
                        case 2: gather_static<Geo, 2>(src, ta); break;
                        case 3: gather_static<Geo, 3>(src, ta); break;
                        case 4: gather_static<Geo, 4>(src, ta); break;
                        case 5: gather_static<Geo, 5>(src, ta); break;
                        case 6: gather_static<Geo, 6>(src, ta); break;
                        case 7: gather_static<Geo, 7>(src, ta); break;
                        case 8: gather_static<Geo, 8>(src, ta); break;
                        default: gather_static<Geo, 9>(src, ta); break;
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {  // 16 K values at a time (register budget)
                        uint32_t hi[16], lo[16];
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4) {
                            const int4 o = reinterpret_cast<const int4 *>(ktab + c * KC + 16 * h)[j4];
                            const int oo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float v = src[oo[i]];
                                hi[4 * j4 + i] = tf32_hi(v);
                                lo[4 * j4 + i] = __float_as_uint(v - __uint_as_float(hi[4 * j4 + i]));
                            }
                        }
                        tmem_st16(ta + 16 * h, hi);
                        tmem_st16(ta + KC + 16 * h, lo);
                    }
                }
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_full + 8 * st);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_xempty + 8 * xb);
        }
        POOL_ITEMS_END
    } else if (warp < kPMmaWarp) {
        // ------------------------------------------------------------ loader
        const int t = tid - kPLoadWarp0 * 32;
        const int half = g.rpitch >> 1;
        const int jcol = t & 63, rg = t >> 6, w4 = g.W >> 2;
        // this thread's staged rows rg + 2u: channel-plane offset and tap row (no division
        // in the tile loop)
        int roff[kPLoadBatch], rky[kPLoadBatch];
#pragma unroll
        for (int u = 0; u < kPLoadBatch; ++u) {
            const int r = rg + 2 * u, ci = r / g.NR;
            roff[u] = ci * g.H * g.W;
            rky[u] = r < g.C * g.NR ? r - ci * g.NR : (1 << 28);  // (past the rows: never in range)
        }
        auto scol = [&](int sc) { return g.par ? (sc & 1) * half + (sc >> 1) : sc; };
        const int sa0 = scol(4 * jcol + g.pw), sa1 = scol(4 * jcol + 1 + g.pw);
        const int sa2 = scol(4 * jcol + 2 + g.pw), sa3 = scol(4 * jcol + 3 + g.pw);
        int it = 0;
        POOL_ITEMS_BEGIN
        const float *xb0 = g.x + (int64_t)b * g.C * g.H * g.W;
        for (int oy = oy_s; oy <= oy_e; oy += g.R, ++it) {
            const int xb = it % kPX;
            mbar_wait_backoff(bar_xempty + 8 * xb, ((it / kPX) & 1) ^ 1);
            float *dst = xs + xb * g.xs_floats;
            const int iy0 = oy * g.sh - g.ph;
            // thread = (row parity rg, float4 column j): rows rg, rg + 2, ... of the
            // C x kh staged rows; all loads of a row group in flight before the stores
            const int rows = g.C * g.NR;
            for (int j = jcol; j < w4; j += 64) {
                float4 v[kPLoadBatch];
#pragma unroll
                for (int u = 0; u < kPLoadBatch; ++u) {
                    const int r = rg + 2 * u;
                    v[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    const int iy = iy0 + rky[u];
                    if ((unsigned)iy < (unsigned)g.H && !(g.dbg & 8))
                        v[u] = __ldg(reinterpret_cast<const float4 *>(
                                         xb0 + roff[u] + (int64_t)iy * g.W) + j);
                }
                const int a0 = j == jcol ? sa0 : scol(4 * j + g.pw), a1 = j == jcol ? sa1 : scol(4 * j + 1 + g.pw);
                const int a2 = j == jcol ? sa2 : scol(4 * j + 2 + g.pw), a3 = j == jcol ? sa3 : scol(4 * j + 3 + g.pw);
#pragma unroll
                for (int u = 0; u < kPLoadBatch; ++u) {
                    const int r = rg + 2 * u;
                    if (r >= rows) break;
                    float *row = dst + r * g.rpitch;
                    row[a0] = v[u].x, row[a1] = v[u].y, row[a2] = v[u].z, row[a3] = v[u].w;
                }
            }
            __syncwarp();
            if ((t & 31) == 0) mbar_arrive(bar_xfull + 8 * xb);
        }
        POOL_ITEMS_END
    } else if (warp == kPMmaWarp) {
        // ------------------------------------------------------------ MMA issue
        const uint64_t dh0 = sw128_desc(s_bhi), dl0 = sw128_desc(s_blo);
        if (lane == 0) {
            int gch = 0, it = 0;
            POOL_ITEMS_BEGIN
            for (int oy = oy_s; oy <= oy_e; oy += g.R, ++it) {
                const int buf = it % kPAcc;
                mbar_wait(bar_tempty + 8 * buf, ((it / kPAcc) & 1) ^ 1);
                fence_after();
                const uint32_t d = tmem + buf * NF;
                for (int c = 0; c < g.nch; ++c, ++gch) {
                    const int st = gch % kPS;
                    mbar_wait(bar_full + 8 * st, (gch / kPS) & 1);
                    fence_after();
                    const uint32_t a = tmem + kPAStage0 + st * 2 * KC;
                    const int nkk = (g.dbg & 2) ? 0 : min(KC / 8, (g.K - c * KC + 7) / 8);  // skip all-zero K steps
                    // descriptors by integer adds on the start-address field (16-byte units):
                    // + 8192 B per chunk, + 32 B per K step
                    const uint64_t ch = dh0 + (uint64_t)(c * (NF * 128 / 16)), cl = dl0 + (uint64_t)(c * (NF * 128 / 16));
#pragma unroll
                    for (int kk = 0; kk < KC / 8; ++kk) {
                        if (kk >= nkk) break;
                        mma_tf32_ts(d, a + kk * 8, ch + 2 * kk, (c | kk) != 0);
                        mma_tf32_ts(d, a + kk * 8, cl + 2 * kk, 1u);
                        mma_tf32_ts(d, a + KC + kk * 8, ch + 2 * kk, 1u);
                    }
                    umma_commit(bar_empty + 8 * st);
                }
                umma_commit(bar_tfull + 8 * buf);
            }
            POOL_ITEMS_END
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3, et = tid - kPEpiWarp0 * 32;
        const int hsel = (warp - kPEpiWarp0) >> 2;  // TMEM columns [32 hsel, 32 hsel + 32)
        const int ox = q * 32 + lane;
        const int px = et & 63, c0 = et >> 6;  // pooled column, channel run c0 * kPCPer + i
        float cur[kPCPer];
        int it = 0;
        POOL_ITEMS_BEGIN
#pragma unroll
        for (int i = 0; i < kPCPer; ++i) cur[i] = -INFINITY;
        float *yb = g.y + (int64_t)b * NF * g.PH * g.PW;
        // sign-pack of an emitted pooled pixel: this thread's kPCPer channels are one
        // kPCPer-bit piece of the pixel's packed NHWC word(s)
        auto put_bits = [&](int py, uint32_t bits, float nf) {
            if (kPCPer != 16 || !g.pack16) return;
            const int64_t pix = ((int64_t)b * g.PH + py) * g.PW + px;
            g.pack16[pix * (NF / 16) + c0] = (uint16_t)bits;
            if (g.pack_flags && nf != 0.0f) atomicOr(g.pack_flags, 1);
        };
        auto emit = [&](int py) {
            if (px >= g.PW) return;
            uint32_t bits = 0;
            float nf = 0.0f;
#pragma unroll
            for (int i = 0; i < kPCPer; ++i) {
                const int c = c0 * kPCPer + i;
                float v = __fmul_rn(cur[i], bnt[c]);
                v = __fadd_rn(__fmul_rn(bnt[3 * NF + c], __fmul_rn(__fsub_rn(v, bnt[NF + c]),
                                                                    bnt[2 * NF + c])),
                              bnt[4 * NF + c]);
                if (g.relu) v = fmaxf(v, 0.0f);
                yb[((int64_t)c * g.PH + py) * g.PW + px] = v;
                bits |= (v >= 0.0f ? 1u : 0u) << i;
                nf = __fmaf_rn(v, 0.0f, nf);
            }
            put_bits(py, bits, nf);
        };
        for (int oy = oy_s; oy <= oy_e; oy += g.R, ++it) {
            const int buf = it % kPAcc;
            // (two row buffers: tile i + 1's values are written while slower warps still pool
            // tile i; the barrier of tile i + 1 orders them against tile i + 2's writes)
            float *rbuf = rbuf0 + (g.rbufs == 2 ? (it & 1) * (NF * kRowPitchR) : 0);
            mbar_wait_sleep(bar_tfull + 8 * buf, (it / kPAcc) & 1);
            fence_after();
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + buf * NF;
#pragma unroll
            {
                constexpr int kCols = NF / (kPEpiW / 4);  // TMEM columns per epilogue warp
                uint32_t v[kCols];
                const int c0col = hsel * kCols;
                if constexpr (kCols == 32) tmem_ld32(ta + c0col, *reinterpret_cast<uint32_t(*)[32]>(v));
                else tmem_ld16(ta + c0col, *reinterpret_cast<uint32_t(*)[16]>(v));
                if (ox < g.R * g.OW) {  // lanes = R conv rows of OW pixels
                    if (g.mode == 1) {  // conv + bias -> tanh (torch.tanh's tanhf), then the pool
#pragma unroll
                        for (int j = 0; j < kCols; ++j) {
                            const float t = __fadd_rn(__uint_as_float(v[j]), bnt[NF + c0col + j]);
                            rbuf[(c0col + j) * kRowPitchR + ox] = g.pool_first ? t : tanhf(t);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < kCols; ++j)
                            rbuf[(c0col + j) * kRowPitchR + ox] =
                                __fmul_rn(__uint_as_float(v[j]), bnt[c0col + j]);
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_tempty + 8 * buf);
            epi_bar<kEW>();
            // horizontal 3-max (window 2px-1 .. 2px+1, clipped) of this conv row, folded
            // into the pooled rows: an odd conv row completes pooled row (oy - 1) / 2
            // and starts (oy + 1) / 2, an even one is the middle row of oy / 2
            if (g.mode == 1) {
                // 2x2/2 pool inside the tile: conv rows (2r, 2r + 1) -> pooled row oy / 2 + r.
                // When the tile's pooled pixels fit the 64 pixel slots of a channel group, each
                // thread takes ONE pooled pixel (row r, column px) instead of walking the rows of
                // its column: twice the active threads, half the serial work (LeNet: 28 pixels)
                const bool flat = (g.R >> 1) * g.PW <= 64;
                const int pp = et & 63;
                const int rf = flat ? pp / g.PW : 0;
                const int px = flat ? pp - rf * g.PW : pp;
                const int r_end = flat ? rf + 1 : g.R;
                if (!(g.dbg & 4) && px < g.PW && (!flat || 2 * rf + 1 < g.R))
                for (int r = rf; r < r_end && 2 * r + 1 < g.R && oy + 2 * r + 1 <= oy_e; ++r) {
                    float *yrow = yb + (int64_t)((oy >> 1) + r) * g.PW + px;
                    const int o0 = 2 * r * g.OW + 2 * px, o1 = o0 + g.OW;
                    uint32_t bits = 0;
                    float nf = 0.0f;
#pragma unroll 8
                    for (int i = 0; i < kPCPer; ++i) {
                        const int c = c0 * kPCPer + i;
                        const float *rr = rbuf + c * kRowPitchR;
                        const float m = fmaxf(fmaxf(rr[o0], rr[o0 + 1]), fmaxf(rr[o1], rr[o1 + 1]));
                        const float v = g.pool_first ? tanhf(m) : m;
                        if (g.y) yrow[(int64_t)c * g.PH * g.PW] = v;
                        bits |= (v >= 0.0f ? 1u : 0u) << i;  // sign(-0) = +1 (binarize, bitpack.py:30-42)
                        nf = __fmaf_rn(v, 0.0f, nf);
                    }
                    if (kPCPer == 8 && g.pack8) {
                        // the next binary layer's QActivation + pack: this thread's 8 channels are
                        // one byte of the pooled pixel's packed NHWC word
                        const int64_t pix = ((int64_t)b * g.PH + (oy >> 1) + r) * g.PW + px;
                        g.pack8[pix * (NF / 8) + c0] = (uint8_t)bits;
                        if (g.pack_flags && nf != 0.0f) atomicOr(g.pack_flags, 1);
                    }
                }
            } else if (px < g.PW && !(g.dbg & 4)) {
                const int xl = 2 * px - 1, xr = 2 * px + 1;
                const bool odd = oy & 1, done = odd && ((oy - 1) >> 1) >= py0;
                float *yrow = yb + (int64_t)((oy - 1) >> 1) * g.PW + px;
                uint32_t bits = 0;
                float nf = 0.0f;
#pragma unroll
                for (int i = 0; i < kPCPer; ++i) {
                    const int c = c0 * kPCPer + i;
                    const float *rr = rbuf + c * kRowPitchR;
                    float m = rr[2 * px];
                    if (xl >= 0) m = fmaxf(m, rr[xl]);
                    if (xr < g.OW) m = fmaxf(m, rr[xr]);
                    if (done) {
                        float v = __fmul_rn(fmaxf(cur[i], m), bnt[c]);
                        v = __fadd_rn(__fmul_rn(bnt[3 * NF + c],
                                                __fmul_rn(__fsub_rn(v, bnt[NF + c]), bnt[2 * NF + c])),
                                      bnt[4 * NF + c]);
                        if (g.relu) v = fmaxf(v, 0.0f);
                        yrow[(int64_t)c * g.PH * g.PW] = v;
                        bits |= (v >= 0.0f ? 1u : 0u) << i;
                        nf = __fmaf_rn(v, 0.0f, nf);
                    }
                    cur[i] = odd ? m : fmaxf(cur[i], m);
                }
                if (done) put_bits((oy - 1) >> 1, bits, nf);
            }
            if (g.rbufs != 2) epi_bar<kEW>();  // the row buffer is free for the next conv row
        }
        if (g.mode == 0 && !(oy_e & 1) && (oy_e >> 1) < py1) emit(oy_e >> 1);  // last pooled row without a row below
        POOL_ITEMS_END
    }
#undef POOL_ITEMS_BEGIN
#undef POOL_ITEMS_END
    fence_before();
    __syncthreads();
    if (warp == kPMmaWarp) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

}  // namespace stem

bool stem_s2_supported(int64_t C, int64_t H, int64_t W, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                       int64_t sw, int64_t ph, int64_t pw);
int launch_stem_s2(const float *x, int64_t B, int64_t H, const float *w, const float *bias,
                   const float *mean, const float *inv, const float *gamma, const float *beta, int relu,
                   int raw, float *y, uint64_t *pack_words, int32_t *pack_flags, cudaStream_t s);

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
    // ResNet-18's stem geometry: the gather-free stride-2 kernel (bnn_stem_s2.cu)
    if (stem_s2_supported(C, H, W, F, kh, kw, sh, sw, ph, pw) && !(reinterpret_cast<uintptr_t>(x) & 7) &&
        !(reinterpret_cast<uintptr_t>(y) & 15))
        return launch_stem_s2(x, B, H, w, bias, nullptr, nullptr, nullptr, nullptr, 0, 1, y, nullptr, nullptr, s);
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


// conv (3xTF32) + BN + ReLU + maxpool 3x3/2/1 fused; BNN_EUNSUP when the shape
// does not fit (the caller then runs the conv and the post-op separately)
int launch_conv_bn_relu_maxpool_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                                   const float *w, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                                   int64_t sw, int64_t ph, int64_t pw, const float *mean,
                                   const float *inv, const float *gamma, const float *beta,
                                   int relu, float *y, cudaStream_t s, int mode,
                                   uint64_t *pack_words, int32_t *pack_flags, int pool_first) {
    using namespace stem;
    const int64_t K = C * kh * kw;
    const int64_t OH = (H + 2 * ph - kh) / sh + 1, OW = (W + 2 * pw - kw) / sw + 1;
    const int64_t PH = mode ? OH / 2 : (OH + 2 - 3) / 2 + 1, PW = mode ? OW / 2 : (OW + 2 - 3) / 2 + 1;
    if (mode && (PH < 1 || PW < 1)) return set_error(BNN_EUNSUP, "fused stem: pool does not fit");
    if (mode == 0 && stem_s2_supported(C, H, W, F, kh, kw, sh, sw, ph, pw) &&
        !(reinterpret_cast<uintptr_t>(x) & 7) && !(reinterpret_cast<uintptr_t>(y) & 15))
        return launch_stem_s2(x, B, H, w, nullptr, mean, inv, gamma, beta, relu, 0, y, pack_words, pack_flags, s);
    if (F != NF || K > kMaxChunks * KC || OW > stem::BM || OW < 2 || OH < 2 || W % 4 != 0 ||
        (reinterpret_cast<uintptr_t>(x) & 15) || PW > 64 || C * H * W >= (1ll << 31) ||
        C * kh > 2 * kPLoadBatch || W / 4 > 64 * 8)
        return set_error(BNN_EUNSUP, "fused stem: unsupported shape");
    PoolGeom g{};
    g.x = x, g.w = w, g.mean = mean, g.inv = inv, g.gamma = gamma, g.beta = beta, g.y = y;
    g.relu = relu;
    g.mode = mode;
    g.pack16 = mode == 0 ? reinterpret_cast<uint16_t *>(pack_words) : nullptr;
    g.pack8 = mode == 1 ? reinterpret_cast<uint8_t *>(pack_words) : nullptr;
    g.pack_flags = pack_flags;
    g.pool_first = mode == 1 && pool_first;
    g.dbg = (int)g_debug.stem_bits;
    g.C = (int)C, g.H = (int)H, g.W = (int)W, g.kh = (int)kh, g.kw = (int)kw, g.sh = (int)sh;
    g.sw = (int)sw, g.ph = (int)ph, g.pw = (int)pw, g.OH = (int)OH, g.OW = (int)OW;
    g.PH = (int)PH, g.PW = (int)PW, g.K = (int)K, g.nch = (int)ceil_div(K, KC);
    g.par = sw == 2;
    g.R = mode ? (int)((stem::BM / OW) & ~1ll) : 1;
    if (g.R < 1) return set_error(BNN_EUNSUP, "fused stem: conv width");
    g.NR = (int)((g.R - 1) * sh + kh);
    if (C * g.NR > 2 * kPLoadBatch) return set_error(BNN_EUNSUP, "fused stem: staged rows");
    const int64_t ws = (OW - 1) * sw + kw;  // staged columns per row (incl. padding)
    int64_t pitch = g.par ? 2 * ceil_div(ws, 2) : ws;
    pitch = ceil_div(pitch, 4) * 4 + (g.par ? 2 : 1);  // spread rows over banks
    if (g.par && (pitch & 1)) pitch += 1;
    if (pw + W > ws + 0 && pw + W > pitch) return set_error(BNN_EUNSUP, "fused stem: row pitch");
    g.rpitch = (int)pitch;
    g.xs_floats = (int)(C * g.NR * pitch);
    // pooled-row bands: about 4 items per SM-wave unit of work, 14 rows for ResNet
    int64_t pyb = PH >= 14 ? 14 : PH;
    g.pyb = (int)pyb;
    g.nbands = (int)ceil_div(PH, pyb);
    if (B * g.nbands >= (1ll << 31)) return set_error(BNN_EUNSUP, "fused stem: too many items");
    g.items = (int)(B * g.nbands);
    g.rbufs = PoolSmem(g.nch, g.xs_floats, 2).bytes <= 227 * 1024 && !(g.dbg & 32) ? 2 : 1;
    const PoolSmem L(g.nch, g.xs_floats, g.rbufs);
    if (L.bytes > 227 * 1024) return set_error(BNN_EUNSUP, "fused stem: shared memory");
    if (B == 0) return BNN_OK;
    const int grid = g.items < sm_count() ? g.items : sm_count();
    if (C == 3 && kh == 7 && kw == 7 && g.par && pitch <= 234) {  // ResNet stem: static offsets
        using G = GeoStride2<3, 7, 7, 234>;
        g.rpitch = 234;
        g.xs_floats = (int)(C * g.NR * 234);
        g.rbufs = PoolSmem(g.nch, g.xs_floats, 2).bytes <= 227 * 1024 && !(g.dbg & 32) ? 2 : 1;
        const PoolSmem L2(g.nch, g.xs_floats, g.rbufs);
        static bool configured = false;
        if (!configured) {
            cudaFuncSetAttribute(conv_pool_kernel<G, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            configured = true;
        }
        conv_pool_kernel<G, 8><<<grid, PEpi<8>::kThreads, L2.bytes, s>>>(g);
    } else {
        static bool configured = false;
        if (!configured) {
            cudaFuncSetAttribute(conv_pool_kernel<GeoDyn, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            cudaFuncSetAttribute(conv_pool_kernel<GeoDyn, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            configured = true;
        }
        if (mode == 1)
            conv_pool_kernel<GeoDyn, 16><<<grid, PEpi<16>::kThreads, L.bytes, s>>>(g);
        else
            conv_pool_kernel<GeoDyn, 8><<<grid, PEpi<8>::kThreads, L.bytes, s>>>(g);
    }
    return check_launch("conv_pool_kernel");
}

}  // namespace bnn



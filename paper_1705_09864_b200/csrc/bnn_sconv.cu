// Small-channel binary convolution on tcgen05 (ResNet-18 layers 1-2 and their 1x1
// downsamples: C = 64 or 128 input channels, F = 64 or 128 filters).
//
// Replaces the same reference path as bnn_umma_impl.cuh -- QConv2d.forward(INFER_PACKED)
// (layers.py:225-245) = im2col (tensor.py:60-78) -> pack_matrix_b (bitpack.py:152-169)
// -> xnor_gemm (gemm.py:128-139) with the G2 "+1" padding -- bit-identically, for the
// shapes whose channel words are too narrow for the 32-byte TMA im2col route.
//
// Orientation: GEMM rows = 128 output pixels per tile (TMEM lanes), columns = the F
// filters.  Per CTA (persistent, one per SM):
//   * the packed weights [F, kh*kw*Cw] u64 (tap-major, bnn_conv_weights_reorder) are
//     expanded ONCE into e2m1 codes in shared memory (SWIZZLE_128B K-major, the MMA's B
//     operand), with their popcounts -- filter-stationary, never re-read;
//   * per tile, one thread issues a single bulk copy (cp.async.bulk, the TMA engine) of
//     the contiguous band of packed NHWC input rows the tile's 128 pixels touch;
//   * 4 expander warps (thread = pixel = TMEM lane) gather their taps from the band
//     (out-of-image taps read the all-ones "+1" word), count popc, expand every bit to
//     an e2m1 nibble and write the row straight into TMEM (tcgen05.st) -- the A operand
//     of tcgen05.mma...kind::mxf4 (A from TMEM, B from SMEM), one kernel row (kw taps)
//     per ring slot;
//   * one thread issues the MMAs (M = 128, N = F, K = 64 per instruction), committing
//     ring slots back to the expanders and finished tiles to the epilogue
//     (double-buffered TMEM accumulators: tile i's epilogue overlaps tile i+1's MMAs);
//   * 8 epilogue warps read the f32 accumulators C = popc(a & b) (tcgen05.ld), decode
//     P = K - popc(pixel) - popc(filter) + 2C (or 2P - K), apply the fused BN in the
//     reference op order (layers.py:598-602), add the residual, store f32 NCHW (for a
//     fixed filter the 32 lanes of a warp are 32 consecutive pixels: coalesced), and
//     build each pixel's sign-pack word in its own lane (the next layer's input).
// The e2m1 codes are those of the kind::mxf4 engine (bnn_umma_impl.cuh): pixel bits
// -> {2, 1, 0.5, 0.5}, filter bits -> {0.5, 1, 2, 2} by bit position, every product of
// two set bits exactly 1.0, f32 accumulation exact for K < 2^24.
#include "bnn_umma_impl.cuh"

namespace bnn {
namespace sconv {

using umma::expand_fp4_a;
using umma::expand_fp4_b;
using umma::fence_after;
using umma::fence_before;
using umma::mbar_arrive;
using umma::mbar_arrive_expect_tx;
using umma::mbar_init;

using umma::mbar_wait_sleep;
using umma::sw128_desc;
using umma::tmem_ld32;
using umma::tmem_st8;
using umma::umma_commit;

constexpr int kRows = 128;        // output pixels per tile (TMEM lanes)
constexpr int kExpHalves = 2;     // expander threads per pixel row: the lo / hi 32 bits of a word
constexpr int kExpWarps = 4 * kExpHalves;  // (two warps per scheduler hide each other's latency)
constexpr int kSetWarps = kExpWarps;  // every expander warp arrives on the tile's barriers
constexpr int kEpiWarps = 8;      // epilogue warps (2 per quadrant)
constexpr int kLoadWarp = kExpWarps;
constexpr int kMmaWarp = kExpWarps + 1;
constexpr int kEpiWarp0 = kExpWarps + 2;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kBandSlots = 3;
constexpr int kPopcBufs = 8;  // pixel-popcount buffers (expanders run up to 8 tiles ahead)



// A-operand ring in shared memory: `slots` chunks of chunk_rows kernel rows (the expanded
// pixel rows, SWIZZLE_128B K-major, 16 KB per 4 K-steps of 64 bits); TMEM holds the
// Cfg::kAcc accumulator buffers [0, kAcc * F) and the UE8M0 scale factors from sf_col
struct TmemPlan {
    int chunk_rows, nchunks, slots, slot_bytes, sf_col;
};

struct Geom {
    const uint64_t *x;      // packed NHWC [B, H, W, Cw]
    const uint64_t *w;      // tap-major weights [F, kh * kw * Cw]
    float *y;               // f32 NCHW [B, F, oh, ow] (may be null: packed output only)
    const float *res;       // residual, same layout as y (may be null)
    int H, W, kh, kw, sh, sw, ph, pw, oh, ow;
    int64_t npix, ntiles;
    int band_bytes;         // bytes of one band slot
    int K;                  // C * kh * kw
    uint64_t *trace;        // debug timeline of CTA 0 (bnn_umma_trace + debug bit 16), or null
    int spin;               // latency-critical waits spin on test_wait (debug bit 1 << 20: off)
    int dbg;                // debug ablations (wrong results): 1 no MMAs, 2 no epilogue work,
                            // 4 no TMEM stores of the expanders
    TmemPlan tp;            // A-ring chunking (tmem_plan)
    unsigned long long *hang;  // debug: records of waits that spun > 2^26 (host-mapped), or null
};

// one elected lane of a converged warp (the warp runs the issue loop with warp-uniform
// values, which the compiler keeps in uniform registers; only the elected lane issues)
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

// debug: %globaltimer of event ev of CTA 0's local tile it (it < 64)
__device__ __forceinline__ void stamp(const Geom &g, int ev, int it) {
    if (g.trace != nullptr && blockIdx.x == 0 && it < 64) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g.trace[ev * 64 + it] = t;  // (ev < 16)
    }
}

template <int kF, int kCw, int kKw>
struct Cfg {
    static constexpr int kRowSteps = kKw * kCw;      // MMAs (K = 64) per kernel row
    static constexpr int kRowCols = kRowSteps * 8;   // TMEM columns per kernel row (32 B / 8 col)
    static constexpr int kAccCols = kF;
    // TMEM accumulator buffers (the MMA runs up to kAcc - 1 tiles ahead of the epilogue)
    static constexpr int kAcc = (512 - 32) / kF >= 4 ? 4 : (512 - 32) / kF;
    static constexpr int kMaxSlots = 8;
    // kind::mxf4, E2M1 x E2M1, UE8M0 scales, f32 accumulate, M = 128, N = kF
    static constexpr uint32_t kIdesc = (1u << 7) | (1u << 10) | ((uint32_t)(kF >> 3) << 17) |
                                       (1u << 23) | ((uint32_t)(kRows >> 4) << 24);
};

constexpr int kMaxChunkRows = 3;
// the largest chunk (kernel rows, <= kMaxChunkRows) of which at least two slots fit in
// `budget` bytes, up to 4 slots
inline bool ring_plan(int F, int kh, int row_steps, int budget, TmemPlan &p) {
    for (int r = kh < kMaxChunkRows ? kh : kMaxChunkRows; r >= 1; --r) {
        const int bytes = ((r * row_steps + 3) / 4) * 16384;
        const int n = budget / bytes;
        if (n >= 2) {
            p.chunk_rows = r;
            p.nchunks = (kh + r - 1) / r;
            p.slots = n > 4 ? 4 : n;
            p.slot_bytes = bytes;
            p.sf_col = ((512 - 32) / F >= 4 ? 4 : (512 - 32) / F) * F;  // after Cfg::kAcc buffers
            return true;
        }
    }
    return false;
}

// shared memory carve-up (runtime: the weight block depends on K, the band on the shape)
struct Smem {
    uint32_t a, w, band, par, aff, thr, popc_f, popc_p, bars, tmem, total;
    __host__ __device__ Smem(int F, int K, int band_bytes, int ring_bytes) {
        const int wblocks = (K + 255) / 256;
        a = 0;                 // A ring (1024-aligned SW128 blocks)
        w = a + ring_bytes;    // expanded weights (SW128 blocks)
        band = w + wblocks * F * 128;
        par = band + kBandSlots * ((band_bytes + 127) / 128) * 128;  // float4 [128] BN
        aff = par + 128 * 16;                                        // float2 [128] scale, shift
        thr = aff + 128 * 8;                                         // float2 [128] sign thresholds
        popc_f = thr + 128 * 8 + 64;                                 // (+ int [8] group flags)
        popc_p = popc_f + 128 * 4;
        bars = popc_p + kPopcBufs * kExpHalves * kRows * 4;
        tmem = bars + 64 * 8;
        total = tmem + 16;
    }
};

template <int kF, int kCw, int kKw, bool kPack>
__global__ void __launch_bounds__(kThreads, 1)
    xnor_sconv_kernel(const __grid_constant__ Geom g, const __grid_constant__ Epilogue ep) {
    using C = Cfg<kF, kCw, kKw>;
    constexpr int kSlots = C::kMaxSlots;  // barrier array size (g.tp.slots are used)
    const int slots = g.tp.slots, nchunks = g.tp.nchunks, crows = g.tp.chunk_rows;
    const uint32_t slot_bytes = g.tp.slot_bytes, sf_col = g.tp.sf_col;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sraw = smem_u32(smem_raw);
    const uint32_t sbase = (sraw + 1023u) & ~1023u;
    uint8_t *sgen = smem_raw + (sbase - sraw);
    const Smem L(kF, g.K, g.band_bytes, g.tp.slots * g.tp.slot_bytes);
    const uint32_t s_w = sbase + L.w;
    const uint32_t s_a = sbase + L.a;
    const uint32_t s_band = sbase + L.band;
    const uint32_t band_pitch = ((g.band_bytes + 127) / 128) * 128;
    int32_t *s_popc_f = reinterpret_cast<int32_t *>(sgen + L.popc_f);
    float4 *s_par = reinterpret_cast<float4 *>(sgen + L.par);  // per filter {mean, inv, gamma, beta}
    float2 *s_aff = reinterpret_cast<float2 *>(sgen + L.aff);  // per filter {scale, shift}
    float2 *s_thr = reinterpret_cast<float2 *>(sgen + L.thr);  // per filter sign threshold {S, V}
    int32_t *s_thr_ok = reinterpret_cast<int32_t *>(sgen + L.thr + 128 * 8);  // [8] per 16 filters
    int32_t *s_popc_p = reinterpret_cast<int32_t *>(sgen + L.popc_p);
    const uint32_t bar_bfull = sbase + L.bars;          // [kBandSlots] band landed
    const uint32_t bar_bempty = bar_bfull + 8 * kBandSlots;  // [kBandSlots] band consumed
    const uint32_t bar_afull = bar_bempty + 8 * kBandSlots;  // [kSlots] A chunk in TMEM
    const uint32_t bar_aempty = bar_afull + 8 * kSlots;      // [kSlots] MMAs read the chunk
    constexpr int kAcc = C::kAcc;
    const uint32_t bar_tfull = bar_aempty + 8 * kSlots;      // [kAcc] accumulator ready
    const uint32_t bar_tempty = bar_tfull + 8 * kAcc;        // [kAcc] accumulator drained
    const uint32_t bar_pfull = bar_tempty + 8 * kAcc;        // [kPopcBufs] pixel popcounts ready
    const uint32_t bar_pempty = bar_pfull + 8 * kPopcBufs;   // [kPopcBufs] popcounts read
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sgen + L.tmem);

    // latency-critical waits spin on test_wait: the suspend-hint try_wait measured
    // ~0.5 us of wake-up latency per wait on the expander -> MMA -> epilogue chain
    // (a wait that has not completed after ~2^28 probes -- seconds -- traps instead of
    // hanging the GPU: a pipeline bug surfaces as a launch error)
    auto mbar_wait = [&](uint32_t bar, uint32_t phase, uint32_t aux = 0, uint32_t backoff = 0) {
        if (!g.spin) {
            umma::mbar_wait(bar, phase);
            return;
        }
        uint32_t done = 0, tries = 0;
        do {
            asm volatile(
                "{\n.reg .pred p;\n"
                "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                "selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(bar), "r"(phase)
                : "memory");
            if (++tries == (1u << 26) && (threadIdx.x & 31) == 0 && g.hang != nullptr) {
                const unsigned k = (unsigned)atomicAdd(&g.hang[0], 1ull) % 256u;
                g.hang[1 + k] = ((unsigned long long)blockIdx.x << 48) |
                                ((unsigned long long)(threadIdx.x >> 5) << 40) |
                                ((unsigned long long)((bar - sbase - L.bars) >> 3) << 32) |
                                ((unsigned long long)phase << 31) | aux;
                __threadfence_system();
            }
            if (tries > (1u << 28)) asm volatile("trap;");
            if (!done && backoff) __nanosleep(backoff);  // (waiters off the critical path)
        } while (!done);
    };
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ohw = g.oh * g.ow;
    const int cw_row = g.W * kCw;  // u64 words per input row

    if (tid == 0) {
        for (int i = 0; i < kBandSlots; ++i) {
            mbar_init(bar_bfull + 8 * i, 1);
            mbar_init(bar_bempty + 8 * i, kSetWarps);
        }
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(bar_afull + 8 * i, kSetWarps);
            mbar_init(bar_aempty + 8 * i, 1);
        }
        for (int i = 0; i < kAcc; ++i) {
            mbar_init(bar_tfull + 8 * i, 1);
            mbar_init(bar_tempty + 8 * i, kEpiWarps);
        }
        for (int i = 0; i < kPopcBufs; ++i) {
            mbar_init(bar_pfull + 8 * i, kSetWarps);
            mbar_init(bar_pempty + 8 * i, kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *s_tmem;
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // (see bnn_wconv.cu)

    // ---- weights: expanded once into the SW128 K-major B operand (+ filter popcounts)
    {
        const int kw32 = g.K / 32;  // u32 words per filter row
        const uint32_t *w32 = reinterpret_cast<const uint32_t *>(g.w);
        for (int f = warp; f < kF; f += kThreads / 32) {
            int32_t pc = 0;
            for (int q = lane; q < kw32; q += 32) {
                const uint32_t v = __ldg(w32 + (int64_t)f * kw32 + q);
                pc += __popc(v);
                uint32_t r4[4];
                expand_fp4_b(v, r4);
                const uint32_t addr = s_w + (q >> 3) * (kF * 128) + f * 128 + (((q & 7) ^ (f & 7)) << 4);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(r4[0]),
                             "r"(r4[1]), "r"(r4[2]), "r"(r4[3]));
            }
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, d);
            if (lane == 0) s_popc_f[f] = pc;
        }
        // per-filter epilogue parameters, read by every lane of the epilogue (broadcast)
        for (int f = tid; f < kF; f += kThreads) {
            float4 bp = make_float4(0.0f, 1.0f, 1.0f, 0.0f);
            if (ep.bn_mean != nullptr) {
                bp.x = ep.bn_mean[f];
                bp.y = ep.bn_inv[f];
                bp.z = ep.bn_gamma[f];
                bp.w = ep.bn_beta[f];
            }
            float2 af = make_float2(1.0f, 0.0f);
            if (ep.scale != nullptr) af.x = ep.scale[f];
            if (ep.shift != nullptr) af.y = ep.shift[f];
            s_par[f] = bp;
            s_aff[f] = af;
        }
        // UE8M0 scale factors = 1.0 in every TMEM column from kSfCol on (both operands)
        if (warp < 4) {
            const uint32_t one[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                     0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
            for (int col = (int)sf_col; col < 512; col += 8)
                tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + col, one);
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        fence_before();
        __syncthreads();
        fence_after();
        // Packed-only outputs need just sign(f(x)) of the epilogue chain f (domain map,
        // affine, BN): every op of f is a monotone f32 rounding, so f is monotone in the
        // exact integer x and {x : f(x) >= 0} is a prefix or suffix of the x range -- one
        // per-filter threshold on a = 2C + (K - popc(pixel)) = P + popc(filter), found by
        // a binary search that evaluates f with the epilogue's own ops (bit-identical to
        // the sign of the computed value).  {S, V}: bit = S * a - V >= 0.  A filter whose
        // outputs can be non-finite keeps the full chain (V = NaN: flag + sign).
        for (int f = tid; f < kF; f += kThreads) {
            const float4 bp = s_par[f];
            const float2 af = s_aff[f];
            const bool dot = ep.domain == BNN_DOT;
            const int K = g.K;
            auto fx = [&](int P) {  // the epilogue chain for popcount-domain value P
                float x = dot ? (float)(2 * P - K) : (float)P;
                if (ep.scale || ep.shift) x = __fadd_rn(__fmul_rn(x, af.x), af.y);
                if (ep.bn_mean) x = __fadd_rn(__fmul_rn(bp.z, __fmul_rn(__fsub_rn(x, bp.x), bp.y)), bp.w);
                return x;
            };
            const float f0 = fx(0), f1 = fx(K);
            float2 t;
            if (!isfinite(f0) || !isfinite(f1)) {
                t = make_float2(0.0f, __int_as_float(0x7fffffff));  // general path
            } else {
                const bool inc = f1 >= f0;
                // first P in [0, K + 1) whose bit differs from the bit at P = 0 ... K's start
                const bool b0 = f0 >= 0.0f;
                int lo = 0, hi = K + 1;  // invariant: bit(P) == b0 for P < lo; differs at hi
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if ((fx(mid) >= 0.0f) == b0) lo = mid + 1;
                    else hi = mid;
                }
                // bits: b0 on [0, lo), !b0 on [lo, K]; inc => b0 == 0 unless constant
                const float U = (float)(lo + s_popc_f[f]);  // threshold on a = P + popc(f)
                if (lo > K) t = make_float2(0.0f, b0 ? -1.0f : 1.0f);      // constant bit b0
                else if (!b0) t = make_float2(1.0f, U);                     // a >= U
                else t = make_float2(-1.0f, -(U - 0.5f));                    // a < U
                (void)inc;
            }
            s_thr[f] = t;
        }
        __syncthreads();
        if (tid < kF / 16) {
            int ok = 1;
            for (int j = 0; j < 16; ++j) ok &= s_thr[tid * 16 + j].y == s_thr[tid * 16 + j].y;
            s_thr_ok[tid] = ok;
        }
        __syncthreads();
    }
    // (the setup above reads load-time constants only: it overlaps the previous kernel's tail)
    asm volatile("griddepcontrol.wait;\n" ::: "memory");

    const int64_t t0 = blockIdx.x, tstep = gridDim.x;
    // the contiguous range of flat input rows (b * H + iy) a tile's pixels touch
    // (index math in f32 reciprocals: npix < 2^24 is a launch precondition, so n * (1/d)
    // is within 1 of n / d and two corrections make it exact -- integer divisions are
    // long dependent chains on the expanders' critical path)
    const uint32_t uohw = (uint32_t)ohw, uow = (uint32_t)g.ow, unpix = (uint32_t)g.npix;
    const float inv_ohw = 1.0f / (float)ohw, inv_ow = 1.0f / (float)g.ow;
    auto fdiv = [](uint32_t n, uint32_t d, float inv) {
        int q = (int)__fmul_rz((float)n, inv);
        int r = (int)n - q * (int)d;
        if (r < 0) { --q; r += (int)d; }
        if (r < 0) { --q; r += (int)d; }
        if (r >= (int)d) { ++q; r -= (int)d; }
        if (r >= (int)d) { ++q; }
        return (uint32_t)q;
    };
    auto band_rows = [&](int64_t tile, int &lo, int &n) {
        const uint32_t m0 = (uint32_t)tile * kRows;
        const uint32_t m1 = (m0 + kRows < unpix ? m0 + kRows : unpix) - 1;
        const int b0 = (int)fdiv(m0, uohw, inv_ohw), b1 = (int)fdiv(m1, uohw, inv_ohw);
        const int oy0 = (int)fdiv(m0 - (uint32_t)b0 * uohw, uow, inv_ow);
        const int oy1 = (int)fdiv(m1 - (uint32_t)b1 * uohw, uow, inv_ow);
        int iy0 = oy0 * g.sh - g.ph, iy1 = oy1 * g.sh - g.ph + g.kh - 1;
        iy0 = iy0 < 0 ? 0 : iy0;
        iy1 = iy1 > g.H - 1 ? g.H - 1 : iy1;
        lo = b0 * g.H + iy0;
        n = b1 * g.H + iy1 - lo + 1;
    };

    if (warp < kExpWarps) {
        // ============================================================ expanders
        // thread = (pixel row, half): half h expands the lo (h = 0) / hi (h = 1) 32 bits of
        // every 64-bit tap word of its pixel
        const int q = warp & 3;
        const int hx = warp >> 2;
        const int row = q * 32 + lane;
        int it = 0;
#pragma unroll 1
        for (int64_t tile = t0; tile < g.ntiles; tile += tstep, ++it) {
            const int bs = it % kBandSlots;
            mbar_wait(bar_bfull + 8 * bs, (uint32_t)(it / kBandSlots) & 1u, it);
            if (q == 0 && lane == 0) stamp(g, 1, it);
            int lo, nrows;
            band_rows(tile, lo, nrows);
            const uint32_t band = s_band + bs * band_pitch;
            const uint32_t m = (uint32_t)tile * kRows + row;
            const bool mok = m < unpix;
            const int b = mok ? (int)fdiv(m, uohw, inv_ohw) : 0;
            const int p = mok ? (int)(m - (uint32_t)b * uohw) : 0;
            const int oy = (int)fdiv((uint32_t)p, uow, inv_ow), ox = p - oy * g.ow;
            const int iy0 = oy * g.sh - g.ph, ix0 = ox * g.sw - g.pw;
            const int rbase = b * g.H - lo;  // band row of image row 0
            int32_t popc = 0;
#pragma unroll 1
            for (int ch = 0; ch < nchunks; ++ch) {
                // chunk ch = kernel rows [i0, i1): one ring slot, one arrival
                const uint32_t gc = (uint32_t)it * (uint32_t)nchunks + (uint32_t)ch;
                const int slot = (int)(gc % (uint32_t)slots);
                const int i0 = ch * crows, i1 = (i0 + crows < g.kh) ? i0 + crows : g.kh;
                // all of the chunk's band words first (independent shared loads in flight)
                // (branch-free: every lane loads from a clamped, always-valid band position
                // and selects the "+1" word for out-of-image taps -- no divergent regions)
                uint32_t v[kMaxChunkRows][kKw][kCw];
#pragma unroll
                for (int r = 0; r < kMaxChunkRows; ++r) {
                    const int iy = iy0 + i0 + r;
                    const bool yok = (i0 + r < i1) && (unsigned)iy < (unsigned)g.H;
                    int brow = rbase + iy;
                    brow = brow < 0 ? 0 : (brow > nrows - 1 ? nrows - 1 : brow);
#pragma unroll
                    for (int j = 0; j < kKw; ++j) {
                        const int ix = ix0 + j;
                        const bool ok = yok && (unsigned)ix < (unsigned)g.W;
                        const int bx = ix < 0 ? 0 : (ix > g.W - 1 ? g.W - 1 : ix);
                        const uint32_t src = band + (uint32_t)((brow * cw_row + bx * kCw) * 8) + 4 * hx;
#pragma unroll
                        for (int c = 0; c < kCw; ++c) {
                            uint32_t w32;
                            asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(w32) : "r"(src + 8 * c));
                            w32 = ok ? w32 : 0xffffffffu;  // out of image: "+1" (G2)
                            v[r][j][c] = mok ? w32 : 0u;    // rows past npix: zero codes
                        }
                    }
                }
                if (i1 == g.kh) {  // the band is no longer needed by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_bempty + 8 * bs);
                }
                if (ch == 0 && warp == 0 && lane == 0) stamp(g, 11, it);
                // the slot's previous chunk has been read by its MMAs
                if (gc >= (uint32_t)slots)
                    mbar_wait(bar_aempty + 8 * slot, ((gc / (uint32_t)slots) - 1) & 1u, gc);
                // pixel row -> e2m1 codes in the slot's SW128 K-major layout: u32 word k of
                // the chunk row -> block k / 8, 16-byte chunk (k % 8) ^ (row % 8)
                const uint32_t rowbase = s_a + slot * slot_bytes + row * 128;
#pragma unroll
                for (int r = 0; r < kMaxChunkRows; ++r) {
                    if (i0 + r >= i1 || (g.dbg & 8)) break;
#pragma unroll
                    for (int j = 0; j < kKw; ++j)
#pragma unroll
                        for (int c = 0; c < kCw; ++c) {
                            const uint32_t w = v[r][j][c];
                            popc += __popc(w);
                            uint32_t r4[4];
                            expand_fp4_a(w, r4);
                            const int k = 2 * ((r * kKw + j) * kCw + c) + hx;
                            const uint32_t addr = rowbase + (k >> 3) * 16384 + (((k & 7) ^ (row & 7)) << 4);
                            if (!(g.dbg & 4))
                                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr),
                                             "r"(r4[0]), "r"(r4[1]), "r"(r4[2]), "r"(r4[3]));
                            else if (r4[0] == 0x12345u && r4[3] == 0x54321u) popc += 7;
                        }
                }
                if (ch == 0 && warp == 0 && lane == 0) stamp(g, 12, it);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_afull + 8 * slot);
                if (ch == 0 && warp == 0 && lane == 0) stamp(g, 13, it);
            }
            if (q == 0 && lane == 0) stamp(g, 2, it);
            // this tile's pixel popcounts for the epilogue (double-buffered)
            const int pb = it % kPopcBufs;
            if (it >= kPopcBufs) mbar_wait(bar_pempty + 8 * pb, (uint32_t)((it / kPopcBufs) - 1) & 1u, it);
            s_popc_p[(pb * kExpHalves + hx) * kRows + row] = popc;
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_pfull + 8 * pb);
        }
    } else if (warp == kLoadWarp) {
        // ============================================================ band loader
        // (the whole warp runs the loop with uniform values; one elected lane issues)
        {
            int it = 0;
#pragma unroll 1
            for (int64_t tile = t0; tile < g.ntiles; tile += tstep, ++it) {
                const int bs = it % kBandSlots;
                if (it >= kBandSlots) mbar_wait(bar_bempty + 8 * bs, (uint32_t)((it / kBandSlots) - 1) & 1u, it, 64);
                int lo, nrows;
                band_rows(tile, lo, nrows);
                const uint32_t bytes = (uint32_t)nrows * (uint32_t)cw_row * 8u;
                if (elect_one()) {
                stamp(g, 0, it);
                mbar_arrive_expect_tx(bar_bfull + 8 * bs, bytes);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                        s_band + bs * band_pitch),
                    "l"(g.x + (int64_t)lo * cw_row), "r"(bytes), "r"(bar_bfull + 8 * bs)
                    : "memory");
                }
                __syncwarp();
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp) {
        // ============================================================ MMA issuer
        // (the whole warp runs the issue loop: descriptors stay warp-uniform, in uniform
        // registers; one elected lane issues each tcgen05.mma / commit)
        {
            int it = 0;
#pragma unroll 1
            for (int64_t tile = t0; tile < g.ntiles; tile += tstep, ++it) {
                const int buf = it % kAcc;
                if (lane == 0) stamp(g, 7, it);
                if (it >= kAcc) {
                    mbar_wait(bar_tempty + 8 * buf, (uint32_t)((it / kAcc) - 1) & 1u, 1000000 + it);
                    fence_after();  // the epilogue's tcgen05.ld of d precede these MMAs
                }
                if (lane == 0) stamp(g, 8, it);
                const uint32_t d = tmem + buf * C::kAccCols;
                int step = 0;  // K step (64 bits) within the tile
#pragma unroll 1
                for (int ch = 0; ch < nchunks; ++ch) {
                    const uint32_t gc = (uint32_t)it * (uint32_t)nchunks + (uint32_t)ch;
                    const int slot = (int)(gc % (uint32_t)slots);
                    mbar_wait(bar_afull + 8 * slot, (gc / (uint32_t)slots) & 1u, 2000000 + gc);
                    if (ch == 0 && lane == 0) stamp(g, 3, it);
                    // (operands are in SMEM, written by st.shared + fence.proxy.async before the
                    // expanders' arrival: no tcgen05 fence per chunk)
                    const int i0 = ch * crows, i1 = (i0 + crows < g.kh) ? i0 + crows : g.kh;
                    const int nsteps = (i1 - i0) * C::kRowSteps;
                    // descriptors: chunk base + compile-time offsets (no per-MMA address math);
                    // the start-address field is addr >> 4 (14 bits, no carry out of it)
                    const uint64_t da0 = sw128_desc(s_a + slot * slot_bytes);
                    const uint64_t db0 = sw128_desc(s_w);
                    if (elect_one()) {
#pragma unroll
                        for (int s2 = 0; s2 < kMaxChunkRows * C::kRowSteps; ++s2) {
                            if (s2 < nsteps && !(g.dbg & 1)) {
                                const int st = step + s2;
                                const uint64_t da = da0 + (uint64_t)((((s2 >> 2) * 16384) + (s2 & 3) * 32) >> 4);
                                const uint64_t db = db0 + (uint64_t)((((st >> 2) * (kF * 128)) + (st & 3) * 32) >> 4);
                                umma::mma_fp4<C::kIdesc>(d, da, db, tmem + sf_col, tmem + sf_col,
                                                         st != 0 ? 1u : 0u);
                            }
                        }
                    }
                    __syncwarp();
                    step += nsteps;
                    if (ch == 0 && lane == 0) stamp(g, 9, it);
                    if (elect_one()) umma_commit(bar_aempty + 8 * slot);
                    __syncwarp();
                    if (ch == 0 && lane == 0) stamp(g, 10, it);
                }
                if (elect_one()) umma_commit(bar_tfull + 8 * buf);
                __syncwarp();
                if (lane == 0) stamp(g, 4, it);
            }
            // keep TMEM allocated until the epilogue drained the last accumulators
            for (int t = it - kAcc; t < it; ++t)
                if (t >= 0) mbar_wait(bar_tempty + 8 * (t % kAcc), (uint32_t)(t / kAcc) & 1u);
        }
        __syncwarp();
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    } else {
        // ============================================================ epilogue
        const int e = warp - kEpiWarp0;
        const int q = warp & 3, h = e >> 2;
        const bool dot = ep.domain == BNN_DOT;
        const bool affine = ep.scale || ep.shift;
        const bool has_bn = ep.bn_mean != nullptr;
        const float kf = (float)g.K;
        int it = 0;
#pragma unroll 1
        for (int64_t tile = t0; tile < g.ntiles; tile += tstep, ++it) {
            const int buf = it % kAcc, pb = it % kPopcBufs;
            mbar_wait(bar_tfull + 8 * buf, (uint32_t)(it / kAcc) & 1u, 3000000 + it, 64);
            mbar_wait(bar_pfull + 8 * pb, (uint32_t)(it / kPopcBufs) & 1u, 4000000 + it, 64);
            if (e == 0 && lane == 0) stamp(g, 5, it);
            fence_after();
            const uint32_t m32 = (uint32_t)tile * kRows + q * 32 + lane;
            const int64_t m = m32;
            const bool mok = m32 < unpix;
            const int64_t b = mok ? (int64_t)fdiv(m32, uohw, inv_ohw) : 0;
            const int64_t p = mok ? (int64_t)(m32 - (uint32_t)b * uohw) : 0;
            const int64_t obase = b * kF * ohw + p;  // (b, filter 0, p) of NCHW y / res
            const float rowf = kf - (float)(s_popc_p[(pb * kExpHalves) * kRows + q * 32 + lane] +
                                            s_popc_p[(pb * kExpHalves + 1) * kRows + q * 32 + lane]);
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_pempty + 8 * pb);  // (the popcounts are in registers)
            // 16-column groups: this warp's groups g = h, h + 2, ... of the quadrant's rows
#pragma unroll 1
            for (int cg = h; cg * 16 < kF && !(g.dbg & 2); cg += kEpiWarps / 4) {
                uint32_t v[16];  // counts C, then (in place) the f32 outputs
                umma::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + buf * C::kAccCols + cg * 16, v);
                if (kPack && g.y == nullptr && g.res == nullptr && s_thr_ok[cg]) {
                    // packed output only: the per-filter sign thresholds (prologue); groups
                    // with a possibly non-finite filter take the full chain below
                    uint32_t half = 0;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float2 t = s_thr[cg * 16 + j];
                        const float a = __fmaf_rn(2.0f, __uint_as_float(v[j]), rowf);  // P + popc(f)
                        half |= (__fmaf_rn(t.x, a, -t.y) >= 0.0f ? 1u : 0u) << j;
                    }
                    if (mok) reinterpret_cast<uint16_t *>(ep.pack_out)[m * 2 * ep.pack_ld32 + cg] = (uint16_t)half;
                    continue;
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int n = cg * 16 + j;
                    // P = K - popc(pixel) - popc(filter) + 2C, exact in f32
                    const float P = __fmaf_rn(2.0f, __uint_as_float(v[j]),
                                              rowf - (float)s_popc_f[n]);
                    float x = dot ? __fmaf_rn(2.0f, P, -kf) : P;
                    if (affine) {
                        const float2 a = s_aff[n];
                        x = __fadd_rn(__fmul_rn(x, a.x), a.y);
                    }
                    if (has_bn) {
                        const float4 bp = s_par[n];  // reference op order, layers.py:598-602
                        x = __fadd_rn(__fmul_rn(bp.z, __fmul_rn(__fsub_rn(x, bp.x), bp.y)), bp.w);
                    }
                    v[j] = __float_as_uint(x);
                }
                if (mok) {
                    const int64_t o = obase + (int64_t)cg * 16 * ohw;
                    if (g.res) {  // all loads in flight before the adds
                        float r[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) r[j] = __ldg(g.res + o + (int64_t)j * ohw);
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            v[j] = __float_as_uint(__fadd_rn(__uint_as_float(v[j]), r[j]));
                    }
                    if (g.y) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) g.y[o + (int64_t)j * ohw] = __uint_as_float(v[j]);
                    }
                    if constexpr (kPack) {
                        uint32_t half = 0;
                        float nf = 0.0f;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const float fj = __uint_as_float(v[j]);
                            half |= (fj >= 0.0f ? 1u : 0u) << j;  // sign(-0) = +1
                            nf = __fmaf_rn(fj, 0.0f, nf);         // NaN iff some f is NaN / Inf
                        }
                        reinterpret_cast<uint16_t *>(ep.pack_out)[m * 2 * ep.pack_ld32 + cg] = (uint16_t)half;
                        if (ep.pack_flags && nf != 0.0f) atomicOr(ep.pack_flags, BNN_FLAG_NONFINITE);
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_tempty + 8 * buf);
            if (e == 0 && lane == 0) stamp(g, 6, it);
        }
    }
    fence_before();
    __syncthreads();
}

}  // namespace sconv

// Eligible shapes: C in {64, 128}, F in {64, 128}, kw * C / 64 <= 8, an even number
// of u64 words per input row (16-byte bulk copies) and a band that fits in SMEM.
// Returns BNN_EUNSUP otherwise (the caller takes the general engine).
int launch_sconv(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
                 const uint64_t *w, int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                 int64_t ph, int64_t pw, int64_t oh, int64_t ow, float *y, const Epilogue &ep,
                 cudaStream_t s, const float *res) {
    using namespace sconv;
    const int64_t Cw = C / 64;
    if (C % 64 != 0 || (Cw != 1 && Cw != 2) || (F != 64 && F != 128) || kw * Cw > 8 ||
        (W * Cw) % 2 != 0 || kh > 16)
        return BNN_EUNSUP;
    if (ep.pack_out && ep.pack_ld32 < F / 32) return BNN_EUNSUP;
    if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return BNN_EUNSUP;
    const int64_t npix = B * oh * ow, ohw = oh * ow;
    const int64_t ntiles = ceil_div(npix, kRows);
    if (npix >= (1ll << 24) || B * H * W * Cw >= (1ll << 31)) return BNN_EUNSUP;
    // the largest band over all tiles (flat input rows b * H + iy), cached per geometry
    // (an eager caller re-launches the same layer every step)
    static thread_local int64_t cache_key[8] = {-1}, cache_rows = 0;
    const int64_t key[8] = {B, H, W, oh, ow, sh, ph, kh};
    int64_t max_rows = 0;
    bool hit = true;
    for (int i = 0; i < 8; ++i) hit = hit && cache_key[i] == key[i];
    if (hit) {
        max_rows = cache_rows;
    } else {
        // a tile's band depends only on its first pixel modulo ohw (and the batch edge):
        // one period of lcm(ohw, kRows) / kRows tiles, plus the last tile, covers all
        int64_t a = ohw, bb = kRows;
        while (bb) { const int64_t r = a % bb; a = bb; bb = r; }
        const int64_t period = ohw / a;  // lcm(ohw, kRows) / kRows
        for (int64_t t = 0; t < ntiles; ++t) {
            if (t > period && t != ntiles - 1) continue;
            const int64_t m0 = t * kRows, m1 = (m0 + kRows < npix ? m0 + kRows : npix) - 1;
            const int64_t b0 = m0 / ohw, b1 = m1 / ohw;
            const int64_t oy0 = (m0 - b0 * ohw) / ow, oy1 = (m1 - b1 * ohw) / ow;
            int64_t iy0 = oy0 * sh - ph, iy1 = oy1 * sh - ph + kh - 1;
            iy0 = iy0 < 0 ? 0 : iy0;
            iy1 = iy1 > H - 1 ? H - 1 : iy1;
            const int64_t rows = b1 * H + iy1 - (b0 * H + iy0) + 1;
            if (rows > max_rows) max_rows = rows;
        }
        for (int i = 0; i < 8; ++i) cache_key[i] = key[i];
        cache_rows = max_rows;
    }
    const int64_t band_bytes = max_rows * W * Cw * 8;
    const int K = (int)(C * kh * kw);
    if (band_bytes <= 0) return BNN_EUNSUP;
    Geom g{};
    g.x = x, g.w = w, g.y = y, g.res = res;
    g.H = (int)H, g.W = (int)W, g.kh = (int)kh, g.kw = (int)kw, g.sh = (int)sh, g.sw = (int)sw;
    g.ph = (int)ph, g.pw = (int)pw, g.oh = (int)oh, g.ow = (int)ow;
    g.npix = npix, g.ntiles = ntiles, g.band_bytes = (int)band_bytes, g.K = K;
    g.trace = (g_debug.umma_bits & 16) ? g_debug.trace_buf : nullptr;
    g.spin = (g_debug.umma_bits & (1 << 20)) ? 0 : 1;
    g.dbg = (int)((g_debug.umma_bits >> 21) & 15);
    g.hang = (g_debug.umma_bits & (1 << 30)) ? reinterpret_cast<unsigned long long *>(g_debug.trace_buf)
                                             : nullptr;
    {
        const Smem L0((int)F, K, (int)band_bytes, 0);  // everything but the A ring
        if (!ring_plan((int)F, (int)kh, (int)(kw * Cw), 227 * 1024 - 2048 - (int)L0.total, g.tp))
            return BNN_EUNSUP;
    }
    const Smem L((int)F, K, (int)band_bytes, g.tp.slots * g.tp.slot_bytes);
    if (L.total + 1024 > 227 * 1024) return BNN_EUNSUP;
    const int smem = (int)L.total + 1024;
    static int sms = 0;
    if (sms == 0) {
        sms = bnn_device_sm_count();
        if (sms <= 0) sms = 148;
    }
    int grid = (int)(ntiles < sms ? ntiles : sms);
    if (g_debug.grid_cap > 0 && grid > g_debug.grid_cap) grid = (int)g_debug.grid_cap;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool pack = ep.pack_out != nullptr;
#define BNN_SCONV(KF, KCW, KKW)                                                                   \
    if (F == KF && Cw == KCW && kw == KKW) {                                                      \
        static bool configured = false;                                                           \
        if (!configured) {                                                                        \
            cudaFuncSetAttribute(xnor_sconv_kernel<KF, KCW, KKW, true>,                           \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);        \
            cudaFuncSetAttribute(xnor_sconv_kernel<KF, KCW, KKW, false>,                          \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);        \
            configured = true;                                                                    \
        }                                                                                         \
        if (pack) cudaLaunchKernelEx(&cfg, xnor_sconv_kernel<KF, KCW, KKW, true>, g, ep);       \
        else cudaLaunchKernelEx(&cfg, xnor_sconv_kernel<KF, KCW, KKW, false>, g, ep);           \
        return check_launch("xnor_sconv_kernel");                                                 \
    }
    BNN_SCONV(64, 1, 3)
    BNN_SCONV(128, 1, 3)
    BNN_SCONV(128, 2, 3)
    BNN_SCONV(64, 2, 3)
    BNN_SCONV(64, 1, 1)
    BNN_SCONV(128, 1, 1)
    BNN_SCONV(128, 2, 1)
    BNN_SCONV(64, 2, 1)
#undef BNN_SCONV
    return BNN_EUNSUP;
}

}  // namespace bnn

// ResNet-18's float stem (conv7x7 / 2, pad 3, 3 -> 64 channels, 224-wide images;
// BASELINE configs[3]: "first conv ... full precision"; reference Conv2d,
// layers.py:81-141) on tcgen05 kind::tf32 WITHOUT an im2col gather.
//
// The trick: stage every input row once in shared memory as 16-byte entries
//     D[q] = (x[2q-4], x[2q-3], x[2q-2], x[2q-1]),  q = 0..113   (zero outside the row)
// so that output pixel p's 8-wide tap window x[2p-4 .. 2p+3] (kw = -1..6, the kw = -1
// weight is 0) is D[p] followed by D[p+2].  A NO-SWIZZLE K-major UMMA descriptor with
// SBO = 128 B (8 pixels x 16 B) and LBO = 32 B (the second 16-byte K chunk starts two
// entries later) reads exactly that: the two K chunks of a K = 8 MMA overlap in
// memory, and the "im2col matrix" of a (channel, kernel row) slice is the staged row
// itself.  (tools/probes/tf32_overlap.cu checks the descriptor and its rate.)
//
// Roles swap with respect to bnn_stem.cu: the WEIGHTS are the A operand, resident in
// TMEM for the whole kernel (128 lanes = 64 filters x {hi, lo} TF32 halves, 21 slices x
// 8 columns), and the 112 pixels of one conv row are the N dimension.  Per conv row:
//     D[lanes hi] = w_hi . (x_hi + x_lo),  D[lanes lo] = w_lo . (x_hi + x_lo)
// as 2 x 21 MMAs of 128 x 112 x 8 (B = the hi / lo staged rows), and the epilogue adds
// the two lane halves: all four terms of (w_hi + w_lo)(x_hi + x_lo), f32 accumulate.
// 42 MMAs x 56 cycles = 2352 cycles per conv row; the staged bytes per conv row are
// 6 new input rows x 2 x 1824 B instead of a 155 KB im2col tile.
//
//   warps 0-7   epilogue: TMEM -> registers (lane = filter half, 57 pixel columns),
//               hi + lo by one shuffle, then either the raw conv row (+ bias) or the
//               fused BN -> ReLU -> maxpool 3x3/2/1 (pool on sign-adjusted values before
//               the monotone BN, as in bnn_stem.cu) with the pooled rows kept in
//               registers, + the sign-packed words of the pooled output
//   warps 8-11  loader: input row pairs -> hi / lo D rows in an 8-slot ring (loads of the
//               next two pairs in flight)
//   warp 12     TMEM allocator + MMA issuer
#include "bnn_umma_impl.cuh"

namespace bnn {
namespace stem2 {

using namespace umma;

constexpr int kC = 3, kKH = 7, kKW = 7, kPad = 3, kW = 224, kOW = 112, kPW = 56, kNF = 64;
constexpr int kSlices = kC * kKH;           // K slices of 8: (channel, kernel row) x kw window
constexpr int kNQ = 114;                    // entries per staged row
constexpr int kRowB = kNQ * 16;             // 1824 bytes
constexpr int kPairB = 2 * kC * 2 * kRowB;  // [row in pair][channel][hi / lo]
constexpr int kNP = 8;                      // ring slots (input row pairs)
constexpr int kAcc = 3;                     // accumulators: TMEM columns 0, 112, 224
constexpr int kACol0 = kAcc * kOW;          // weights: columns [336, 504)
static_assert(kACol0 + 8 * kSlices <= 512, "TMEM budget");
constexpr int kEpiWarps = 8, kLoadWarp0 = 8, kLoadWarps = 4, kMmaWarp = 12, kMmaWarps = 2;
constexpr int kThreads = (kMmaWarp + kMmaWarps) * 32;
constexpr int kTPitch = 58;  // per-warp store transpose buffer: 16 filters x kTPitch floats
// kind::tf32: D f32, A / B TF32, K-major, N = 112, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kOW >> 3) << 17) |
                            ((uint32_t)(128 >> 4) << 24);
constexpr int kOffTr = kNP * kPairB;
constexpr int kOffBars = kOffTr + kEpiWarps * 16 * kTPitch * 4;
constexpr int kNumBars = 2 * kNP + 2 * kAcc + 2;
constexpr int kSmemBytes = kOffBars + kNumBars * 8 + 16 + 128;
static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");

struct Geom {
    const float *x, *w, *bias, *mean, *inv, *gamma, *beta;
    float *y;
    uint16_t *pack16;
    int32_t *pack_flags;
    int relu, raw;
    int H, OH, PH;
    int rpb, nbands, items;  // rows per band (raw: conv rows, pooled: pooled rows)
    int dbg;  // BNN_DEBUG_STEM_BITS (wrong results): 1 no input loads, 2 no MMAs, 4 no epilogue math / stores
    long long *trace;  // BNN_DEBUG_STEM_BITS & 8 with bnn_umma_trace: CTA 0 writes clock64 at [event * 64 + row]
};

struct Rows {
    int b, oy_s, oy_e, py0, py1;
};
__device__ __forceinline__ void trace(const Geom &g, int ev, int idx) {
    if (g.trace && blockIdx.x == 0 && idx < 64) g.trace[ev * 64 + idx] = clock64();
}
__device__ __forceinline__ Rows item_rows(const Geom &g, int item) {
    Rows r;
    r.b = item / g.nbands;
    const int band = item - r.b * g.nbands;
    if (g.raw) {
        r.oy_s = band * g.rpb, r.oy_e = min(g.OH - 1, r.oy_s + g.rpb - 1);
        r.py0 = r.py1 = 0;
    } else {
        r.py0 = band * g.rpb, r.py1 = min(g.PH, r.py0 + g.rpb);
        r.oy_s = max(0, 2 * r.py0 - 1), r.oy_e = min(g.OH - 1, 2 * r.py1 - 1);
    }
    return r;
}

// plain parked wait (umma::mbar_wait reads the watchdog pointer from global memory on
// every call: an L1 miss per wait here, where the loader streams the images through L1)
__device__ __forceinline__ void wait_parked(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase), "r"(1000000u)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ uint32_t tf32_hi(float v) { return __float_as_uint(v) & 0xFFFFE000u; }
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

// the position of an input row pair in the loader's stream
struct PairPos {
    int item, b, jp, jp_end;
};

__global__ void __launch_bounds__(kThreads, 1) stem_s2_kernel(const __grid_constant__ Geom g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 127u) & ~127u;
    uint8_t *smem = smem_raw + (base - raw);
    const uint32_t bar_full = base + kOffBars, bar_empty = bar_full + 8 * kNP;
    const uint32_t bar_tfull = bar_empty + 8 * kNP, bar_tempty = bar_tfull + 8 * kAcc;
    const uint32_t bar_stagger = bar_tempty + 8 * kAcc;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + kOffBars + kNumBars * 8);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) trace(g, 7, 0);
    if (tid == 0) {
        for (int s = 0; s < kNP; ++s) {
            mbar_init(bar_full + 8 * s, kLoadWarps);
            mbar_init(bar_empty + 8 * s, 2);  // both MMA issuers (see the release rule below)
        }
        for (int b = 0; b < kAcc; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, kEpiWarps);
        }
        mbar_init(bar_stagger, 1);
        mbar_init(bar_stagger + 8, 1);
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

    // weights -> TMEM, once: lane 32 q + l holds filter 16 q + (l & 15), TF32 half l >> 4;
    // slice s = (c, ky): columns kACol0 + 8 s + j, j = kx + 1 (j = 0: zero)
    if (warp < 4) {
        const int f = 16 * warp + (lane & 15), part = lane >> 4;
        const float *wf = g.w + f * (kC * kKH * kKW);
#pragma unroll 1
        for (int s = 0; s < kSlices; ++s) {
            uint32_t v[8];
            v[0] = 0u;
#pragma unroll
            for (int j = 1; j < 8; ++j) {
                const float wv = __ldg(wf + s * kKW + (j - 1));
                const uint32_t hi = tf32_hi(wv);
                v[j] = part ? __float_as_uint(wv - __uint_as_float(hi)) : hi;
            }
            tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kACol0 + 8 * s, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();

    if (warp >= kLoadWarp0 && warp < kLoadWarp0 + kLoadWarps) {
        // ------------------------------------------------------------ loader
        const int q = tid - kLoadWarp0 * 32;  // entry index
        const int xi0 = 2 * q - 4;
        const bool act = q < kNQ;
        const bool va = act && xi0 >= 0 && xi0 < kW, vb = act && xi0 + 2 >= 0 && xi0 + 2 < kW;
        auto start = [&](int item) {
            PairPos p{item, 0, 0, -1};
            if (item < g.items) {
                const Rows r = item_rows(g, item);
                p.b = r.b, p.jp = r.oy_s, p.jp_end = r.oy_e + 3;
            }
            return p;
        };
        auto next = [&](const PairPos &p) {
            if (p.item >= g.items) return p;
            if (p.jp < p.jp_end) return PairPos{p.item, p.b, p.jp + 1, p.jp_end};
            return start(p.item + (int)gridDim.x);
        };
        auto load = [&](const PairPos &p, float2(&v)[12]) {
            const bool live = p.item < g.items && !(g.dbg & 1);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int y = 2 * p.jp - kPad + r;
                const bool ok = live && (unsigned)y < (unsigned)g.H;
#pragma unroll
                for (int c = 0; c < kC; ++c) {
                    const float *src = g.x + ((int64_t)(p.b * kC + c) * g.H + y) * kW + xi0;
                    v[(r * kC + c) * 2] = make_float2(0.0f, 0.0f);
                    v[(r * kC + c) * 2 + 1] = make_float2(0.0f, 0.0f);
                    if (ok && va) v[(r * kC + c) * 2] = __ldg(reinterpret_cast<const float2 *>(src));
                    if (ok && vb) v[(r * kC + c) * 2 + 1] = __ldg(reinterpret_cast<const float2 *>(src + 2));
                }
            }
        };
        PairPos p0 = start(blockIdx.x), p1 = next(p0), p2 = next(p1);
        float2 v0[12], v1[12], v2[12];
        load(p0, v0);
        load(p1, v1);
        int pc = 0;
        while (p0.item < g.items) {
            load(p2, v2);
            const int slot = pc % kNP;
            wait_parked(bar_empty + 8 * slot, ((pc / kNP) & 1) ^ 1);
            if (q == 0) trace(g, 0, pc);
            if (act && !(g.dbg & 64)) {
                const uint32_t dst = base + slot * kPairB + q * 16;
#pragma unroll
                for (int rc = 0; rc < 2 * kC; ++rc) {
                    const float f[4] = {v0[2 * rc].x, v0[2 * rc].y, v0[2 * rc + 1].x, v0[2 * rc + 1].y};
                    uint32_t hi[4], lo[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        hi[i] = tf32_hi(f[i]);
                        lo[i] = __float_as_uint(f[i] - __uint_as_float(hi[i]));
                    }
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(dst + (2 * rc) * kRowB),
                                 "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3])
                                 : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(dst + (2 * rc + 1) * kRowB),
                                 "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3])
                                 : "memory");
                }
            }
            // the MMA (async proxy) reads what the generic proxy just wrote
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_full + 8 * slot);
            if (q == 0) trace(g, 1, pc);
            ++pc;
            p0 = p1, p1 = p2, p2 = next(p2);
#pragma unroll
            for (int i = 0; i < 12; ++i) v0[i] = v1[i], v1[i] = v2[i];
        }
    } else if (warp >= kMmaWarp) {
        // ------------------------------------------------------------ MMA issue
        // Two issuer threads take alternate conv rows, unsynchronised: a single thread
        // issues one MMA per ~60 cycles plus ~360 cycles of barrier work per row and
        // starves the pipe (56 cycles per MMA).  Rows use different accumulators, so
        // their MMAs may interleave freely.  tcgen05.commit only tracks the issuing
        // thread's MMAs, hence every ring slot is released by two commits: one from each
        // of the last two rows that read it (count 2; the first row of a band, which has
        // no predecessor, commits twice).
        const int which = warp - kMmaWarp;
        // (the whole warp runs the loop with warp-uniform values -- descriptors and TMEM addresses
        // stay in uniform registers, no R2UR per MMA operand; one elected lane issues)
        {
            // no-swizzle K-major descriptor: LBO = 32 B (K chunk 1 = two entries on),
            // SBO = 128 B (8 pixels), version 1
            const uint64_t dbase = ((uint64_t)(32 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
            auto rel = [&](int p) {
                if (elect_one()) umma_commit(bar_empty + 8 * (p % kNP));
                __syncwarp();
            };
            int pc0 = 0, it = 0;
            for (int item = blockIdx.x; item < g.items; item += gridDim.x) {
                const Rows r = item_rows(g, item);
                const int n = r.oy_e - r.oy_s + 1;
                for (int rr = 0; rr < n; ++rr, ++it) {
                    if ((it & 1) != which) continue;
                    const int buf = it % kAcc;
                    wait_parked(bar_tempty + 8 * buf, ((it / kAcc) & 1) ^ 1);
                    const int pc = pc0 + rr;  // the pair holding input rows 2 oy - 3, 2 oy - 2
                    wait_parked(bar_full + 8 * ((pc + 3) % kNP), ((pc + 3) / kNP) & 1);
                    // half-row stagger, enforced every row: a row starts only once the other
                    // issuer is half way through the row before it.  In phase (where equal
                    // sharing of the pipe would keep them) both issuers would do their per-row
                    // barrier work at the same time with the pipe idle.
                    if (it > 0) wait_parked(bar_stagger + 8 * (which ^ 1), ((it - 1) >> 1) & 1);
                    fence_after();
                    if (which == 0 && lane == 0) trace(g, 2, it);
                    uint64_t sb[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        sb[i] = dbase + (uint64_t)((base + ((pc + i) % kNP) * kPairB) >> 4);
                    const uint32_t d = tmem + buf * kOW;
                    if (elect_one()) {
#pragma unroll
                        for (int s = 0; s < kSlices; ++s) {
                            if (s == kSlices / 2) mbar_arrive(bar_stagger + 8 * which);
                            if (g.dbg & 2) continue;
                            const int c = s / kKH, ky = s % kKH;
                            const uint64_t dh = sb[ky >> 1] + (uint64_t)((((ky & 1) * kC + c) * 2 * kRowB) >> 4);
                            mma_ts(d, tmem + kACol0 + 8 * s, dh, s != 0);
                            mma_ts(d, tmem + kACol0 + 8 * s, dh + (uint64_t)(kRowB >> 4), 1u);
                        }
                    }
                    __syncwarp();
                    // pair p is last read by row min(p, last row) and the row before it
                    rel(pc);
                    if (rr == 0) rel(pc);
                    if (rr == n - 1) {
                        for (int k = 1; k <= 3; ++k) {
                            rel(pc + k);
                            if (n == 1) rel(pc + k);
                        }
                    } else if (rr + 1 < n - 1) {
                        rel(pc + 1);
                    } else {  // the next row is the band's last: its own pair and its look-ahead pairs
                        for (int k = 1; k <= 4; ++k) rel(pc + k);
                    }
                    if (elect_one()) umma_commit(bar_tfull + 8 * buf);
                    __syncwarp();
                    if (which == 0 && lane == 0) trace(g, 3, it);
                }
                pc0 += n + 3;
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3, h = warp >> 2;      // TMEM lane quadrant, pixel half
        const int f = 16 * q + (lane & 15), sub = lane >> 4;
        const bool low = sub == 0;
        const float sgn = g.raw ? 1.0f : (__ldg(g.gamma + f) < 0.0f ? -1.0f : 1.0f);
        const float bn_mean = g.raw ? 0.0f : __ldg(g.mean + f), bn_inv = g.raw ? 0.0f : __ldg(g.inv + f);
        const float bn_gamma = g.raw ? 0.0f : __ldg(g.gamma + f), bn_beta = g.raw ? 0.0f : __ldg(g.beta + f);
        const float bias = (g.raw && g.bias) ? __ldg(g.bias + f) : 0.0f;
        const int pcol0 = 28 * h + 14 * sub;  // and pooled columns pcol0 .. pcol0 + 13
        float *tb = reinterpret_cast<float *>(smem + kOffTr) + warp * 16 * kTPitch;  // this warp's store transpose
        const int fl = lane & 15;
        float cur[14];
        int it = 0;
        for (int item = blockIdx.x; item < g.items; item += gridDim.x) {
            const Rows r = item_rows(g, item);
#pragma unroll
            for (int i = 0; i < 14; ++i) cur[i] = -INFINITY;
            // BN -> ReLU of a finished pooled row (undo the sign), store it and its sign bits
            auto finish = [&](int py, const float(&mx)[14]) {
                float o[14];
                uint32_t mine = 0;
                float nf = 0.0f;
#pragma unroll
                for (int j = 0; j < 14; ++j) {
                    float v = __fmul_rn(mx[j], sgn);
                    v = __fadd_rn(__fmul_rn(bn_gamma, __fmul_rn(__fsub_rn(v, bn_mean), bn_inv)), bn_beta);
                    if (g.relu) v = fmaxf(v, 0.0f);
                    o[j] = v;
                    if (g.pack16) {
                        const uint32_t bal = __ballot_sync(0xffffffffu, v >= 0.0f);
                        if ((lane & 15) == j) mine = low ? (bal & 0xffffu) : (bal >> 16);
                        nf = __fmaf_rn(v, 0.0f, nf);
                    }
                }
                // through the warp's transpose buffer: one 112-byte run per filter and store
                // instead of 32 scattered 8-byte pieces
#pragma unroll
                for (int j = 0; j < 14; ++j) tb[fl * kTPitch + 14 * sub + j] = o[j];
                __syncwarp();
                if (lane < 28) {
                    float *yw = g.y + (((int64_t)r.b * kNF + 16 * q) * g.PH + py) * kPW + 28 * h + lane;
#pragma unroll
                    for (int k = 0; k < 16; ++k) yw[(int64_t)k * g.PH * kPW] = tb[k * kTPitch + lane];
                }
                __syncwarp();
                if (g.pack16) {
                    if ((lane & 15) < 14) {
                        const int64_t pix = ((int64_t)r.b * g.PH + py) * kPW + pcol0 + (lane & 15);
                        g.pack16[pix * (kNF / 16) + q] = (uint16_t)mine;
                    }
                    if (g.pack_flags && nf != 0.0f) atomicOr(g.pack_flags, 1);
                }
            };
            for (int oy = r.oy_s; oy <= r.oy_e; ++oy, ++it) {
                const int buf = it % kAcc;
                wait_parked(bar_tfull + 8 * buf, (it / kAcc) & 1);
                fence_after();
                if (tid == 0) trace(g, 4, it);
                if (tid == 0 && it >= 64 && (it & 7) == 0) trace(g, 7, 2 + ((it - 64) >> 3));
                // v[i] <-> conv column 56 h - 1 + i
                uint32_t v[57];
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + buf * kOW + 56 * h;
#pragma unroll
                for (int k = 0; k < 7; ++k) v[1 + 8 * k] = 0u;  // (debug bit 32 leaves them unloaded)
#pragma unroll
                for (int k = 0; k < 7; ++k)
                    if (!(g.dbg & 32)) ld8(ta + 8 * k, v + 1 + 8 * k);
                v[0] = 0u;
                if (h && !(g.dbg & 32)) {
                    uint32_t t8[8];
                    ld8(ta - 8, t8);
                    v[0] = t8[7];
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_tempty + 8 * buf);
                if (tid == 0) trace(g, 5, it);
                if (g.dbg & 4) continue;
                // hi + lo lane halves; the low 16 lanes keep columns v[0..28], the high 16
                // lanes v[28..56]: s[i] <-> conv column col0 - 1 + i
                float s[29];
#pragma unroll
                for (int i = 0; i < 29; ++i) {
                    const uint32_t send = low ? v[28 + i] : v[i];
                    const uint32_t keep = low ? v[i] : v[28 + i];
                    const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 16);
                    // (w_hi part) + (w_lo part), in this order on both lane halves
                    const float a = __uint_as_float(low ? keep : got), b = __uint_as_float(low ? got : keep);
                    s[i] = __fadd_rn(a, b);
                }
                if (g.raw) {
#pragma unroll
                    for (int i = 0; i < 28; i += 2)
                        *reinterpret_cast<float2 *>(tb + fl * kTPitch + 28 * sub + i) =
                            make_float2(__fadd_rn(s[1 + i], bias), __fadd_rn(s[2 + i], bias));
                    __syncwarp();
                    if (lane < 28) {  // 224 contiguous bytes per filter and store
                        float *yw = g.y + (((int64_t)r.b * kNF + 16 * q) * g.OH + oy) * kOW + 56 * h + 2 * lane;
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            __stcs(reinterpret_cast<float2 *>(yw + (int64_t)k * g.OH * kOW),
                                   *reinterpret_cast<const float2 *>(tb + k * kTPitch + 2 * lane));
                    }
                    __syncwarp();
                    continue;
                }
#pragma unroll
                for (int i = 0; i < 29; ++i) s[i] = __fmul_rn(s[i], sgn);
                if (h == 0 && low) s[0] = -INFINITY;  // left image border
                const bool odd = oy & 1, done = odd && ((oy - 1) >> 1) >= r.py0;
                float m[14];
#pragma unroll
                for (int j = 0; j < 14; ++j) m[j] = fmaxf(fmaxf(s[2 * j], s[2 * j + 1]), s[2 * j + 2]);
                if (done) {
                    float mx[14];
#pragma unroll
                    for (int j = 0; j < 14; ++j) mx[j] = fmaxf(cur[j], m[j]);
                    finish((oy - 1) >> 1, mx);
                }
#pragma unroll
                for (int j = 0; j < 14; ++j) cur[j] = odd ? m[j] : fmaxf(cur[j], m[j]);
                if (tid == 0) trace(g, 6, it);
            }
            // last pooled row without a conv row below it (odd OH)
            if (!g.raw && !(r.oy_e & 1) && (r.oy_e >> 1) < r.py1) finish(r.oy_e >> 1, cur);
        }
    }
    fence_before();
    __syncthreads();
    if (tid == 0) trace(g, 7, 1);
    if (warp == kMmaWarp) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

}  // namespace stem2

bool stem_s2_supported(int64_t C, int64_t H, int64_t W, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                       int64_t sw, int64_t ph, int64_t pw) {
    using namespace stem2;
    return C == kC && W == kW && F == kNF && kh == kKH && kw == kKW && sh == 2 && sw == 2 && ph == kPad &&
           pw == kPad && H >= 1 && !(g_debug.stem_bits & 16);
}

// raw != 0: y = conv(x) (+ bias) [B, 64, OH, 112]; raw == 0: y = maxpool3x3/2/1(relu?(bn(conv(x))))
// [B, 64, PH, 56], optionally with its sign-packed NHWC words
int launch_stem_s2(const float *x, int64_t B, int64_t H, const float *w, const float *bias,
                   const float *mean, const float *inv, const float *gamma, const float *beta, int relu,
                   int raw, float *y, uint64_t *pack_words, int32_t *pack_flags, cudaStream_t s) {
    using namespace stem2;
    if ((reinterpret_cast<uintptr_t>(x) & 7) || (reinterpret_cast<uintptr_t>(y) & 15))
        return set_error(BNN_EUNSUP, "stride-2 stem: unaligned tensors");
    Geom g{};
    g.x = x, g.w = w, g.bias = bias, g.mean = mean, g.inv = inv, g.gamma = gamma, g.beta = beta, g.y = y;
    g.pack16 = raw ? nullptr : reinterpret_cast<uint16_t *>(pack_words);
    g.pack_flags = pack_flags;
    g.relu = relu, g.raw = raw;
    g.dbg = (int)(g_debug.stem_bits & (7 | 32 | 64));  // 32: no TMEM loads, 64: no loader stores
    g.trace = (g_debug.stem_bits & 8) ? reinterpret_cast<long long *>(g_debug.trace_buf) : nullptr;
    g.H = (int)H, g.OH = (int)((H + 2 * kPad - kKH) / 2 + 1), g.PH = (g.OH - 1) / 2 + 1;
    g.rpb = raw ? 28 : 14;
    g.nbands = (int)ceil_div(raw ? g.OH : g.PH, g.rpb);
    if (B * g.nbands >= (1ll << 31) || B * kC * H * kW >= (1ll << 40))
        return set_error(BNN_EUNSUP, "stride-2 stem: too many items");
    g.items = (int)(B * g.nbands);
    if (g.items == 0) return BNN_OK;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(stem_s2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        configured = true;
    }
    const int grid = g.items < sm_count() ? g.items : sm_count();
    stem_s2_kernel<<<grid, kThreads, kSmemBytes, s>>>(g);
    return check_launch("stem_s2_kernel");
}

}  // namespace bnn

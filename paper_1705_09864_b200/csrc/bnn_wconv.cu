// Shifted-window binary convolution on tcgen05 (stride-1 convs of ResNet-18 layers 1-2:
// C, F in {64, 128}, 3x3 / pad 1 and friends): every input pixel is expanded to e2m1
// codes ONCE, and the im2col matrix of a filter tap is the expanded band itself at a
// shifted start address.
//
// Replaces the same reference path as bnn_sconv.cu / bnn_umma_impl.cuh --
// QConv2d.forward(INFER_PACKED) (layers.py:225-245) = im2col (tensor.py:60-78) ->
// pack_matrix_b (bitpack.py:152-169) -> xnor_gemm (gemm.py:128-139) with the G2 "+1"
// padding -- bit-identically.
//
// Geometry: the batch is one raster of PADDED positions, t = R * Wp + col with
// Wp = W + 2 pw and R = b * Hp + (padded row), Hp = H + 2 ph; halo positions hold the
// all-ones "+1" word (sign(0) = +1).  For stride 1, output position t reads
// tap (ky, kx) at padded position t + ky * Wp + kx -- the same shift for every t.  A GEMM
// tile is 128 consecutive positions (TMEM lanes; positions whose (row, col) fall outside
// OH x OW are computed and dropped, a few percent), the N dimension is the F filters.
//
// Per CTA (persistent, a contiguous range of tiles, processed in items of `tpi` tiles):
//   * weights: expanded once into the SW128 K-major B operand (filter-stationary), with
//     popcounts and the per-filter monotone sign thresholds (as in bnn_sconv.cu);
//   * 4 loader warps expand the item's band of padded rows -- one u64 load per pixel,
//     4-7 ALU ops and one st.shared.v4 per 32 channels -- into C / 32 planes of 16-byte
//     entries (plane c = channels 32 c .. 32 c + 31 of every position, 16-byte pitch) and
//     write the pixel's popcount; double-buffered bands;
//   * one thread issues, per tile and tap, C / 64 MMAs (kind::mxf4, M = 128, N = F,
//     K = 64) whose A operand is a NO-SWIZZLE K-major descriptor over planes (2j, 2j + 1):
//     SBO = 128 B (8 positions), LBO = the plane stride, start = plane + 16 * (tile
//     position + ky * Wp + kx).  No per-tap expansion, no im2col rows anywhere;
//   * 8 epilogue warps: C = popc(a & b) from TMEM, pixel popcount = sum of the taps'
//     popcounts, P = K - popc(pixel) - popc(filter) + 2C, fused BN / residual / f32 NCHW
//     stores / sign-pack exactly as bnn_sconv.cu.
#include "bnn_umma_impl.cuh"

namespace bnn {
namespace wconv {

using umma::expand_fp4_a;
using umma::expand_fp4_b;
using umma::fence_after;
using umma::fence_before;
using umma::mbar_arrive;
using umma::mbar_init;
using umma::sw128_desc;
using umma::umma_commit;

constexpr int kRows = 128;
// (12 warps: registers are allocated per 4 warps, so a 13th warp would cap every thread at 128)
constexpr int kEpiWarps = 8, kLoadWarp0 = 8, kLoadWarps = 3, kMmaWarp = 11;
constexpr int kThreads = (kMmaWarp + 1) * 32;
constexpr int kBands = 2;

struct Geom {
    const uint64_t *x;  // packed NHWC [B, H, W, Cw]
    const uint64_t *w;  // tap-major weights [F, kh * kw * Cw]
    float *y;           // f32 NCHW [B, F, OH, OW] (may be null)
    const float *res;   // residual, same layout (may be null)
    int B, H, W, Hp, Wp, OH, OW, kh, kw, ph, pw, K;
    int Ftot, fgroups, nranges;  // all filters; groups of kF filters; tile ranges (grid = fgroups * nranges)
    int total_rows;     // B * Hp
    int P;              // positions: total_rows * Wp
    int ntiles, tpi;
    int band_rows, band_pos, plane_bytes;  // per band buffer: rows, rows * Wp, band_pos * 16
    long long *trace;   // debug timeline of CTA 0 (bnn_umma_trace + debug bit 16): clock64 at [event * 64 + idx]
    int dbg;            // debug ablations (wrong results): 1 no MMAs, 2 no epilogue work, 4 no band loads,
                        // 8 no band expansion at all
};

__device__ __forceinline__ void stamp(const Geom &g, int ev, int idx) {
    if (g.trace != nullptr && blockIdx.x == 0 && idx < 64) g.trace[ev * 64 + idx] = clock64();
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

template <int kF>
struct Cfg {
    static constexpr int kAcc = (512 - 32) / kF >= 4 ? 4 : (512 - 32) / kF;
    static constexpr int kSfCol = kAcc * kF;
    // kind::mxf4, E2M1 x E2M1, UE8M0 scales, f32 accumulate, M = 128, N = kF
    static constexpr uint32_t kIdesc = (1u << 7) | (1u << 10) | ((uint32_t)(kF >> 3) << 17) | (1u << 23) |
                                       ((uint32_t)(kRows >> 4) << 24);
};

struct Smem {
    uint32_t w, band, pc, par, aff, thr, thu, popc_f, popc_ff, bars, tmem, total;
    __host__ __device__ Smem(int F, int K, int planes, int plane_bytes, int band_pos) {
        const int wblocks = (K + 255) / 256;
        w = 0;                                        // expanded weights (SW128 blocks, 1024-aligned)
        band = w + wblocks * F * 128;                 // [kBands][planes][band_pos] 16-byte entries
        pc = band + kBands * planes * plane_bytes;    // [kBands][band_pos] pixel popcounts
        par = (pc + kBands * band_pos * 4 + 15) & ~15u;  // float4 [128] BN
        aff = par + 128 * 16;                         // float2 [128] scale, shift
        thr = aff + 128 * 8;                          // float2 [128] sign thresholds (+ int [8] flags)
        thu = thr + 128 * 8 + 64;                     // float [128] compare thresholds U, u64 [2] flip masks
        popc_f = thu + 128 * 4 + 16;
        popc_ff = popc_f + 128 * 4;                   // the same as f32 (no I2F per output element)
        bars = popc_ff + 128 * 4;
        tmem = bars + 32 * 8;
        total = tmem + 16;
    }
};

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
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t *v) {  // (no wait: batch several)
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
// base + j * stride_bytes as ONE IMAD.WIDE (j folds to an immediate after unrolling): the NCHW
// filter stride of the epilogue's residual loads / f32 stores, instead of a 4-instruction
// 64-bit add + scale per address
template <typename T>
__device__ __forceinline__ T *at_stride(T *base, int stride_bytes, int j) {
    uint64_t d;
    asm("mad.wide.s32 %0, %1, %2, %3;\n" : "=l"(d) : "r"(stride_bytes), "r"(j), "l"((uint64_t)base));
    return reinterpret_cast<T *>(d);
}
__device__ __forceinline__ void wait_spin(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
    } while (!done);
}

template <int kF, int kCw, bool kPack>
__global__ void __launch_bounds__(kThreads, 1)
    xnor_wconv_kernel(const __grid_constant__ Geom g, const __grid_constant__ Epilogue ep) {
    using C = Cfg<kF>;
    constexpr int kAcc = C::kAcc, kPlanes = 2 * kCw;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sraw = smem_u32(smem_raw);
    const uint32_t sbase = (sraw + 1023u) & ~1023u;
    uint8_t *sgen = smem_raw + (sbase - sraw);
    const Smem L(kF, g.K, kPlanes, g.plane_bytes, g.band_pos);
    const uint32_t s_w = sbase + L.w, s_band = sbase + L.band;
    int32_t *s_pc = reinterpret_cast<int32_t *>(sgen + L.pc);
    float4 *s_par = reinterpret_cast<float4 *>(sgen + L.par);
    float2 *s_aff = reinterpret_cast<float2 *>(sgen + L.aff);
    float2 *s_thr = reinterpret_cast<float2 *>(sgen + L.thr);
    int32_t *s_thr_ok = reinterpret_cast<int32_t *>(sgen + L.thr + 128 * 8);
    float *s_thu = reinterpret_cast<float *>(sgen + L.thu);
    uint32_t *s_flip = reinterpret_cast<uint32_t *>(sgen + L.thu + 128 * 4);  // [kF / 32]
    int32_t *s_popc_f = reinterpret_cast<int32_t *>(sgen + L.popc_f);
    float *s_popc_ff = reinterpret_cast<float *>(sgen + L.popc_ff);
    const uint32_t bar_bfull = sbase + L.bars;               // [kBands] band expanded
    const uint32_t bar_bempty = bar_bfull + 8 * kBands;      // [kBands] MMAs + epilogue done with it
    const uint32_t bar_tfull = bar_bempty + 8 * kBands;      // [kAcc] accumulator ready
    const uint32_t bar_tempty = bar_tfull + 8 * kAcc;        // [kAcc] accumulator drained
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sgen + L.tmem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ohw = g.OH * g.OW;
    const int ohw4 = ohw * 4;  // (bytes; positions < 2^24)
    const int fg = blockIdx.x % g.fgroups, rg = blockIdx.x / g.fgroups;  // filter group, tile range
    const int f0 = fg * kF;  // this CTA's first filter
    if (tid == 0) stamp(g, 7, 0);

    if (tid == 0) {
        for (int i = 0; i < kBands; ++i) {
            mbar_init(bar_bfull + 8 * i, kLoadWarps);
            mbar_init(bar_bempty + 8 * i, 1 + kEpiWarps);
        }
        for (int i = 0; i < kAcc; ++i) {
            mbar_init(bar_tfull + 8 * i, 1);
            mbar_init(bar_tempty + 8 * i, kEpiWarps / 2);  // the four quadrant warps of the tile's parity
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
    // programmatic dependent launch: let the next kernel's CTAs start on SMs this grid frees (its own
    // griddepcontrol.wait still holds its reads / writes until this grid has completed)
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

    if (tid == 0) stamp(g, 7, 3);
    // ---- weights: expanded once into the SW128 K-major B operand (+ filter popcounts),
    // per-filter epilogue parameters and sign thresholds (same construction as bnn_sconv.cu)
    {
        const int kw32 = g.K / 32;
        const uint32_t *w32 = reinterpret_cast<const uint32_t *>(g.w);
        // (flat over the group's kF x kw32 words, eight loads in flight per thread: the
        // group's rows are contiguous in the tap-major weight array; (filter, word) advance
        // incrementally, no division per word)
        const int total = kF * kw32;
        const uint32_t *wg = w32 + (int64_t)f0 * kw32;
        const int df = kThreads / kw32, dq = kThreads - df * kw32;
        int wf = tid / kw32, wq = tid - wf * kw32;
#pragma unroll 1
        for (int base = tid; base < total; base += 8 * kThreads) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int idx = base + u * kThreads;
                v[u] = idx < total ? __ldg(wg + idx) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (base + u * kThreads < total) {
                    uint32_t r4[4];
                    expand_fp4_b(v[u], r4);
                    const uint32_t addr = s_w + (wq >> 3) * (kF * 128) + wf * 128 + (((wq & 7) ^ (wf & 7)) << 4);
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(r4[0]),
                                 "r"(r4[1]), "r"(r4[2]), "r"(r4[3]));
                }
                wf += df, wq += dq;
                if (wq >= kw32) wq -= kw32, ++wf;
            }
        }
        if (tid == 0) stamp(g, 7, 6);
        // filter popcounts: a warp per filter (the words are L1 / L2 hits now), four filters'
        // loads in flight
#pragma unroll 1
        for (int fb = warp * 4; fb < kF; fb += (kThreads / 32) * 4) {
            int32_t pc[4] = {0, 0, 0, 0};
            uint32_t wv[4][5];  // (kw32 <= 160: C * kh * kw <= 5120; all loads in flight)
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const int q = lane + 32 * i;
                    wv[u][i] = (fb + u < kF && q < kw32) ? __ldg(wg + (fb + u) * kw32 + q) : 0u;
                }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 5; ++i) pc[u] += __popc(wv[u][i]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int sum = __reduce_add_sync(0xffffffffu, pc[u]);
                if (lane == 0 && fb + u < kF) s_popc_f[fb + u] = sum, s_popc_ff[fb + u] = (float)sum;
            }
        }
        if (tid == 0) stamp(g, 7, 4);
        for (int f = tid; f < kF; f += kThreads) {
            float4 bp = make_float4(0.0f, 1.0f, 1.0f, 0.0f);
            if (ep.bn_mean != nullptr) {
                bp.x = ep.bn_mean[f0 + f];
                bp.y = ep.bn_inv[f0 + f];
                bp.z = ep.bn_gamma[f0 + f];
                bp.w = ep.bn_beta[f0 + f];
            }
            float2 af = make_float2(1.0f, 0.0f);
            if (ep.scale != nullptr) af.x = ep.scale[f0 + f];
            if (ep.shift != nullptr) af.y = ep.shift[f0 + f];
            s_par[f] = bp;
            s_aff[f] = af;
        }
        if (warp < 4) {  // UE8M0 scale factors = 1.0 in every TMEM column from kSfCol on
            const uint32_t one[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                     0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
            for (int col = C::kSfCol; col < 512; col += 8)
                umma::tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + col, one);
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        fence_before();
        __syncthreads();
        fence_after();
        if (tid == 0) stamp(g, 7, 5);
        // monotone sign thresholds for packed-only outputs: bit = S * a - V >= 0 on
        // a = 2C + (K - popc(pixel)) = P + popc(filter) (see bnn_sconv.cu)
        for (int f = tid; f < kF; f += kThreads) {
            const float4 bp = s_par[f];
            const float2 af = s_aff[f];
            const bool dot = ep.domain == BNN_DOT;
            const int K = g.K;
            auto fx = [&](int P) {
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
                const bool b0 = f0 >= 0.0f;
                int lo = 0, hi = K + 1;  // bit(P) == b0 for P < lo; differs at hi
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if ((fx(mid) >= 0.0f) == b0) lo = mid + 1;
                    else hi = mid;
                }
                const float U = (float)(lo + s_popc_f[f]);
                if (lo > K) t = make_float2(0.0f, b0 ? -1.0f : 1.0f);
                else if (!b0) t = make_float2(1.0f, U);
                else t = make_float2(-1.0f, -(U - 0.5f));
            }
            s_thr[f] = t;
        }
        __syncthreads();
        if (tid < kF / 16) {
            int ok = 1;
            for (int j = 0; j < 16; ++j) ok &= s_thr[tid * 16 + j].y == s_thr[tid * 16 + j].y;
            s_thr_ok[tid] = ok;
        }
        // the same test as one compare per element: bit = (a >= U) ^ flip  (a and U are
        // integers: S = -1 means a < U; constant bits are U = -inf / +inf)
        if (tid < kF) {  // (warp w = filters 32 w .. 32 w + 31)
            const float2 t = s_thr[tid];
            float U;
            if (t.x > 0.0f) U = t.y;
            else if (t.x < 0.0f) U = -t.y + 0.5f;
            else U = t.y < 0.0f ? -INFINITY : INFINITY;
            s_thu[tid] = U;
            const uint32_t fl = __ballot_sync(0xffffffffu, t.x < 0.0f);
            if (lane == 0) s_flip[warp] = fl;
        }
        __syncthreads();
    }
    // everything above (barriers, TMEM, the weight group's expansion, per-filter parameters and
    // thresholds) reads only load-time constants and overlaps the previous kernel's tail; the
    // activations, the shortcut and the outputs are touched after this point
    asm volatile("griddepcontrol.wait;\n" ::: "memory");

    if (tid == 0) stamp(g, 7, 1);
    // this CTA's contiguous tile range, in items of tpi tiles
    const int tb = (int)((int64_t)rg * g.ntiles / g.nranges);
    const int te = (int)((int64_t)(rg + 1) * g.ntiles / g.nranges);
    const int Wp = g.Wp;
    // first padded row and number of rows of the band of tiles [T0, T1)
    // items: the first one is short, so that the MMAs start after a small band
    auto item_end = [&](int T0, int ii) { return min(te, T0 + (ii == 0 ? min(2, g.tpi) : g.tpi)); };
    auto band_of = [&](int T0, int T1, int &Ra, int &nrows) {
        Ra = (T0 * kRows) / Wp;
        const int last = T1 * kRows - 1 + (g.kh - 1) * Wp + (g.kw - 1);
        nrows = last / Wp - Ra + 1;
    };

    if (warp >= kLoadWarp0 && warp < kLoadWarp0 + kLoadWarps) {
        // ============================================================ band expanders
        const int lw = warp - kLoadWarp0;
        int ii = 0;
#pragma unroll 1
        for (int T0 = tb, T1 = tb; T0 < te; T0 = T1, ++ii) {
            T1 = item_end(T0, ii);
            const int bb = ii & 1;
            int Ra, nrows;
            band_of(T0, T1, Ra, nrows);
            wait_parked(bar_bempty + 8 * bb, ((ii >> 1) & 1) ^ 1);
            if (lw == 0 && lane == 0) stamp(g, 0, ii);
            const uint32_t band = s_band + bb * kPlanes * g.plane_bytes;
            int32_t *pcb = s_pc + bb * g.band_pos;
            // kU rows (two 32-column passes each) per iteration: all loads in flight before
            // the first expansion (Wp <= 64 is a launch precondition)
            constexpr int kU = kCw <= 2 ? 4 : (kCw == 4 ? 2 : 1);
#pragma unroll 1
            for (int r0 = lw; r0 < nrows && !(g.dbg & 8); r0 += kU * kLoadWarps) {
                uint64_t wd[kU][2][kCw];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const int r = r0 + u * kLoadWarps, R = Ra + r;
                    const int b = R / g.Hp, iy = R - b * g.Hp - g.ph;
                    const bool rok = r < nrows && R < g.total_rows && (unsigned)iy < (unsigned)g.H && !(g.dbg & 4);
                    const uint64_t *xrow = g.x + ((int64_t)b * g.H + iy) * g.W * kCw;
#pragma unroll
                    for (int it = 0; it < 2; ++it) {
                        const int ix = lane + 32 * it - g.pw;
                        const bool ok = rok && (unsigned)ix < (unsigned)g.W && lane + 32 * it < Wp;
#pragma unroll
                        for (int c = 0; c < kCw; ++c) wd[u][it][c] = ~0ull;  // out of image: "+1" (G2)
                        if (ok) {
                            if constexpr (kCw >= 2) {
#pragma unroll
                                for (int c = 0; c < kCw; c += 2) {
                                    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2 *>(
                                        xrow + (int64_t)ix * kCw + c));
                                    wd[u][it][c] = v.x, wd[u][it][c + 1] = v.y;
                                }
                            } else {
                                wd[u][it][0] = __ldg(xrow + ix);
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const int r = r0 + u * kLoadWarps;
                    if (r >= nrows) break;
#pragma unroll
                    for (int it = 0; it < 2; ++it) {
                        const int col = lane + 32 * it;
                        if (col >= Wp) break;
                        const int pos = r * Wp + col;
                        int32_t pc = 0;
#pragma unroll
                        for (int c = 0; c < kCw; ++c) {
                            pc += __popcll(wd[u][it][c]);
#pragma unroll
                            for (int hx = 0; hx < 2; ++hx) {
                                uint32_t r4[4];
                                expand_fp4_a((uint32_t)(wd[u][it][c] >> (32 * hx)), r4);
                                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                                                 band + (2 * c + hx) * g.plane_bytes + pos * 16),
                                             "r"(r4[0]), "r"(r4[1]), "r"(r4[2]), "r"(r4[3])
                                             : "memory");
                            }
                        }
                        pcb[pos] = pc;
                    }
                }
            }
            // the MMA (async proxy) reads what the generic proxy just wrote
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_bfull + 8 * bb);
            if (lw == 0 && lane == 0) stamp(g, 1, ii);
        }
    } else if (warp == kMmaWarp) {
        // ============================================================ MMA issuer
        // (the whole warp runs the loop with warp-uniform values, which the compiler keeps
        // in uniform registers -- a single divergent lane pays an R2UR per MMA operand;
        // one elected lane issues each tcgen05.mma / commit)
        {
            // A: no-swizzle K-major, LBO = plane stride (K chunk 1 = the next plane), SBO = 128 B
            const uint64_t da_base = ((uint64_t)((uint32_t)g.plane_bytes >> 4) << 16) |
                                     ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
            const uint64_t db0 = sw128_desc(s_w);
            int ii = 0, tc = 0;
#pragma unroll 1
            for (int T0 = tb, T1 = tb; T0 < te; T0 = T1, ++ii) {
                T1 = item_end(T0, ii);
                const int bb = ii & 1;
                int Ra, nrows;
                band_of(T0, T1, Ra, nrows);
                wait_spin(bar_bfull + 8 * bb, (ii >> 1) & 1);
                const uint32_t band = s_band + bb * kPlanes * g.plane_bytes;
#pragma unroll 1
                for (int T = T0; T < T1; ++T, ++tc) {
                    const int buf = tc % kAcc;
                    wait_spin(bar_tempty + 8 * buf, ((tc / kAcc) & 1) ^ 1);
                    fence_after();
                    if (lane == 0) stamp(g, 2, tc);
                    const uint32_t d = tmem + buf * kF;
                    const uint32_t a0 = band + (uint32_t)(T * kRows - Ra * Wp) * 16;
                    // descriptor = {lo: start >> 4 | LBO << 16, hi: SBO | version}; 3x3 kernels
                    // (the ResNet shapes) issue from compile-time tap / K-step offsets
                    const uint32_t da_hi = (uint32_t)(da_base >> 32);
                    const uint32_t da_lo = (uint32_t)da_base | (a0 >> 4);
                    auto issue = [&](uint32_t lo, int st) {
                        const uint64_t da = ((uint64_t)da_hi << 32) | lo;
                        const uint64_t db = db0 + (uint64_t)((((st >> 2) * (kF * 128)) + (st & 3) * 32) >> 4);
                        umma::mma_fp4<C::kIdesc>(d, da, db, tmem + C::kSfCol, tmem + C::kSfCol, st != 0 ? 1u : 0u);
                    };
                    const uint32_t plane2 = (uint32_t)(2 * g.plane_bytes) >> 4;
                    if (!elect_one() || (g.dbg & 1)) {
                    } else if (g.kh == 3 && g.kw == 3) {
                        const uint32_t row_lo[3] = {da_lo, da_lo + (uint32_t)Wp, da_lo + 2u * (uint32_t)Wp};
#pragma unroll
                        for (int tap = 0; tap < 9; ++tap)
#pragma unroll
                            for (int j = 0; j < kCw; ++j)
                                issue(row_lo[tap / 3] + (tap % 3) + j * plane2, tap * kCw + j);
                    } else {
                        int st = 0;
#pragma unroll 1
                        for (int ky = 0; ky < g.kh; ++ky)
#pragma unroll 1
                            for (int kx = 0; kx < g.kw; ++kx)
#pragma unroll
                                for (int j = 0; j < kCw; ++j, ++st)
                                    issue(da_lo + (uint32_t)(ky * Wp + kx) + j * plane2, st);
                    }
                    __syncwarp();
                    if (elect_one()) umma_commit(bar_tfull + 8 * buf);
                    __syncwarp();
                    if (lane == 0) stamp(g, 3, tc);
                }
                if (elect_one()) umma_commit(bar_bempty + 8 * bb);
                __syncwarp();
            }
            // keep TMEM allocated until the epilogue drained the last accumulators
            for (int t = tc - kAcc; t < tc; ++t)
                if (t >= 0) wait_parked(bar_tempty + 8 * (t % kAcc), (uint32_t)(t / kAcc) & 1u);
        }
        __syncwarp();
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    } else {
        // ============================================================ epilogue
        // warp (q, h): TMEM lane quadrant q, tiles of parity h (CTA-local tile counter) --
        // two tiles are in the epilogue at a time, each warp walking all of its tile's
        // filter columns, so one tile's serial latencies (coordinates, TMEM loads, residual
        // loads) hide behind the other tile's work
        const int q = warp & 3, h = warp >> 2;
        const bool dot = ep.domain == BNN_DOT;
        const bool affine = ep.scale || ep.shift;
        const bool has_bn = ep.bn_mean != nullptr;
        const bool pack_only = kPack && g.y == nullptr && g.res == nullptr;
        const float kf = (float)g.K;
        // exact n / d for n < 2^24 by an f32 reciprocal and two corrections
        const float inv_wp = 1.0f / (float)Wp, inv_hp = 1.0f / (float)g.Hp;
        auto fdiv = [](uint32_t n, uint32_t d, float inv) {
            int qq = (int)__fmul_rz((float)n, inv);
            int r = (int)n - qq * (int)d;
            if (r < 0) { --qq; r += (int)d; }
            if (r < 0) { --qq; r += (int)d; }
            if (r >= (int)d) { ++qq; r -= (int)d; }
            if (r >= (int)d) { ++qq; }
            return (uint32_t)qq;
        };
        // this warp's tiles are tb + h, tb + h + 2, ...: padded-raster coordinates of its lane's
        // position, advanced by 256 positions per tile instead of two divisions
        const uint32_t dR = 256u / (uint32_t)Wp, dcol = 256u - dR * (uint32_t)Wp;
        uint32_t cR, ccol, cb, coy;
        {
            const uint32_t t = (uint32_t)(tb + h) * kRows + q * 32 + lane;
            cR = fdiv(t, (uint32_t)Wp, inv_wp), ccol = t - cR * Wp;
            cb = fdiv(cR, (uint32_t)g.Hp, inv_hp), coy = cR - cb * g.Hp;
        }
        uint64_t *pack64 = reinterpret_cast<uint64_t *>(ep.pack_out);
        const int64_t pack_ld64 = ep.pack_ld32 >> 1;
        int ii = 0, tc = 0;
        // address of filter column j of an NCHW value: one IMAD.WIDE for 128-filter groups
        // (measured: layer 2's shortcut conv 83 -> 77 us, and r[] stays in registers); the
        // 64-filter kernel measured faster with the compiler's own address chains (106 vs 111 us)
        auto res_at = [&](auto *base, int j) {
            if constexpr (kF >= 128) return at_stride(base, ohw4, j);
            else return base + (int64_t)j * ohw;
        };
#pragma unroll 1
        for (int T0 = tb, T1 = tb; T0 < te; T0 = T1, ++ii) {
            T1 = item_end(T0, ii);
            const int bb = ii & 1;
            int Ra, nrows;
            band_of(T0, T1, Ra, nrows);
            wait_parked(bar_bfull + 8 * bb, (ii >> 1) & 1);  // (the band's popcounts)
            const int32_t *pcb = s_pc + bb * g.band_pos;
            bool released = false;
#pragma unroll 1
            for (int T = T0; T < T1; ++T, ++tc) {
                if ((tc & 1) != h) continue;
                const int buf = tc % kAcc;
                const uint32_t t = (uint32_t)T * kRows + q * 32 + lane;  // padded position
                const uint32_t col = ccol, b = cb, oy = coy;
                {   // advance to this warp's next tile
                    ccol += dcol;
                    uint32_t step = dR;
                    if (ccol >= (uint32_t)Wp) ccol -= Wp, ++step;
                    cR += step, coy += step;
                    while (coy >= (uint32_t)g.Hp) coy -= g.Hp, ++cb;
                }
                const bool mok = t < (uint32_t)g.P && oy < (uint32_t)g.OH && col < (uint32_t)g.OW;
                const int64_t m = ((int64_t)b * g.OH + oy) * g.OW + col;  // pixel index (NHWC order)
                const int64_t obase = ((int64_t)b * g.Ftot + f0) * ohw + (int64_t)oy * g.OW + col;
                if (g.res != nullptr && T + 2 < te && !(g.dbg & 64)) {
                    // warm L2 with the shortcut values of this warp's NEXT tile (T + 2, whose raster
                    // coordinates the advance above just produced): the f32 + shortcut epilogue is
                    // DRAM-latency-bound.  Lane l covers filters l, l + 32, ... at the first and last
                    // valid position of the warp's 32 (its span is at most two 128-byte lines per filter)
                    const bool nv = t + 2 * kRows < (uint32_t)g.P && coy < (uint32_t)g.OH && ccol < (uint32_t)g.OW;
                    const uint32_t vm = __ballot_sync(0xffffffffu, nv);
                    if (vm != 0) {
                        const int64_t nb = ((int64_t)cb * g.Ftot + f0) * ohw + (int64_t)coy * g.OW + ccol;
                        const int64_t n_lo = __shfl_sync(0xffffffffu, nb, __ffs(vm) - 1);
                        const int64_t n_hi = __shfl_sync(0xffffffffu, nb, 31 - __clz(vm));
#pragma unroll
                        for (int j = 0; j < kF; j += 32) {
                            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(g.res + n_lo + (int64_t)(j + lane) * ohw));
                            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(g.res + n_hi + (int64_t)(j + lane) * ohw));
                        }
                    }
                }
                int32_t pcs = 0;
                {
                    const int32_t *pw0 = pcb + ((int)t - Ra * Wp);
                    if (g.kh == 3 && g.kw == 3) {  // (nine independent loads)
#pragma unroll
                        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                            for (int kx = 0; kx < 3; ++kx) pcs += pw0[ky * Wp + kx];
                    } else {
                        for (int ky = 0; ky < g.kh; ++ky)
                            for (int kx = 0; kx < g.kw; ++kx) pcs += pw0[ky * Wp + kx];
                    }
                }
                const float rowf = kf - (float)pcs;
                if (T + 2 >= T1) {  // this warp's last tile of the item: the band's popcounts are consumed
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_bempty + 8 * bb);
                    released = true;
                }
                if (q == 0 && lane == 0) stamp(g, 4, tc);
                // the first 64 columns' residuals: in flight while the tile's MMAs finish
                float r[64];
                const bool use_res = g.res != nullptr && mok;
                if (use_res) {
#pragma unroll
                    for (int j = 0; j < 64; ++j) r[j] = __ldg(res_at(g.res + obase, j));
                }
                if (g.dbg & 4) wait_parked(bar_tfull + 8 * buf, (uint32_t)(tc / kAcc) & 1u);
                else {
                    if (lane == 0) wait_spin(bar_tfull + 8 * buf, (uint32_t)(tc / kAcc) & 1u);  // (one prober per warp)
                    __syncwarp();
                }
                fence_after();
                if (q == 0 && lane == 0) stamp(g, 5, tc);
                const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + buf * kF;
#pragma unroll 1
                for (int c0 = 0; c0 < kF && !(g.dbg & 2); c0 += 64) {
                    uint64_t bits = 0;
                    const bool thr_ok = s_thr_ok[c0 / 16] & s_thr_ok[c0 / 16 + 1] & s_thr_ok[c0 / 16 + 2] &
                                        s_thr_ok[c0 / 16 + 3];
                    if (pack_only && thr_ok) {
                        // packed output only: per-filter sign thresholds on a = P + popc(f)
                        uint32_t v[64];
#pragma unroll
                        for (int k = 0; k < 4; ++k) ld16(tacc + c0 + 16 * k, v + 16 * k);
                        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                        uint32_t w2[2] = {0u, 0u};
#pragma unroll
                        for (int j = 0; j < 64; ++j) {
                            const float a = __fmaf_rn(2.0f, __uint_as_float(v[j]), rowf);
                            uint32_t dmask;  // all ones iff a >= U
                            asm("set.ge.u32.f32 %0, %1, %2;\n" : "=r"(dmask) : "f"(a), "f"(s_thu[c0 + j]));
                            w2[j >> 5] |= dmask & (1u << (j & 31));
                        }
                        bits = ((uint64_t)(w2[1] ^ s_flip[(c0 >> 5) + 1]) << 32) | (w2[0] ^ s_flip[c0 >> 5]);
                        if (mok) pack64[m * pack_ld64 + ((f0 + c0) >> 6)] = bits;
                        continue;
                    }
                    float nf = 0.0f;
                    if (use_res && c0 != 0) {
#pragma unroll
                        for (int j = 0; j < 64; ++j)
                            r[j] = __ldg(res_at(g.res + obase + (int64_t)c0 * ohw, j));
                    }
#pragma unroll
                    for (int c1 = c0; c1 < c0 + 64; c1 += 32) {
                        uint32_t v[32];  // counts C, then (in place) the f32 outputs
                        ld16(tacc + c1, v);
                        ld16(tacc + c1 + 16, v + 16);
                        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int n = c1 + j;
                            // P = K - popc(pixel) - popc(filter) + 2C, exact in f32
                            const float P = __fmaf_rn(2.0f, __uint_as_float(v[j]), rowf - s_popc_ff[n]);
                            float x = dot ? __fmaf_rn(2.0f, P, -kf) : P;
                            if (affine) {
                                const float2 a = s_aff[n];
                                x = __fadd_rn(__fmul_rn(x, a.x), a.y);
                            }
                            if (has_bn) {
                                const float4 bp = s_par[n];  // reference op order, layers.py:598-602
                                x = __fadd_rn(__fmul_rn(bp.z, __fmul_rn(__fsub_rn(x, bp.x), bp.y)), bp.w);
                            }
                            if (use_res) x = __fadd_rn(x, r[(c1 - c0) + j]);
                            v[j] = __float_as_uint(x);
                        }
                        if (mok) {
                            if (g.y) {
                                float *yo = g.y + obase + (int64_t)c1 * ohw;
#pragma unroll
                                for (int j = 0; j < 32; ++j) *res_at(yo, j) = __uint_as_float(v[j]);
                            }
                            if constexpr (kPack) {
                                uint32_t w32 = 0;
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    const float fj = __uint_as_float(v[j]);
                                    if (fj >= 0.0f) w32 |= 1u << j;   // sign(-0) = +1
                                    nf = __fmaf_rn(fj, 0.0f, nf);     // NaN iff some f is NaN / Inf
                                }
                                bits |= (uint64_t)w32 << (c1 - c0);
                            }
                        }
                    }
                    if constexpr (kPack) {
                        if (mok) {
                            pack64[m * pack_ld64 + ((f0 + c0) >> 6)] = bits;
                            if (ep.pack_flags && nf != 0.0f) atomicOr(ep.pack_flags, BNN_FLAG_NONFINITE);
                        }
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_tempty + 8 * buf);
                if (q == 0 && lane == 0) stamp(g, 6, tc);
            }
            if (!released) {  // (no tile of this warp's parity in the item)
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_bempty + 8 * bb);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (tid == 0) stamp(g, 7, 2);
}

}  // namespace wconv

// Eligible: stride 1, C a multiple of 64 up to 512, F a multiple of 64, kh, kw <= 5 with
// C * kh * kw <= 5120 (LeNet's 5x5 conv: 38 vs 102 us on bnn_sconv.cu), padding <=
// kernel - 1, padded width <= 64, positions < 2^24, and two band buffers that fit in SMEM next to
// one filter group's expanded weights (groups of 128 filters when they fit, else 64; a CTA
// owns one filter group and a contiguous range of tiles).  Returns BNN_EUNSUP otherwise (the
// caller tries bnn_sconv.cu, then the general engine).
int launch_wconv(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W, const uint64_t *w,
                 int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                 int64_t oh, int64_t ow, float *y, const Epilogue &ep, cudaStream_t s, const float *res) {
    using namespace wconv;
    const int64_t Cw = C / 64;
    if (sh != 1 || sw != 1 || C % 64 != 0 || (Cw != 1 && Cw != 2 && Cw != 4 && Cw != 8) || F % 64 != 0 ||
        kh > 5 || kw > 5 || C * kh * kw > 5120 || ph > kh - 1 || pw > kw - 1 ||
        (g_debug.umma_bits & (1 << 19)))
        return BNN_EUNSUP;
    // C = 256 (filter groups of 128): faster than the TMA im2col engine on ResNet layer 3
    // (27 vs 40 us packed-only, 44 vs 67 us with the shortcut) once the per-CTA weight expansion
    // was batched; C = 512 does not fit next to two band buffers and falls through below.
    // Debug bit 17 forces the general engine for C >= 256.
    if (Cw > 2 && (g_debug.umma_bits & (1 << 17))) return BNN_EUNSUP;
    if (ep.pack_out && (ep.pack_ld32 < F / 32 || (ep.pack_ld32 & 1) ||
                        (reinterpret_cast<uintptr_t>(ep.pack_out) & 7)))
        return BNN_EUNSUP;
    if ((reinterpret_cast<uintptr_t>(x) & 15) != 0 && Cw >= 2) return BNN_EUNSUP;
    const int64_t Hp = H + 2 * ph, Wp = W + 2 * pw;
    const int64_t total_rows = B * Hp, P = total_rows * Wp;
    if (P <= 0) return BNN_OK;
    if (P + 128 >= (1ll << 24) || B * H * W * Cw >= (1ll << 31) || Wp > 64) return BNN_EUNSUP;
    if (oh != Hp - kh + 1 || ow != Wp - kw + 1) return BNN_EUNSUP;
    Geom g{};
    g.x = x, g.w = w, g.y = y, g.res = res;
    g.B = (int)B, g.H = (int)H, g.W = (int)W, g.Hp = (int)Hp, g.Wp = (int)Wp, g.OH = (int)oh, g.OW = (int)ow;
    g.kh = (int)kh, g.kw = (int)kw, g.ph = (int)ph, g.pw = (int)pw, g.K = (int)(C * kh * kw);
    g.total_rows = (int)total_rows, g.P = (int)P;
    g.ntiles = (int)ceil_div(P, kRows);
    g.Ftot = (int)F;
    g.dbg = (int)((g_debug.umma_bits >> 21) & 15);
    g.trace = (g_debug.umma_bits & 16) ? reinterpret_cast<long long *>(g_debug.trace_buf) : nullptr;
    const int planes = (int)(2 * Cw);
    // filter group size and the largest tpi <= 16 whose two band buffers fit
    int FG = 0, tpi = 0;
    for (int fgs = 128; fgs >= 64 && tpi == 0; fgs -= 64) {
        if (F % fgs != 0) continue;
        for (int t = 16; t >= 1; --t) {
            const int rows = (int)((t * kRows + (kh - 1) * Wp + (kw - 1) + Wp - 1) / Wp + 1);
            const int pos = (int)(rows * Wp), pb = pos * 16;
            const Smem L(fgs, g.K, planes, pb, pos);
            if (L.total + 1024 <= 225 * 1024 && pb < (1 << 18)) {
                FG = fgs, tpi = t, g.band_rows = rows, g.band_pos = pos, g.plane_bytes = pb;
                break;
            }
        }
    }
    if (tpi == 0) return BNN_EUNSUP;
    g.fgroups = (int)(F / FG);
    {
        // a CTA's range should split into >= 3 items, so that the band loads of an item overlap
        // the MMAs / epilogue of the previous one (ResNet-18 layer 2 at batch 256, 12 tiles per
        // CTA: items of 4 tiles 70 us against 76 us with one 10-tile item; layer 1, 45 tiles
        // per CTA, keeps large bands: fewer halo rows expanded twice)
        int sms0 = bnn_device_sm_count();
        if (sms0 <= 0) sms0 = 148;
        if (g_debug.grid_cap > 0 && sms0 > g_debug.grid_cap) sms0 = (int)g_debug.grid_cap;
        int nr = sms0 / g.fgroups < 1 ? 1 : sms0 / g.fgroups;
        if (nr > g.ntiles) nr = g.ntiles;
        const int per = g.ntiles / nr, want = per / 3 < 2 ? 2 : per / 3;
        if (want < tpi) {
            tpi = want;
            const int rows = (int)((tpi * kRows + (kh - 1) * Wp + (kw - 1) + Wp - 1) / Wp + 1);
            g.band_rows = rows, g.band_pos = (int)(rows * Wp), g.plane_bytes = g.band_pos * 16;
        }
    }
    g.tpi = tpi;
    const Smem L(FG, g.K, planes, g.plane_bytes, g.band_pos);
    const int smem = (int)L.total + 1024;
    int sms = bnn_device_sm_count();
    if (sms <= 0) sms = 148;
    if (g_debug.grid_cap > 0 && sms > g_debug.grid_cap) sms = (int)g_debug.grid_cap;
    g.nranges = sms / g.fgroups < 1 ? 1 : sms / g.fgroups;
    if (g.nranges > g.ntiles) g.nranges = g.ntiles;
    // C = 256 with only a few tiles per CTA (BASELINE configs[1]: 3): the per-CTA weight expansion
    // and the f32 store tail dominate and the TMA im2col engine is faster (30.6 vs 21 us cold)
    if (Cw > 2 && g.ntiles < 5 * g.nranges) return BNN_EUNSUP;
    const int grid = g.nranges * g.fgroups;
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
#define BNN_WCONV(KF, KCW)                                                                          \
    if (FG == KF && Cw == KCW) {                                                                    \
        static bool configured = false;                                                             \
        if (!configured) {                                                                          \
            cudaFuncSetAttribute(xnor_wconv_kernel<KF, KCW, true>,                                  \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);          \
            cudaFuncSetAttribute(xnor_wconv_kernel<KF, KCW, false>,                                 \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);          \
            configured = true;                                                                      \
        }                                                                                           \
        if (pack) cudaLaunchKernelEx(&cfg, xnor_wconv_kernel<KF, KCW, true>, g, ep);              \
        else cudaLaunchKernelEx(&cfg, xnor_wconv_kernel<KF, KCW, false>, g, ep);                  \
        return check_launch("xnor_wconv_kernel");                                                   \
    }
    BNN_WCONV(64, 1)
    BNN_WCONV(128, 1)
    BNN_WCONV(64, 2)
    BNN_WCONV(128, 2)
    BNN_WCONV(64, 4)
    BNN_WCONV(128, 4)
    BNN_WCONV(64, 8)
    BNN_WCONV(128, 8)
#undef BNN_WCONV
    return BNN_EUNSUP;
}

}  // namespace bnn

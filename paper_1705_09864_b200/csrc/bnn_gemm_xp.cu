// Large xnor-popcount GEMMs on pre-expanded operands (bnn_xnor_gemm_ws): the
// bits of both packed operands are expanded ONCE, by an HBM-bound pass, into
// e2m1 codes +1.0 / -1.0 (k >= K: 0.0) in a caller-provided workspace, and a
// persistent 2-CTA tcgen05 GEMM (cta_group::2, kind::mxf4, 256 x BN tiles)
// streams the codes straight from the workspace into SWIZZLE_128B operand
// tiles with TMA.  The f32 accumulator is then the signed dot product
// D = sum_k a_k b_k = 2P - K itself (gemm.py:3-8, 128-139: P = K - popcount(a ^ b)),
// exact for K < 2^24, so no row popcounts and no in-CTA expansion are needed.
//
// Why: the in-CTA expansion of bnn_umma_impl.cuh moves ~112 KB through shared
// memory per 448 tensor cycles (TMA write, expander reads, expanded stores, MMA
// reads) and is SMEM-bound near 0.45 of the kind::mxf4 issue rate.  Here a CTA
// of the pair moves 30 KB in and 30 KB out per 448 cycles, the B operand is
// shared by the two SMs of the pair, and no warp touches operand data.
//
// Same results as bnn_xnor_gemm (bit-identical f32), same reference functions
// (gemm.py:80-159, 226-291).  Epilogues other than the plain DOT / POPCOUNT
// decode return BNN_EUNSUP from the launcher and the caller falls back to the
// packed engine.
#include "bnn_umma_impl.cuh"

namespace bnn {
namespace xp {

using namespace umma;

// ------------------------------------------------------------------ expansion
struct ExpandOp {
    const uint2 *src;  // [rows, ld64] packed u64 words
    uint4 *dst;        // [rows, kw32] 16-byte groups of 32 e2m1 codes
    int64_t ld64, rows;
};

// u32 word w (bits 32 w .. 32 w + 31 of a row) -> 16 bytes: register j, nibble n <- bit
// 4 n + j as the e2m1 code 0x2 (+1.0) for a set bit, 0xA (-1.0) for a clear bit and
// 0x0 for positions >= K (tail bits of the last words, whatever the pad fill was).
// Both operands use the same permutation of K, which a dot product does not see.
__device__ __forceinline__ uint4 expand_pm1(uint32_t x, int64_t left) {
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = 0xAAAAAAAAu ^ (((x >> j) & 0x11111111u) << 3);
    if (left < 32) {
        const uint32_t vm = left <= 0 ? 0u : ((1u << left) - 1u);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] &= ((vm >> j) & 0x11111111u) * 0xFu;
    }
    return make_uint4(v[0], v[1], v[2], v[3]);
}

// one 256-bit store (32-byte aligned): a warp writes 1 KB runs of whole sectors per instruction
__device__ __forceinline__ void st256(uint4 *dst, const uint4 &lo, const uint4 &hi) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"l"(dst), "r"(lo.x),
                 "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
                 : "memory");
}

// HBM-bound pass over both operands: a thread takes one u64 word of kRows consecutive
// rows (kRows loads in flight), a warp writes 1 KB runs of codes
constexpr int kExpRows = 4;
__global__ void __launch_bounds__(128) expand_pm1_kernel(ExpandOp a, ExpandOp b, int64_t kw64,
                                                         int64_t K) {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // (the GEMM's setup overlaps this pass)
    const ExpandOp op = blockIdx.z == 0 ? a : b;
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= kw64) return;
    for (int64_t r0 = (int64_t)blockIdx.y * kExpRows; r0 < op.rows; r0 += (int64_t)gridDim.y * kExpRows) {
        uint2 x[kExpRows];
#pragma unroll
        for (int i = 0; i < kExpRows; ++i)
            x[i] = r0 + i < op.rows ? __ldg(op.src + (r0 + i) * op.ld64 + w) : make_uint2(0u, 0u);
#pragma unroll
        for (int i = 0; i < kExpRows; ++i) {
            if (r0 + i >= op.rows) break;
            st256(op.dst + (r0 + i) * 2 * kw64 + 2 * w, expand_pm1(x[i].x, K - 64 * w),
                  expand_pm1(x[i].y, K - 64 * w - 32));
        }
    }
}

// Multi-bit operands (bits == 2): planes 0 / 1 of a code c = b0 + 2 b1 -> the e2m1 code of
// the code's grid VALUE numerator: unsigned grid c in {0, 1, 2, 3}, signed grid 2c - 3 in
// {-3, -1, +1, +3} (all exact in e2m1), so the MMA accumulates sum_k v_a v_b directly
// (layers.py:240-242, 370-377 numerator; the division by L^2 is the epilogue's one rounding).
struct ExpandOp2 {
    const uint2 *p0, *p1;  // bit planes [rows, ld64]
    uint4 *dst;
    int64_t ld64, rows;
    int32_t is_signed;
};
__device__ __forceinline__ uint4 expand_code2_val(uint32_t w0, uint32_t w1, int64_t left, bool sgn) {
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t b0 = (w0 >> j) & 0x11111111u, b1 = (w1 >> j) & 0x11111111u;
        if (sgn) {  // c: 0 -> 0xD (-3), 1 -> 0xA (-1), 2 -> 0x2 (+1), 3 -> 0x5 (+3)
            const uint32_t x = b0 ^ b1, nx = x ^ 0x11111111u;
            v[j] = nx | (x << 1) | (nx << 2) | ((b1 ^ 0x11111111u) << 3);
        } else {    // c: 0 -> 0x0, 1 -> 0x2 (1), 2 -> 0x4 (2), 3 -> 0x5 (3)
            v[j] = (b0 & b1) | ((b0 & ~b1) << 1) | (b1 << 2);
        }
    }
    if (left < 32) {
        const uint32_t vm = left <= 0 ? 0u : ((1u << left) - 1u);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] &= ((vm >> j) & 0x11111111u) * 0xFu;
    }
    return make_uint4(v[0], v[1], v[2], v[3]);
}
__global__ void __launch_bounds__(128) expand_code2_kernel(ExpandOp2 a, ExpandOp2 b, int64_t kw64,
                                                           int64_t K) {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const ExpandOp2 op = blockIdx.z == 0 ? a : b;
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= kw64) return;
    for (int64_t r = blockIdx.y; r < op.rows; r += gridDim.y) {
        const uint2 x0 = __ldg(op.p0 + r * op.ld64 + w), x1 = __ldg(op.p1 + r * op.ld64 + w);
        st256(op.dst + r * 2 * kw64 + 2 * w, expand_code2_val(x0.x, x1.x, K - 64 * w, op.is_signed),
              expand_code2_val(x0.y, x1.y, K - 64 * w - 32, op.is_signed));
    }
}

// ------------------------------------------------------------------ GEMM
// kStaged: outputs leave through a per-warp SMEM block and TMA stores (6 operand stages fit);
// otherwise straight from registers (16 B per row per instruction; outputs TMA cannot address)
// and the 32 KB of staging become a 7th operand stage
template <int BN, bool kStaged>
struct Cfg {
    static_assert(BN % 32 == 0 && BN >= 64 && BN <= 224, "pair tile N");
    static constexpr int kStages = kStaged ? 6 : 7;
    static constexpr int kABytes = BM * 128;           // this CTA's 128 A rows x 256 codes
    static constexpr int kBRows = BN / 2;              // this CTA's half of the B rows
    static constexpr int kBBytes = kBRows * 128;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static_assert(kStageBytes % 1024 == 0, "SW128 atoms");
    static constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2, kEpiWarps = 4;
    static constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
    static constexpr int kStgBytes = 32 * 128;         // one 32 x 32 f32 block
    static constexpr int off_stage = 0;
    static constexpr int off_epi = kStages * kStageBytes;
    static constexpr int off_bars = off_epi + (kStaged ? kEpiWarps * 2 * kStgBytes : 0);
    static constexpr int kNumBars = 2 * kStages + 4;
    static constexpr int off_tmem = off_bars + kNumBars * 8;
    static constexpr int kSmemBytes = off_tmem + 16 + 1024;
    static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
    static constexpr int kSfCol = 2 * BN;              // UE8M0 scales (all 1.0) from here
    static_assert(kSfCol + 64 <= 512, "TMEM budget");
    // kind::mxf4: E2M1 x E2M1, UE8M0 scales, f32 accumulate, M = 256 (pair), N = BN
    static constexpr uint32_t kIdesc = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                       (1u << 23) | ((uint32_t)(2 * BM >> 4) << 24);
};

struct Params {
    float *C;
    int64_t ldc_m, ldc_n, M, N;
    int32_t kstages, tiles_m, ntiles;
    int32_t k_logical, domain;  // domain 2: out = accumulator * scale (multi-bit numerator / L^2)
    float scale;
    int32_t tma_store, vec4, park;
};

// TMA load into this CTA's SMEM, completing on the mbarrier of the pair's leader CTA
// (same offset, CTA-rank bit of the shared::cluster address cleared)
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                                 uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// the same, multicast to the CTAs of `mask` (same SMEM offset in each; every destination's
// bytes complete on the barrier of its own pair's leader)
__device__ __forceinline__ void tma_load_2d_pair_mc(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                                    uint32_t bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void umma_commit_mask(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            bar),
        "h"(mask)
        : "memory");
}

// kQuad: clusters of FOUR CTAs = two pairs working on vertically adjacent tiles (same B tile).
// Each CTA fetches a quarter of the B tile and multicasts it to the CTA of the same pair rank
// in the other pair, so a CTA pulls 128 + BN/4 instead of 128 + BN/2 rows per stage through the
// L2 -> SM fabric (the measured bound of the pair kernel).  A stage may be refilled only when
// BOTH pairs' MMAs have retired it: every commit is multicast to all four CTAs' empty barriers.
template <int BN, bool kStaged, bool kQuad>
__global__ void __launch_bounds__(Cfg<BN, kStaged>::kThreads, 1)
    xnor_xp_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                   const __grid_constant__ CUtensorMap omap, Params p, uint64_t *trace_buf) {
    using C = Cfg<BN, kStaged>;
    constexpr int S = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase_raw = smem_u32(smem_raw);
    const uint32_t sbase = (sbase_raw + 1023u) & ~1023u;
    uint8_t *sgen = smem_raw + (sbase - sbase_raw);
    const uint32_t s_stage = sbase + C::off_stage;
    const uint32_t s_epi = sbase + C::off_epi;
    const uint32_t bar_full = sbase + C::off_bars;   // [S] leader: both CTAs' TMA bytes landed
    const uint32_t bar_empty = bar_full + S * 8;     // [S] MMAs that read the stage retired
    const uint32_t bar_tfull = bar_empty + S * 8;    // [2] accumulator complete
    const uint32_t bar_tempty = bar_tfull + 2 * 8;   // [2] leader: both CTAs' epilogues drained it
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sgen + C::off_tmem);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t clrank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(clrank));
    const uint32_t crank = clrank & 1u;           // rank in the CTA pair; rank 0 issues the MMAs
    const uint32_t qidx = kQuad ? clrank >> 1 : 0u;  // which pair of the cluster
    const uint32_t lead = clrank & ~1u;           // cluster rank of this pair's leader
    constexpr int kCl = kQuad ? 4 : 2;
    const int t0 = (int)(blockIdx.x / kCl), tstep = (int)(gridDim.x / kCl);
    // quad: the tile loop runs over super-tiles of two vertically adjacent tiles
    const int tiles_mu = kQuad ? (p.tiles_m + 1) / 2 : p.tiles_m;
    const int nunits = kQuad ? tiles_mu * (p.ntiles / p.tiles_m) : p.ntiles;
    const uint32_t kstages = (uint32_t)p.kstages;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, kQuad ? 2 : 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, 2 * C::kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&amap)));
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&bmap)));
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&omap)));
    }
    if (warp == C::kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *s_tmem;
    if (warp >= C::kEpiWarp0) {  // block scales 2^0 in this CTA's TMEM lanes
        const uint32_t one[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
        for (int col = C::kSfCol; col < 512; col += 8)
            tmem_st8(tmem + ((uint32_t)((warp & 3) * 32) << 16) + col, one);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    fence_before();
    __syncthreads();
    cluster_sync();  // the peer's barriers and scales exist before any remote arrival / MMA
    fence_after();
    // programmatic dependent launch: the setup above overlapped the expansion pass; its codes
    // (and the previous users of the output buffer) are complete from here on
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (trace_buf && tid == 0) trace_at(trace_buf, 1);

    if (warp == C::kTmaWarp) {
        // ================================================================ TMA producer
        if (lane == 0) {
            uint32_t g = 0;
            const uint32_t lead_full = bar_full & 0xFEFFFFFFu;
#pragma unroll 1
            for (int tile = t0; tile < nunits; tile += tstep) {
                const int tm = (tile % tiles_mu) * (kQuad ? 2 : 1) + (int)qidx, tn = tile / tiles_mu;
                const int arow = tm * 2 * BM + (int)crank * BM;  // (past M in an odd last super-tile: zero fill)
                const int brow = tn * BN + (int)crank * C::kBRows + (int)qidx * (C::kBRows / 2);
#pragma unroll 1
                for (uint32_t ks = 0; ks < kstages; ++ks, ++g) {
                    const uint32_t s = g % S;
                    if (g >= S) {
                        if (p.park) mbar_wait(bar_empty + 8 * s, ((g / S) - 1) & 1u);
                        else mbar_wait_spin(bar_empty + 8 * s, ((g / S) - 1) & 1u);
                    }
                    if (crank == 0) mbar_arrive_expect_tx(bar_full + 8 * s, 2 * C::kStageBytes);
                    const uint32_t dst = s_stage + s * C::kStageBytes;
                    tma_load_2d_pair(dst, &amap, (int)(ks * 128), arow, lead_full + 8 * s);
                    if constexpr (kQuad)
                        tma_load_2d_pair_mc(dst + C::kABytes + qidx * (C::kBRows / 2) * 128, &bmap, (int)(ks * 128),
                                            brow, lead_full + 8 * s, (uint16_t)(5u << crank));
                    else
                        tma_load_2d_pair(dst + C::kABytes, &bmap, (int)(ks * 128), brow, lead_full + 8 * s);
                }
            }
        }
        __syncwarp();
    } else if (warp == C::kMmaWarp) {
        // ================================================================ MMA issuer (leader CTA)
        if (crank == 0) {
            uint32_t g = 0;
            int it = 0;
            const uint32_t sfc = tmem + C::kSfCol;
#pragma unroll 1
            for (int tile = t0; tile < nunits; tile += tstep, ++it) {
                const int buf = it & 1;
                if (it >= 2) mbar_wait_cluster(bar_tempty + 8 * buf, (uint32_t)((it >> 1) - 1) & 1u);
                fence_after();
                const uint32_t d = tmem + buf * BN;
#pragma unroll 1
                for (uint32_t ks = 0; ks < kstages; ++ks, ++g) {
                    const uint32_t s = g % S;
                    if (p.park) mbar_wait(bar_full + 8 * s, (g / S) & 1u);
                    else mbar_wait_spin(bar_full + 8 * s, (g / S) & 1u);
                    fence_after();
                    const uint32_t a_addr = s_stage + s * C::kStageBytes;
                    const uint64_t da = sw128_desc(a_addr), db = sw128_desc(a_addr + C::kABytes);
                    if (elect_one_sync()) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_fp4_pair<C::kIdesc>(d, da + 2 * kk, db + 2 * kk, sfc, sfc,
                                                    (ks | (uint32_t)kk) != 0 ? 1u : 0u);
                        umma_commit_mask(bar_empty + 8 * s, kQuad ? (uint16_t)0xF : (uint16_t)3);
                    }
                    __syncwarp();
                }
                if (elect_one_sync()) umma_commit_mask(bar_tfull + 8 * buf, (uint16_t)(3u << lead));
                __syncwarp();
            }
        }
    } else {
        // ================================================================ epilogue
        const int e = warp - C::kEpiWarp0, q = warp & 3;
        const uint32_t stg0 = s_epi + e * 2 * C::kStgBytes;
        const uint32_t lead_tempty = mapa_shared(bar_tempty, lead);
        const bool dot = p.domain == BNN_DOT, scaled = p.domain == 2;
        const float kf = (float)p.k_logical;
        int it = 0;
        uint32_t nst = 0;  // staged blocks so far (staging buffer parity)
#pragma unroll 1
        for (int tile = t0; tile < nunits; tile += tstep, ++it) {
            const int buf = it & 1;
            const int tm = (tile % tiles_mu) * (kQuad ? 2 : 1) + (int)qidx, tn = tile / tiles_mu;
            const int64_t mq = (int64_t)tm * 2 * BM + crank * BM + q * 32, n0 = (int64_t)tn * BN;
            const int64_t m = mq + lane;
            mbar_wait_sleep(bar_tfull + 8 * buf, (uint32_t)(it >> 1) & 1u);
            fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + buf * BN;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(taddr + c * 32, v);
                const int64_t nc = n0 + c * 32;
                if (mq >= p.M || nc >= p.N) continue;  // (warp-uniform)
                float f[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float dsum = __uint_as_float(v[j]);
                    f[j] = scaled ? __fmul_rn(dsum, p.scale) : (dot ? dsum : __fmul_rn(__fadd_rn(dsum, kf), 0.5f));
                }
                if (kStaged && p.tma_store) {
                    const uint32_t stg = stg0 + (nst & 1u) * C::kStgBytes;
                    ++nst;
                    if (lane == 0) bulk_wait_read<1>();  // the store two blocks back has read its buffer
                    __syncwarp();
                    const uint32_t row = stg + lane * 128;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                                         row + ((j ^ (lane & 7)) << 4)),
                                     "f"(f[4 * j]), "f"(f[4 * j + 1]), "f"(f[4 * j + 2]), "f"(f[4 * j + 3]));
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {  // (the TMA unit clips rows past M and columns past N)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                                reinterpret_cast<uint64_t>(&omap)),
                            "r"((int)nc), "r"((int)mq), "r"(stg)
                            : "memory");
                        bulk_commit();
                    }
                } else if (m < p.M) {
                    float *col = p.C + m * p.ldc_m + nc * p.ldc_n;
                    if (p.vec4 && nc + 32 <= p.N) {  // row-major: 128 contiguous bytes per lane
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            reinterpret_cast<float4 *>(col)[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
                    } else {  // [N, M] outputs: lanes = consecutive addresses (any strides work)
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (nc + j < p.N) col[j * p.ldc_n] = f[j];
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(lead_tempty + 8 * buf);
        }
        if (lane == 0) bulk_wait_all();
    }

    fence_before();
    __syncthreads();
    cluster_sync();  // the peer reads this CTA's SMEM and arrives on its barriers until here
    if (warp == C::kMmaWarp) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
    if (trace_buf && tid == 0) trace_at(trace_buf, 12);
}

// [rows, kb bytes] u8 view of an expanded operand; box = 128 bytes x box_rows, SWIZZLE_128B
static int encode_codes(CUtensorMap &map, const void *base, int64_t rows, int64_t kb, int box_rows) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return set_error(BNN_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)kb, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)kb};
    const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box,
                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(BNN_ECUDA, "cuTensorMapEncodeTiled failed (codes)");
    return BNN_OK;
}

template <int BN, bool kStaged, bool kQuad>
static int launch_cfg(const void *ea, const void *eb, int64_t kb, const GemmStore &st, const Epilogue &ep,
                      int64_t M, int64_t N, cudaStream_t s) {
    using C = Cfg<BN, kStaged>;
    auto kern = xnor_xp_kernel<BN, kStaged, kQuad>;
    constexpr int kCl = kQuad ? 4 : 2;
    CUtensorMap amap, bmap;
    int rc = encode_codes(amap, ea, M, kb, BM);
    if (rc == BNN_OK) rc = encode_codes(bmap, eb, N, kb, kQuad ? C::kBRows / 2 : C::kBRows);
    if (rc != BNN_OK) return rc;
    const int64_t tiles_m = ceil_div(M, 2 * BM), tiles_n = ceil_div(N, BN);
    const int64_t ntiles = tiles_m * tiles_n;
    if (ntiles > (1ll << 30)) return set_error(BNN_EUNSUP, "too many tiles");
    Params p{};
    p.C = st.C, p.ldc_m = st.ldc_m, p.ldc_n = st.ldc_n, p.M = M, p.N = N;
    p.kstages = (int32_t)ceil_div(kb, 128), p.tiles_m = (int32_t)tiles_m, p.ntiles = (int32_t)ntiles;
    p.k_logical = ep.k_logical, p.domain = ep.domain;
    p.scale = ep.inv_gamma;
    p.tma_store = st.has_map;
    p.park = (umma_dbg() & (1 << 21)) ? 1 : 0;
    p.vec4 = st.ldc_n == 1 && st.ldc_m % 4 == 0 && (reinterpret_cast<uintptr_t>(st.C) & 15) == 0;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    // clusters that can be co-resident (one CTA per SM; a cluster lives inside one GPC)
    static int max_clusters = -1;
    if (max_clusters < 0) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        cfg.gridDim = dim3((unsigned)(sm_count() / kCl * kCl));
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = sm_count() / kCl;
        }
        max_clusters = n;
    }
    const int64_t units = kQuad ? ceil_div(tiles_m, 2) * tiles_n : ntiles;
    int grid = (int)(units < max_clusters ? units : max_clusters) * kCl;
    if (g_debug.grid_cap > 0 && grid > g_debug.grid_cap) grid = (int)((g_debug.grid_cap + kCl - 1) / kCl * kCl);
    cfg.gridDim = dim3((unsigned)grid);
    cudaLaunchKernelEx(&cfg, kern, amap, bmap, st.omap, p, g_debug.trace_buf);
    return check_launch("xnor_xp_kernel");
}

}  // namespace xp

static int launch_tiles(const void *ea, const void *eb, int64_t kb, const GemmStore &st, const Epilogue &ep,
                        int64_t M, int64_t N, cudaStream_t s) {
    using namespace xp;
    // tile N from {224, 192, 160, 128}: waves over the SM pairs x the cycles of a K = 256 stage.
    // A stage is bound by the SM's shared-memory port, not the tensor pipe: the TMA writes
    // (128 + N/2) rows of 128 B and the MMA reads 128 + N rows (its own A rows and ALL of B, the
    // peer's half included) = 128 B x (256 + 1.5 N) at 128 B/clk, against 2 N tensor cycles
    // (profiles/r02: 578 cycles per stage measured at N = 224, tensor pipe 79% active)
    static const int cands[] = {224, 192, 160, 128};
    const int64_t pairs = sm_count() / 2, tm = ceil_div(M, 2 * umma::BM);
    int best = 224;
    int64_t best_cost = -1;
    for (int bn : cands) {
        const int64_t cost = ceil_div(tm * ceil_div(N, bn), pairs) * (512 + 3 * bn);
        if (best_cost < 0 || cost < best_cost) best = bn, best_cost = cost;
    }
    if (g_debug.fp4_bn == 128 || g_debug.fp4_bn == 160 || g_debug.fp4_bn == 192 || g_debug.fp4_bn == 224)
        best = (int)g_debug.fp4_bn;
    // row-major outputs leave through SMEM staging + TMA stores (6 operand stages); register
    // stores with a 7th stage measured slower (8192^3: 207 vs 198 us, 4096^3: 54 vs 44 us;
    // debug bit 1 << 20 selects them, bit 1 << 21 parks the TMA / MMA waits instead of spinning)
    const bool staged = st.has_map && !(umma_dbg() & (1 << 20));
    // clusters of two pairs sharing the B tile by TMA multicast: bit-exact but measured SLOWER
    // (8192^3: 211 vs 197 us) -- fewer rows cross the L2 -> SM fabric, yet every CTA's SMEM still
    // takes the same writes and MMA reads, which is what bounds a stage; debug bit 1 << 26 only
    const bool quad = staged && M > 2 * umma::BM && (umma_dbg() & (1 << 26)) != 0;
    if (quad) {
        switch (best) {
            case 128: return launch_cfg<128, true, true>(ea, eb, kb, st, ep, M, N, s);
            case 160: return launch_cfg<160, true, true>(ea, eb, kb, st, ep, M, N, s);
            case 192: return launch_cfg<192, true, true>(ea, eb, kb, st, ep, M, N, s);
            default: return launch_cfg<224, true, true>(ea, eb, kb, st, ep, M, N, s);
        }
    }
    switch (best) {
        case 128: return staged ? launch_cfg<128, true, false>(ea, eb, kb, st, ep, M, N, s) : launch_cfg<128, false, false>(ea, eb, kb, st, ep, M, N, s);
        case 160: return staged ? launch_cfg<160, true, false>(ea, eb, kb, st, ep, M, N, s) : launch_cfg<160, false, false>(ea, eb, kb, st, ep, M, N, s);
        case 192: return staged ? launch_cfg<192, true, false>(ea, eb, kb, st, ep, M, N, s) : launch_cfg<192, false, false>(ea, eb, kb, st, ep, M, N, s);
        default: return staged ? launch_cfg<224, true, false>(ea, eb, kb, st, ep, M, N, s) : launch_cfg<224, false, false>(ea, eb, kb, st, ep, M, N, s);
    }
}

int64_t xnor_gemm_xp_workspace(int64_t M, int64_t N, int64_t K) {
    const int64_t kw32 = 2 * ceil_div(K, 64);
    return (M + N) * kw32 * 16;
}

// BNN_EUNSUP: shape / epilogue / workspace not eligible (the caller runs the packed engine)
int launch_xnor_gemm_xp(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                        int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n, const Epilogue &ep,
                        cudaStream_t s, const float *res, void *ws, int64_t ws_bytes) {
    using namespace xp;
    if (ep.scale || ep.shift || ep.bn_mean || ep.pack_out || res || !C) return BNN_EUNSUP;
    if (ep.a_alpha != 1 || ep.a_beta != 0 || ep.b_alpha != 1 || ep.b_beta != 0) return BNN_EUNSUP;
    if (!ws || ws_bytes < xnor_gemm_xp_workspace(M, N, K) || (reinterpret_cast<uintptr_t>(ws) & 127))
        return BNN_EUNSUP;
    if (M > (1ll << 30) || N > (1ll << 30)) return BNN_EUNSUP;
    const int64_t kw32 = 2 * ceil_div(K, 64), kb = kw32 * 16;
    GemmStore st{};
    st.C = C, st.ldc_m = ldc_m, st.ldc_n = ldc_n, st.M = M, st.N = N;
    if (ldc_n == 1) encode_out(st);  // (row-major outputs TMA cannot address: plain stores)
    uint8_t *ea = static_cast<uint8_t *>(ws), *eb = ea + M * kb;
    ExpandOp oa{reinterpret_cast<const uint2 *>(A), reinterpret_cast<uint4 *>(ea), lda, M};
    ExpandOp ob{reinterpret_cast<const uint2 *>(B), reinterpret_cast<uint4 *>(eb), ldb, N};
    const int64_t rows = M > N ? M : N, kw64 = kw32 / 2, rgroups = ceil_div(rows, kExpRows);
    dim3 grid((unsigned)ceil_div(kw64, 128), (unsigned)(rgroups < 32768 ? rgroups : 32768), 2);
    expand_pm1_kernel<<<grid, 128, 0, s>>>(oa, ob, kw64, K);
    int rc = check_launch("expand_pm1_kernel");
    if (rc != BNN_OK) return rc;
    return launch_tiles(ea, eb, kb, st, ep, M, N, s);
}

// Multi-bit GEMM (bits == 2) on the same engine: ep carries the grid constants (a_alpha = 2 /
// a_beta = -3 for the signed grid) and inv_gamma = 1 / L^2; domain 2 = scaled accumulator.
// BNN_EUNSUP when 9 K >= 2^24 (the f32 accumulator would round) or the workspace is too small.
int launch_bitplane_gemm_xp(const uint64_t *A, int64_t lda, int64_t a_plane, const uint64_t *B, int64_t ldb,
                            int64_t b_plane, int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m,
                            int64_t ldc_n, const Epilogue &ep_in, cudaStream_t s, void *ws,
                            int64_t ws_bytes) {
    using namespace xp;
    if (!C || 9 * K >= (1ll << 24)) return BNN_EUNSUP;
    if (!ws || ws_bytes < xnor_gemm_xp_workspace(M, N, K) || (reinterpret_cast<uintptr_t>(ws) & 127))
        return BNN_EUNSUP;
    if (M > (1ll << 30) || N > (1ll << 30)) return BNN_EUNSUP;
    const int64_t kw32 = 2 * ceil_div(K, 64), kb = kw32 * 16, kw64 = kw32 / 2;
    GemmStore st{};
    st.C = C, st.ldc_m = ldc_m, st.ldc_n = ldc_n, st.M = M, st.N = N;
    if (ldc_n == 1) encode_out(st);
    uint8_t *ea = static_cast<uint8_t *>(ws), *eb = ea + M * kb;
    ExpandOp2 oa{reinterpret_cast<const uint2 *>(A), reinterpret_cast<const uint2 *>(A + a_plane),
                 reinterpret_cast<uint4 *>(ea), lda, M, ep_in.a_alpha == 2};
    ExpandOp2 ob{reinterpret_cast<const uint2 *>(B), reinterpret_cast<const uint2 *>(B + b_plane),
                 reinterpret_cast<uint4 *>(eb), ldb, N, ep_in.b_alpha == 2};
    const int64_t rows = M > N ? M : N;
    dim3 grid((unsigned)ceil_div(kw64, 128), (unsigned)(rows < 32768 ? rows : 32768), 2);
    expand_code2_kernel<<<grid, 128, 0, s>>>(oa, ob, kw64, K);
    int rc = check_launch("expand_code2_kernel");
    if (rc != BNN_OK) return rc;
    Epilogue ep = ep_in;
    ep.domain = 2;
    return launch_tiles(ea, eb, kb, st, ep, M, N, s);
}

// ================================================================== convolution
// Stride-s convs with C % 256 == 0 on the same engine (bnn_bconv2d_ws): the packed NHWC
// activations are expanded once into e2m1 codes with a physical halo of +1.0 codes (the
// reference's zero-pad-then-binarize, tensor.py:73-74 + bitpack.py:39), the weights into
// [F, K/2] code rows, and the GEMM's A operand (rows = output pixels, one TMEM lane each) is
// fetched by im2col-mode TMA loads of 128 pixels x 128 bytes (256 channels of one filter tap)
// per CTA and stage; B = a BN-row slice of the filters.  Lanes = pixels, so for every filter a
// warp reads / writes 32 consecutive pixels of the NCHW output and shortcut (coalesced), and a
// pixel's 32 sign bits are one u32 of the next layer's packed NHWC input, built in-lane.
// Epilogue in the reference op order (layers.py:225-245, 598-602): value -> scale / shift ->
// BatchNorm -> + shortcut -> f32 store and / or sign-pack.
namespace xp {

struct ConvExpand {
    const uint2 *x;   // packed NHWC [B, H, W, cw64]
    uint4 *e;         // codes [B, Hp, Wp, 2 cw64] uint4 (C / 2 bytes per pixel)
    const uint2 *w;   // packed weights [F, kw64]
    uint4 *we;        // codes [F, 2 kw64] uint4
    int64_t npad, wwords;  // B * Hp * Wp * cw64 activation items, F * kw64 weight items
    int32_t H, W, Hp, Wp, ph, pw, cw64;
};

__global__ void __launch_bounds__(256) expand_conv_kernel(ConvExpand c) {
    // programmatic dependent launch on both sides: the conv's setup may start while this pass
    // runs; this pass reads the previous layer's packed output only after that layer completed
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.y == 1) {  // weights: every bit is a valid +-1
        if (i >= c.wwords) return;
        const uint2 v = __ldg(c.w + i);
        st256(c.we + 2 * i, expand_pm1(v.x, 64), expand_pm1(v.y, 64));
        return;
    }
    if (i >= c.npad) return;
    const int64_t pix = i / c.cw64;
    const int wd = (int)(i - pix * c.cw64);
    const int xx = (int)(pix % c.Wp);
    const int64_t t = pix / c.Wp;
    const int yy = (int)(t % c.Hp);
    const int64_t b = t / c.Hp;
    const int iy = yy - c.ph, ix = xx - c.pw;
    uint4 lo, hi;
    if ((unsigned)iy < (unsigned)c.H && (unsigned)ix < (unsigned)c.W) {
        const uint2 v = __ldg(c.x + ((b * c.H + iy) * c.W + ix) * c.cw64 + wd);
        lo = expand_pm1(v.x, 64);
        hi = expand_pm1(v.y, 64);
    } else {
        lo = hi = make_uint4(0x22222222u, 0x22222222u, 0x22222222u, 0x22222222u);  // halo: +1
    }
    st256(c.e + 2 * i, lo, hi);
}

template <int BN>
struct ConvCfg {
    static_assert(BN % 32 == 0 && BN >= 64 && BN <= 224, "pair tile N");
    static constexpr int kStages = 6;
    static constexpr int kABytes = BM * 128;  // this CTA's 128 pixels x 256 channel codes
    static constexpr int kBRows = BN / 2;     // this CTA's half of the filter rows
    static constexpr int kStageBytes = kABytes + kBRows * 128;
    // two epilogue warps per TMEM lane quadrant (alternate 32-filter chunks): a tile has only
    // kh * kw * C / 256 stages, so its epilogue must finish within a few microseconds
    static constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2, kEpiWarps = 8;
    static constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
    static constexpr int kMaxF = 1024;        // per-filter epilogue parameters staged in SMEM
    static constexpr int off_par = kStages * kStageBytes;  // [6][kMaxF] f32
    static constexpr int off_bars = off_par + 6 * kMaxF * 4;
    static constexpr int kNumBars = 2 * kStages + 4;
    static constexpr int off_tmem = off_bars + kNumBars * 8;
    static constexpr int kSmemBytes = off_tmem + 16 + 1024;
    static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
    static constexpr int kSfCol = 2 * BN;
    static constexpr uint32_t kIdesc = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                       (1u << 23) | ((uint32_t)(2 * BM >> 4) << 24);
};

struct ConvParams {
    float *y;
    const float *res;
    uint32_t *pack_out;
    int64_t pack_ld32;
    int32_t *pack_flags;
    const float *scale, *shift, *bn_mean, *bn_inv, *bn_gamma, *bn_beta;
    int64_t npix, ohw;
    int32_t F, ow, sh, sw, kw, chunks;  // chunks = C / 256 (stages per filter tap)
    int32_t kstages, tiles_m, ntiles, k_logical, domain;
    int32_t raster, wp, dbg;
};

__device__ __forceinline__ void tma_load_im2col_pair(uint32_t dst, const CUtensorMap *map, int c, int w,
                                                     int h, int n, uint16_t off_w, uint16_t off_h,
                                                     uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.im2col.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar), "h"(off_w),
        "h"(off_h)
        : "memory");
}

template <int BN>
__global__ void __launch_bounds__(ConvCfg<BN>::kThreads, 1)
    xconv_xp_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                    const __grid_constant__ CUtensorMap rmap, ConvParams p) {
    using C = ConvCfg<BN>;
    constexpr int S = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase_raw = smem_u32(smem_raw);
    const uint32_t sbase = (sbase_raw + 1023u) & ~1023u;
    uint8_t *sgen = smem_raw + (sbase - sbase_raw);
    const uint32_t s_stage = sbase;
    float *s_par = reinterpret_cast<float *>(sgen + C::off_par);
    const uint32_t bar_full = sbase + C::off_bars;
    const uint32_t bar_empty = bar_full + S * 8;
    const uint32_t bar_tfull = bar_empty + S * 8;
    const uint32_t bar_tempty = bar_tfull + 2 * 8;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sgen + C::off_tmem);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t crank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
    const int t0 = (int)(blockIdx.x >> 1), tstep = (int)(gridDim.x >> 1);
    const uint32_t kstages = (uint32_t)p.kstages;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, 2 * C::kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&amap)));
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&bmap)));
    }
    if (warp == C::kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    // per-filter epilogue parameters (identity where absent): scale, shift, mean, inv_std, gamma, beta
    for (int f = tid; f < p.F; f += blockDim.x) {
        s_par[f] = p.scale ? __ldg(p.scale + f) : 1.0f;
        s_par[C::kMaxF + f] = p.shift ? __ldg(p.shift + f) : 0.0f;
        s_par[2 * C::kMaxF + f] = p.bn_mean ? __ldg(p.bn_mean + f) : 0.0f;
        s_par[3 * C::kMaxF + f] = p.bn_mean ? __ldg(p.bn_inv + f) : 1.0f;
        s_par[4 * C::kMaxF + f] = p.bn_mean ? __ldg(p.bn_gamma + f) : 1.0f;
        s_par[5 * C::kMaxF + f] = p.bn_mean ? __ldg(p.bn_beta + f) : 0.0f;
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *s_tmem;
    if (warp >= C::kEpiWarp0 && warp < C::kEpiWarp0 + 4) {
        const uint32_t one[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
        for (int col = C::kSfCol; col < 512; col += 8)
            tmem_st8(tmem + ((uint32_t)((warp & 3) * 32) << 16) + col, one);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    fence_before();
    __syncthreads();
    cluster_sync();
    fence_after();
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // (the expansion pass before us)

    if (warp == C::kTmaWarp) {
        // ================================================================ TMA producer
        if (lane == 0) {
            uint32_t g = 0;
            const uint32_t lead_full = bar_full & 0xFEFFFFFFu;
#pragma unroll 1
            for (int tile = t0; tile < p.ntiles; tile += tstep) {
                const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
                // this CTA's first output pixel -> window corner in the padded input
                int64_t n0 = (int64_t)tm * 2 * BM + crank * BM;
                if (n0 >= p.npix) n0 = 0;  // (a half-tile past the end: its rows are never stored)
                const int cb = (int)(n0 / p.ohw);
                const int pp = (int)(n0 - (int64_t)cb * p.ohw);
                const int cy = (pp / p.ow) * p.sh, cx = (pp % p.ow) * p.sw;
                const int brow = tn * BN + (int)crank * C::kBRows;
                int chunk = 0, ti = 0, tj = 0;
#pragma unroll 1
                for (uint32_t ks = 0; ks < kstages; ++ks, ++g) {
                    const uint32_t s = g % S;
                    if (g >= S) mbar_wait_spin(bar_empty + 8 * s, ((g / S) - 1) & 1u);
                    if (crank == 0) mbar_arrive_expect_tx(bar_full + 8 * s, 2 * C::kStageBytes);
                    const uint32_t dst = s_stage + s * C::kStageBytes;
                    if (p.raster)  // (timing experiment: tiled loads of the same bytes)
                        tma_load_2d_pair(dst, &rmap, chunk * 128, (int)n0 + ti * p.wp + tj, lead_full + 8 * s);
                    else
                        tma_load_im2col_pair(dst, &amap, chunk * 128, cx, cy, cb, (uint16_t)tj, (uint16_t)ti,
                                             lead_full + 8 * s);
                    tma_load_2d_pair(dst + C::kABytes, &bmap, (int)(ks * 128), brow, lead_full + 8 * s);
                    if (++chunk == p.chunks) {
                        chunk = 0;
                        if (++tj == p.kw) tj = 0, ++ti;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == C::kMmaWarp) {
        // ================================================================ MMA issuer (leader CTA)
        if (crank == 0) {
            uint32_t g = 0;
            int it = 0;
            const uint32_t sfc = tmem + C::kSfCol;
#pragma unroll 1
            for (int tile = t0; tile < p.ntiles; tile += tstep, ++it) {
                const int buf = it & 1;
                if (it >= 2) mbar_wait_cluster(bar_tempty + 8 * buf, (uint32_t)((it >> 1) - 1) & 1u);
                fence_after();
                const uint32_t d = tmem + buf * BN;
#pragma unroll 1
                for (uint32_t ks = 0; ks < kstages; ++ks, ++g) {
                    const uint32_t s = g % S;
                    mbar_wait_spin(bar_full + 8 * s, (g / S) & 1u);
                    fence_after();
                    const uint32_t a_addr = s_stage + s * C::kStageBytes;
                    const uint64_t da = sw128_desc(a_addr), db = sw128_desc(a_addr + C::kABytes);
                    if (elect_one_sync()) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_fp4_pair<C::kIdesc>(d, da + 2 * kk, db + 2 * kk, sfc, sfc,
                                                    (ks | (uint32_t)kk) != 0 ? 1u : 0u);
                        umma_commit_pair(bar_empty + 8 * s);
                    }
                    __syncwarp();
                }
                if (elect_one_sync()) umma_commit_pair(bar_tfull + 8 * buf);
                __syncwarp();
            }
        }
    } else {
        // ================================================================ epilogue (lane = pixel)
        const int q = warp & 3, half = (warp - C::kEpiWarp0) >> 2;
        const uint32_t lead_tempty = mapa_shared(bar_tempty, 0);
        const bool dot = p.domain == BNN_DOT;
        const bool affine = p.scale != nullptr || p.shift != nullptr, has_bn = p.bn_mean != nullptr;
        const float kf = (float)p.k_logical;
        int it = 0;
#pragma unroll 1
        for (int tile = t0; tile < p.ntiles; tile += tstep, ++it) {
            const int buf = it & 1;
            const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
            const int64_t n = (int64_t)tm * 2 * BM + crank * BM + q * 32 + lane;  // output pixel
            const bool nok = n < p.npix;
            const int64_t nn = nok ? n : 0;
            const int64_t b = nn / p.ohw;
            const int64_t base = b * p.F * p.ohw + (nn - b * p.ohw);  // + f * ohw
            mbar_wait_sleep(bar_tfull + 8 * buf, (uint32_t)(it >> 1) & 1u);
            fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + buf * BN;
#pragma unroll 1
            for (int c = half; c < BN / 32; c += 2) {
                if (p.dbg & 2) break;
                uint32_t v[32];
                tmem_ld32(taddr + c * 32, v);
                const int f0 = tn * BN + c * 32;
                if (f0 >= p.F) continue;  // (warp-uniform; F % 32 == 0)
                float f[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    float x = __uint_as_float(v[j]);
                    if (!dot) x = __fmul_rn(__fadd_rn(x, kf), 0.5f);
                    if (affine) x = __fadd_rn(__fmul_rn(x, s_par[f0 + j]), s_par[C::kMaxF + f0 + j]);
                    if (has_bn)
                        x = __fadd_rn(__fmul_rn(s_par[4 * C::kMaxF + f0 + j],
                                                __fmul_rn(__fsub_rn(x, s_par[2 * C::kMaxF + f0 + j]),
                                                          s_par[3 * C::kMaxF + f0 + j])),
                                      s_par[5 * C::kMaxF + f0 + j]);
                    f[j] = x;
                }
                if (nok) {
                    const int64_t o = base + (int64_t)f0 * p.ohw;
                    if (p.res) {  // all 32 loads in flight before any use
                        float r[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) r[j] = __ldg(p.res + o + j * p.ohw);
#pragma unroll
                        for (int j = 0; j < 32; ++j) f[j] = __fadd_rn(f[j], r[j]);
                    }
                    if (p.y && !(p.dbg & 1)) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) p.y[o + j * p.ohw] = f[j];
                    }
                    if (p.pack_out) {
                        uint32_t word = 0;
                        float nf = 0.0f;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            word |= (f[j] >= 0.0f ? 1u : 0u) << j;
                            nf = __fmaf_rn(f[j], 0.0f, nf);
                        }
                        p.pack_out[n * p.pack_ld32 + (f0 >> 5)] = word;
                        if (p.pack_flags && nf != 0.0f) atomicOr(p.pack_flags, 1);
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(lead_tempty + 8 * buf);
        }
    }

    fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == C::kMmaWarp) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

typedef CUresult (*EncodeIm2colU8Fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                     const cuuint64_t *, const cuuint64_t *, const int *, const int *,
                                     cuuint32_t, cuuint32_t, const cuuint32_t *, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// im2col map over the halo'd code tensor {C/2 bytes, Wp, Hp, B}: 128 pixels x 128 bytes per load,
// window corners traversed with the conv strides, no out-of-bounds taps (the halo is physical)
static int encode_codes_im2col(CUtensorMap &map, const void *e, int64_t cb, int64_t Wp, int64_t Hp,
                               int64_t B, int64_t ow, int64_t oh, int64_t sw, int64_t sh) {
    static EncodeIm2colU8Fn fn = nullptr;
    if (!fn) {
        void *q = nullptr;
        cudaDriverEntryPointQueryResult r;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &q, cudaEnableDefault, &r) == cudaSuccess &&
            r == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeIm2colU8Fn>(q);
    }
    if (!fn) return set_error(BNN_ECUDA, "cuTensorMapEncodeIm2col unavailable");
    const cuuint64_t dims[4] = {(cuuint64_t)cb, (cuuint64_t)Wp, (cuuint64_t)Hp, (cuuint64_t)B};
    const cuuint64_t strides[3] = {(cuuint64_t)cb, (cuuint64_t)(cb * Wp), (cuuint64_t)(cb * Wp * Hp)};
    const int lower[2] = {0, 0};
    const int upper[2] = {(int)((ow - 1) * sw - (Wp - 1)), (int)((oh - 1) * sh - (Hp - 1))};
    const cuuint32_t estr[4] = {1, (cuuint32_t)sw, (cuuint32_t)sh, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(e), dims, strides, lower,
                    upper, 128, (cuuint32_t)BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(BNN_ECUDA, "cuTensorMapEncodeIm2col failed (codes)");
    return BNN_OK;
}

template <int BN>
static int launch_conv_cfg(const CUtensorMap &amap, const CUtensorMap &rmap, const void *we, int64_t kb,
                           const ConvParams &p_in, cudaStream_t s) {
    using C = ConvCfg<BN>;
    auto kern = xconv_xp_kernel<BN>;
    CUtensorMap bmap;
    int rc = encode_codes(bmap, we, p_in.F, kb, C::kBRows);
    if (rc != BNN_OK) return rc;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        configured = true;
    }
    ConvParams p = p_in;
    const int64_t tiles_m = ceil_div(p.npix, 2 * BM), tiles_n = ceil_div((int64_t)p.F, BN);
    if (tiles_m * tiles_n > (1ll << 30)) return set_error(BNN_EUNSUP, "too many tiles");
    p.tiles_m = (int32_t)tiles_m, p.ntiles = (int32_t)(tiles_m * tiles_n);
    const int64_t pairs = sm_count() / 2;
    int grid = (int)(p.ntiles < pairs ? p.ntiles : pairs) * 2;
    if (g_debug.grid_cap > 0 && grid > g_debug.grid_cap) grid = (int)((g_debug.grid_cap + 1) & ~1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, kern, amap, bmap, rmap, p);
    return check_launch("xconv_xp_kernel");
}

}  // namespace xp

static bool conv_xp_shape_ok(int64_t C, int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw) {
    return C % 256 == 0 && F % 64 == 0 && F <= xp::ConvCfg<128>::kMaxF && sh <= 8 && sw <= 8 &&
           kh <= 128 && kw <= 128;
}

int64_t bconv2d_xp_workspace(int64_t B, int64_t C, int64_t H, int64_t W, int64_t F, int64_t kh, int64_t kw,
                             int64_t ph, int64_t pw) {
    const int64_t e = B * (H + 2 * ph) * (W + 2 * pw) * (C / 2);
    return ((e + 1023) / 1024) * 1024 + F * kh * kw * (C / 2);
}

// BNN_EUNSUP: geometry / workspace not eligible (the caller runs the packed engines)
int launch_bconv2d_xp(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W, const uint64_t *w,
                      int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                      int64_t oh, int64_t ow, float *y, const Epilogue &ep, cudaStream_t s,
                      const float *res, void *ws, int64_t ws_bytes) {
    using namespace xp;
    if (!conv_xp_shape_ok(C, F, kh, kw, sh, sw)) return BNN_EUNSUP;
    if (!ws || ws_bytes < bconv2d_xp_workspace(B, C, H, W, F, kh, kw, ph, pw) ||
        (reinterpret_cast<uintptr_t>(ws) & 127))
        return BNN_EUNSUP;
    if (ep.a_alpha != 1 || ep.a_beta != 0 || ep.b_alpha != 1 || ep.b_beta != 0) return BNN_EUNSUP;
    const int64_t Hp = H + 2 * ph, Wp = W + 2 * pw, cb = C / 2, cw64 = C / 64;
    const int64_t up_w = (ow - 1) * sw - (Wp - 1), up_h = (oh - 1) * sh - (Hp - 1);
    if (up_w < -128 || up_w > 0 || up_h < -128 || up_h > 0 || Wp > 65535 || Hp > 65535) return BNN_EUNSUP;
    const int64_t npix = B * oh * ow, K = C * kh * kw, kb = K / 2;
    if (npix > (1ll << 30) || B * Hp * Wp * cw64 > (1ll << 40)) return BNN_EUNSUP;
    uint8_t *e = static_cast<uint8_t *>(ws);
    uint8_t *we = e + ((B * Hp * Wp * cb + 1023) / 1024) * 1024;
    ConvExpand ce{reinterpret_cast<const uint2 *>(x), reinterpret_cast<uint4 *>(e),
                  reinterpret_cast<const uint2 *>(w), reinterpret_cast<uint4 *>(we),
                  B * Hp * Wp * cw64, F * (K / 64), (int32_t)H, (int32_t)W, (int32_t)Hp, (int32_t)Wp,
                  (int32_t)ph, (int32_t)pw, (int32_t)cw64};
    const int64_t items = ce.npad > ce.wwords ? ce.npad : ce.wwords;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)ceil_div(items, 256), 2);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, expand_conv_kernel, ce);
    }
    int rc = check_launch("expand_conv_kernel");
    if (rc != BNN_OK) return rc;
    CUtensorMap amap;
    rc = encode_codes_im2col(amap, e, cb, Wp, Hp, B, ow, oh, sw, sh);
    if (rc != BNN_OK) return rc;
    CUtensorMap rmap;
    rc = encode_codes(rmap, e, B * Hp * Wp, cb, BM);
    if (rc != BNN_OK) return rc;
    ConvParams p{};
    p.raster = (umma_dbg() & (1 << 22)) ? 1 : 0, p.wp = (int32_t)Wp;
    p.dbg = (umma_dbg() >> 23) & 3;  // timing experiments: 1 = no global stores, 2 = no epilogue work
    p.y = y, p.res = res, p.pack_out = ep.pack_out, p.pack_ld32 = ep.pack_ld32, p.pack_flags = ep.pack_flags;
    p.scale = ep.scale, p.shift = ep.shift, p.bn_mean = ep.bn_mean, p.bn_inv = ep.bn_inv;
    p.bn_gamma = ep.bn_gamma, p.bn_beta = ep.bn_beta;
    p.npix = npix, p.ohw = oh * ow, p.F = (int32_t)F, p.ow = (int32_t)ow, p.sh = (int32_t)sh;
    p.sw = (int32_t)sw, p.kw = (int32_t)kw, p.chunks = (int32_t)(C / 256);
    p.kstages = (int32_t)(kh * kw * (C / 256)), p.k_logical = ep.k_logical, p.domain = ep.domain;
    // filter tile from {224, 192, 160, 128}: waves over the SM pairs x the stage cost model
    static const int cands[] = {224, 192, 160, 128};
    const int64_t pairs = sm_count() / 2, tm = ceil_div(npix, 2 * umma::BM);
    int best = 128;
    int64_t best_cost = -1;
    for (int bn : cands) {
        const int64_t cost = ceil_div(tm * ceil_div(F, bn), pairs) * (512 + 3 * bn);
        if (best_cost < 0 || cost <= best_cost) best = bn, best_cost = cost;
    }
    switch (best) {
        case 128: return launch_conv_cfg<128>(amap, rmap, we, kb, p, s);
        case 160: return launch_conv_cfg<160>(amap, rmap, we, kb, p, s);
        case 192: return launch_conv_cfg<192>(amap, rmap, we, kb, p, s);
        default: return launch_conv_cfg<224>(amap, rmap, we, kb, p, s);
    }
}

}  // namespace bnn

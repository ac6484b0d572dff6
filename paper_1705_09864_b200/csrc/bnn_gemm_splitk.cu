// Small binary GEMMs (BASELINE configs[0]: QFullyConnected 4096 -> 1024, batch 256): one
// launch with IN-KERNEL split-K.  The general engine runs such shapes as 128 x 16 tiles
// whose 16 serial superstages set the time (~20 us); here a cluster of 8 CTAs owns one
// 128-row tile of A and splits K eight ways:
//   * every CTA loads its K slice of the packed operands with plain coalesced loads,
//     expands the bits to e2m1 codes in shared memory (SWIZZLE_128B K-major) and counts the
//     row popcounts of its slice;
//   * one thread issues the slice's MMAs (kind::mxf4, M = 128, N = the padded batch,
//     K = 64 per instruction) into one TMEM accumulator;
//   * the CTA turns its counts into the exact integer partial X = popc(a) + popc(b) - 2C
//     (popc(a ^ b) over its slice) and leaves it in its shared memory;
//   * after a cluster barrier, CTA r sums the eight partials of its eighth of the columns
//     through distributed shared memory in a fixed order (integers in f32: exact and
//     deterministic), applies the epilogue (P = k_eff - X, dot / affine / BN) and stores.
// Same reference path as bnn_umma_impl.cuh: xnor_gemm (gemm.py:128-139) behind
// QDense.forward (layers.py:361-369); bit-identical by construction.
#include "bnn_umma_impl.cuh"

namespace bnn {
namespace splitk {

using umma::expand_fp4_a;
using umma::expand_fp4_b;
using umma::fence_after;
using umma::fence_before;
using umma::mbar_init;
using umma::sw128_desc;
using umma::umma_commit;

constexpr int kS = 8;        // cluster size = K splits
constexpr int kRows = 128;   // A rows per tile (TMEM lanes)
constexpr int kMaxN = 256;   // padded B rows (MMA N)
constexpr int kMaxWpc = 8;   // u64 words of K per CTA
constexpr int kThreads = 256;
constexpr int kSfCol = 256;

struct Geom {
    const uint64_t *A, *B;
    int64_t lda, ldb;
    int M, N, Npad, W, wpc;  // W = u64 words per row; wpc = words per CTA (rank r: [r wpc, (r+1) wpc))
    float *C;
    int64_t ldc_m, ldc_n;
    const float *res;
    long long *trace;  // debug (bnn_umma_trace + debug bit 16): CTA 0's clock64 per phase
};
__device__ __forceinline__ void stamp(const Geom &g, int ev) {
    if (g.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0) g.trace[ev] = clock64();
}

// operands: [block of 4 K steps][row][128 B]; partials reuse the same memory as f32 [Npad][128]
constexpr int kOffA = 0;
constexpr int kOffB = kOffA + 2 * kRows * 128;
constexpr int kOffX = 0;
constexpr int kOperandBytes = kOffB + 2 * kMaxN * 128;            // 96 KB
constexpr int kXBytes = kMaxN * kRows * 4;                        // 128 KB
constexpr int kOffPop = kXBytes > kOperandBytes ? kXBytes : kOperandBytes;  // int [128] + int [256]
constexpr int kOffBar = kOffPop + (kRows + kMaxN) * 4 + (kRows + kMaxN / kS) * 4;  // (+ s_tot)
constexpr int kSmemBytes = kOffBar + 32 + 1024;

// kFast: wpc == 8 (every rank owns 8 whole words) and 16-byte aligned operand rows: two words per
// load, row popcounts by shuffles, no divisions
template <int kNpad, bool kFast>
__global__ void __launch_bounds__(kThreads, 1) xnor_splitk_kernel(const __grid_constant__ Geom g,
                                                                  const __grid_constant__ Epilogue ep) {
    // kind::mxf4, E2M1 x E2M1, UE8M0 scales, f32 accumulate, M = 128, N = kNpad
    constexpr uint32_t kIdesc = (1u << 7) | (1u << 10) | ((uint32_t)(kNpad >> 3) << 17) | (1u << 23) |
                                ((uint32_t)(kRows >> 4) << 24);
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sraw = smem_u32(smem_raw);
    const uint32_t sbase = (sraw + 1023u) & ~1023u;
    uint8_t *sgen = smem_raw + (sbase - sraw);
    const uint32_t s_a = sbase + kOffA, s_b = sbase + kOffB;
    float *s_x = reinterpret_cast<float *>(sgen + kOffX);
    int32_t *s_pa = reinterpret_cast<int32_t *>(sgen + kOffPop), *s_pb = s_pa + kRows;
    const uint32_t bar = sbase + kOffBar;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sgen + kOffBar + 16);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
    const int tile = blockIdx.x / kS;
    const int m0 = tile * kRows;

    stamp(g, 0);
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int i = tid; i < kRows + kMaxN; i += kThreads) s_pa[i] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *s_tmem;
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // (the pack kernel before us)
    if (warp < 4) {  // UE8M0 scale factors = 1.0
        const uint32_t one[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
        for (int col = kSfCol; col < 512; col += 8) umma::tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + col, one);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }

    stamp(g, 1);
    // ---- this CTA's K slice of both operands: load, count, expand
    const int w0 = (int)rank * g.wpc;
    const int nw = max(0, min(g.W, w0 + g.wpc) - w0);  // words of this slice (0: nothing to add)
    if constexpr (kFast) {
        // unit = (row, pair of u64 words): 4 units per row, (128 + kNpad) rows, all loads in flight
        constexpr int kUnits = (kRows + kNpad) * 4, kPer = (kUnits + kThreads - 1) / kThreads;
        ulonglong2 v[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int idx = tid + u * kThreads, row = idx >> 2, wq = (idx & 3) * 2;
            v[u] = make_ulonglong2(0ull, 0ull);
            if (idx < kUnits) {
                if (row < kRows) {
                    if (m0 + row < g.M)
                        v[u] = __ldg(reinterpret_cast<const ulonglong2 *>(g.A + (int64_t)(m0 + row) * g.lda + w0 + wq));
                } else if (row - kRows < g.N) {
                    v[u] = __ldg(reinterpret_cast<const ulonglong2 *>(g.B + (int64_t)(row - kRows) * g.ldb + w0 + wq));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int idx = tid + u * kThreads, row = idx >> 2, wq = (idx & 3) * 2;
            const bool isa = row < kRows;
            const int r = isa ? row : row - kRows;
            const uint32_t base = (isa ? s_a : s_b) + r * 128;
            const uint32_t rows = isa ? kRows : kNpad;
            const uint32_t w4[4] = {(uint32_t)v[u].x, (uint32_t)(v[u].x >> 32), (uint32_t)v[u].y, (uint32_t)(v[u].y >> 32)};
            if (idx < kUnits) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int k = 2 * wq + i;  // u32 word of the slice: block k / 8, chunk k % 8
                    uint32_t r4[4];
                    if (isa) expand_fp4_a(w4[i], r4);
                    else expand_fp4_b(w4[i], r4);
                    const uint32_t addr = base + (k >> 3) * (rows * 128) + (((k & 7) ^ (r & 7)) << 4);
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(r4[0]), "r"(r4[1]),
                                 "r"(r4[2]), "r"(r4[3])
                                 : "memory");
                }
            }
            // row popcount of the slice: the four lanes of a row
            int pc = __popcll(v[u].x) + __popcll(v[u].y);
            pc += __shfl_xor_sync(0xffffffffu, pc, 1);
            pc += __shfl_xor_sync(0xffffffffu, pc, 2);
            if ((tid & 3) == 0 && idx < kUnits) (isa ? s_pa : s_pb)[r] = pc;
        }
    } else
    {
        const int total = (kRows + kNpad) * g.wpc;
        constexpr int kBatch = 6;
#pragma unroll 1
        for (int base = tid; base < total; base += kBatch * kThreads) {
            uint64_t v[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int idx = base + u * kThreads;
                const int row = idx / g.wpc, wq = idx - row * g.wpc;
                v[u] = 0ull;
                if (idx < total && wq < nw) {
                    if (row < kRows) {
                        if (m0 + row < g.M) v[u] = __ldg(g.A + (int64_t)(m0 + row) * g.lda + w0 + wq);
                    } else if (row - kRows < g.N) {
                        v[u] = __ldg(g.B + (int64_t)(row - kRows) * g.ldb + w0 + wq);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int idx = base + u * kThreads;
                if (idx >= total) break;
                const int row = idx / g.wpc, wq = idx - row * g.wpc;
                const bool isa = row < kRows;
                const int r = isa ? row : row - kRows;
                const uint32_t rows = isa ? kRows : kNpad;
                const uint32_t opb = isa ? s_a : s_b;
#pragma unroll
                for (int hx = 0; hx < 2; ++hx) {
                    const uint32_t w32 = (uint32_t)(v[u] >> (32 * hx));
                    const int k = 2 * wq + hx;  // u32 word of the slice: block k / 8, chunk k % 8
                    uint32_t r4[4];
                    if (isa) expand_fp4_a(w32, r4);
                    else expand_fp4_b(w32, r4);
                    const uint32_t addr = opb + (k >> 3) * (rows * 128) + r * 128 + (((k & 7) ^ (r & 7)) << 4);
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(r4[0]), "r"(r4[1]),
                                 "r"(r4[2]), "r"(r4[3])
                                 : "memory");
                }
                const int pc = __popcll(v[u]);
                if (pc) atomicAdd(isa ? &s_pa[r] : &s_pb[r], pc);
            }
        }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();

    stamp(g, 2);
    // ---- MMAs of the slice (K = 64 per instruction), then wait for them
    if (tid == 0) {
        const uint64_t da0 = sw128_desc(s_a), db0 = sw128_desc(s_b);
        for (int st = 0; st < g.wpc; ++st) {
            const uint64_t da = da0 + (uint64_t)((((st >> 2) * (kRows * 128)) + (st & 3) * 32) >> 4);
            const uint64_t db = db0 + (uint64_t)((((st >> 2) * (kNpad * 128)) + (st & 3) * 32) >> 4);
            umma::mma_fp4<kIdesc>(tmem, da, db, tmem + kSfCol, tmem + kSfCol, st != 0 ? 1u : 0u);
        }
        umma_commit(bar);
    }
    {
        uint32_t done = 0;
        do {
            asm volatile(
                "{\n.reg .pred p;\n"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                "selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(bar), "r"(0u)
                : "memory");
        } while (!done);
    }
    fence_after();

    stamp(g, 3);
    // ---- this slice's counts C[m][n] = popc(a & b) <= 512 -> s_x16[n][m] as u16 (DSMEM moves
    // 17-21 B/clk per SM: half the bytes of f32; the operands are consumed, their memory is
    // reused); the row popcounts stay in s_pa / s_pb for the reducers
    {
        uint16_t *s_x16 = reinterpret_cast<uint16_t *>(s_x);
        const int q = warp & 3, h = warp >> 2;  // lane quadrant, column half
        const int m = q * 32 + lane;
        constexpr int kHalf = kNpad / 2;
#pragma unroll 1
        for (int c = 0; c < kHalf; c += 32) {
            uint32_t v[32];
            umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + h * kHalf + c, v);
#pragma unroll
            for (int j = 0; j < 32; ++j)
                s_x16[(h * kHalf + c + j) * kRows + m] = (uint16_t)__float2uint_rn(__uint_as_float(v[j]));
        }
    }
    fence_before();
    stamp(g, 4);
    umma::cluster_sync();
    stamp(g, 5);

    // ---- CTA `rank` sums the eight partials of its eighth of the columns (DSMEM):
    // X = sum popc(a) + sum popc(b) - 2 sum C in integers (exact, order-free), then the epilogue.
    // Thread = 8 rows (one 16-byte load of u16 counts per peer and column) x columns cl, cl + 16, ...
    {
        constexpr int kCols = kNpad / kS;
        const int m8 = tid & 15, cl = tid >> 4;
        uint32_t peer_x[kS], peer_p[kS];
#pragma unroll
        for (int j = 0; j < kS; ++j) {
            peer_x[j] = umma::mapa_shared(sbase + kOffX, (uint32_t)j);
            peer_p[j] = umma::mapa_shared(sbase + kOffPop, (uint32_t)j);
        }
        // total row popcounts, once per CTA (every other thread would re-read them over DSMEM, whose
        // 17-21 B/clk per SM is this phase's bound): rows m by threads 0..127, this rank's columns
        // by the next kCols threads -> s_tot[0..127], s_tot[128 + column]
        int32_t *s_tot = s_pa + kRows + kMaxN;
        if (tid < kRows + kCols) {
            const uint32_t off = tid < kRows ? (uint32_t)(4 * tid)
                                             : (uint32_t)(4 * (kRows + (int)rank * kCols + (tid - kRows)));
            int sum = 0;
#pragma unroll
            for (int j = 0; j < kS; ++j) {
                int t;
                asm volatile("ld.shared::cluster.s32 %0, [%1];\n" : "=r"(t) : "r"(peer_p[j] + off));
                sum += t;
            }
            s_tot[tid] = sum;
        }
        const float keff = (float)ep.k_eff, klog = (float)ep.k_logical;
        constexpr int kIter = (kCols + 15) / 16;
        uint4 c[kIter][kS];
#pragma unroll
        for (int it = 0; it < kIter; ++it) {
            const int cn = cl + 16 * it;
            const int n = (int)rank * kCols + (cn < kCols ? cn : 0);
#pragma unroll
            for (int j = 0; j < kS; ++j) {
                asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                             : "=r"(c[it][j].x), "=r"(c[it][j].y), "=r"(c[it][j].z), "=r"(c[it][j].w)
                             : "r"(peer_x[j] + (uint32_t)((n * kRows + 8 * m8) * 2)));
            }
        }
        __syncthreads();  // s_tot
        int pa[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pa[i] = s_tot[8 * m8 + i];
#pragma unroll
        for (int it = 0; it < kIter; ++it) {
            const int cn = cl + 16 * it;
            const int n = (int)rank * kCols + cn;
            if (cn >= kCols || n >= g.N) continue;
            // packed u16 pairs add without carries: 8 slices x <= 512 < 65536
            uint32_t w4[4] = {c[it][0].x, c[it][0].y, c[it][0].z, c[it][0].w};
            const int pb = s_tot[kRows + cn];
#pragma unroll
            for (int j = 1; j < kS; ++j)
                w4[0] += c[it][j].x, w4[1] += c[it][j].y, w4[2] += c[it][j].z, w4[3] += c[it][j].w;
            float o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int m = min(m0 + 8 * m8 + i, g.M - 1);
                const int cs = (int)((w4[i >> 1] >> (16 * (i & 1))) & 0xffffu);
                // X = popc(a) + popc(b) - 2C; the epilogue chain is Epilogue::apply's (bnn_common.cuh)
                o[i] = ep.apply(pa[i] + pb - 2 * cs, m);
            }
            const int m = m0 + 8 * m8;
            const int64_t at = (int64_t)m * g.ldc_m + (int64_t)n * g.ldc_n;
            if (g.ldc_m == 1 && m + 7 < g.M && !g.res && ((at & 3) == 0)) {
                *reinterpret_cast<float4 *>(g.C + at) = make_float4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<float4 *>(g.C + at + 4) = make_float4(o[4], o[5], o[6], o[7]);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (m + i < g.M) {
                        const int64_t a2 = at + (int64_t)i * g.ldc_m;
                        g.C[a2] = g.res ? __fadd_rn(o[i], __ldg(g.res + a2)) : o[i];
                    }
            }
        }
    }
    stamp(g, 6);
    // nobody leaves while a peer may still read its partials
    umma::cluster_sync();
    stamp(g, 7);
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

}  // namespace splitk

// Eligible: binary (1-bit) operands, no fused sign-pack, N <= 256, K <= 4096 (8 u64 words per
// CTA), at most 18 row tiles (one 8-CTA cluster each), C 16-byte aligned.  BNN_EUNSUP otherwise.
int launch_xnor_gemm_splitk(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                            int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n,
                            const Epilogue &ep, cudaStream_t s, const float *res) {
    using namespace splitk;
    const int64_t W = ceil_div(K, 64);
    const int64_t tiles = ceil_div(M, kRows);
    if (N > kMaxN || W > kS * kMaxWpc || W < 16 || tiles > 18 || tiles < 1 || ep.pack_out != nullptr ||
        ep.a_alpha != 1 || ep.a_beta != 0 || ep.b_alpha != 1 || ep.b_beta != 0 || C == nullptr ||
        (reinterpret_cast<uintptr_t>(C) & 15) != 0 ||
        (g_debug.umma_bits & (1 << 15)))
        return BNN_EUNSUP;
    Geom g{};
    g.A = A, g.B = B, g.lda = lda, g.ldb = ldb, g.M = (int)M, g.N = (int)N, g.W = (int)W;
    g.wpc = (int)ceil_div(W, kS);
    g.Npad = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
    g.C = C, g.ldc_m = ldc_m, g.ldc_n = ldc_n, g.res = res;
    g.trace = (g_debug.umma_bits & 16) ? reinterpret_cast<long long *>(g_debug.trace_buf) : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(tiles * kS));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kS, attr[0].val.clusterDim.y = 1, attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const bool fast = g.wpc == 8 && W == 64 && lda % 2 == 0 && ldb % 2 == 0 &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
#define BNN_SPLITK(NP)                                                                               \
    if (g.Npad == NP) {                                                                              \
        static bool configured = false;                                                              \
        if (!configured) {                                                                           \
            cudaFuncSetAttribute(xnor_splitk_kernel<NP, true>,                                       \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);           \
            cudaFuncSetAttribute(xnor_splitk_kernel<NP, false>,                                      \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);           \
            configured = true;                                                                       \
        }                                                                                            \
        if (fast) cudaLaunchKernelEx(&cfg, xnor_splitk_kernel<NP, true>, g, ep);                     \
        else cudaLaunchKernelEx(&cfg, xnor_splitk_kernel<NP, false>, g, ep);                         \
        return check_launch("xnor_splitk_kernel");                                                   \
    }
    BNN_SPLITK(64)
    BNN_SPLITK(128)
    BNN_SPLITK(256)
#undef BNN_SPLITK
    return BNN_EUNSUP;
}

}  // namespace bnn

// (bnn_umma_impl.cuh: kernel + launch templates, included by bnn_gemm_umma.cu and
// bnn_gemm_umma_pk.cu -- the sign-pack epilogue instantiations live in their own
// translation unit so the two sets compile in parallel)
//
// xnor-popcount GEMM / implicit-im2col binary conv on the 5th-gen tensor
// cores (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM), the BNN_ALGO_UMMA
// engine.  Replaces the same reference functions as bnn_gemm_popc.cu
// (gemm.py:80-159, layers.py:225-245); results are bit-identical.
//
// B200 has no binary tensor-core MMA (b1 mma.sync is emulated on sm_100a,
// SURVEY 0), so each CTA expands its packed operands to bytes right before
// the MMA consumes them.  The expansion is one LOP3 per 4 bytes.  For u32
// word w, register r in 0..7 and byte j in 0..3, byte j of register r
// stands for bit 8j + r of w:
//     B (activations):  w & (0x01010101 << r)        -> bit * 2^r
//     A (weights):      w' & (0x80808080 >> r)       -> bit * 2^(7-r)
// where w' = w with the bits of every byte reversed (BREV + PRMT, 2 ops per
// A word).  Every product is therefore 2^7 * [a_k = 1 and b_k = 1] and the
// s32 accumulator holds 128 * C with C = popc(a & b) (exact for K < 2^24).
// Both operands use the same K permutation (byte 4r + j of a word's 32
// expanded bytes <- bit 8j + r), and a sum over K is permutation invariant.
// The xnor count is then recovered as in the north star's .and.popc form:
//     X = popc(a) + popc(b) - 2C,   P = k_eff - X
// with popc(a), popc(b) counted by the producer threads as they expand.
//
// Persistent, warp-specialised CTA (one per SM) looping over 128 x BN output
// tiles; K is streamed in 128-bit slices (128 expanded bytes per row).
//   warps [0, P)   producers, one operand row each (128 A rows + BN B rows):
//                  cp.async packed words into a private PD-deep ring (running
//                  ahead across tile boundaries), expand, write the stage:
//                  B rows -> SWIZZLE_128B K-major SMEM (st.shared.v4);
//                  A rows -> SMEM as well (kATmem = false) or straight into
//                  TMEM with tcgen05.st (kATmem = true: the MMA then reads A
//                  from TMEM and only B crosses shared memory);
//                  then arrive on full[s].
//   warp P         TMEM allocator + single-thread tcgen05.mma issuer (4 MMAs
//                  of K=32 per stage; commit -> empty[s]; per tile commit ->
//                  tmem_full[buf]).
//   warps P+1..P+8 epilogue: tcgen05.ld 32x32b.x16 of accumulator buffer
//                  buf (double-buffered, so it overlaps the next tile's MMA),
//                  decode, transpose through SMEM, coalesced 128-byte stores;
//                  arrive tmem_empty[buf].
#pragma once
#include <cuda.h>

#include <cstdlib>
#include <type_traits>

#include "bnn_loaders.cuh"

// build-time tuning knobs of the kind::mxf4 engine (tools/build_variant.sh)
#ifndef BNN_WAIT_SLEEP_NS
#define BNN_WAIT_SLEEP_NS 0  // (32: measured -12% at 8192^3 -- polling warps take the expanders' issue slots)
#endif
#ifndef BNN_FP4_ES
#define BNN_FP4_ES 3
#endif
#ifndef BNN_PAIR_ES
#define BNN_PAIR_ES 5  // expanded buffers of a CTA pair: hide the cluster-scope arrival latency
#endif
#ifndef BNN_MARK_FENCE
#define BNN_MARK_FENCE 1
#endif
#ifndef BNN_FP4_PAIR_KW32
// K words (u32) from which 2-CTA pairs are used (M >= 256).  Off by default: every
// superstage of a pair needs one cluster-scope release/arrive from the peer CTA,
// measured at ~0.7 us each, which caps the pair below the single-CTA engine
// (8192^3: 2.5 vs 3.7 POPS).  BNN_PAIR_KW32=<n> enables it for experiments.
#define BNN_FP4_PAIR_KW32 (1ll << 40)
#endif
#ifndef BNN_FP4_SETS_KW32
#define BNN_FP4_SETS_KW32 192  // K words (u32) from which two expander sets are used
#endif
#ifndef BNN_FP4_TMA_SLOTS
#define BNN_FP4_TMA_SLOTS 4
#endif

namespace bnn {

// Dense packed operand [rows, ld32] u32 fetched by the tensor-memory
// accelerator: a 2-D tensor map over the kw32 valid words of every row; one
// cp.async.bulk.tensor per operand per superstage writes the rows' packed
// words (row-major, 16 B per stage per row, SWIZZLE_32B when a superstage is
// two stages) and signals an mbarrier with complete_tx.  Rows past the end and
// words past kw32 are zero-filled by the TMA unit, which the and-popcount
// decode ignores (a zero word matches a zero word).
struct TmaRows {
    static constexpr bool kTma = true;
    CUtensorMap map;
    const uint32_t *base;
    int64_t ld32, rows, kw32;
    // (the cp.async loader interface, unused on the TMA path)
    struct Cursor {};
    __device__ Cursor row(int64_t) const { return {}; }
    template <int kVec>
    __device__ void load(Cursor &, int, uint32_t, int = 0) const {}
};

// Implicit-im2col activations for the TMA path: an im2col tensor map over
// the packed NHWC words {cs32, W, H, B}; one load per superstage fetches, for
// BN consecutive output pixels, the 32 bytes of channel words of one filter
// tap (cp.async.bulk.tensor.4d.im2col with the tap as the im2col offset).
// Out-of-image taps come back zero-filled; the expander thread of that pixel
// row knows its window corner and the superstage's tap, and substitutes the
// all-ones word -- the reference's "+1" padding (tensor.py:73-74 +
// bitpack.py:39).  Requires cs32 % 8 == 0 (C a multiple of 256), so a
// superstage never straddles two taps and no channel tail exists.
struct TmaConv {
    static constexpr bool kTma = true;
    CUtensorMap map;
    const uint32_t *x;
    int64_t npix;
    int H, W, cs32, kw, sh, sw, ph, pw, oh, ow;
    struct Cursor {};
    __device__ Cursor row(int64_t) const { return {}; }
    template <int kVec>
    __device__ void load(Cursor &, int, uint32_t, int = 0) const {}
};

namespace umma {

constexpr int BM = 128;

// Debug timeline (bnn_umma_trace): when a buffer is set, CTA c records
// %globaltimer at slot s into trace_buf[c * kTraceSlots + s] (kernel argument,
// null in production).
constexpr int kTraceSlots = 16;
__device__ __forceinline__ void trace_at(uint64_t *buf, int slot) {
    if (buf) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        buf[blockIdx.x * kTraceSlots + slot] = t;
    }
}
constexpr int kWordsPerStage = 4;  // u32 words of K per row per stage
constexpr int kRowBytes = 128;     // expanded bytes per row per stage

template <int BN, bool kATmem, int kPlanes = 1, bool kTma = false, bool kFp4 = false,
          int kSetsT = 1, bool kPair = false>
struct Cfg {
    // kPair: a cluster of two CTAs computes a 256 x BN tile with tcgen05.mma.cta_group::2
    // (issued by the even CTA); each CTA expands its 128 A rows and half of the BN B rows,
    // so per MAC the B-operand expansion, SMEM stores and SMEM operand reads halve
    static_assert(!kPair || (kFp4 && kTma && kSetsT == 1 && BN <= 256), "pair: fp4, TMA, one set");
    static constexpr int kBRows = kPair ? BN / 2 : BN;  // B rows expanded by this CTA
    static constexpr int kTmBM = kPair ? 2 * BM : BM;    // tile rows
    static_assert(BN % 16 == 0 && BN >= 16 && (BN <= 256 || (kFp4 && BN % 32 == 0 && BN <= 384)),
                  "UMMA N for M=128 (wide fp4 tiles: two MMAs of N/2)");
    // tiles wider than one MMA (fp4, N <= 384) issue two MMAs of N/2 per K step into
    // adjacent TMEM column ranges; their single accumulator buffer is meant for
    // shapes that fit in one wave of CTAs
    static constexpr int kMmaN = BN > 256 ? BN / 2 : BN;
    static constexpr int kNMma = BN / kMmaN;
    static_assert(!kFp4 || (kPlanes == 1 && kTma && !(kATmem && kPair)), "fp4 engine: TMA-fed");
    static constexpr int kProducers = BM + kBRows;             // one thread per operand row
    static constexpr int kProducerWarps = (kProducers + 31) / 32;
    // kind::mxf4: two expander sets take alternate superstages, so each warp's
    // barrier round trip (slot wait, popcounts, release, buffer wait, proxy fence,
    // arrival) overlaps the other set's
    static constexpr int kSets = kSetsT;
    static_assert(kSets == 1 || (kSets == 2 && kFp4), "expander sets: kind::mxf4 engine only");
    static constexpr int kExpWarps = kProducerWarps * kSets;
    static constexpr int kTmaWarp = kExpWarps;  // one elected lane issues the TMA loads
    static constexpr int kMmaWarp = kTmaWarp + 1;
    static constexpr int kEpiWarp0 = kMmaWarp + 1;
    // 2 epilogue warps per TMEM lane quadrant; 1 with two expander sets (register budget)
    static constexpr int kEpiWarps = kSets == 2 ? 4 : 8;
    static constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
    // K is consumed in 128-bit stages grouped into superstages of kSub stages:
    // every barrier round trip (expanded-buffer wait, proxy fence, full arrival,
    // MMA commit) is paid once per superstage
    static constexpr int kSub = (kATmem || kFp4) ? 2 : 1;
    static constexpr int PD = (kATmem && kPlanes == 1) ? 8 : 4;  // per-thread packed ring (stages)
    static_assert((PD & (PD - 1)) == 0 && PD >= 2 * kSub, "packed ring depth");
    // bytes of one row per 128-bit stage: u8 expansion 128, e2m1 expansion 64 (an
    // fp4 superstage row is one 128-byte SW128 row; A rows precede B rows)
    static constexpr int kStageRow = kFp4 ? 64 : kRowBytes;
    static constexpr int kStageA = kATmem ? 0 : BM * kStageRow;
    static constexpr int kStageB = kBRows * kStageRow;
    static constexpr int kStageBytes = kStageA + kStageB;
    static constexpr int kSuperBytes = kSub * kStageBytes;
    static constexpr int ES = (kATmem && !kFp4) ? 2 : (kATmem ? ((512 - 2 * BN - 32) / 32 < 4 ? (512 - 2 * BN - 32) / 32 : 4) : (kPair ? BNN_PAIR_ES : (kFp4 ? (BN > 256 ? 2 : (BN <= 176 ? BNN_FP4_ES : 3)) : 3)));  // expanded superstage buffers
    static constexpr int kFp4A = kATmem ? 0 : BM * 128;  // fp4: A block of a superstage buffer
    // fp4 with A in TMEM: one 128-byte row per superstage = 32 TMEM columns per stage buffer
    static constexpr int kAStageCols = kFp4 ? 32 : kSub * 32;
    // TMEM: 2 accumulator buffers of BN columns (+ ES x kSub A stages of 32 columns)
    static constexpr int kAccCols = BN;
    static constexpr int kAccBufs = BN > 256 ? 1 : 2;  // TMEM accumulator buffers
    static constexpr int kAStageCol = 2 * BN;
    static constexpr int kTmemCols = 512;
    static constexpr int kSfCol = (BN > 256 ? 1 : 2) * BN + (kATmem ? ES * kAStageCols : 0);  // fp4: UE8M0 scales (all 1.0) from here
    // (fp4 scale factors: 64 columns reserved, 32 with A in TMEM -- every byte from kSfCol
    // on holds the UE8M0 value 1.0, and SFA / SFB of one MMA span a few columns)
    static_assert((BN > 256 ? 1 : 2) * BN + (kATmem ? ES * kAStageCols : 0) + (kFp4 ? (kATmem ? 32 : 64) : 0) <= 512,
                  "TMEM budget");
    // shared memory carve-up (offsets from the 1024-aligned base)
    // epilogue staging: per warp 32 rows x 32 f32 = 4 KB in the SWIZZLE_128B layout
    // (16-B chunk c of row r at (c ^ (r & 7))): conflict-free row writes and
    // transposed reads, and the layout a TMA store consumes
    static constexpr int kStgBytes = 32 * 128;
    static constexpr int off_exp = 0;
    static constexpr int off_pk = ES * kSuperBytes;
    // packed staging: per-thread cp.async rings (PD stages x 16 B per row), or
    // with TMA kTmaSlots superstage slots of [A rows | B rows] x kSub x 16 B
    static constexpr int kTmaSlots = (kFp4 && BN > 256) ? 3 : ((kFp4 && BN <= 176) ? BNN_FP4_TMA_SLOTS : 4);
    static constexpr int kTmaA = BM * kSub * 16, kTmaB = kBRows * kSub * 16;
    static constexpr int kTmaBoxB = BN > 256 ? BN / 2 : kBRows;  // tiled TMA boxes are <= 256 rows
    static constexpr int kTmaSlotBytes = ((kTmaA + kTmaB + 1023) / 1024) * 1024;
    static constexpr int kPkBytes = kTma ? kTmaSlots * kTmaSlotBytes
                                         : PD * kProducerWarps * 32 * 16 * kPlanes;
    static constexpr int off_popc_a = off_pk + kPkBytes;
    static constexpr int off_popc_b = off_popc_a + kSets * 2 * BM * 4;  // [set][buf][row]
    static constexpr int off_epi = ((off_popc_b + kSets * 2 * kBRows * 4 + 1023) / 1024) * 1024;
    static constexpr int off_bars = off_epi + kEpiWarps * kStgBytes;
    static constexpr int kNumBars = 2 * ES + 6 + 2 * kTmaSlots;
    static constexpr int off_tmem = off_bars + kNumBars * 8;
    static constexpr int kSmemBytes = off_tmem + 16 + 1024;
    static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
    static constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) |
                                       ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    // kind::mxf4: E2M1 x E2M1 (format 1), UE8M0 scales (bit 23), f32 accumulate
    static constexpr uint32_t kIdescFp4 = (1u << 7) | (1u << 10) | ((uint32_t)(kMmaN >> 3) << 17) |
                                          (1u << 23) | ((uint32_t)(kTmBM >> 4) << 24);
};

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// arrive after `dep` has been computed (a register dependency orders it after the
// instructions that produced dep, e.g. the consumers of a buffer being released)
__device__ __forceinline__ void mbar_arrive_dep(uint32_t bar, int32_t dep) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n// dep %1\n" ::"r"(bar), "r"(dep)
                 : "memory");
}
// debug watchdog (bnn_umma_watchdog): a wait that
// does not complete within ~2 s logs (block, warp, barrier offset, parity) and traps
static __device__ uint64_t *g_wait_log = nullptr;
static __device__ __noinline__ void wait_timeout(uint32_t bar, uint32_t phase, uint32_t tries) {
    if (tries == (1u << 22) + 1 && g_wait_log && (threadIdx.x & 31) == 0) {  // record once per warp
        const uint32_t slot = atomicAdd(reinterpret_cast<unsigned int *>(g_wait_log), 1u) % 64u;
        g_wait_log[1 + slot] = ((uint64_t)blockIdx.x << 48) | ((uint64_t)(threadIdx.x >> 5) << 40) |
                               ((uint64_t)(bar & 0xFFFFF) << 8) | phase;
        uint64_t state;
        asm volatile("ld.shared.b64 %0, [%1];\n" : "=l"(state) : "r"(bar));
        if (slot < 32) g_wait_log[65 + 8 * 16 + slot] = state;  // raw mbarrier word
        __threadfence_system();
    }
    if (tries > (1u << 23)) asm volatile("trap;");  // every stuck warp has recorded by now
}
// cluster (2-CTA pair) helpers: address of the same shared variable in CTA `rank`,
// release/acquire arrivals and waits at cluster scope
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    uint32_t tries = 0;
    const bool watch = g_wait_log != nullptr;  // (one global load per wait, not per probe)
    do {
        if (watch && ++tries > (1u << 22)) wait_timeout(bar, phase, tries);
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                     : "memory");
}
template <uint32_t kIdesc>
__device__ __forceinline__ void mma_fp4_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            bar),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_im2col_4d(uint32_t dst, const CUtensorMap *map, int c,
                                                   int w, int h, int n, uint16_t off_w,
                                                   uint16_t off_h, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar),
        "h"(off_w), "h"(off_h)
        : "memory");
}
// debug progress marks next to the watchdog log: g_wait_log[65 + 8 * block + k] = v
__device__ __forceinline__ void progress_mark(int k, uint64_t v) {
    if (g_wait_log && blockIdx.x < 16) {
        g_wait_log[65 + 8 * blockIdx.x + k] = v;
        if (BNN_MARK_FENCE) __threadfence_system();
    }
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    // the suspend-time hint parks the warp in try_wait until the phase
    // completes instead of re-issuing the probe (spinning warps steal issue
    // slots from the expanders sharing their scheduler)
    uint32_t done = 0;
    uint32_t tries = 0;
    const bool watch = g_wait_log != nullptr;  // (one global load per wait, not per probe)
    do {
        if (watch && ++tries > (1u << 22)) wait_timeout(bar, phase, tries);
#if BNN_WAIT_SLEEP_NS
        // short sleeps between probes instead of parking in try_wait: parked warps on one
        // barrier wake up one after another (the last of an expander set ~1 us after the
        // first, tools/umma_stages_conv.py), and the stragglers pace every superstage
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
        if (!done) __nanosleep(BNN_WAIT_SLEEP_NS);
#else
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase), "r"(0x989680u)
            : "memory");
#endif
    } while (!done);
}
// latency-critical waits: spin on test_wait (no suspension, so no wake-up latency
// after the phase completes)
__device__ __forceinline__ void mbar_wait_spin(uint32_t bar, uint32_t phase) {
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
// long waits (epilogue): the thread sleeps in try_wait until the phase completes
// instead of spinning on the issue slots the producers need
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    uint32_t tries = 0;
    const bool watch = g_wait_log != nullptr;  // (one global load per wait, not per probe)
    do {
        if (watch && ++tries > (1u << 22)) wait_timeout(bar, phase, tries);
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase), "r"(1000000u)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (8-row atoms of 1024 B)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);  // start address
    d |= (uint64_t)1 << 16;                   // LBO (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;         // SBO: 8-row group stride
    d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
    return d;
}

template <uint32_t kIdesc>
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}
template <uint32_t kIdesc>
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ bool elect_one_sync() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// bulk async copy SMEM -> global (TMA engine), per-thread bulk groups
__device__ __forceinline__ void bulk_store(void *gdst, uint32_t ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
                 "r"(ssrc), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
        : "memory");
}

template <bool kIsA>
__device__ __forceinline__ void expand8(uint32_t w, uint32_t (&r)[8]) {
    if (kIsA) w = __byte_perm(__brev(w), 0, 0x0123);  // reverse the bits of each byte
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = kIsA ? (w & (0x80808080u >> i)) : (w & (0x01010101u << i));
}

// e2m1 (fp4) expansion, 8 nibbles per register: register r, nibble n <- bit 4n + r
// of the word, as codes whose values multiply to 1 for every (A, B) pair of set
// bits, so the f32 accumulator is popc(a & b) exactly:
//     B: bit 4n+r -> 0.5, 1, 2, 2    A: bit 4n+r -> 2, 1, 0.5, 0.5
// (e2m1 codes 1 = 0.5, 2 = 1.0, 4 = 2.0); one or two ALU ops per register
__device__ __forceinline__ void expand_fp4_b(uint32_t w, uint32_t (&r)[4]) {
    r[0] = w & 0x11111111u;
    r[1] = w & 0x22222222u;
    r[2] = w & 0x44444444u;
    r[3] = (w >> 1) & 0x44444444u;
}
__device__ __forceinline__ void expand_fp4_a(uint32_t w, uint32_t (&r)[4]) {
    r[0] = (w << 2) & 0x44444444u;
    r[1] = w & 0x22222222u;
    r[2] = (w >> 2) & 0x11111111u;
    r[3] = (w >> 3) & 0x11111111u;
}

template <uint32_t kIdesc>
__device__ __forceinline__ void mma_fp4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate), "r"(sfa), "r"(sfb));
}

// kind::mxf4 with the expanded A operand in TMEM (32 columns per 128-byte K row)
template <uint32_t kIdesc>
__device__ __forceinline__ void mma_fp4_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                           uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(
            tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(kIdesc), "r"(accumulate), "r"(sfa), "r"(sfb));
}

// two bit planes -> u8 codes 0..3 (same K permutation as expand8; no scaling:
// the MMA then accumulates sum(code_a * code_b) directly)
__device__ __forceinline__ void expand_code2(uint32_t w0, uint32_t w1, uint32_t (&r)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
        r[i] = ((w0 >> i) & 0x01010101u) | (((w1 >> i) << 1) & 0x02020202u);
}

// 32 expanded bytes of word q -> two 16-byte chunks of a SW128 K-major row
__device__ __forceinline__ void store_row32(const uint32_t (&r)[8], uint32_t row_base, int row,
                                            int q) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int chunk = (2 * q + h) ^ (row & 7);
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(row_base + chunk * 16),
                     "r"(r[4 * h]), "r"(r[4 * h + 1]), "r"(r[4 * h + 2]), "r"(r[4 * h + 3]));
    }
}

struct TileMap {
    int tiles_m, ntiles;
    // dense kind::mxf4 operands: superstages fetched per TMA load (1 or 2).  The TMA unit is
    // row-rate bound on 32-byte rows (352 rows per superstage ~ 545 ns at 8192^3, exactly the
    // superstage cadence): 64-byte rows (SWIZZLE_64B) halve the rows per K
    int wide = 1;
    __device__ void decode(int t, int &tm, int &tn) const {
        tm = t % tiles_m;
        tn = t / tiles_m;
    }
};

template <class L>
struct is_tma { static constexpr bool value = false; };
template <>
struct is_tma<TmaRows> { static constexpr bool value = true; };
template <>
struct is_tma<TmaConv> { static constexpr bool value = true; };

template <int BN, bool kATmem, int kVec, class ALoad, class BLoad, class Store, int kPlanes = 1,
          bool kFp4 = false, int kSets = 1, bool kPair = false>
__global__ void __launch_bounds__(Cfg<BN, kATmem, kPlanes, is_tma<ALoad>::value, kFp4, kSets, kPair>::kThreads, 1)
    xnor_umma_kernel(const __grid_constant__ ALoad aload, const __grid_constant__ BLoad bload,
                     const __grid_constant__ Store store, Epilogue ep, int64_t kw32, TileMap tmap,
                     uint64_t *trace_buf, int dbg) {
    auto trace = [&](int slot) { trace_at(trace_buf, slot); };
    // per-superstage pipeline timeline of CTA 0 (debug: dbg bit 16; u64 [4096 + ev * 256 + g])
    const bool stage_trace = trace_buf != nullptr && (dbg & 16) && blockIdx.x < 2;
    auto tr = [&](int ev, uint32_t g) {  // blocks 0 and 1 (both CTAs of the first pair)
        if (stage_trace && g < 256) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace_buf[4096 + blockIdx.x * 4096 + ev * 256 + g] = t;
        }
    };
    constexpr bool kTma = is_tma<ALoad>::value;
    static_assert(kTma == is_tma<BLoad>::value && (!kTma || kPlanes == 1), "TMA: both operands");
    using C = Cfg<BN, kATmem, kPlanes, kTma, kFp4, kSets, kPair>;
    constexpr int ES = C::ES;
    constexpr bool kWideOk = kTma && kFp4 && !kATmem && BN <= 256 && C::kSub == 2 &&
                             !std::is_same<BLoad, TmaConv>::value;
    const uint32_t wide = kWideOk ? (uint32_t)tmap.wide : 1u;  // superstages per TMA load
    const uint32_t nslots = (uint32_t)C::kTmaSlots / wide;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase_raw = smem_u32(smem_raw);
    const uint32_t sbase = (sbase_raw + 1023u) & ~1023u;
    uint8_t *sgen = smem_raw + (sbase - sbase_raw);
    const uint32_t s_exp = sbase + C::off_exp;
    const uint32_t s_pk = sbase + C::off_pk;
    int32_t *s_popc_a = reinterpret_cast<int32_t *>(sgen + C::off_popc_a);
    int32_t *s_popc_b = reinterpret_cast<int32_t *>(sgen + C::off_popc_b);
    const uint32_t s_epi = sbase + C::off_epi;
    const uint32_t bar_full = sbase + C::off_bars;      // [ES]
    const uint32_t bar_empty = bar_full + ES * 8;       // [ES]
    const uint32_t bar_tfull = bar_empty + ES * 8;      // [2] MMA -> epilogue
    const uint32_t bar_tempty = bar_tfull + 2 * 8;      // [2] epilogue -> MMA / producers
    const uint32_t bar_pfull = bar_tempty + 2 * 8;      // [2] producers' popcounts ready
    const uint32_t bar_ld = bar_pfull + 2 * 8;          // [kTmaSlots] TMA bytes landed
    const uint32_t bar_free = bar_ld + C::kTmaSlots * 8; // [kTmaSlots] expanders read the slot
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sgen + C::off_tmem);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t ktiles = ceil_div(kw32, kWordsPerStage);
    uint32_t crank = 0;  // rank in the CTA pair (kPair); rank 0 issues the MMAs
    if constexpr (kPair) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
    const uint32_t peer = crank ^ 1u;
    const int t0 = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;       // first tile
    const int tstep = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;      // tile stride

    if (tid == 0) {
        trace(0);
        for (int s = 0; s < ES; ++s) {
            // pair: the leader's full[] takes its own warps + one relayed arrival from the peer
            mbar_init(bar_full + 8 * s, C::kProducerWarps + ((kPair && crank == 0) ? 1 : 0));
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, (kPair ? 2 : 1) * C::kEpiWarps);
            mbar_init(bar_pfull + 8 * b, (kPair ? 2 : 1) * C::kExpWarps);
        }
        for (int r = 0; r < C::kTmaSlots; ++r) {
            mbar_init(bar_ld + 8 * r, 1);
            mbar_init(bar_free + 8 * r, C::kProducerWarps * wide);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == C::kMmaWarp) {
        if constexpr (kPair) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             smem_u32(s_tmem)),
                         "n"(C::kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             smem_u32(s_tmem)),
                         "n"(C::kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
        }
    }
    if constexpr (kTma) {
        if (tid == 0) {  // descriptor prefetch does not depend on the previous kernel
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&aload.map)));
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&bload.map)));
        }
    }
    fence_before();
    __syncthreads();
    if constexpr (kPair) cluster_sync();  // the peer's barriers exist before any remote arrival
    fence_after();
    const uint32_t tmem = *s_tmem;
    // programmatic dependent launch: the setup above (barriers, TMEM allocation,
    // descriptor prefetch) overlaps the previous kernel's tail; operand reads and
    // output writes start only once that kernel's results are visible
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // (the next kernel's setup may start)
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (tid == 0) trace(1);

    if (warp < C::kExpWarps) {
        // ================================================================ producers
        if constexpr (kFp4) {
            // UE8M0 block scales = 2^0 in every TMEM column from kSfCol on (both
            // operands' scale vectors point there); ordered before the MMAs by the
            // first full[] arrival of these warps
            if (warp < 4) {
                const uint32_t one[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                         0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
                for (int col = C::kSfCol; col < C::kTmemCols; col += 8)
                    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + col, one);
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                fence_before();
            }
        }
        const int set = warp / C::kProducerWarps;                    // expander set
        const int ptid = tid - set * C::kProducerWarps * 32;         // thread within the set
        const bool is_a = ptid < BM;
        const bool active = ptid < C::kProducers;  // the last warp may be partly idle
        // A rows written to TMEM belong to the warp's lane quadrant (warp % 4): with two
        // expander sets the second set's A warps start at a quadrant offset
        const int row = is_a ? ((kATmem && kFp4) ? (warp & 3) * 32 + lane : ptid) : ptid - BM;
        const uint32_t ring = s_pk + tid * 16 * kPlanes;  // slot-major private ring
        constexpr uint32_t kRingSlot = C::kProducerWarps * 32 * 16 * kPlanes;
        // fetch iterator (runs PD - kSub stages ahead, across tile boundaries)
        int f_tile = t0;
        uint32_t f_kt = 0;
        const uint32_t kt32 = (uint32_t)ktiles;
        typename ALoad::Cursor fa{};
        typename BLoad::Cursor fb{};
        auto set_cursor = [&](int t) {
            if (t >= tmap.ntiles || !active) return;
            int tm, tn;
            tmap.decode(t, tm, tn);
            if (is_a) fa = aload.row((int64_t)tm * C::kTmBM + crank * BM + row);
            else fb = bload.row((int64_t)tn * BN + crank * C::kBRows + row);
        };
        set_cursor(f_tile);
        uint32_t f_count = 0;  // stages fetched so far
        auto fetch_next = [&]() {
            if (f_tile < tmap.ntiles && active) {
                const uint32_t dst = ring + (f_count & (C::PD - 1)) * kRingSlot;
#pragma unroll
                for (int pl = 0; pl < kPlanes; ++pl)
#pragma unroll
                    for (int p = 0; p < kWordsPerStage / kVec; ++p) {
                        const int w = (int)(f_kt * kWordsPerStage + p * kVec);
                        const uint32_t d = dst + pl * 16 + p * kVec * 4;
                        if (is_a) aload.template load<kVec>(fa, w, d, pl);
                        else bload.template load<kVec>(fb, w, d, pl);
                    }
                ++f_count;
                if (++f_kt == kt32) {
                    f_kt = 0;
                    f_tile += tstep;
                    set_cursor(f_tile);
                }
            }
            cp_async_commit();
        };
        if constexpr (!kTma) {
#pragma unroll 1
            for (int p = 0; p < C::PD - C::kSub; ++p) fetch_next();
        }

        constexpr uint32_t kSub = C::kSub;
        // the operand role is warp-uniform (warps 0..3 = A rows, the rest B rows):
        // instantiate the pipeline loop per role so neither role executes the
        // other's (if-converted) expansion code
        auto run = [&](auto role) {
            constexpr bool is_a = decltype(role)::value;
            uint32_t gk = 0;  // global stage counter (packed ring)
            uint32_t gs = 0;  // global superstage counter (expanded buffers / phases)
            int it = 0;
    #pragma unroll 1
            for (int tile = t0; tile < tmap.ntiles; tile += tstep, ++it) {
                int32_t my_popc = 0;
                // im2col route: this B row's window corner and the running tap
                int c_iy0 = 0, c_ix0 = 0, c_cw = 0, c_i = 0, c_j = 0;
                if constexpr (std::is_same<BLoad, TmaConv>::value) {
                    int tm, tn;
                    tmap.decode(tile, tm, tn);
                    const int64_t ohw = (int64_t)bload.oh * bload.ow;
                    const int64_t n = (int64_t)tn * BN + crank * C::kBRows + (is_a ? 0 : row);
                    const int p = (int)(n % ohw);
                    c_iy0 = (p / bload.ow) * bload.sh - bload.ph;
                    c_ix0 = (p % bload.ow) * bload.sw - bload.pw;
                }
    #pragma unroll 1
                for (uint32_t kt = 0; kt < kt32; kt += kSub, ++gs) {
                    const uint32_t nsub = kt32 - kt < kSub ? kt32 - kt : kSub;
                    if constexpr (C::kSets > 1) {
                        if ((int)(gs % C::kSets) != set) {  // the other set's superstage
                            if constexpr (std::is_same<BLoad, TmaConv>::value) {
                                c_cw += 4 * kSub;
                                if (c_cw == bload.cs32) {
                                    c_cw = 0;
                                    if (++c_j == bload.kw) c_j = 0, ++c_i;
                                }
                            }
                            gk += nsub;
                            continue;
                        }
                    }
                    uint32_t wv[kSub][4], wv1[kSub][4] = {};
                    if constexpr (kTma) {
                        // this superstage's packed rows, landed by the TMA warp
                        const uint32_t gl = gs / wide, ts = gl % nslots;
                        mbar_wait(bar_ld + 8 * ts, (gl / nslots) & 1u);
                        if (lane == 0 && (warp == 0 || warp == C::kProducerWarps - 1)) tr(warp ? 6 : 3, gs);
                        const uint32_t rbase = s_pk + ts * C::kTmaSlotBytes * wide +
                                               (is_a ? row * kSub * 16 * wide
                                                     : C::kTmaA * wide + row * kSub * 16 * wide);
    #pragma unroll
                        for (uint32_t u = 0; u < kSub; ++u) {
                            // SWIZZLE_32B (kSub == 2): 16-B chunk u of row r sits at u ^ bit 2 of r;
                            // wide loads (64-byte rows, SWIZZLE_64B): chunk c = 2 (gs % 2) + u of row r
                            // sits at c ^ bits 1-2 of r
                            const uint32_t a = rbase + (wide == 2 ? (((gs & 1u) * kSub + u) ^ ((row >> 1) & 3)) * 16
                                                                  : (kSub == 2 ? ((u ^ ((row >> 2) & 1)) * 16) : 0));
                            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                                         : "=r"(wv[u][0]), "=r"(wv[u][1]), "=r"(wv[u][2]), "=r"(wv[u][3])
                                         : "r"(a)
                                         : "memory");
                        }
                        if constexpr (std::is_same<BLoad, TmaConv>::value) {
                            // padding: this pixel's window tap outside the image reads as +1
                            if (!is_a) {
                                const bool oob = (unsigned)(c_iy0 + c_i) >= (unsigned)bload.H ||
                                                 (unsigned)(c_ix0 + c_j) >= (unsigned)bload.W;
    #pragma unroll
                                for (uint32_t u = 0; u < kSub; ++u)
    #pragma unroll
                                    for (int q = 0; q < 4; ++q)
                                        if (oob) wv[u][q] = 0xffffffffu;
                            }
                            c_cw += 4 * kSub;
                            if (c_cw == bload.cs32) {
                                c_cw = 0;
                                if (++c_j == bload.kw) c_j = 0, ++c_i;
                            }
                        }
                        // row popcount now: it consumes every loaded word, so once the POPCs
                        // have issued the slot's ld.shared data is in registers and the TMA
                        // slot can be handed back before the expansion
                        int32_t sp = 0;
#pragma unroll
                        for (uint32_t u = 0; u < kSub; ++u)
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                if (u < nsub) sp += __popc(wv[u][q]);
                        my_popc += sp;
                        __syncwarp();
                        if (lane == 0) mbar_arrive_dep(bar_free + 8 * ts, sp);
                    } else {
                        // keep PD - kSub stages in flight beyond this superstage
    #pragma unroll
                        for (uint32_t u = 0; u < kSub; ++u)
                            if (u < nsub) fetch_next();
                        if (lane == 0 && warp == C::kProducerWarps - 1) tr(0, gs);
                        cp_async_wait<C::PD - C::kSub>();
                        if (lane == 0 && (warp == 0 || warp == C::kProducerWarps - 1)) tr(warp ? 6 : 3, gs);
    #pragma unroll
                        for (uint32_t u = 0; u < kSub; ++u) {
                            if (u >= nsub) break;
                            const uint32_t slot = ring + ((gk + u) & (C::PD - 1)) * kRingSlot;
                            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                                         : "=r"(wv[u][0]), "=r"(wv[u][1]), "=r"(wv[u][2]), "=r"(wv[u][3])
                                         : "r"(slot));
                            if constexpr (kPlanes == 2)
                                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                                             : "=r"(wv1[u][0]), "=r"(wv1[u][1]), "=r"(wv1[u][2]),
                                               "=r"(wv1[u][3])
                                             : "r"(slot + 16));
                        }
                    }
                    // expanded registers of word q of stage u for this operand side
                    auto expand = [&](uint32_t u, int q, bool as_a, uint32_t (&r)[8]) {
                        if constexpr (kPlanes == 2) {
                            my_popc += __popc(wv[u][q]) + 2 * __popc(wv1[u][q]);  // code sum
                            expand_code2(wv[u][q], wv1[u][q], r);
                        } else {
                            if constexpr (!kTma) my_popc += __popc(wv[u][q]);
                            if (as_a) expand8<true>(wv[u][q], r);
                            else expand8<false>(wv[u][q], r);
                        }
                    };
                    const int sb = (int)(gs % ES);
                    if (gs >= ES) mbar_wait(bar_empty + 8 * sb, ((gs / ES) - 1) & 1u);
                    if (lane == 0 && (warp == 0 || warp == C::kProducerWarps - 1)) tr(warp ? 4 : 1, gs);
                    if constexpr (kFp4 && kATmem) {
                        if (is_a) {  // e2m1 A row -> this lane's TMEM lane, 32 columns per superstage
                            const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) +
                                                   C::kAStageCol + sb * C::kAStageCols;
#pragma unroll
                            for (uint32_t u = 0; u < kSub; ++u) {
                                uint32_t r8[8];
#pragma unroll
                                for (int j = 0; j < 4; j += 2) {
                                    expand_fp4_a(u < nsub ? wv[u][j] : 0u, *reinterpret_cast<uint32_t(*)[4]>(&r8[0]));
                                    expand_fp4_a(u < nsub ? wv[u][j + 1] : 0u, *reinterpret_cast<uint32_t(*)[4]>(&r8[4]));
                                    if (!(dbg & 4)) tmem_st8(taddr + (4 * u + j) * 4, r8);
                                }
                            }
                        }
                    }
                    if constexpr (kFp4) {
                        // one 128-byte SW128 row per superstage: word q (stage q / 4) -> chunk q
                        const uint32_t row_base = s_exp + sb * C::kSuperBytes +
                                                  (is_a ? row * 128 : C::kFp4A + row * 128);
    #pragma unroll
                        for (uint32_t u = 0; u < kSub; ++u) {
                            if (u >= nsub || !active || (kATmem && is_a)) break;
    #pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const uint32_t w = wv[u][j];
                                uint32_t r4[4];
                                if (is_a) expand_fp4_a(w, r4);
                                else expand_fp4_b(w, r4);
                                const int q = 4 * (int)u + j;
                                if (!(dbg & 1))
                                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                                                     row_base + ((q ^ (row & 7)) << 4)),
                                                 "r"(r4[0]), "r"(r4[1]), "r"(r4[2]), "r"(r4[3]));
                            }
                        }
                    }
    #pragma unroll
                    for (uint32_t u = 0; u < kSub; ++u) {
                        if (kFp4 || u >= nsub || !active) break;
                        const uint32_t stage = s_exp + sb * C::kSuperBytes + u * C::kStageBytes;
                        if (is_a) {
                            if constexpr (kATmem) {
                                // warps 0..3 own TMEM lanes 0..127 = A rows 0..127
                                const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) +
                                                       C::kAStageCol + (sb * kSub + u) * 32;
    #pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    uint32_t r[8];
                                    expand(u, q, true, r);
                                    if (!(dbg & 4)) tmem_st8(taddr + q * 8, r);
                                }
                            } else {
                                const uint32_t row_base = stage + row * kRowBytes;
    #pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    uint32_t r[8];
                                    expand(u, q, true, r);
                                    store_row32(r, row_base, row, q);
                                }
                            }
                        } else {
                            const uint32_t row_base = stage + C::kStageA + row * kRowBytes;
    #pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                uint32_t r[8];
                                expand(u, q, false, r);
                                if (!(dbg & 1)) store_row32(r, row_base, row, q);
                                else if (r[0] == 0x12345678u && r[7] == 0x9abcdef0u) store_row32(r, row_base, row, q);
                            }
                        }
                    }
                    if (kATmem && is_a) {
                        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                        fence_before();
                    } else {
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    }
                    __syncwarp();  // every lane's writes + fence precede the warp's arrival
                    if (lane == 0 && (warp == 0 || warp == C::kProducerWarps - 1)) tr(warp ? 5 : 2, gs);
                    else if (lane == 0 && (warp % C::kProducerWarps) >= 1 && (warp % C::kProducerWarps) <= 7)
                        tr(8 + (warp % C::kProducerWarps), gs);  // (debug timeline: the other warps' arrivals)
                    if (lane == 0) {
                        mbar_arrive(bar_full + 8 * sb);  // (pair: rank 1 relays to the leader)
                    }
                    gk += nsub;
                }
                // hand this tile's row popcounts to the epilogue (double-buffered)
                const int buf = it % C::kAccBufs;
                if (it >= C::kAccBufs)
                    mbar_wait(bar_tempty + 8 * buf, (uint32_t)((it / C::kAccBufs) - 1) & 1u);
                if (is_a) s_popc_a[(set * 2 + buf) * BM + row] = my_popc;
                else if (active)  // (f32 bits on the fp4 engine, whose epilogue decodes in f32)
                    s_popc_b[(set * 2 + buf) * C::kBRows + row] = kFp4 ? __float_as_int((float)my_popc) : my_popc;
                __syncwarp();
                if (lane == 0) {
                    if constexpr (kPair) {  // both CTAs' epilogues read these B popcounts
                        mbar_arrive_cluster(mapa_shared(bar_pfull + 8 * buf, crank));
                        mbar_arrive_cluster(mapa_shared(bar_pfull + 8 * buf, peer));
                    } else {
                        mbar_arrive(bar_pfull + 8 * buf);
                    }
                }
            }
        };
        if (is_a) run(std::true_type{});
        else run(std::false_type{});
        cp_async_wait<0>();
    } else if (warp == C::kTmaWarp) {
        // ================================================================ TMA issuer
        if constexpr (kTma) {
            if (lane == 0) {
                asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&aload.map)));
                asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&bload.map)));
                const uint32_t kt32 = (uint32_t)ktiles;
                uint32_t g = 0;
#pragma unroll 1
                for (int tile = t0; tile < tmap.ntiles; tile += tstep) {
                    int tm, tn;
                    tmap.decode(tile, tm, tn);
                    // im2col start: the tile's first output pixel (b, oy, ox) -> window corner
                    int cw = 0, ci = 0, cj = 0, cx = 0, cy = 0, cb = 0;
                    if constexpr (std::is_same<BLoad, TmaConv>::value) {
                        const int64_t n0 = (int64_t)tn * BN + crank * C::kBRows;
                        const int64_t ohw = (int64_t)bload.oh * bload.ow;
                        cb = (int)(n0 / ohw);
                        const int p = (int)(n0 - (int64_t)cb * ohw);
                        cy = (p / bload.ow) * bload.sh - bload.ph;
                        cx = (p % bload.ow) * bload.sw - bload.pw;
                    }
#pragma unroll 1
                    for (uint32_t kt = 0; kt < kt32; kt += C::kSub, ++g) {
                        if (wide == 2 && (g & 1u)) continue;  // fetched with the superstage before it
                        const uint32_t gl = g / wide, ts = gl % nslots;
                        if (gl >= nslots) mbar_wait(bar_free + 8 * ts, ((gl / nslots) - 1) & 1u);
                        uint32_t dst = s_pk + ts * C::kTmaSlotBytes * wide;
                        uint32_t ldbar = bar_ld + 8 * ts;
                        if (kPair && (dbg & 131072)) {  // debug: explicit shared::cluster addresses
                            dst = mapa_shared(dst, crank);
                            ldbar = mapa_shared(ldbar, crank);
                        }
                        tr(0, g);
                        if (g == 0) progress_mark(0, 1000 + (uint64_t)tm * 100 + tn);
                        mbar_arrive_expect_tx(bar_ld + 8 * ts, (C::kTmaA + C::kTmaB) * wide);
                        tma_load_2d(dst, &aload.map, (int)(kt * kWordsPerStage),
                                    tm * C::kTmBM + (int)crank * BM, ldbar);
                        if constexpr (std::is_same<BLoad, TmaConv>::value) {
                            // superstage kt: tap (ci, cj), channel words cw .. cw + 8
                            tma_load_im2col_4d(dst + C::kTmaA, &bload.map, cw, cx, cy, cb,
                                               (uint16_t)cj, (uint16_t)ci, bar_ld + 8 * ts);
                            cw += 4 * C::kSub;
                            if (cw == bload.cs32) {
                                cw = 0;
                                if (++cj == bload.kw) cj = 0, ++ci;
                            }
                        } else {
                            tma_load_2d(dst + C::kTmaA * wide, &bload.map, (int)(kt * kWordsPerStage),
                                        tn * BN + (int)crank * C::kBRows, ldbar);
                            if constexpr (BN > 256)  // second box of a wide tile
                                tma_load_2d(dst + C::kTmaA + C::kTmaBoxB * C::kSub * 16, &bload.map,
                                            (int)(kt * kWordsPerStage), tn * BN + C::kTmaBoxB,
                                            bar_ld + 8 * ts);
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == C::kMmaWarp) {
        // ================================================================ MMA issuer
        // (the whole warp runs the loop with warp-uniform values, which the compiler keeps in
        // uniform registers -- a single divergent lane pays an R2UR per MMA operand and falls
        // behind the tensor pipe on wide tiles; one elected lane issues each MMA / commit)
        {
            uint32_t gs = 0;
            const uint32_t kt32 = (uint32_t)ktiles;
            constexpr uint32_t kSub = C::kSub;
            int it = 0;
#pragma unroll 1
            for (int tile = t0; tile < tmap.ntiles; tile += tstep, ++it) {
                if (kPair && crank != 0) {
                    // rank 1 relays: once its expanders filled superstage gs locally, one
                    // cluster-scope arrival on the leader's full[] (cumulative release)
#pragma unroll 1
                    for (uint32_t kt = 0; kt < kt32; kt += kSub, ++gs) {
                        const int sb = (int)(gs % ES);
                        mbar_wait(bar_full + 8 * sb, (gs / ES) & 1u);
                        if (lane == 0) mbar_arrive_cluster(mapa_shared(bar_full + 8 * sb, 0));
                        __syncwarp();
                    }
                    continue;
                }
                const int buf = it % C::kAccBufs;
                if (it >= C::kAccBufs)
                    mbar_wait(bar_tempty + 8 * buf, (uint32_t)((it / C::kAccBufs) - 1) & 1u);
                fence_after();
                const uint32_t d = tmem + buf * C::kAccCols;
#pragma unroll 1
                for (uint32_t kt = 0; kt < kt32; kt += kSub, ++gs) {
                    const uint32_t nsub = kt32 - kt < kSub ? kt32 - kt : kSub;
                    const int sb = (int)(gs % ES);
                    if (gs == 0 && lane == 0) progress_mark(1, 1);
                    if constexpr (kPair) mbar_wait_cluster(bar_full + 8 * sb, (gs / ES) & 1u);
                    else mbar_wait(bar_full + 8 * sb, (gs / ES) & 1u);
                    if (gs == 0 && lane == 0) progress_mark(2, 2);
                    if (lane == 0) tr(7, gs);
                    if (gs == 0 && lane == 0) trace(2);
                    fence_after();
                    const bool leader = elect_one_sync();
                    if constexpr (kFp4) {
                        // K = 64 e2m1 per MMA = 32 bytes of the superstage row
                        const uint32_t a_addr = s_exp + sb * C::kSuperBytes;
                        const uint32_t b_addr = a_addr + C::kFp4A;
                        // descriptors: base + constant start-address increments (16-byte
                        // units; 32 B per K = 64 step) -- no per-MMA descriptor arithmetic
                        // on the issue thread's critical path
                        const uint64_t da = sw128_desc(a_addr), db = sw128_desc(b_addr);
                        const uint64_t db2 = sw128_desc(b_addr + C::kMmaN * 128);
                        const uint32_t sfc = tmem + C::kSfCol;
                        const uint32_t ta = tmem + C::kAStageCol + sb * C::kAStageCols;
                        const int nk = ((dbg & 2) || !leader) ? 0 : 2 * (int)nsub;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            if (kk >= nk) break;
                            const uint32_t acc = (kt | kk) != 0 ? 1u : 0u;
                            if constexpr (kPair) {  // 256 x BN: A and B halves from both CTAs
                                mma_fp4_pair<C::kIdescFp4>(d, da + 2 * kk, db + 2 * kk, sfc, sfc, acc);
                                continue;
                            }
                            if constexpr (kATmem)
                                mma_fp4_ts<C::kIdescFp4>(d, ta + kk * 8, db + 2 * kk, sfc, sfc, acc);
                            else
                                mma_fp4<C::kIdescFp4>(d, da + 2 * kk, db + 2 * kk, sfc, sfc, acc);
                            if constexpr (C::kNMma == 2)  // columns [N/2, N): B rows N/2..N-1
                                mma_fp4<C::kIdescFp4>(d + C::kMmaN, da + 2 * kk, db2 + 2 * kk, sfc,
                                                      sfc, acc);
                        }
                    }
#pragma unroll
                    for (uint32_t u = 0; u < kSub; ++u) {
                        if (kFp4 || u >= nsub || !leader) break;
                        const uint32_t stage = s_exp + sb * C::kSuperBytes + u * C::kStageBytes;
                        const uint32_t b_addr = stage + C::kStageA;
                        const uint64_t da = sw128_desc(stage), db = sw128_desc(b_addr);
                        const uint32_t ta = tmem + C::kAStageCol + (sb * kSub + u) * 32;
#pragma unroll
                        for (int kk = 0; kk < kRowBytes / 32; ++kk) {
                            if (dbg & 2) break;
                            const uint32_t acc = ((kt + u) | kk) != 0 ? 1u : 0u;
                            if constexpr (kATmem)
                                mma_ts<C::kIdesc>(d, ta + kk * 8, db + 2 * kk, acc);
                            else
                                mma_ss<C::kIdesc>(d, da + 2 * kk, db + 2 * kk, acc);
                        }
                    }
                    if (leader) {
                        if constexpr (kPair) umma_commit_pair(bar_empty + 8 * sb);
                        else umma_commit(bar_empty + 8 * sb);
                    }
                    __syncwarp();
                    if (lane == 0) tr(8, gs);
                }
                if (elect_one_sync()) {
                    if constexpr (kPair) umma_commit_pair(bar_tfull + 8 * buf);
                    else umma_commit(bar_tfull + 8 * buf);
                }
                __syncwarp();
                if (it < 3 && lane == 0) trace(3 + 3 * it);
            }
            // release TMEM as soon as the epilogue has drained the last two
            // accumulators, overlapping the dealloc with the final stores
            for (int t = it - C::kAccBufs; t < it; ++t)
                if (t >= 0)
                    mbar_wait(bar_tempty + 8 * (t % C::kAccBufs), (uint32_t)(t / C::kAccBufs) & 1u);
        }
        __syncwarp();
        fence_after();
        if constexpr (kPair)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                         "n"(C::kTmemCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                         "n"(C::kTmemCols));
        if (lane == 0) trace(13);
    } else {
        // ================================================================ epilogue
        // 8 warps: quadrant q = warp % 4 owns TMEM lanes (= tile rows) 32q..32q+31;
        // the two warps of a quadrant take alternating 32-column chunks.  Lane r
        // decodes its row's 32 accumulators in registers and writes them to a
        // padded SMEM row; the warp then re-reads the 32x32 block transposed so
        // each st.global.v4 instruction covers four full 128-byte row segments.
        const int e = warp - C::kEpiWarp0;
        const int q = warp & 3, h = e >> 2;
        const uint32_t stg = s_epi + e * C::kStgBytes;
        const bool ncontig = store.n_contiguous();
        const int64_t M = store.rows(), N = store.cols();
        const int64_t ms = store.m_stride();
        // (swapped conv orientation: the per-filter parameters are per column, applied
        // after the decode)
        const bool affine = (ep.scale || ep.shift) && !Store::kSwap;
        const bool dot = ep.domain == BNN_DOT;
        const bool magic = ep.k_logical < (1 << 21);  // int -> f32 via the 2^23 trick
        const bool plain = (magic || kFp4) && !affine && (ep.bn_mean == nullptr || Store::kSwap);  // straight-line decode
        int it = 0;
#pragma unroll 1
        for (int tile = t0; tile < tmap.ntiles; tile += tstep, ++it) {
            const int buf = it % C::kAccBufs;
            int tm, tn;
            tmap.decode(tile, tm, tn);
            const int64_t mq = (int64_t)tm * C::kTmBM + crank * BM + q * 32, n0 = (int64_t)tn * BN;
            const int64_t m = mq + lane;
            if (!Store::kSwap && store.res && ncontig && m < M) {
                // warm L2 with this tile's residual blocks while the MMAs run: lane r
                // prefetches row m's 128-byte segment of each of its 32-column chunks
                if constexpr (!Store::kSwap) {
                    for (int c = h; c * 32 < BN; c += C::kEpiWarps / 4) {
                        const int64_t nc = n0 + c * 32;
                        if (nc >= N) break;
                        const float *pr = store.res + store.col_off(nc) + m * ms;
                        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pr));
                    }
                }
            }
            if constexpr (Store::kSwap) {
                // swapped orientation: for filter nc + lane the warp's 32 pixels are one
                // contiguous 128-byte run of the residual (one prefetch per lane)
                if (store.res && mq < M) {
                    for (int c = h; c * 32 < BN; c += C::kEpiWarps / 4) {
                        const int64_t nc = n0 + c * 32;
                        if (nc + lane >= N) break;
                        const float *pr = store.res + store.row_off(mq) + (nc + lane) * store.ohw;
                        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pr));
                    }
                }
            }
            mbar_wait_sleep(bar_tfull + 8 * buf, (uint32_t)(it / C::kAccBufs) & 1u);
            mbar_wait_sleep(bar_pfull + 8 * buf, (uint32_t)(it / C::kAccBufs) & 1u);
            fence_after();
            if (e == 0 && lane == 0 && it < 3) trace(4 + 3 * it);
            if (dbg & 2048) {  // debug: skip the whole epilogue (wrong outputs)
                fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (kPair) {  // the leader's MMA and both CTAs' producers wait
                        mbar_arrive_cluster(mapa_shared(bar_tempty + 8 * buf, crank));
                        mbar_arrive_cluster(mapa_shared(bar_tempty + 8 * buf, peer));
                    } else {
                        mbar_arrive(bar_tempty + 8 * buf);
                    }
                }
                continue;
            }
            const bool mok = m < M;
            // per-row constants: P = kb - pb[n] + 2C, with 2C = acc >> 6 (acc = 128 C)
            int32_t popa = s_popc_a[buf * BM + q * 32 + lane];
            if constexpr (C::kSets > 1) popa += s_popc_a[(2 + buf) * BM + q * 32 + lane];
            const int32_t kb = ep.k_eff - popa;
            const int32_t rowc = (dot ? 2 * kb - ep.k_logical : kb) + 0x4B400000;
            const uint32_t vsh = dot ? 5u : 6u, psh = dot ? 1u : 0u;
            const float rowf = (float)(dot ? 2 * kb - ep.k_logical : kb);  // fp4 decode
            const float cmul = dot ? 4.0f : 2.0f, pmul = dot ? 2.0f : 1.0f;
            // multi-bit decode constants (kPlanes == 2): s_popc_* hold code sums
            const int32_t abab = ep.a_alpha * ep.b_alpha;
            const int32_t rowterm = ep.a_alpha * ep.b_beta * popa +
                                    ep.k_logical * ep.a_beta * ep.b_beta;
            const float sc = (mok && ep.scale) ? __ldg(ep.scale + m) : 1.0f;
            const float sh = (mok && ep.shift) ? __ldg(ep.shift + m) : 0.0f;
            const bool has_bn = ep.bn_mean != nullptr && !Store::kSwap;
            const float bm = (mok && has_bn) ? __ldg(ep.bn_mean + m) : 0.0f;
            const float bi = (mok && has_bn) ? __ldg(ep.bn_inv + m) : 1.0f;
            const float bg = (mok && has_bn) ? __ldg(ep.bn_gamma + m) : 1.0f;
            const float bb = (mok && has_bn) ? __ldg(ep.bn_beta + m) : 0.0f;
            const int32_t *pb = s_popc_b + buf * C::kBRows;
            const int32_t *pb1 = s_popc_b + (2 + buf) * C::kBRows;  // second expander set (kSets == 2)
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + buf * C::kAccCols;
#pragma unroll 1
            for (int c = h; c * 32 < BN; c += C::kEpiWarps / 4) {
                uint32_t v[32];
                const int w = BN - c * 32 < 32 ? BN - c * 32 : 32;
                if (w == 32) {
                    tmem_ld32(taddr + c * 32, v);
                } else {
                    uint32_t v16[16];
                    tmem_ld16(taddr + c * 32, v16);
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = v16[j], v[16 + j] = 0;
                }
                const int64_t nc = n0 + c * 32;
                if (mq >= M || nc >= N) {  // warp-uniform
                    // a quadrant past M inside the last packed word: its 32 bits are 0
                    // (words from ceil(M/64) on are not touched)
                    if constexpr (Store::kSwap) {  // filters past F inside the last word: 0
                        if (Store::kPack && m < M && nc >= N && (nc >> 6) < ((N + 63) >> 6))
                            ep.pack_out[m * ep.pack_ld32 + (nc >> 5)] = 0u;
                    } else if (Store::kPack && ep.pack_out && nc < N && (mq >> 6) < ((M + 63) >> 6) &&
                               lane < w && nc + lane < N) {
                        ep.pack_out[(nc + lane) * ep.pack_ld32 + (mq >> 5)] = 0u;
                    }
                    continue;
                }
                float f[32];
                if constexpr (kPlanes == 2) {
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        const int4 pb4 = *reinterpret_cast<const int4 *>(pb + c * 32 + 4 * j4);
                        const int32_t pbv[4] = {pb4.x, pb4.y, pb4.z, pb4.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            // exact integer numerator, one rounding: (.) / (gA gB)
                            const int32_t num = abab * (int32_t)v[4 * j4 + i] + rowterm +
                                                ep.a_beta * ep.b_alpha * pbv[i];
                            f[4 * j4 + i] = __fmul_rn((float)num, ep.inv_gamma);
                        }
                    }
                } else if (kFp4) {
                    // f32 accumulator C = popc(a & b): P = kb - pb + 2C, or 2P - K =
                    // (2kb - K) - 2pb + 4C, every term an exact f32 integer
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        float4 pb4;
                        if constexpr (kPair) {
                            // B popcounts of columns [r * N/2, (r+1) * N/2) live in CTA r
                            const int col = c * 32 + 4 * j4;
                            const uint32_t owner = (uint32_t)(col / C::kBRows);
                            const uint32_t a = mapa_shared(
                                smem_u32(pb + (col - (int)owner * C::kBRows)), owner);
                            asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                                         : "=f"(pb4.x), "=f"(pb4.y), "=f"(pb4.z), "=f"(pb4.w)
                                         : "r"(a));
                        } else {
                            pb4 = *reinterpret_cast<const float4 *>(pb + c * 32 + 4 * j4);
                        }
                        if constexpr (C::kSets > 1) {
                            const float4 q4 = *reinterpret_cast<const float4 *>(pb1 + c * 32 + 4 * j4);
                            pb4.x += q4.x; pb4.y += q4.y; pb4.z += q4.z; pb4.w += q4.w;
                        }
                        const float pbv[4] = {pb4.x, pb4.y, pb4.z, pb4.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            float x = __fmaf_rn(cmul, __uint_as_float(v[4 * j4 + i]),
                                                __fmaf_rn(-pmul, pbv[i], rowf));
                            if (!plain) {
                                if (affine) x = __fadd_rn(__fmul_rn(x, sc), sh);
                                if (has_bn)
                                    x = __fadd_rn(__fmul_rn(bg, __fmul_rn(__fsub_rn(x, bm), bi)), bb);
                            }
                            f[4 * j4 + i] = x;
                        }
                    }
                } else if (plain) {
                    // P = kb - pb + 2C (2C = acc >> 6), or 2P - K = (2kb - K) - 2pb + (acc >> 5),
                    // with the 2^23 bias of the int -> f32 trick folded into the row constant
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        const int4 pb4 = *reinterpret_cast<const int4 *>(pb + c * 32 + 4 * j4);
                        const int32_t pbv[4] = {pb4.x, pb4.y, pb4.z, pb4.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            f[4 * j4 + i] = __int_as_float(rowc + (int32_t)(v[4 * j4 + i] >> vsh) -
                                                           (pbv[i] << psh)) -
                                            12582912.0f;
                    }
                } else {
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        const int4 pb4 = *reinterpret_cast<const int4 *>(pb + c * 32 + 4 * j4);
                        const int32_t pbv[4] = {pb4.x, pb4.y, pb4.z, pb4.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int j = 4 * j4 + i;
                            int32_t val = kb - pbv[i] + (int32_t)(v[j] >> 6);
                            if (dot) val = 2 * val - ep.k_logical;
                            float x = magic ? __int_as_float(val + 0x4B400000) - 12582912.0f
                                            : (float)val;
                            if (affine) x = __fadd_rn(__fmul_rn(x, sc), sh);
                            if (has_bn)
                                x = __fadd_rn(__fmul_rn(bg, __fmul_rn(__fsub_rn(x, bm), bi)), bb);
                            f[j] = x;
                        }
                    }
                }
                // fused residual add in the row layout when the sign-pack needs the
                // final values (the staged stores then skip their own residual add)
                if constexpr (Store::kSwap) {
                    // rows = pixels (lane m), columns = filters nc + j: per-filter affine /
                    // BN in the reference op order, then (shortcut,) sign-pack of the
                    // pixel's 32 filters in-lane, and coalesced NCHW stores (for each
                    // filter the warp writes 32 consecutive pixels)
                    const int64_t nvalid = N - nc < w ? N - nc : w;
                    if (ep.scale || ep.shift || ep.bn_mean) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int64_t p = nc + (j < nvalid ? j : 0);
                            float x = f[j];
                            if (ep.scale) x = __fmul_rn(x, __ldg(ep.scale + p));
                            if (ep.shift) x = __fadd_rn(x, __ldg(ep.shift + p));
                            if (ep.bn_mean)
                                x = __fadd_rn(__fmul_rn(__ldg(ep.bn_gamma + p),
                                                        __fmul_rn(__fsub_rn(x, __ldg(ep.bn_mean + p)),
                                                                  __ldg(ep.bn_inv + p))),
                                              __ldg(ep.bn_beta + p));
                            f[j] = x;
                        }
                    }
                    if (mok) {
                        const int64_t ro = store.row_off(m) + nc * store.ohw;
                        if (store.res) {  // all 32 loads in flight before any store
                            float r[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                r[j] = j < nvalid ? __ldg(store.res + ro + j * store.ohw) : 0.0f;
#pragma unroll
                            for (int j = 0; j < 32; ++j) f[j] = __fadd_rn(f[j], r[j]);
                        }
                        if (!Store::kPack || store.has_out()) {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (j < nvalid) store.y[ro + j * store.ohw] = f[j];
                        }
                        if constexpr (Store::kPack) {
                            uint32_t word = 0;
                            float nf = 0.0f;
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (j < nvalid) {
                                    word |= (f[j] >= 0.0f ? 1u : 0u) << j;
                                    nf = __fmaf_rn(f[j], 0.0f, nf);
                                }
                            ep.pack_out[m * ep.pack_ld32 + (nc >> 5)] = word;
                            if (ep.pack_flags && nf != 0.0f) atomicOr(ep.pack_flags, 1);
                        }
                    }
                } else {
                // next layer's QActivation + pack: column j's 32 rows -> one u32 word
                // (ballot); lane j keeps column j's word.  Rows past M pack as 0 (their
                // values are not stored); columns past the tile / N hold garbage and
                // are zeroed (warp-uniform, tail chunks only) so that nf = sum of 0 * g
                // is NaN iff a stored value is NaN / Inf
                auto emit_pack = [&](float (&g)[32]) {
                    if (!mok) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) g[j] = -1.0f;
                    }
                    const int64_t nvalid = N - nc < w ? N - nc : w;
                    if (nvalid < 32) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (j >= nvalid) g[j] = 0.0f;
                    }
                    uint32_t word = 0;
                    float nf = 0.0f;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t bits = __ballot_sync(0xffffffffu, g[j] >= 0.0f);
                        nf = __fmaf_rn(g[j], 0.0f, nf);
                        if (lane == j) word = bits;
                    }
                    if (lane < w && nc + lane < N)
                        ep.pack_out[(nc + lane) * ep.pack_ld32 + (mq >> 5)] = word;
                    if (ep.pack_flags && __any_sync(0xffffffffu, nf != 0.0f) && lane == 0)
                        atomicOr(ep.pack_flags, 1);
                };
                // residual + sign-pack: row-layout outputs add the residual here; staged
                // (column-contiguous) outputs add it in the coalesced transposed phase,
                // write the sums back to the staging block and pack from there (late)
                bool res_added = false, pack_late = false;
                if constexpr (Store::kPack) {
                    if (store.res && !ncontig) {
                        if (mok) store.add_res_row(m, nc, w, f);
                        res_added = true;
                    }
                    pack_late = store.res && ncontig;
                    if (!pack_late) emit_pack(f);
                }
                if ((dbg & 1024) || (Store::kPack && !store.has_out() && !pack_late)) {
                } else if (ncontig) {
                    // staged 32 x 32 block: lane r writes its row (SW128 chunk swizzle)
                    const uint32_t row = stg + lane * 128;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                                         row + ((j ^ (lane & 7)) << 4)),
                                     "f"(f[4 * j]), "f"(f[4 * j + 1]), "f"(f[4 * j + 2]),
                                     "f"(f[4 * j + 3]));
                    // TMA store of the whole block when the output has a map and the block
                    // does not straddle an image (conv) -- the TMA unit clips rows past M
                    // and columns past N
                    bool tma_st = store.has_map && !store.res && w == 32;  // (whole block in the tile)
                    int64_t tb = 0, tp = nc;
                    if constexpr (Store::kConv) {
                        tb = nc / store.ohw;
                        tp = nc - tb * store.ohw;
                        tma_st = tma_st && tp + 32 <= store.ohw;
                    }
                    if (tma_st) {
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                        __syncwarp();
                        if (lane == 0) {
                            const uint64_t map = reinterpret_cast<uint64_t>(&store.omap);
                            if constexpr (Store::kConv)
                                asm volatile(
                                    "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map),
                                    "r"((int)tp), "r"((int)mq), "r"((int)tb), "r"(stg)
                                    : "memory");
                            else
                                asm volatile(
                                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map),
                                    "r"((int)tp), "r"((int)mq), "r"(stg)
                                    : "memory");
                            bulk_commit();
                            bulk_wait_read<0>();  // staging reusable for the next block
                        }
                        __syncwarp();
                        continue;
                    }
                    __syncwarp();
                    // transposed write-out: lane = (row quarter, 4-column segment)
                    const int seg = lane & 7, rsub = lane >> 3;
                    const int64_t n = nc + 4 * seg;
                    const bool out_f32 = !Store::kPack || store.has_out();
                    if (4 * seg < w && n < N) {
                        float *col = nullptr;
                        const bool v4 = out_f32 ? store.col4(n, col) : false;
                        // row 4 rr + rsub, chunk seg (rows 4 rr + rsub have r & 7 = 4 (rr & 1) + rsub)
                        auto src_of = [&](int rr) {
                            const int r = 4 * rr + rsub;
                            return stg + r * 128 + ((seg ^ (r & 7)) << 4);
                        };
                        // late sign-pack: the residual sums go back to the staging block
                        auto keep = [&](int rr, const float4 &t) {
                            if (Store::kPack && pack_late)
                                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(src_of(rr)),
                                             "f"(t.x), "f"(t.y), "f"(t.z), "f"(t.w));
                        };
                        if (v4 && mq + 32 <= M) {
                            // common case: 8 unpredicated 16-byte stores, pointer bumps only
                            float *dst = col + (mq + rsub) * ms;
                            const int64_t step = 4 * ms;
                            if (store.res) {
                                // fused residual add: all 8 loads in flight before the
                                // stores (the output may alias nothing, but the compiler
                                // cannot know, and would serialise load -> store pairs)
                                float4 r[8];
                                const float *rs = store.res_of(dst);
#pragma unroll
                                for (int rr = 0; rr < 8; ++rr)
                                    r[rr] = __ldg(reinterpret_cast<const float4 *>(rs + rr * step));
#pragma unroll
                                for (int rr = 0; rr < 8; ++rr) {
                                    float4 t;
                                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                                                 : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w)
                                                 : "r"(src_of(rr)));
                                    t.x = __fadd_rn(t.x, r[rr].x); t.y = __fadd_rn(t.y, r[rr].y);
                                    t.z = __fadd_rn(t.z, r[rr].z); t.w = __fadd_rn(t.w, r[rr].w);
                                    *reinterpret_cast<float4 *>(dst) = t;
                                    keep(rr, t);
                                    dst += step;
                                }
                            } else {
#pragma unroll
                                for (int rr = 0; rr < 8; ++rr) {
                                    float4 t;
                                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                                                 : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w)
                                                 : "r"(src_of(rr)));
                                    *reinterpret_cast<float4 *>(dst) = t;
                                    keep(rr, t);
                                    dst += step;
                                }
                            }
                        } else {
                            // the lane's 4 columns: element offsets of row 0 (one division per
                            // lane, not per element), -1 past the tile / N
                            int64_t coff[4];
                            if (!v4) {
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    coff[i] = (4 * seg + i < w && n + i < N) ? store.col_off(n + i) : -1;
                            }
                            for (int rr = 0; rr < 8; ++rr) {
                                const int r = 4 * rr + rsub;
                                const int64_t mr = mq + r;
                                if (mr >= M) break;
                                float4 t;
                                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                                             : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w)
                                             : "r"(src_of(rr)));
                                if (v4) {
                                    float *dst = col + mr * ms;
                                    if (store.res) {
                                        const float4 r = __ldg(reinterpret_cast<const float4 *>(store.res_of(dst)));
                                        t.x = __fadd_rn(t.x, r.x); t.y = __fadd_rn(t.y, r.y);
                                        t.z = __fadd_rn(t.z, r.z); t.w = __fadd_rn(t.w, r.w);
                                    }
                                    *reinterpret_cast<float4 *>(dst) = t;
                                } else {
                                    float tv[4] = {t.x, t.y, t.z, t.w};
                                    const int64_t ro = mr * ms;
#pragma unroll
                                    for (int i = 0; i < 4; ++i)
                                        if (coff[i] >= 0) {
                                            if (store.res) tv[i] = __fadd_rn(tv[i], __ldg(store.res + coff[i] + ro));
                                            if (out_f32) store.out_ptr()[coff[i] + ro] = tv[i];
                                        }
                                    t = make_float4(tv[0], tv[1], tv[2], tv[3]);
                                }
                                keep(rr, t);
                            }
                        }
                    }
                    __syncwarp();
                    if constexpr (Store::kPack) {
                        if (pack_late) {  // lane r re-reads its row: the final values
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                                             : "=f"(f[4 * j]), "=f"(f[4 * j + 1]), "=f"(f[4 * j + 2]),
                                               "=f"(f[4 * j + 3])
                                             : "r"(row + ((j ^ (lane & 7)) << 4)));
                            emit_pack(f);
                            __syncwarp();
                        }
                    }
                } else if (mok) {
                    // rows contiguous in memory (e.g. an [N, M] output): lanes = rows
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < w && nc + j < N) {
                            if (res_added) store.put_raw(m, nc + j, f[j]);
                            else store.put(m, nc + j, f[j]);
                        }
                }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) {
                    if constexpr (kPair) {  // the leader's MMA and both CTAs' producers wait
                        mbar_arrive_cluster(mapa_shared(bar_tempty + 8 * buf, crank));
                        mbar_arrive_cluster(mapa_shared(bar_tempty + 8 * buf, peer));
                    } else {
                        mbar_arrive(bar_tempty + 8 * buf);
                    }
                }
            if (e == 0 && lane == 0 && it < 3) trace(5 + 3 * it);
        }
        if (lane == 0) bulk_wait_all();  // TMA stores of this warp complete before exit
    }

    fence_before();
    __syncthreads();
    // a CTA of a pair stays resident until its peer no longer reads its SMEM or
    // arrives on its barriers
    if constexpr (kPair) cluster_sync();
    if (tid == 0) trace(12);
}

}  // namespace umma

// debug bit flags (bnn_debug_set(BNN_DEBUG_UMMA_BITS); some give wrong results)
static inline int umma_dbg() { return (int)g_debug.umma_bits; }

static int sm_count() {
    static int n = 0;
    if (n == 0) {
        n = bnn_device_sm_count();
        if (n <= 0) n = 148;
    }
    return n;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// [rows, kw32] u32 view with row pitch ld32 words; box = box_words x box_rows
static int encode_rows(TmaRows &t, int box_words, int box_rows) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return set_error(BNN_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)t.kw32, (cuuint64_t)t.rows};
    const cuuint64_t strides[1] = {(cuuint64_t)t.ld32 * 4};
    const cuuint32_t box[2] = {(cuuint32_t)box_words, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = box_words * 4 == 32   ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : box_words * 4 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = fn(&t.map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t *>(t.base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(BNN_ECUDA, "cuTensorMapEncodeTiled failed");
    return BNN_OK;
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const int *, const int *,
                                   cuuint32_t, cuuint32_t, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
static int encode_conv(TmaConv &t, int box_words, int box_pixels, int64_t B) {
    static EncodeIm2colFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeIm2colFn>(p);
    }
    if (!fn) return set_error(BNN_ECUDA, "cuTensorMapEncodeIm2col unavailable");
    const cuuint64_t dims[4] = {(cuuint64_t)t.cs32, (cuuint64_t)t.W, (cuuint64_t)t.H, (cuuint64_t)B};
    const cuuint64_t strides[3] = {(cuuint64_t)t.cs32 * 4, (cuuint64_t)t.cs32 * 4 * t.W,
                                   (cuuint64_t)t.cs32 * 4 * t.W * t.H};
    // window corners traversed per image: first (-ph, -pw), last ((oh-1)sh - ph, (ow-1)sw - pw),
    // the upper corner given relative to (H - 1, W - 1); order W, H (innermost first)
    const int lower[2] = {-t.pw, -t.ph};
    const int upper[2] = {(t.ow - 1) * t.sw - t.pw - (t.W - 1), (t.oh - 1) * t.sh - t.ph - (t.H - 1)};
    const cuuint32_t estr[4] = {1, (cuuint32_t)t.sw, (cuuint32_t)t.sh, 1};
    CUresult r = fn(&t.map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t *>(t.x), dims,
                    strides, lower, upper, (cuuint32_t)box_words, (cuuint32_t)box_pixels, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    box_words * 4 == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(BNN_ECUDA, "cuTensorMapEncodeIm2col failed");
    return BNN_OK;
}

// TMA store maps of the epilogue (32 x 32 f32 boxes, SWIZZLE_128B); silently
// skipped (regular stores) when the output does not meet the TMA constraints
static void encode_out(GemmStore &st) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn || !st.C || st.ldc_n != 1 || (st.ldc_m * 4) % 16 ||
        (reinterpret_cast<uintptr_t>(st.C) & 15) || st.N > (1ll << 32) || st.M > (1ll << 32))
        return;
    const cuuint64_t dims[2] = {(cuuint64_t)st.N, (cuuint64_t)st.M};
    const cuuint64_t strides[1] = {(cuuint64_t)st.ldc_m * 4};
    const cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
    if (fn(&st.omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, st.C, dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        st.has_map = 1;
}
static void encode_out(ConvStore &st) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn || !st.y || (st.ohw * 4) % 16 || (reinterpret_cast<uintptr_t>(st.y) & 15)) return;
    const int64_t B = st.npix / st.ohw;
    const cuuint64_t dims[3] = {(cuuint64_t)st.ohw, (cuuint64_t)st.F, (cuuint64_t)B};
    const cuuint64_t strides[2] = {(cuuint64_t)st.ohw * 4, (cuuint64_t)(st.F * st.ohw * 4)};
    const cuuint32_t box[3] = {32, 32, 1}, estr[3] = {1, 1, 1};
    if (fn(&st.omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, st.y, dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        st.has_map = 1;
}

template <int BN, bool kATmem, int kVec, class ALoad, class BLoad, class Store, int kPlanes = 1,
          bool kFp4 = false, int kSets = 1, bool kPair = false>
static int launch_umma_cfg(const ALoad &a_in, const BLoad &b_in, const Store &st, const Epilogue &ep,
                           int64_t M, int64_t N, int64_t kw32, cudaStream_t s) {
    constexpr bool kTma = umma::is_tma<ALoad>::value;
    using C = umma::Cfg<BN, kATmem, kPlanes, kTma, kFp4, kSets, kPair>;
    auto kern = umma::xnor_umma_kernel<BN, kATmem, kVec, ALoad, BLoad, Store, kPlanes, kFp4, kSets, kPair>;
    ALoad a = a_in;
    BLoad b = b_in;
    // dense kind::mxf4 operands with K a multiple of 512 bits: two superstages per TMA load --
    // built and parity-tested, but measured 3-5% slower at 8192^3 / 16384^3 (the TMA round trip drops
    // from ~1.5 to ~0.9 us, yet the superstage cadence stays ~545 ns: the row rate of the TMA unit
    // is not what paces the pipeline), so it is opt-in (debug bit 16384)
    constexpr bool kWideOk = kTma && kFp4 && !kATmem && BN <= 256 && C::kSub == 2 &&
                             !std::is_same<BLoad, TmaConv>::value && C::kTmaSlots % 2 == 0;
    const int wide = (kWideOk && kw32 % 16 == 0 && (umma_dbg() & 16384)) ? 2 : 1;
    if constexpr (kTma) {
        int rc = encode_rows(a, 4 * C::kSub * wide, umma::BM);
        if constexpr (std::is_same<BLoad, TmaConv>::value) {
            static_assert(C::kSub == 2, "im2col TMA: one 32-byte tap chunk per superstage");
            if (rc == BNN_OK) rc = encode_conv(b, 4 * C::kSub, C::kBRows, b.npix / ((int64_t)b.oh * b.ow));
        } else {
            if (rc == BNN_OK) rc = encode_rows(b, 4 * C::kSub * wide, C::kTmaBoxB);
        }
        if (rc != BNN_OK) return rc;
    }
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        configured = true;
    }
    const int64_t tiles_m = ceil_div(M, C::kTmBM), tiles_n = ceil_div(N, BN);
    const int64_t ntiles = tiles_m * tiles_n;
    if (ntiles > (1ll << 30)) return set_error(BNN_EUNSUP, "too many tiles");
    umma::TileMap tmap{(int)tiles_m, (int)ntiles};
    tmap.wide = wide;
    // one CTA (pair of CTAs) per SM (pair of SMs), persistent over the tiles
    const int64_t units = kPair ? sm_count() / 2 : sm_count();
    int grid = (int)((ntiles < units ? ntiles : units) * (kPair ? 2 : 1));
    if (g_debug.grid_cap > 0 && grid > g_debug.grid_cap) grid = (int)((g_debug.grid_cap + 1) & ~1);
    const bool force_cluster = !kPair && (umma_dbg() & 32768);  // debug: cluster launch of 1-CTA code
    if (force_cluster) grid = (grid + 1) & ~1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (umma_dbg() & 65536) ? 0 : 1;  // debug: no PDL
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (kPair || force_cluster) ? 2 : 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (kPair || force_cluster) ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, a, b, st, ep, kw32, tmap, g_debug.trace_buf, umma_dbg());
    return check_launch("xnor_umma_kernel");
}

// engine variants (per call: algo = BNN_ALGO_UMMA_V0 + v, carried in Epilogue::variant):
//   0: 128x256 tiles, u8 expansion, A and B through SMEM (kind::i8)
//   1: u8 expansion, A in TMEM, B through SMEM (kind::i8), tile N chosen per shape
//      from {128, 160, 176, 192} to minimise (waves x N) on the SMs of this GPU
//   2: e2m1 expansion, A and B through SMEM (kind::mxf4, 2x the i8 MMA rate and
//      half the expanded bytes) for TMA-fed operands, tile N from {128 .. 224};
//      cp.async-fed shapes fall back to variant 1 (variant 0 for <= 64 filters)
//   3: kind::mxf4 with the expanded A operand in TMEM (TMA-fed shapes, N tiles <= 192)
//   4: variant 2, and convs with <= 64 filters always in the swapped orientation
//      (rows = pixels, 128 x 64 tiles); variant 2 takes it only for convs with a
//      fused shortcut add, where it beats variant 0

static int choose_bn(int64_t M, int64_t N, bool fp4 = false, bool wide = false) {
    static const int cands[] = {192, 176, 160, 128};
    // (small N tiles give small problems enough CTAs: every tile runs the full K loop)
    static const int cands4[] = {224, 208, 192, 176, 160, 128, 96, 64, 32, 16};
    if (fp4) {
        const int force = (int)g_debug.fp4_bn;  // tuning / debug override of the tile N
        if (force > 0 && (force <= 224 || wide)) return force;  // (wide tiles: one expander set)
        const int64_t sms = sm_count(), tm = ceil_div(M, umma::BM);
        int best = 192;
        int64_t best_cost = -1;
        for (int bn : cands4) {
            const int64_t waves = ceil_div(tm * ceil_div(N, bn), sms);
            const int64_t cost = waves * (bn + 32);
            if (best_cost < 0 || cost < best_cost) best = bn, best_cost = cost;
        }
        // wide tiles (two MMAs, one accumulator buffer): only when they fit in one wave
        static const int wide_cands[] = {320, 352, 384};
        if (wide)
            for (int bn : wide_cands) {
                if (tm * ceil_div(N, bn) > sms) continue;
                const int64_t cost = bn + 32;
                if (cost < best_cost) best = bn, best_cost = cost;
            }
        return best;
    }
    const int64_t sms = sm_count(), tm = ceil_div(M, umma::BM);
    int best = 192;
    int64_t best_cost = -1;
    for (int bn : cands) {
        const int64_t waves = ceil_div(tm * ceil_div(N, bn), sms);
        const int64_t cost = waves * (bn + 32);  // + fixed per-tile overhead in columns
        if (best_cost < 0 || cost < best_cost) best = bn, best_cost = cost;
    }
    return best;
}

// 2-CTA pairs (256-row tiles): BN from {128, 160, 192, 224}, minimising waves x (BN + 32)
// over the SM pairs
template <class ALoad, class BLoad, class Store>
static int launch_fp4_pair(const ALoad &a, const BLoad &b, const Store &st, const Epilogue &ep,
                           int64_t M, int64_t N, int64_t kw32, cudaStream_t s) {
    static const int cands[] = {224, 192, 160, 128};
    const int64_t pairs = sm_count() / 2, tm = ceil_div(M, 2 * umma::BM);
    int best = 224;
    int64_t best_cost = -1;
    for (int bn : cands) {
        const int64_t cost = ceil_div(tm * ceil_div(N, bn), pairs) * (bn + 32);
        if (best_cost < 0 || cost < best_cost) best = bn, best_cost = cost;
    }
    using S = Store;
    switch (best) {
        case 128: return launch_umma_cfg<128, false, 4, ALoad, BLoad, S, 1, true, 1, true>(a, b, st, ep, M, N, kw32, s);
        case 160: return launch_umma_cfg<160, false, 4, ALoad, BLoad, S, 1, true, 1, true>(a, b, st, ep, M, N, kw32, s);
        case 192: return launch_umma_cfg<192, false, 4, ALoad, BLoad, S, 1, true, 1, true>(a, b, st, ep, M, N, kw32, s);
        default: return launch_umma_cfg<224, false, 4, ALoad, BLoad, S, 1, true, 1, true>(a, b, st, ep, M, N, kw32, s);
    }
}

template <int kSets, class ALoad, class BLoad, class Store>
static int launch_fp4(const ALoad &a, const BLoad &b, const Store &st, const Epilogue &ep, int64_t M,
                      int64_t N, int64_t kw32, cudaStream_t s) {
    using S = Store;
    switch (choose_bn(M, N, true, kSets == 1)) {
        case 320: if constexpr (kSets == 1) return launch_umma_cfg<320, false, 4, ALoad, BLoad, S, 1, true, 1>(a, b, st, ep, M, N, kw32, s); else break;
        case 352: if constexpr (kSets == 1) return launch_umma_cfg<352, false, 4, ALoad, BLoad, S, 1, true, 1>(a, b, st, ep, M, N, kw32, s); else break;
        case 384: if constexpr (kSets == 1) return launch_umma_cfg<384, false, 4, ALoad, BLoad, S, 1, true, 1>(a, b, st, ep, M, N, kw32, s); else break;
        case 16: return launch_umma_cfg<16, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 32: return launch_umma_cfg<32, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 64: return launch_umma_cfg<64, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 96: return launch_umma_cfg<96, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 128: return launch_umma_cfg<128, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 160: return launch_umma_cfg<160, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 176: return launch_umma_cfg<176, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 192: return launch_umma_cfg<192, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 208: return launch_umma_cfg<208, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        default: return launch_umma_cfg<224, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
    }
    // (wide tiles with two expander sets: not instantiated, take the widest narrow tile)
    return launch_umma_cfg<224, false, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
}

// variant 3: kind::mxf4 with the expanded A operand in TMEM (tcgen05.st) instead of
// SMEM -- per superstage the SMEM data path then carries only the B operand's
// expansion and MMA reads (the A side moves to TMEM); N <= 192 (TMEM budget)
template <int kSets, class ALoad, class BLoad, class Store>
static int launch_fp4_tm(const ALoad &a, const BLoad &b, const Store &st, const Epilogue &ep,
                         int64_t M, int64_t N, int64_t kw32, cudaStream_t s) {
    static const int cands[] = {192, 160, 128, 64};
    const int64_t sms = sm_count(), tm = ceil_div(M, umma::BM);
    int best = 192;
    int64_t best_cost = -1;
    for (int bn : cands) {
        const int64_t cost = ceil_div(tm * ceil_div(N, bn), sms) * (bn + 32);
        if (best_cost < 0 || cost < best_cost) best = bn, best_cost = cost;
    }
    using S = Store;
    switch (best) {
        case 64: return launch_umma_cfg<64, true, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 128: return launch_umma_cfg<128, true, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        case 160: return launch_umma_cfg<160, true, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
        default: return launch_umma_cfg<192, true, 4, ALoad, BLoad, S, 1, true, kSets>(a, b, st, ep, M, N, kw32, s);
    }
}

template <int kVec, class ALoad, class BLoad, class Store>
static int launch_umma(const ALoad &a, const BLoad &b, const Store &st, const Epilogue &ep,
                       int64_t M, int64_t N, int64_t kw32, cudaStream_t s) {
    if constexpr (!std::is_same<BLoad, TmaConv>::value) {
        // variant 0 (128 x 256 tiles, A and B through SMEM) also by default for cp.async-fed
        // shapes with M <= 64 (e.g. ResNet-18 layer1 convs, 64 filters): measured 1.1-1.4x
        // the A-in-TMEM engine there (tools/l1_variants.sh)
        // (and for every cp.async-fed conv: C % 256 != 0; measured 1.0-1.1x, profiles/r01)
        const bool small_m = (ep.variant == 2 || ep.variant == 4) &&
                             (M <= 64 || std::is_same<BLoad, ConvRows>::value) &&
                             !umma::is_tma<ALoad>::value;
        if (ep.variant == 0 || small_m)
            return launch_umma_cfg<256, false, kVec>(a, b, st, ep, M, N, kw32, s);
    }
    if constexpr (umma::is_tma<ALoad>::value) {
        if (ep.variant == 3) {
            if (kw32 >= BNN_FP4_SETS_KW32) return launch_fp4_tm<2>(a, b, st, ep, M, N, kw32, s);
            return launch_fp4_tm<1>(a, b, st, ep, M, N, kw32, s);
        }
        if (ep.variant == 2 || ep.variant == 4) {
            // long K (>= 24 superstages per tile): two expander sets on alternate
            // superstages; short K: one set and 8 epilogue warps (tiles end often)
            // long K and M >= 256: CTA pairs (cta_group::2); long K otherwise: two expander sets
            const int64_t pair_kw32 = g_debug.pair_kw32 > 0 ? g_debug.pair_kw32 : BNN_FP4_PAIR_KW32;
            if (kw32 >= pair_kw32 && M >= 2 * umma::BM && !(umma_dbg() & 8192))
                return launch_fp4_pair(a, b, st, ep, M, N, kw32, s);
            if (kw32 >= BNN_FP4_SETS_KW32) return launch_fp4<2>(a, b, st, ep, M, N, kw32, s);
            return launch_fp4<1>(a, b, st, ep, M, N, kw32, s);
        }
    }
    switch (choose_bn(M, N)) {
        case 128: return launch_umma_cfg<128, true, kVec>(a, b, st, ep, M, N, kw32, s);
        case 160: return launch_umma_cfg<160, true, kVec>(a, b, st, ep, M, N, kw32, s);
        case 176: return launch_umma_cfg<176, true, kVec>(a, b, st, ep, M, N, kw32, s);
        default: return launch_umma_cfg<192, true, kVec>(a, b, st, ep, M, N, kw32, s);
    }
}

template <class GS>
static int launch_xnor_gemm_umma_t(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                          int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n,
                          const Epilogue &ep, cudaStream_t s, const float *res) {
    const int64_t kw32 = 2 * ceil_div(K, 64);
    DenseRows a{reinterpret_cast<const uint32_t *>(A), 2 * lda, M, kw32};
    DenseRows b{reinterpret_cast<const uint32_t *>(B), 2 * ldb, N, kw32};
    GS st{};
    st.C = C, st.ldc_m = ldc_m, st.ldc_n = ldc_n, st.M = M, st.N = N, st.res = res;
    if (!(umma_dbg() & 4096)) encode_out(st);
    const bool vec4 = (lda % 2 == 0) && (ldb % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
    if (vec4 && !(umma_dbg() & 256)) {
        // TMA needs 16-B aligned bases and row pitches (even u64 leading dims)
        TmaRows ta{}, tb{};
        ta.base = a.base, ta.ld32 = a.ld32, ta.rows = M, ta.kw32 = kw32;
        tb.base = b.base, tb.ld32 = b.ld32, tb.rows = N, tb.kw32 = kw32;
        return launch_umma<4>(ta, tb, st, ep, M, N, kw32, s);
    }
    return vec4 ? launch_umma<4>(a, b, st, ep, M, N, kw32, s)
                : launch_umma<2>(a, b, st, ep, M, N, kw32, s);
}

// small-channel convs (C, F in {64, 128}): filter-stationary kernel with pixels as the
// TMEM A operand (bnn_sconv.cu); BNN_EUNSUP for other shapes
int launch_sconv(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
                 const uint64_t *w, int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                 int64_t ph, int64_t pw, int64_t oh, int64_t ow, float *y, const Epilogue &ep,
                 cudaStream_t s, const float *res);

// stride-1 small-channel convs: shifted-window kernel (bnn_wconv.cu), every pixel expanded once
int launch_wconv(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W, const uint64_t *w,
                 int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                 int64_t oh, int64_t ow, float *y, const Epilogue &ep, cudaStream_t s, const float *res);

template <class CS>
static int launch_bconv2d_umma_t(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
                        const uint64_t *w, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                        int64_t sw, int64_t ph, int64_t pw, int64_t oh, int64_t ow, float *y,
                        const Epilogue &ep, cudaStream_t s, const float *res) {
    if (ep.variant == 2 && !(umma_dbg() & 262144)) {
        const int rw = launch_wconv(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, oh, ow, y, ep, s, res);
        if (rw != BNN_EUNSUP) return rw;
        const int rc = launch_sconv(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, oh, ow, y, ep, s,
                                    res);
        if (rc != BNN_EUNSUP) return rc;
    }
    const int64_t cw64 = ceil_div(C, 64);
    const int64_t cs32 = 2 * cw64;
    const int64_t kw32 = kh * kw * cs32;
    const int64_t npix = B * oh * ow;
    DenseRows a{reinterpret_cast<const uint32_t *>(w), kw32, F, kw32};
    ConvRows b{reinterpret_cast<const uint32_t *>(x), npix, (int)H, (int)W, (int)cs32, (int)C,
               (int)kw, (int)sh, (int)sw, (int)ph, (int)pw, (int)oh, (int)ow, kw32};
    CS st{};
    st.y = y, st.F = F, st.ohw = oh * ow, st.npix = npix, st.res = res;
    if (!(umma_dbg() & 4096)) encode_out(st);
    const bool vec4 = (cw64 % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) == 0;
    // im2col TMA: whole 32-byte tap chunks (C % 256 == 0), corner offsets and
    // strides within the tensor-map limits, A-in-TMEM engine (superstages of 2)
    const int64_t up_w = (ow - 1) * sw - pw - (W - 1), up_h = (oh - 1) * sh - ph - (H - 1);
    const bool im2col = vec4 && cs32 % 8 == 0 && ep.variant >= 1 && !(umma_dbg() & 256) &&
                        ph <= 128 && pw <= 128 && up_w >= -128 && up_w <= 127 && up_h >= -128 &&
                        up_h <= 127 && sh <= 8 && sw <= 8 && kh <= 128 && kw <= 128;
    if (im2col) {
        TmaRows ta{};
        ta.base = a.base, ta.ld32 = kw32, ta.rows = F, ta.kw32 = kw32;
        TmaConv tb{};
        tb.x = reinterpret_cast<const uint32_t *>(x), tb.npix = npix, tb.H = (int)H, tb.W = (int)W;
        tb.cs32 = (int)cs32, tb.kw = (int)kw, tb.sh = (int)sh, tb.sw = (int)sw, tb.ph = (int)ph;
        tb.pw = (int)pw, tb.oh = (int)oh, tb.ow = (int)ow;
        return launch_umma<4>(ta, tb, st, ep, F, npix, kw32, s);
    }
    // <= 64 filters: swapped orientation (rows = pixels, cp.async im2col rows as the A
    // operand, 128 x 64 tiles with A in TMEM): every TMEM lane and epilogue warp busy
    // instead of half of them (tools/layer_bench.py)
    // (measured on ResNet's layer 1: the swapped route wins with a shortcut add --
    // 333 vs 381 us --, variant 0 without -- 200 vs 242 us; profiles/r01)
    if (F <= 64 && (ep.variant == 4 || (ep.variant == 2 && res != nullptr))) {
        using ST = typename std::conditional<CS::kPack, ConvStoreTPk, ConvStoreT>::type;
        ST ts{};
        ts.y = y, ts.F = F, ts.ohw = oh * ow, ts.npix = npix, ts.res = res;
        return vec4 ? launch_umma_cfg<64, true, 4, ConvRows, DenseRows, ST>(b, a, ts, ep, npix, F, kw32, s)
                    : launch_umma_cfg<64, true, 2, ConvRows, DenseRows, ST>(b, a, ts, ep, npix, F, kw32, s);
    }
    return vec4 ? launch_umma<4>(a, b, st, ep, F, npix, kw32, s)
                : launch_umma<2>(a, b, st, ep, F, npix, kw32, s);
}

}  // namespace bnn

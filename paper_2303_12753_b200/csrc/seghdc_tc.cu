// tcgen05 round kernel: assign_labels (clusterer.cpp:132-162) fused with the accumulation of
// update_centroids (clusterer.cpp:164-188) on the 5th-generation tensor cores, as a block-scaled
// FP4 product (kind::mxf4, e2m1 x e2m1 -> f32, every scale factor 1.0) that is exact by
// construction.
//
// Per CTA (one per SM) and per tile of 128 pixels (the MMA's M):
//   producer warp   2-D TMA (cp.async.bulk.tensor, 128B swizzle) of 128 pixel rows x 32 words
//                   ("chunk") into an NSTAGE-deep smem ring; once, the centroid B image.
//   unpack warps    3 per TMEM lane quarter: thread = pixel row. Each 32-bit HV word w becomes
//                   four A registers of eight e2m1 nibbles, one HV bit per nibble:
//                     w & 0x22222222          bits 4j+1 as 1.0      (w << 1) & 0x22222222  bits 4j   as 1.0
//                     w & 0x44444444          bits 4j+2 as 2.0      (w >> 1) & 0x44444444  bits 4j+3 as 2.0
//                   stored to TMEM with tcgen05.st (A lives in TMEM, one buffer per chunk).
//   MMA warps       per k-step of 64 HV dims ONE tcgen05.mma.kind::mxf4 M128 N16 K64 against
//                   B = the centroid digits d (weight-1 nibbles) or d/2 (weight-2 nibbles), so
//                   every product is bit * d exactly; two warps take alternate chunks into their
//                   own accumulators. tcgen05.commit frees the A buffer / publishes the tile.
//   epilogue warps  one per lane quarter: tcgen05.ld of the 2 x 16 accumulator columns of its
//                   pixel, exact integer dots, 128-bit argmax, labels, counts, update list.
//   fold warps      incremental re-bundling of cluster 1: only pixels whose membership of
//                   cluster 1 changed this round are folded into Harley-Seal counters (thread
//                   = word column, rows read back from L2): a pixel entering adds its HV, a
//                   pixel leaving adds its complement, and the flush subtracts the number of
//                   leavers, so the exchange buffer receives the exact delta of cluster 1's
//                   member sums (k_finish keeps the running sums; cluster 0 = colsum - S1).
//                   After the first rounds almost no pixel changes and the fold is idle.
// Centroid entries z are written in balanced base 8, z = sum_p d_p 8^p with d_p in [-4, 3]
// (kP8 = 8 digits cover z <= 3 (8^8 - 1) / 7): every digit and every half-digit is an e2m1
// value, each digit column's dot is an integer of magnitude <= 4 D < 2^24 (exact in f32), and
// the epilogue recombines the digit dots in int64.
// All hand-offs are mbarriers; the counters and counts leave through the exchange buffer
// exactly as in the IMMA kernel (seghdc_kernels.cu), so results are bit-identical.
#include <cuda.h>

#include <algorithm>

#include "kernels.cuh"
#include "launch.h"

namespace seghdc_dev {
namespace {

constexpr uint32_t kTP = 128;      // pixels per tile (MMA M)
constexpr uint32_t kCW = 32;       // HV words per chunk (one 128-byte swizzle span per row)
constexpr uint32_t kKS = kCW / 2;  // k-steps (64 HV dims) per chunk
constexpr uint32_t kChunkBytes = kTP * kCW * 4;
constexpr uint32_t kP8 = 8;        // balanced base-8 digits per centroid entry (K <= 4 layouts)
// warp layout of the unsplit kernel (SM sub-partition = warp % 4): [0, 12) unpack (3 per lane
// quarter), [12, 16) epilogue (one per lane quarter), 16/17/21/22 fold, 18/19 MMA issue
// (sub-partitions 2 and 3, away from the producer), 20 producer. Two MMA-issuing warps split the
// chunks of a tile (even / odd) into two accumulators, halving the issue load on any one
// sub-partition. The dimension-split kernel (SPLIT = 4, below) has no fold warps: [0, 8) unpack
// (2 per lane quarter), [8, 12) epilogue, 12 MMA, 13 producer.
constexpr uint32_t kNRW = 4;
// chunks per tile: at least 2, so the two MMA warps of the K <= 2 layout (alternating chunks)
// both write their accumulators; a short HV's second chunk is all zeros (TMA out-of-bounds fill)
__host__ __device__ __forceinline__ uint32_t tc_chunks(uint32_t W32) {
    const uint32_t c = (W32 + kCW - 1) / kCW;
    return c < 2 ? 2u : c;
}
__device__ __forceinline__ int fold_index(uint32_t warp) {
    return warp == 16 ? 0 : warp == 17 ? 1 : warp == 21 ? 2 : warp == 22 ? 3 : -1;
}
// TMEM columns: A buffers [128*i, 128*i+128), then accumulators D[tile parity][MMA warp]
// (N columns each), then the (all 1.0) scale factors of A and B
constexpr uint32_t kTmemCols = 512;
// Per-layout configuration. N = NDIG digit columns per cluster x KC clusters: 16 (K <= 2) and 32
// (K <= 4) with 8 digits and the whole B image resident; 64 (K <= 8, 8 base-9 digits: entries up to
// 21.5M, i.e. images of 2^24 pixels) with SPLIT = 4: a cluster of 4 CTAs shares each 128-pixel
// tile, CTA q owning a quarter of the HV dimensions (and only that quarter of the B image), and
// the partial dots meet in distributed shared memory.
template <uint32_t NCOL, uint32_t SPLIT = 1>
struct TcCfg {
    static constexpr uint32_t N = NCOL;
    // the split layout uses balanced base 9 (digits -4..4: each digit and half-digit is still an
    // e2m1 value), so 8 digits cover entries up to 4 (9^8 - 1) / 8 = 21.5M (images of 2^24
    // pixels) with N = 8 x 8 = 64 columns instead of 9 base-8 digits (N = 72)
    static constexpr uint32_t BASE = (SPLIT > 1 || NCOL == 64) ? 9 : 8;
    static constexpr uint32_t NDIG = kP8;
    static constexpr uint32_t KC = NCOL / NDIG;              // clusters of the layout
    static constexpr uint32_t KB = NCOL * 32;                // B image bytes per k-step: N rows x 64 e2m1
#ifndef SEGHDC_SPLIT_AB3
    static constexpr uint32_t AB = (SPLIT > 1 || NCOL == 64) ? 2 : 3;  // A buffers in TMEM (128 columns each)
#else  // experiment: 3 A buffers and one accumulator set in the split layout (32 warps)
    static constexpr uint32_t AB = 3;
#endif
#ifdef SEGHDC_C3_UH2
    // experiment: the K <= 4 layout (no fold warps) with two unpack warps per chunk
    static constexpr bool FOLD = NCOL == 16 && SPLIT == 1;    // fold warps (incremental K == 2 schedule)
    static constexpr uint32_t UH = (SPLIT > 1 || !FOLD) ? 2 : 1;  // unpack warps sharing one chunk (halves)
#else
    static constexpr bool FOLD = SPLIT == 1 && NCOL <= 32;    // fold warps (incremental K == 2 schedule)
    static constexpr uint32_t UH = (SPLIT > 1 || NCOL == 64) ? 2 : 1;  // unpack warps sharing one chunk (halves)
#endif
    static constexpr uint32_t UW = AB * UH;                  // unpack warps per TMEM lane quarter
#ifndef SEGHDC_NO_HALVES
    // in the layouts with two unpack warps per chunk (split, N = 64), each half chunk is its own
    // hand-off (full / free barriers per half, 8 MMAs + a commit per half): the MMAs of a half
    // start as soon as its two warps are done (C4 rounds 5-8 % faster; measured slower where one
    // warp unpacks a whole chunk, so those layouts keep whole-chunk hand-offs)
    static constexpr bool HALVES = UH == 2;
#else
    static constexpr bool HALVES = false;
#endif
#ifdef SEGHDC_QUARTERS  // experiment: quarter-chunk hand-offs (4 MMAs + a commit each)
    static constexpr uint32_t PARTS = HALVES ? 4 : 1;
#else
    static constexpr uint32_t PARTS = HALVES ? 2 : 1;        // hand-offs per chunk
#endif
    static constexpr uint32_t NAF = PARTS * AB;              // a_free barriers
#if defined(SEGHDC_SPLIT_AB3)
    static constexpr uint32_t DB = SPLIT > 1 ? 1 : 2;
#elif !defined(SEGHDC_C3_NMW2)
    static constexpr uint32_t DB = 2;                        // accumulator sets (by tile parity)
#else
    static constexpr uint32_t DB = (NCOL == 32 && SPLIT == 1) ? 1 : 2;
#endif
    static constexpr uint32_t Stages = NCOL == 16 ? 9 : (SPLIT > 1 || NCOL == 64) ? (AB == 3 ? 3 : 4) : 3;  // smem ring depth (16 KB each):
                                                             // the larger B image takes the rest; a multiple
                                                             // of AB, so slot g % Stages is unpacked by phase g % AB
#ifndef SEGHDC_C3_NMW2
    static constexpr uint32_t NMW = NCOL == 16 ? 2 : 1;      // MMA-issuing warps (alternate chunks)
#else
    static constexpr uint32_t NMW = (NCOL == 16 || (NCOL == 32 && SPLIT == 1)) ? 2 : 1;
#endif
#ifdef SEGHDC_PAIR
    // CTA pairs (cta_group::2, M = 256): the 4-CTA cluster is two pairs; pair p multiplies the two
    // tiles of a 256-pixel super-tile (one per CTA, in that CTA's TMEM) against dimension half p,
    // each CTA holding half of the digit columns of B, so every MMA reads 1 KB of B per SM, not 2
    static constexpr bool PAIR = SPLIT == 4;
#else
    static constexpr bool PAIR = false;
#endif
    static constexpr uint32_t DS = PAIR ? 2 : SPLIT;         // dimension split of the cluster
#ifdef SEGHDC_COOP
    // the unpack warps of a lane quarter share EVERY chunk (16-byte pieces u, u + AB, ... each)
    // instead of owning whole chunks: a chunk is complete after a third of the time, so its MMAs
    // overlap the next chunk's unpack instead of all AB buffers filling, then all draining
    static constexpr bool COOP = !HALVES;
#else
    static constexpr bool COOP = false;
#endif
    static constexpr uint32_t WEpi = 4 * UW;                 // first epilogue warp
    static constexpr uint32_t WMma0 = (SPLIT > 1 || !FOLD) ? WEpi + 4 : 18;
    static constexpr uint32_t WProd = (SPLIT > 1 || !FOLD) ? WEpi + 4 + NMW : 20;
    static constexpr uint32_t WFin = WEpi + 6;               // SPLIT: 2 finalizer warps (labels), by tile parity
    static constexpr uint32_t Warps = SPLIT > 1 ? WEpi + 8 : FOLD ? 23 : WEpi + 5 + NMW;
    static constexpr uint32_t ColD = 128 * AB;
    static constexpr uint32_t ColSF = ColD + DB * NMW * NCOL;  // after D[DB tile parities][NMW]
    static_assert(Stages % AB == 0, "ring slots follow the unpack phases");
    static_assert(ColSF + 16 <= kTmemCols, "TMEM budget");
    static_assert(SPLIT == 1 || Warps == 4 * UW + 8, "split layout: unpack, 4 epilogue, MMA, producer, 2 finalizers");
};
constexpr uint32_t kKB = TcCfg<16>::KB;  // the K <= 2 image (k_finish_tc)

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// dot_c = sum_p v_p BASE^p from the 8 digit-column dots of one cluster (f32 accumulators holding
// exact integers, |v_p| <= 4 x the dimensions one CTA multiplies). Digits are first combined in
// groups of 3, 3 and 2 with FFMA, which stays exact while 4 dims (1 + BASE + BASE^2) < 2^24
// (dims < 46k at base 9; every tcgen05 layout keeps a CTA's dimensions below 25k), so a cluster
// costs 5 FFMA + 3 F2I + 2 IMAD.WIDE instead of 8 conversions and 8 64-bit multiply-adds.
template <uint32_t BASE>
__device__ __forceinline__ long long combine_digits(const float (&v)[8]) {
    constexpr float B = float(BASE);
    const float g0 = fmaf(fmaf(v[2], B, v[1]), B, v[0]);
    const float g1 = fmaf(fmaf(v[5], B, v[4]), B, v[3]);
    const float g2 = fmaf(v[7], B, v[6]);
    constexpr long long B3 = (long long)BASE * BASE * BASE, B6 = B3 * B3;
    return (long long)__float2int_rn(g0) + (long long)__float2int_rn(g1) * B3 + (long long)__float2int_rn(g2) * B6;
}
// One chunk (kKS k-steps) of MMAs, issued by an elected lane of the calling warp from a single
// asm block: addresses advance inside PTX, so the whole block runs on the uniform datapath.
// Per k-step ONE block-scaled FP4 MMA: A = 8 TMEM columns (64 e2m1), B = kN x 64 e2m1 at b;
// the scale factors (all ue8m0 127 = 1.0) sit at sf.
#define SEGHDC_KSTEP                                                                                  \
    "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [a], b, %3, [%4], [%5], p;\n\t" \
    "add.u64 b, b, %6;\n\tadd.u32 a, a, 8;\n\tsetp.ne.b32 p, 1, 0;\n\t"
template <uint32_t KB>
__device__ __forceinline__ void tc_mma_chunk(uint32_t d_t, uint32_t a_t, uint64_t bdesc, uint32_t idesc, uint32_t sf,
                                             uint32_t accum) {
    static_assert(kKS == 16, "tc_mma_chunk issues 16 k-steps");
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %7, 0;\n\t"
        "mov.b32 a, %1;\n\tmov.b64 b, %2;\n\t" SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP
            SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP
                SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP "}" ::"r"(d_t),
        "r"(a_t), "l"(bdesc), "r"(idesc), "r"(sf), "r"(sf + 4), "n"(KB >> 4), "r"(accum)
        : "memory");
}
template <uint32_t KB>
__device__ __forceinline__ void tc_mma_half(uint32_t d_t, uint32_t a_t, uint64_t bdesc, uint32_t idesc, uint32_t sf,
                                            uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %7, 0;\n\t"
        "mov.b32 a, %1;\n\tmov.b64 b, %2;\n\t" SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP
            SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP "}" ::"r"(d_t),
        "r"(a_t), "l"(bdesc), "r"(idesc), "r"(sf), "r"(sf + 4), "n"(KB >> 4), "r"(accum)
        : "memory");
}
template <uint32_t KB>
__device__ __forceinline__ void tc_mma_quarter(uint32_t d_t, uint32_t a_t, uint64_t bdesc, uint32_t idesc, uint32_t sf,
                                               uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %7, 0;\n\t"
        "mov.b32 a, %1;\n\tmov.b64 b, %2;\n\t" SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP SEGHDC_KSTEP "}" ::"r"(d_t),
        "r"(a_t), "l"(bdesc), "r"(idesc), "r"(sf), "r"(sf + 4), "n"(KB >> 4), "r"(accum)
        : "memory");
}
#undef SEGHDC_KSTEP
// commit all prior MMAs of the calling thread to an mbarrier (elected lane)
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
// Lean issue (the default): ONE elected thread issues NSTEP k-steps from warp-uniform operands, so
// ptxas keeps every address in uniform registers (UTCOMMA + UIADD3 per k-step). The asm-block
// variants above predicate each MMA on the per-thread elect result, which costs ~15 instructions
// and 5 R2UR per MMA: measured 48-60 cycles per MMA inside the busy round kernel against the
// tensor pipe's 12 / 16 / 32 (N = 16 / 32 / 64; tools/probes/mma_floor.cu).
__device__ __forceinline__ bool tc_elect() {
    uint32_t e;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
    return e != 0;
}
template <uint32_t KB, uint32_t NSTEP>
__device__ __forceinline__ void tc_mma_steps(uint32_t d_t, uint32_t a_t, uint64_t bdesc, uint32_t idesc, uint32_t sf,
                                             uint32_t accum) {
#pragma unroll
    for (uint32_t ks = 0; ks < NSTEP; ++ks)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n\t}" ::"r"(d_t),
            "r"(a_t + 8 * ks), "l"(bdesc + uint64_t(ks) * (KB >> 4)), "r"(idesc), "r"(sf), "r"(sf + 4),
            "r"(ks ? 1u : accum)
            : "memory");
}
// the pair forms: M = 256 over both CTAs' TMEM, issued by the leader; the commit arrives on the
// same barrier of every CTA in `mask` (cluster ranks)
template <uint32_t KB, uint32_t NSTEP>
__device__ __forceinline__ void tc_mma_steps_pair(uint32_t d_t, uint32_t a_t, uint64_t bdesc, uint32_t idesc, uint32_t sf,
                                                  uint32_t accum) {
#pragma unroll
    for (uint32_t ks = 0; ks < NSTEP; ++ks)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n\t}" ::"r"(d_t),
            "r"(a_t + 8 * ks), "l"(bdesc + uint64_t(ks) * (KB >> 5)), "r"(idesc), "r"(sf), "r"(sf + 4),
            "r"(ks ? 1u : accum)
            : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"(mask)
                 : "memory");
}
// commit by the calling (already elected) thread
__device__ __forceinline__ void tc_commit_one(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// L2 prefetch of a future chunk (no shared memory, no barrier): the ring's TMA load of that chunk
// then hits L2, so a shallow ring (large B image) still keeps enough bytes in flight
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// smem matrix descriptor: K-major, no swizzle, core matrices of 8 rows x 16 B; LBO = 128 (next
// core matrix along K), SBO = 256 (next 8 rows), version 1 (tcgen05)
__device__ __forceinline__ uint64_t bdesc_at(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
}
// instruction descriptor, block-scaled kinds: A/B format E2M1 (1) at bits 7 / 10, both K-major,
// N >> 3 at bit 17, scale format UE8M0 (bit 23), M >> 4 at bit 24, scale-factor ids 0, K = 64
constexpr uint32_t idesc_mxf4(uint32_t n, uint32_t m) {
    return (1u << 7) | (1u << 10) | ((n >> 3) << 17) | (1u << 23) | ((m >> 4) << 24);
}

#ifdef SEGHDC_HANGDBG
// diagnostic build only: bounded mbarrier waits. Timeouts are logged (block, warp, barrier id,
// parity, iteration) into host-mapped memory, then the kernel traps, so the log survives.
__device__ unsigned int* g_hang;  // [0] count, then 5 words per record
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity, uint32_t id, uint32_t it) {
    uint32_t ok = 0;
    for (uint32_t round = 0; round < 4 && !ok; ++round) {
        for (uint32_t i = 0; i < (1u << 22) && !ok; ++i)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (!ok && round == 0 && (threadIdx.x & 31) == 0) {  // log once, keep waiting so others log too
            const unsigned k = atomicAdd(&g_hang[0], 1u);
            if (k < 200) {
                volatile unsigned* r = g_hang + 1 + 5 * k;
                r[0] = blockIdx.x; r[1] = threadIdx.x >> 5; r[2] = id; r[3] = parity; r[4] = it;
                __threadfence_system();
            }
        }
    }
    if (!ok) asm volatile("trap;");
}
#define TCW(id, it, bar, par) (PRG((id) * 100000 + (it)), tc_wait(bar, par, id, it), PRG((id) * 100000 + (it) + 50000))
// per-warp progress of block 0 (host-mapped): last code written by lane 0
#define PRG(code) ((blockIdx.x == 0 && (threadIdx.x & 31) == 0) ? (void)(((volatile unsigned*)g_hang)[4096 + (threadIdx.x >> 5)] = (code)) : (void)0)
#else
#define TCW(id, it, bar, par) mbar_wait(bar, par)
#define PRG(code) ((void)0)
#endif
// Hand-offs whose arrivals come from whole warps (slot_free, a_full, d_free): one elected arrival
// per warp after a __syncwarp instead of 32 (128-256 serialised shared-memory atomics per hand-off
// otherwise). SEGHDC_LANE_ARRIVE restores per-lane arrivals (A/B builds).
#ifndef SEGHDC_LANE_ARRIVE
constexpr uint32_t kArrivePerWarp = 1;
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
#else
constexpr uint32_t kArrivePerWarp = 32;
__device__ __forceinline__ void warp_arrive(uint64_t* bar) { mbar_arrive(bar); }
#endif
// the same towards CTA `rank` of the cluster (pairs: the peer's warps report to the leader's barriers)
__device__ __forceinline__ void warp_arrive_at(uint64_t* bar, uint32_t rank, bool remote);
// the A-buffer hand-offs (unpack <-> MMA): polling waits under SEGHDC_SPIN_AB=1/2/3 (experiment;
// 1: MMA warp's a_full, 2: unpack warps' a_free, 3: both)
#ifndef SEGHDC_SPIN_AB
#define SEGHDC_SPIN_AB 0
#endif
#if !defined(SEGHDC_HANGDBG)
#define TCW_AFULL(id, it, bar, par) ((SEGHDC_SPIN_AB & 1) ? mbar_wait_spin(bar, par) : mbar_wait(bar, par))
#define TCW_AFREE(id, it, bar, par) ((SEGHDC_SPIN_AB & 2) ? mbar_wait_spin(bar, par) : mbar_wait(bar, par))
#else
#define TCW_AFULL TCW
#define TCW_AFREE TCW
#endif

template <uint32_t NCOL, uint32_t SPLIT = 1>
struct TcSmem {
    using Cfg = TcCfg<NCOL, SPLIT>;
    static constexpr size_t ring = 0;  // [Stages][128][32] u32, 1024-aligned (128B swizzle)
    __host__ __device__ static size_t b(uint32_t nks) { return size_t(Cfg::Stages) * kChunkBytes; }              // [nks][KB] B image
    __host__ __device__ static size_t list(uint32_t nks) { return b(nks) + size_t(nks) * Cfg::KB; }             // [2][4][32] u32
    __host__ __device__ static size_t listn(uint32_t nks) { return list(nks) + (SPLIT > 1 ? 0 : 2 * 4 * 32 * 4); }  // [2][4] u32
    __host__ __device__ static size_t misc(uint32_t nks) { return listn(nks) + 2 * 4 * 4; }                        // tmem base, skip
    // SPLIT: partial dots of the 4 CTAs for this CTA's lane quarter, [2][src][KC][32] i64
    __host__ __device__ static size_t xb(uint32_t nks) { return misc(nks) + 16; }
    __host__ __device__ static size_t bars(uint32_t nks) {
        return (xb(nks) + (SPLIT > 1 ? 2 * size_t(SPLIT) * 32 * Cfg::KC * 8 : 0) + 7) & ~size_t(7);
    }
    static constexpr uint32_t nbars =
        2 * Cfg::Stages + (Cfg::PARTS > 2 ? Cfg::PARTS : 2) * Cfg::AB + Cfg::NAF + 2 + 2 + 2 + 2 + 1 +
        (SPLIT > 1 ? 2 * (2 + SPLIT) + 1 : 0);  // x_full [2][2] (pairs; [2] otherwise), x_free [2][SPLIT], b_peer
    __host__ __device__ static size_t total(uint32_t nks) { return bars(nks) + nbars * 8; }
};

// distributed shared memory (SPLIT kernel): the address of the same smem object in CTA `rank`
// of the cluster, remote stores and cluster-scope mbarrier arrive / wait
__device__ __forceinline__ uint32_t cl_mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_st_u64(uint32_t addr, unsigned long long a) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(a) : "memory");
}
// asynchronous remote store that completes `bytes` on the destination CTA's mbarrier when the data
// has landed: the sender neither waits for an acknowledgement nor issues a release
__device__ __forceinline__ void cl_st_async_u64(uint32_t addr, unsigned long long a, uint32_t remote_bar) {
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr), "l"(a),
                 "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void cl_arrive(uint32_t remote_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void cl_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nCLW_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra CLW_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void warp_arrive_at(uint64_t* bar, uint32_t rank, bool remote) {
    __syncwarp();
    if (kArrivePerWarp == 32 || (threadIdx.x & 31) == 0) {
        if (remote) cl_arrive(cl_mapa(smem_u32(bar), rank));
        else mbar_arrive(bar);
    }
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace

#ifdef SEGHDC_TRACE
__device__ unsigned long long g_trace_tc[148 * 64 * 8];
__device__ int g_trace_round;  // 0: trace every launch (the last one wins), r: only round r
#define TC_ON (g_trace_round == 0 || int(round) == g_trace_round)
#define TC_TR(ev, it)                                                                 \
    do {                                                                              \
        if (lane == 0 && blockIdx.x < 148 && (it) < 60 && TC_ON)                      \
            g_trace_tc[(size_t(blockIdx.x) * 64 + (it)) * 8 + (ev)] = clock64();      \
    } while (0)
static cudaEvent_t* g_tc_events = nullptr;
void read_trace_tc(void* dst) {
    cudaMemcpyFromSymbol(dst, g_trace_tc, sizeof(g_trace_tc));
    if (g_tc_events) {  // last launch: event ms of [stamp0], [round], [stamp1] into slot 60 of CTA 0
        cudaEventSynchronize(g_tc_events[3]);
        unsigned long long* o = static_cast<unsigned long long*>(dst) + 60 * 8;
        for (int i = 0; i < 3; ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, g_tc_events[i], g_tc_events[i + 1]);
            o[i] = (unsigned long long)(ms * 1e6);  // ns
        }
    }
}
// kernel-level events in slot 63 with %globaltimer (ns, comparable across SMs)
#define TC_TG(ev)                                                                     \
    do {                                                                              \
        if (lane == 0 && blockIdx.x < 148 && TC_ON) {                                 \
            unsigned long long t_;                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
            g_trace_tc[(size_t(blockIdx.x) * 64 + 63) * 8 + (ev)] = t_;               \
        }                                                                             \
    } while (0)
// accumulated wait cycles in slot 62: 0 unpack slot_full, 1 unpack a_free, 2 MMA a_full,
// 3 MMA issue (wait-free part), 4 producer slot_free, 5 epilogue d_full
#define TC_ACC(ev, cyc)                                                               \
    do {                                                                              \
        if (lane == 0 && blockIdx.x < 148 && TC_ON)                                   \
            atomicAdd(&g_trace_tc[(size_t(blockIdx.x) * 64 + 62) * 8 + (ev)], (cyc));  \
    } while (0)
#define TC_CLK(v) const unsigned long long v = clock64()
// more accumulated cycles in slot 60 (split layout): 0 epilogue TMEM loads, 1 digit recombination,
// 2 remote stores + arrive, 3 finalizer x_full wait, 4 finalizer sum + argmax + labels, 5 lists
#define TC_ACC2(ev, cyc)                                                              \
    do {                                                                              \
        if (lane == 0 && blockIdx.x < 148 && TC_ON)                                   \
            atomicAdd(&g_trace_tc[(size_t(blockIdx.x) * 64 + 60) * 8 + (ev)], (cyc));  \
    } while (0)
#else
#define TC_TR(ev, it) ((void)0)
#define TC_TG(ev) ((void)0)
#define TC_ACC(ev, cyc) ((void)0)
#define TC_ACC2(ev, cyc) ((void)0)
#define TC_CLK(v) ((void)0)
#endif

// WR: count 128-bit comparator wraps (diagnostic; instantiated only where the host's bound says
// a wrap is possible, because the counting costs the split layout registers)
template <bool UPD, int H, uint32_t NCOL, uint32_t SPLIT, bool WR>
__global__ void __launch_bounds__(TcCfg<NCOL, SPLIT>::Warps * 32, 1)
    k_round_tc(const __grid_constant__ CUtensorMap tmap, const uint32_t* __restrict__ grid, uint64_t n, uint32_t S32,
               uint32_t W32, uint32_t K, const uint8_t* __restrict__ bimg, uint32_t nks, uint32_t* labels,
               void* state, uint32_t round, int do_update, uint32_t* __restrict__ xchg, uint32_t Dp,
               uint32_t* __restrict__ flist, uint32_t* __restrict__ flist_count, uint32_t serpentine, uint32_t pf,
               const unsigned long long* __restrict__ lh_slot) {
    constexpr uint32_t NRT = kNRW * 32;
    constexpr int CPTMAX = 3;  // fold columns per thread: W32 <= 3 * NRW * 32 (tc_supported)
    using Cfg = TcCfg<NCOL, SPLIT>;
    using Smem = TcSmem<NCOL, SPLIT>;
    constexpr uint32_t kStages = Cfg::Stages, NMW = Cfg::NMW, KC = Cfg::KC, NDIG = Cfg::NDIG;
    constexpr uint32_t kAB = Cfg::AB, kUH = Cfg::UH, kWEpi = Cfg::WEpi, kWMma0 = Cfg::WMma0, kWProd = Cfg::WProd;
    constexpr uint32_t kColD = Cfg::ColD;
#ifdef SEGHDC_SPLIT_LDG
    constexpr bool kLdg = SPLIT > 1;  // experiment: the unpack warps load A rows from global memory
#else
    constexpr bool kLdg = false;
#endif
    static_assert(!UPD || (NCOL == 16 && SPLIT == 1), "the incremental fold is the K == 2 schedule");
    extern __shared__ __align__(1024) uint8_t smem[];
    StateView st = StateView::at(state, K);

    // the warp index through a shuffle: ptxas then knows it is warp-uniform and keeps the role
    // branches and the MMA warps' operand addresses on the uniform datapath
    const uint32_t tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const uint32_t parity = round & 1;
    uint32_t* tail = xchg + size_t(K) * Dp;  // [K counts | changed]
    if (warp == 0) TC_TG(0);
    uint8_t* ring = smem + Smem::ring;
    uint8_t* sB = smem + Smem::b(nks);
    uint32_t* s_list = reinterpret_cast<uint32_t*>(smem + Smem::list(nks));
    uint32_t* s_listn = reinterpret_cast<uint32_t*>(smem + Smem::listn(nks));
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + Smem::misc(nks));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars(nks));
    uint64_t* slot_full = bars;                 // [kStages] TMA landed
    uint64_t* slot_free = bars + kStages;       // [kStages] unpack warps read the chunk
    // a_full[ab][m]: chunk g (buffer ab = g % kAB) written for MMA warp m = g % 2. One barrier
    // per (buffer, consumer) keeps every parity wait in order (a shared barrier consumed by two
    // warps alternately would alias phases)
    uint64_t* a_full = bars + 2 * kStages;      // [kAB][2] A buffer written (tcgen05.st)
    uint64_t* a_free = a_full + (Cfg::PARTS > 2 ? Cfg::PARTS : 2) * kAB;  // [kAB] MMAs on the A buffer done; [PARTS kAB] by part
    uint64_t* d_full = a_free + Cfg::NAF;       // [2] tile accumulator complete (commit)
    uint64_t* d_free = d_full + 2;              // [2] epilogue read the accumulator
    uint64_t* list_ready = d_free + 2;          // [2] labels + update list written
    uint64_t* list_free = list_ready + 2;       // [2] fold warps done with the list
    uint64_t* b_full = list_free + 2;           // B image landed
    uint64_t* x_full = b_full + 1;              // SPLIT: [2] the 4 partial dots of this CTA's lane quarter landed (pairs: [2][2], by quarter)
    uint64_t* x_free = x_full + 4;              // SPLIT: [2][dest] dest CTA consumed what this CTA's epilogue warp sent
    uint64_t* b_peer = x_free + 2 * SPLIT;      // pairs (leader): the peer's half of the B slice landed
    const uint32_t qrank = SPLIT > 1 ? cl_rank() : 0u;  // SPLIT: dimension quarter = rank in the cluster
    const uint32_t cid = blockIdx.x / SPLIT, ncl = gridDim.x / SPLIT;  // tiles go to clusters
    // pairs: CTA (pr, pe) = rank 2 pr + pe multiplies tile pe of every super-tile (256 pixels)
    // against dimension half pr; pe == 0 leads the pair (issues the MMAs)
    constexpr bool kPair = Cfg::PAIR;
    const uint32_t pr = qrank >> 1, pe = qrank & 1, leader_rank = qrank & ~1u;
    const uint32_t dq = kPair ? pr : qrank;     // this CTA's part of the dimension split

    const uint32_t nch_all = tc_chunks(W32);  // chunks per tile
    // SPLIT: this CTA's chunks [ch0, ch0 + nch) of every tile; its B image slice starts at ch0
    const uint32_t ch0 = dq * nch_all / Cfg::DS, nch = (dq + 1) * nch_all / Cfg::DS - ch0;
    const uint64_t ntiles_px = (n + kTP - 1) / kTP;
    const uint64_t ntiles = kPair ? (ntiles_px + 1) / 2 : ntiles_px;  // pairs: super-tiles of two tiles
    const uint32_t my_tiles = cid < ntiles ? uint32_t((ntiles - 1 - cid) / ncl + 1) : 0;
    // serpentine traversal: odd rounds walk the tiles from the end of the grid, even rounds from
    // the start, so each round begins with the ~100 MB the previous pass (the encode, or the
    // previous round) left in L2 and only the rest streams from HBM
    const bool reverse = serpentine && (round & 1) != 0;
    auto tile_px0 = [&](uint32_t it) -> uint64_t {
        const uint64_t t = cid + uint64_t(it) * ncl;
        return ((reverse ? ntiles - 1 - t : t) * (kPair ? 2 : 1) + (kPair ? pe : 0)) * kTP;
    };

    if (tid == 0) {
        for (uint32_t s = 0; s < kStages; ++s) {
            mbar_init(&slot_full[s], 1);
            mbar_init(&slot_free[s], 4 * kArrivePerWarp * (Cfg::COOP ? Cfg::UW : kUH));
        }
        for (uint32_t b = 0; b < (Cfg::PARTS > 2 ? Cfg::PARTS : 2) * kAB; ++b)  // PARTS > 1: a_full[PARTS b + part]
            mbar_init(&a_full[b], (kPair ? 2 : 1) * 4 * kArrivePerWarp * (Cfg::HALVES ? 1 : Cfg::COOP ? Cfg::UW : kUH));  // pairs: both CTAs' warps
        for (uint32_t b = 0; b < Cfg::NAF; ++b) mbar_init(&a_free[b], 1);
        for (uint32_t b = 0; b < 2; ++b) {
            mbar_init(&d_full[b], NMW);  // every MMA warp commits
            mbar_init(&d_free[b], (kPair ? 2 : 1) * 4 * kArrivePerWarp);
            mbar_init(&list_ready[b], 4 * 32);
            mbar_init(&list_free[b], NRT);
        }
        mbar_init(b_full, 1);
        if (SPLIT > 1) {
            for (uint32_t b = 0; b < 4; ++b) mbar_init(&x_full[b], 1);  // the finalizer arms it with the senders' bytes
            for (uint32_t b = 0; b < 2 * SPLIT; ++b) mbar_init(&x_free[b], 1);
            mbar_init(b_peer, 1);
        }
        mbar_fence_init();
        s_listn[0] = s_listn[1] = 0;
    }
    if (kPair) {  // both CTAs of a pair are resident before either allocates the pair's TMEM
        __syncthreads();
        cl_sync();
    }
    if (warp == kWMma0) {
        if constexpr (kPair) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_misc)),
                         "n"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_misc)),
                         "n"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (SPLIT > 1) cl_sync();  // every CTA's barriers are initialised before any remote arrive
    tc_fence_after();
    const uint32_t tbase = s_misc[0];
    if (warp < 4) {  // scale factors of A and B: every ue8m0 byte 127 (2^0), whatever the layout
        uint32_t one[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) one[q] = 0x7F7F7F7Fu;
        tc_st16(tbase + ((32 * warp) << 16) + Cfg::ColSF, one);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // programmatic dependent launch: everything above (barriers, TMEM, scale factors) overlaps
    // the previous kernel; state, B image, labels and the exchange buffer are read after it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const bool done = *reinterpret_cast<volatile uint32_t*>(&st.hdr->done) != 0;
    // last round of a run_pipeline call: the labels also go straight into the caller's
    // page-locked buffer (a device-mapped host pointer, written before the graph launch), so the
    // download overlaps the round instead of following it
    uint32_t* const labels_host = lh_slot ? reinterpret_cast<uint32_t*>(*lh_slot) : nullptr;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (done) {  // early stop reached (clusterer.cpp:213): nothing left to do
        if (kPair) cl_sync();  // the pair's TMEM is freed once both CTAs are here
        if (warp == kWMma0)
        {
            if constexpr (kPair) {
                asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
            } else {
                asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
            }
        }
        return;
    }
    if (blockIdx.x == 0 && tid == 0) st.hdr->rounds_run = round;
    if (warp == 0) TC_TG(1);
    // flist != nullptr (round 1: every member of cluster 1 enters): the changed pixels are
    // appended to a global list that k_fold_list folds with the whole GPU after this kernel,
    // instead of the fold warps reading them back tile by tile
#ifdef SEGHDC_EXP_NOGRID
    const bool folding = false;  // timing experiment: labels are meaningless, nothing to fold
#else
    const bool folding = UPD && do_update && flist == nullptr;
#endif

    if (warp < kWEpi) {
        // ------------------------------------------------------------------------ unpack warps
        // warp (qd, u) unpacks the 32 rows of lane quarter qd of every chunk g with
        // g % kAB == u / kUH (words [32 hf / kUH, 32 (hf + 1) / kUH) of the chunk, hf = u % kUH),
        // so kAB chunks are in flight per quarter (each warp's chain of LDS -> masks ->
        // tcgen05.st -> wait::st is latency-bound; SPLIT halves it with two warps per chunk)
        const uint32_t qd = warp & 3, u = warp >> 2;  // lane quarter, chunk phase x half
        const uint32_t ph = u / kUH, hf = u % kUH;
        const uint32_t r = 32 * qd + lane;            // pixel row of the tile
        const uint32_t lane_addr = tbase + ((32 * qd) << 16);
        const uint32_t nchunks = my_tiles * nch;
        // kLdg: the warp's 64 bytes of each chunk row come from global memory, one chunk ahead
        uint4 nv[4];
        auto ld_row = [&](uint32_t gg, uint4 (&o)[4]) {
            const uint64_t pr = tile_px0(gg / nch) + r;
            if (pr < n) {
                const uint4* p4 = reinterpret_cast<const uint4*>(grid + pr * S32 + (ch0 + gg % nch) * kCW + hf * 16);
#pragma unroll
                for (int j = 0; j < 4; ++j) o[j] = __ldg(p4 + j);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) o[j] = make_uint4(0u, 0u, 0u, 0u);
            }
        };
        if constexpr (kLdg) {
            if (ph < nchunks) ld_row(ph, nv);
        }
        for (uint32_t g = Cfg::COOP ? 0 : ph; g < nchunks; g += Cfg::COOP ? 1 : kAB) {
            const uint32_t s = g % kStages, ab = g % kAB;
            uint4 cv[4];
            if constexpr (kLdg) {
#pragma unroll
                for (int j = 0; j < 4; ++j) cv[j] = nv[j];
                if (g + kAB < nchunks) ld_row(g + kAB, nv);
            }
            TC_CLK(c0);
            if (!kLdg) TCW(1, g, &slot_full[s], (g / kStages) & 1);  // slot s only ever carries this warp's chunks
            TC_CLK(c1);
            if (warp == 0 && g == 0) TC_TG(3);
            constexpr uint32_t kPPW = Cfg::PARTS > 1 ? Cfg::PARTS / 2 : 1;  // parts per unpack warp
            TCW_AFREE(2, g, &a_free[Cfg::HALVES ? Cfg::PARTS * ab + kPPW * hf : ab], ((g / kAB) & 1) ^ 1);
            __syncwarp();  // lanes leave the spin loops independently; tcgen05.st is .sync.aligned
            TC_CLK(c2);
            if (warp == 0) { TC_ACC(0, c1 - c0); TC_ACC(1, c2 - c1); }
            tc_fence_after();
            if (warp == 0 && g % nch == 0) TC_TR(1, g / nch);
            const uint8_t* row = ring + size_t(s) * kChunkBytes + r * 128;
            // both shifts run on the FMA pipe (IMAD.SHL, IMAD.HI with an opaque 2^31), leaving the
            // ALU pipe the four masks per word
            const uint32_t half = opaque(0x80000000u), two = opaque(2u);
#pragma unroll
            for (uint32_t c16i = hf * (8 / kUH); c16i < (hf + 1) * (8 / kUH); ++c16i) {  // 16-byte pieces: 4 words = 2 k-steps
                // COOP: this warp's pieces u, u + AB, ... of every chunk
                const uint32_t c16 = Cfg::COOP ? u + c16i * kAB : c16i;
                if (Cfg::COOP && (c16i >= (8 + kAB - 1) / kAB || c16 >= 8)) continue;
#if defined(SEGHDC_EXP_NOGRID)  // timing experiment: no grid at all (no TMA, no smem), words from a hash
                const uint32_t hq = uint32_t(tile_px0(g / nch) + r) * 2654435761u ^ ((g % nch) * 8 + c16) * 40503u;
                const uint4 v = make_uint4(hq, hq * 3u, hq ^ 0x9E3779B9u, hq + 0x7F4A7C15u);
#elif !defined(SEGHDC_EXP_NOLDS)  // timing experiment only: no shared-memory reads in the unpack
                uint4 v;
                if constexpr (kLdg) v = cv[(c16 - hf * (8 / kUH)) & 3];
                else v = *reinterpret_cast<const uint4*>(row + ((c16 ^ (r & 7)) << 4));
#else
                const uint4 v = make_uint4(0u, 0u, 0u, 0u);  // all-zero A: every dot 0, labels settle at 0
#endif
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
                uint32_t a[16];
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // A column 4i + c: class c of word i (see header)
                    a[4 * i + 0] = w4[i] & 0x22222222u;
                    a[4 * i + 1] = w4[i] & 0x44444444u;
                    a[4 * i + 2] = (w4[i] * two) & 0x22222222u;
                    a[4 * i + 3] = __umulhi(w4[i], half) & 0x44444444u;
                }
#ifndef SEGHDC_EXP_NOSTTM  // timing experiment only: no A stores into TMEM
                tc_st16(lane_addr + ab * 128 + c16 * 16, a);  // k-steps 2*c16, 2*c16+1: 8 columns each
#else
                if (a[0] == 0x12345678u) tc_st16(lane_addr + ab * 128 + c16 * 16, a);
#endif
                if constexpr (Cfg::PARTS == 4) {  // quarter done: hand it off, claim the next one
                    if (((c16 + 1) & 1) == 0 && c16 + 1 < (hf + 1) * (8 / kUH)) {
                        const uint32_t qp = Cfg::PARTS * ab + c16 / 2;
                        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                        tc_fence_before();
                        warp_arrive_at(&a_full[qp], leader_rank, kPair && pe != 0);
                        TCW(2, g, &a_free[qp + 1], ((g / kAB) & 1) ^ 1);
                        __syncwarp();
                        tc_fence_after();
                    }
                }
            }
            PRG(10 * 100000 + g);
#ifndef SEGHDC_EXP_NOWAITST  // timing experiment only: hand the buffer off without waiting for the stores
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#endif
            PRG(11 * 100000 + g);
            if (!kLdg) warp_arrive(&slot_free[s]);
            tc_fence_before();
            warp_arrive_at(&a_full[Cfg::HALVES ? Cfg::PARTS * ab + kPPW * hf + (kPPW - 1) : 2 * ab + (g % NMW)], leader_rank,
                           kPair && pe != 0);
            if (warp == 0 && g % nch == nch - 1) TC_TR(2, g / nch);
        }
    } else if (SPLIT > 1 && warp < kWEpi + 4) {
        // ------------------------------------------------------- split layout: epilogue senders
        // One warp per lane quarter qd: the partial dots of its 32 pixels (this CTA's quarter of
        // the dimensions) go to CTA qd of the cluster, slot [tile parity][this CTA], with
        // asynchronous remote stores that complete bytes on that CTA's x_full barrier. The warp
        // never waits for the stores (a release + arrive cost a DSMEM round trip per tile, and
        // this warp is the split layout's critical path).
        if constexpr (SPLIT > 1) {
            const uint32_t qd = warp & 3;
            const uint32_t lane_addr = tbase + ((32 * qd) << 16);
            long long* xbuf = reinterpret_cast<long long*>(smem + Smem::xb(nks));
            // destination of lane quarter qd's partial dots: CTA qd, slot [this CTA]; pairs: the CTA
            // with this CTA's tile (same pe) in pair qd / 2, which finalizes quarters 2 (qd / 2) and
            // 2 (qd / 2) + 1 of it: slot [quarter qd % 2][this pair]
            const uint32_t xrank = kPair ? 2 * (qd >> 1) + pe : qd;
            const uint32_t xslot = kPair ? (qd & 1) * 2 + pr : qrank;
            const uint32_t xdst = cl_mapa(smem_u32(xbuf + (xslot * KC) * 32 + lane), xrank);
            const uint32_t xfull_dst = cl_mapa(smem_u32(x_full), xrank) + (kPair ? (qd & 1) * 8 : 0);
            static_assert(SPLIT == 1 || (NDIG == 8 && NCOL == 64), "two loads of 32 columns = 4 clusters each");
            for (uint32_t it = 0; it < my_tiles; ++it) {
                const uint32_t db = it & 1, dd = it % Cfg::DB, dpar = (it / Cfg::DB) & 1;
                TC_CLK(c0);
                TCW(3, it, &d_full[dd], dpar);
                __syncwarp();  // converge before the .sync.aligned tcgen05.ld
                TC_CLK(c1);
                if (qd == 0) TC_ACC(5, c1 - c0);
                tc_fence_after();
                if (qd == 0) TC_TR(4, it);
                long long d[KC];
                TC_CLK(ce0);
#pragma unroll
                for (uint32_t grp = 0; grp < 2; ++grp) {
                    uint32_t r32[32];
                    tc_ld16(lane_addr + kColD + dd * NCOL + 32 * grp, r32);
                    tc_ld16(lane_addr + kColD + dd * NCOL + 32 * grp + 16, r32 + 16);
                    tc_wait_ld();
                    if (grp == 1) {  // the accumulator set is free once the second group sits in registers
                        tc_fence_before();
                        warp_arrive_at(&d_free[dd], leader_rank, kPair && pe != 0);
                    }
#pragma unroll
                    for (uint32_t cc = 0; cc < 4; ++cc) {
                        float v[8];
#pragma unroll
                        for (uint32_t p = 0; p < 8; ++p) v[p] = __uint_as_float(r32[8 * cc + p]);
                        d[4 * grp + cc] = combine_digits<Cfg::BASE>(v);
                    }
                }
                TC_CLK(cx0);
                if (qd == 0) TC_ACC2(0, cx0 - ce0);
                cl_wait(&x_free[db * SPLIT + qd], ((it >> 1) & 1) ^ 1);
                TC_CLK(cx1);
                if (qd == 0) TC_ACC(7, cx1 - cx0);
                const uint32_t o = db * (SPLIT * KC * 32 * 8);
#pragma unroll
                for (uint32_t c = 0; c < KC; ++c)
                    cl_st_async_u64(xdst + o + c * 256, (unsigned long long)d[c], xfull_dst + db * (kPair ? 16 : 8));
                {
                    TC_CLK(cs1);
                    if (qd == 0) TC_ACC2(2, cs1 - cx1);
                }
                if (qd == 0) TC_TR(5, it);
            }
            if (qd == 0) TC_TG(4);
        }
    } else if (warp < kWEpi + 4 || (SPLIT > 1 && warp >= Cfg::WFin)) {
        // ---------------------------------------------------------------------- epilogue warps
        // SPLIT: the epilogue warps (one per lane quarter qd) send the partial dots of their 32
        // pixels (this CTA's quarter of the dimensions) to CTA qd of the cluster; the finalizer
        // warp receives the 4 partials of this CTA's own lane quarter (qrank) and labels them.
        // The exchange buffer is double-buffered by tile parity, [2][src][KC][32] i64.
        const bool finw = SPLIT > 1;  // split layout: only the finalizers get here; warp f takes the tiles of parity f
        // finalizer lane quarter: this CTA's own (rank) one; pairs: quarters 2 pr and 2 pr + 1 of
        // this CTA's tile, one per finalizer warp
        const uint32_t fq = finw ? warp - Cfg::WFin : 0u;
        const uint32_t qd = finw ? (kPair ? 2 * pr + fq : qrank) : (warp & 3);
        const uint32_t lane_addr = tbase + ((32 * qd) << 16);
        const bool fin = SPLIT == 1 || finw;  // this warp labels pixels
        long long* xbuf = reinterpret_cast<long long*>(smem + Smem::xb(nks));
        uint32_t xdst = 0, xfull_dst = 0;
        if (SPLIT > 1 && !finw) {
            xdst = cl_mapa(smem_u32(xbuf + (qrank * KC) * 32 + lane), qd);
            xfull_dst = cl_mapa(smem_u32(x_full), qd);
        }
        unsigned long long n2[KC];
#pragma unroll
        for (uint32_t c = 0; c < KC; ++c) n2[c] = c < K ? st.norm2[parity * K + c] : 0ull;
        const bool count_wraps = WR && fin && wraps_possible(n2, K < KC ? K : KC, 32 * W32);
        uint32_t changed = 0, nwrap = 0, ccount[KC];
#pragma unroll
        for (uint32_t c = 0; c < KC; ++c) ccount[c] = 0;
        for (uint32_t it = 0; it < my_tiles; ++it) {
            const uint32_t db = it & 1;  // exchange slot / finalizer
            if (finw && !kPair && db != fq) continue;  // (pairs: both warps take every tile, a quarter each)
            const uint32_t dd = it % Cfg::DB, dpar = (it / Cfg::DB) & 1;  // accumulator set, its phase
            const uint64_t px0 = tile_px0(it);
            const uint64_t px = px0 + 32 * qd + lane;
            const bool live = px < n;
            SG_CHECK(!(fin && live) || px < n);
            // round 1: every label is 0xFFFFFFFF ("no cluster") by definition; the buffer is not read
            // (and not cleared beforehand for tcgen05 plans)
            const uint32_t old = (fin && live) ? (round == 1 ? 0xFFFFFFFFu : labels[px]) : 0u;
            long long d[KC];
            if (!finw) {
                TC_CLK(c0);
                TCW(3, it, &d_full[dd], dpar);
                __syncwarp();  // converge before the .sync.aligned tcgen05.ld
                TC_CLK(c1);
                if (qd == 0) TC_ACC(5, c1 - c0);
                tc_fence_after();
                if (qd == 0) TC_TR(4, it);
                if constexpr (SPLIT > 1) {
                    // (the split layout's senders have their own branch above)
                } else {
                    uint32_t acc[NMW][NCOL];  // the MMA warps' accumulators of this tile
#pragma unroll
                    for (uint32_t mw = 0; mw < NMW; ++mw)
#pragma unroll
                        for (uint32_t c16 = 0; c16 < NCOL / 16; ++c16) {
                            tc_ld16(lane_addr + kColD + (NMW * dd + mw) * NCOL + 16 * c16, acc[mw] + 16 * c16);
                            if (NCOL % 16 != 0 && c16 == NCOL / 16 - 1)  // N % 16 == 8: the last 8 columns
                                tc_ld8(lane_addr + kColD + (NMW * dd + mw) * NCOL + 16 * (c16 + 1), acc[mw] + 16 * (c16 + 1));
                        }
                    tc_wait_ld();
                    tc_fence_before();
                    warp_arrive(&d_free[dd]);
                    // exact dots: column n = NDIG * c + p holds sum_i y_i d_p(z_c[i]) (an integer in
                    // f32, summed over the MMA warps' accumulators); dot_c = sum_p digit_dot_p * BASE^p
                    static_assert(NDIG == 8, "combine_digits takes 8 digit columns");
#pragma unroll
                    for (uint32_t c = 0; c < KC; ++c) {
                        float v[8];
#pragma unroll
                        for (uint32_t p = 0; p < 8; ++p) {
                            v[p] = __uint_as_float(acc[0][NDIG * c + p]);
#pragma unroll
                            for (uint32_t mw = 1; mw < NMW; ++mw) v[p] += __uint_as_float(acc[mw][NDIG * c + p]);
                        }
                        d[c] = combine_digits<Cfg::BASE>(v);
                    }
                }
            }
            if constexpr (SPLIT > 1) {
                // arm this tile's phase with the bytes the 4 senders deliver, then wait for them
                constexpr uint32_t kSrc = kPair ? 2 : SPLIT;  // CTAs sharing this tile
                uint64_t* xf = &x_full[kPair ? db * 2 + fq : db];
                if (lane == 0) mbar_expect_tx(xf, kSrc * 32 * KC * 8);
                TC_CLK(cw0);
                cl_wait(xf, (it >> 1) & 1);
                {
                    TC_CLK(cw1);
                    TC_ACC2(3, cw1 - cw0);
                }
                SG_CHECK(Smem::xb(nks) + (size_t(db + 1) * SPLIT * KC * 32) * 8 <= Smem::bars(nks));
                const long long* xb = xbuf + db * (SPLIT * KC * 32) + lane;
#pragma unroll
                for (uint32_t c = 0; c < KC; ++c) {
                    long long t = 0;
#pragma unroll
                    for (uint32_t src = 0; src < kSrc; ++src) t += xb[(((kPair ? fq * 2 : 0) + src) * KC + c) * 32];
                    d[c] = t;
                }
                __syncwarp();
                // slots free again: tell every sender of this quarter
                if (lane < kSrc)
                    cl_arrive(cl_mapa(smem_u32(&x_free[db * SPLIT + qd]), kPair ? 2 * lane + pe : lane));
            }
            // assign_labels (clusterer.cpp:146-158): first strictly closer centroid wins
            uint32_t best = 0;
            unsigned long long bd = (unsigned long long)d[0], bn = n2[0];
#pragma unroll
#pragma unroll
            for (uint32_t c = 1; c < KC; ++c)
                if (c < K && strictly_closer((unsigned long long)d[c], n2[c], bd, bn)) {
                    best = c;
                    bd = (unsigned long long)d[c];
                    bn = n2[c];
                }
            if (count_wraps && live) {  // copies: d and n2 themselves stay in registers
                long long dw[KC];
                unsigned long long nw[KC];
#pragma unroll
                for (uint32_t c = 0; c < KC; ++c) dw[c] = d[c], nw[c] = n2[c];
                nwrap += count_wraps_seq<KC>(dw, nw, K);
            }
            if (live) {
                labels[px] = best;
                if (labels_host) labels_host[px] = best;
                changed += old != best;
#pragma unroll
                for (uint32_t c = 0; c < KC; ++c) ccount[c] += best == c;
            }
            if (SPLIT == 1 && Cfg::FOLD) TCW(4, it, &list_free[db], ((it >> 1) & 1) ^ 1);
            // incremental re-bundling: pixels whose membership of a tracked cluster c >= 1 changed
            // (old = 0xFFFFFFFF before round 1); entering pixels add their HV, leaving pixels their
            // complement (flag). Global lists (one per tracked cluster, n entries apart) for
            // k_fold_list, or the tile's shared list for the fold warps (K == 2).
            // the warp's touched clusters >= 1 in one reduction: after the first rounds almost no
            // warp holds a changed pixel, and a changed one touches one or two clusters
            uint32_t touched = 0;
#if defined(SEGHDC_EXP_NOMMA) || defined(SEGHDC_EXP_NOLDS) || defined(SEGHDC_EXP_NOSTTM) || defined(SEGHDC_EXP_NOGRID) || \
    defined(SEGHDC_EXP_NOFLIST)
            if (false) {  // timing experiments: results are meaningless, keep the lists out of it
#else
            if (flist != nullptr && do_update && __ballot_sync(0xffffffffu, live && old != best)) {
                const uint32_t mine =
                    (live && old != best) ? ((1u << best) | (old < KC ? (1u << old) : 0u)) : 0u;
                touched = __reduce_or_sync(0xffffffffu, mine) & ~1u;
            }
            if (touched) {
#endif
                while (touched) {
                    const uint32_t c = __ffs(touched) - 1;
                    touched &= touched - 1;
                    if (c >= K) break;
                    const bool enter = live && best == c && old != c, leave = live && old == c && best != c;
                    const uint32_t m = __ballot_sync(0xffffffffu, enter || leave);
                    if (!m) continue;
                    uint32_t base = 0;
                    if (lane == 0) base = atomicAdd(flist_count + (c - 1), uint32_t(__popc(m)));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    SG_CHECK(!(enter || leave) || base + __popc(m & ((1u << lane) - 1)) < n);
                    if (enter || leave)
                        flist[size_t(c - 1) * n + base + __popc(m & ((1u << lane) - 1))] =
                            uint32_t(px) | (leave ? 0x80000000u : 0u);
                }
            }
            if constexpr (UPD) {
                const bool enter = live && best == 1 && old != 1, leave = live && old == 1 && best != 1;
                const bool take = folding && (enter || leave);
                // one compacted list per tile: the four quarters reserve their ranges with an
                // shared-memory atomic (the fold warps reset the count once they have read it)
                const uint32_t m = __ballot_sync(0xffffffffu, take);
                uint32_t base = 0;
                if (lane == 0 && m) base = atomicAdd(&s_listn[db], uint32_t(__popc(m)));
                base = __shfl_sync(0xffffffffu, base, 0);
                SG_CHECK(!take || base + __popc(m & ((1u << lane) - 1)) < kTP);
                if (take) s_list[db * kTP + base + __popc(m & ((1u << lane) - 1))] = (32 * qd + lane) | (leave ? 0x100u : 0u);
            }
            if (SPLIT == 1 && Cfg::FOLD) mbar_arrive(&list_ready[db]);
            if (qd == 0) TC_TR(5, it);
        }
        for (int o = 16; o; o >>= 1) {
            changed += __shfl_xor_sync(0xffffffffu, changed, o);
            nwrap += __shfl_xor_sync(0xffffffffu, nwrap, o);
#pragma unroll
            for (uint32_t c = 0; c < KC; ++c) ccount[c] += __shfl_xor_sync(0xffffffffu, ccount[c], o);
        }
        if (qd == 0) TC_TG(4);
        if (lane == 0) {
            if (nwrap) atomicAdd(st.wraps + (round - 1), (unsigned long long)nwrap);
            if (changed) atomicAdd(tail + K, changed);
#pragma unroll
            for (uint32_t c = 0; c < KC; ++c)
                if (c < K && ccount[c]) atomicAdd(tail + c, ccount[c]);
        }
    } else if (warp >= kWMma0 && warp < kWMma0 + NMW) {
        // ------------------------------------------------------------------------ MMA warps
        // warp m issues the chunks g = m, m+2, ... (global chunk parity) into accumulator
        // D[db][m] of their tile; the whole warp walks the loop (barrier waits are
        // warp-uniform), one elected lane issues inside tc_mma_chunk / tc_commit
        constexpr uint32_t idesc = idesc_mxf4(NCOL, kTP);
        const uint32_t m = warp - kWMma0;
        const uint32_t b0 = smem_u32(sB);
        TCW(5, 0, b_full, 0);
        __syncwarp();
        TC_TG(2);
        if constexpr (kPair) {
            // the leader issues M = 256 MMAs over both CTAs' A buffers and accumulators; its commits
            // arrive on the a_free / d_full barriers of both CTAs. The peer's warps report to the
            // leader's a_full / d_free barriers; its MMA warp only reports its B half.
            if (pe != 0) {
                if (lane == 0) cl_arrive(cl_mapa(smem_u32(b_peer), leader_rank));
            } else {
                cl_wait(b_peer, 0);
                __syncwarp();
                constexpr uint32_t idesc2 = idesc_mxf4(NCOL, 2 * kTP);
                constexpr uint32_t kStepsPP = kKS / Cfg::PARTS, kKBH = Cfg::KB / 2;  // B bytes per k-step and CTA
                const uint16_t mask = uint16_t(3u << leader_rank);
                for (uint32_t it = 0; it < my_tiles; ++it) {
                    const uint32_t db = it % Cfg::DB;
                    const uint32_t d_t = tbase + kColD + db * NCOL;
                    cl_wait(&d_free[db], ((it / Cfg::DB) & 1) ^ 1);
                    __syncwarp();
                    for (uint32_t ch = 0; ch < nch; ++ch) {
                        const uint32_t g = it * nch + ch, ab = g % kAB;
#pragma unroll
                        for (uint32_t pt = 0; pt < Cfg::PARTS; ++pt) {
                            cl_wait(&a_full[Cfg::PARTS * ab + pt], (g / kAB) & 1);
                            __syncwarp();
                            tc_fence_after();
                            if (tc_elect()) {
                                tc_mma_steps_pair<Cfg::KB, kStepsPP>(
                                    d_t, tbase + ab * 128 + pt * (128 / Cfg::PARTS),
                                    bdesc_at(b0 + (ch * kKS + pt * kStepsPP) * kKBH), idesc2, tbase + Cfg::ColSF,
                                    (ch || pt) ? 1u : 0u);
                                tc_commit_pair(&a_free[Cfg::PARTS * ab + pt], mask);
                            }
                            __syncwarp();
                        }
                    }
                    if (tc_elect()) tc_commit_pair(&d_full[db], mask);
                    __syncwarp();
                    if (m == 0) TC_TR(3, it);
                }
            }
        } else
        for (uint32_t it = 0; it < my_tiles; ++it) {
            const uint32_t db = it % Cfg::DB;  // accumulator set
            const uint32_t d_t = tbase + kColD + (NMW * db + m) * NCOL;
            TC_CLK(cf0);
            TCW(6, it, &d_free[db], ((it / Cfg::DB) & 1) ^ 1);
            __syncwarp();
            {
                TC_CLK(cf1);
                if (m == 0) TC_ACC(6, cf1 - cf0);
            }
            const uint32_t first = (NMW + m - (it * nch) % NMW) % NMW;
            for (uint32_t ch = first; ch < nch; ch += NMW) {  // chunks with g % NMW == m
                const uint32_t g = it * nch + ch, ab = g % kAB;
                TC_CLK(c0);
                // a_full[2 ab + m] carries chunks g = x + lcm(NMW, kAB) t
                constexpr uint32_t kLcm = (kAB % NMW == 0) ? kAB : NMW * kAB;
                if constexpr (Cfg::HALVES) {  // each half chunk as soon as its unpack warps are done
                    static_assert(!Cfg::HALVES || NMW == 1, "half-chunk hand-offs assume one MMA warp");
#pragma unroll
                    for (uint32_t pt = 0; pt < Cfg::PARTS; ++pt) {
                        TCW_AFULL(7, g, &a_full[Cfg::PARTS * ab + pt], (g / kLcm) & 1);
                        __syncwarp();
                        tc_fence_after();
#ifndef SEGHDC_EXP_NOMMA
                        constexpr uint32_t kStepsPP = kKS / Cfg::PARTS;
                        const uint32_t acc = (ch >= NMW || pt) ? 1u : 0u;
                        const uint64_t bd = bdesc_at(b0 + (ch * kKS + pt * kStepsPP) * Cfg::KB);
#ifdef SEGHDC_OLD_ISSUE
                        if constexpr (Cfg::PARTS == 4)
                            tc_mma_quarter<Cfg::KB>(d_t, tbase + ab * 128 + pt * 32, bd, idesc, tbase + Cfg::ColSF, acc);
                        else
                            tc_mma_half<Cfg::KB>(d_t, tbase + ab * 128 + pt * 64, bd, idesc, tbase + Cfg::ColSF, acc);
#else
                        if (tc_elect()) {
                            tc_mma_steps<Cfg::KB, kStepsPP>(d_t, tbase + ab * 128 + pt * (128 / Cfg::PARTS), bd, idesc,
                                                            tbase + Cfg::ColSF, acc);
                            tc_commit_one(&a_free[Cfg::PARTS * ab + pt]);
                        }
                        __syncwarp();
                        continue;
#endif
#endif
                        tc_commit(&a_free[Cfg::PARTS * ab + pt]);
                    }
                    continue;
                }
                TCW_AFULL(7, g, &a_full[2 * ab + m], (g / kLcm) & 1);
                __syncwarp();  // converge before elect.sync / tcgen05.mma
                TC_CLK(c1);
                if (m == 0) TC_ACC(2, c1 - c0);
                tc_fence_after();
                PRG(12 * 100000 + g);
#if defined(SEGHDC_EXP_NOMMA)  // timing experiment only: the pipeline without the tensor-core work
                tc_commit(&a_free[ab]);
#elif defined(SEGHDC_OLD_ISSUE)
                tc_mma_chunk<Cfg::KB>(d_t, tbase + ab * 128, bdesc_at(b0 + ch * kKS * Cfg::KB), idesc,
                                      tbase + Cfg::ColSF, ch >= NMW);
                tc_commit(&a_free[ab]);
#else
                if (tc_elect()) {
                    tc_mma_steps<Cfg::KB, kKS>(d_t, tbase + ab * 128, bdesc_at(b0 + ch * kKS * Cfg::KB), idesc,
                                               tbase + Cfg::ColSF, ch >= NMW ? 1u : 0u);
                    tc_commit_one(&a_free[ab]);
                }
                __syncwarp();
#endif
                PRG(13 * 100000 + g);
                {
                    TC_CLK(c2);
                    if (m == 0) TC_ACC(3, c2 - c1);
                }
            }
            tc_commit(&d_full[db]);
            if (m == 0) TC_TR(3, it);
        }
        __syncwarp();
    } else if (warp == kWProd) {
        // ----------------------------------------------------------------------- producer warp
        if (lane == 0) {
            // this CTA's slice (SPLIT) or the whole image; pairs: half of the digit columns of the
            // pair's dimension half, contiguous in the pair layout [column half][k-step][KB / 2]
            const uint32_t bbytes = nch * kKS * (kPair ? Cfg::KB / 2 : Cfg::KB);
            const size_t boff = kPair ? size_t(pe) * (size_t(nch_all) * kKS * (Cfg::KB / 2)) + size_t(ch0) * kKS * (Cfg::KB / 2)
                                      : size_t(ch0) * kKS * Cfg::KB;
            // the grid streams through L2 with evict_first (measured: evict_last on the tiles read
            // last slows every round; evict_first takes round 1 from 98 to 82 us at C1)
            const uint64_t pol_stream = policy_evict_first();
            mbar_expect_tx(b_full, bbytes);
            bulk_g2s(sB, bimg + boff, bbytes, b_full);
            uint32_t g = 0;
            const uint32_t nchunks = kLdg ? 0u : my_tiles * nch;  // kLdg: the unpack warps load A
            for (uint32_t q = 0; q < pf && q < nchunks; ++q)
                tma_prefetch_2d(&tmap, int((ch0 + q % nch) * kCW), int(tile_px0(q / nch)));
            for (uint32_t it = 0; it < (kLdg ? 0u : my_tiles); ++it) {
                const int y = int(tile_px0(it));
                for (uint32_t ch = 0; ch < nch; ++ch, ++g) {
                    const uint32_t s = g % kStages;
                    if (pf && g + pf < nchunks) {  // chunk g + pf into L2 now
                        const uint32_t gp = g + pf;
                        tma_prefetch_2d(&tmap, int((ch0 + gp % nch) * kCW), int(tile_px0(gp / nch)));
                    }
                    TC_CLK(c0);
                    TCW(8, g, &slot_free[s], ((g / kStages) & 1) ^ 1);
                    TC_CLK(c1);
                    TC_ACC(4, c1 - c0);
                    if (ch == 0) TC_TR(0, it);
#ifdef SEGHDC_EXP_NOGRID  // timing experiment: the slot is "full" without any data
                    (void)y;
                    mbar_arrive(&slot_full[s]);
#else
                    mbar_expect_tx(&slot_full[s], kChunkBytes);
                    tma_load_2d_hint(ring + size_t(s) * kChunkBytes, &tmap, int((ch0 + ch) * kCW), y, &slot_full[s],
                                     pol_stream);
#endif
                }
            }
        }
        __syncwarp();
    }

    // ---------------------------------------------------------------------------- fold warps
    BitCounter<UPD ? H : 1> cnt[CPTMAX];
    const int fw = (SPLIT == 1 && Cfg::FOLD) ? fold_index(warp) : -1;
    const uint32_t rt = uint32_t(fw) * 32 + lane;
    const uint32_t cpt = (W32 + NRT - 1) / NRT;
    uint32_t nleave = 0;  // leaving pixels folded by this CTA (same count in every fold thread)
    if (fw >= 0) {
        if constexpr (UPD)
#pragma unroll
            for (int c = 0; c < CPTMAX; ++c) cnt[c].reset();
        for (uint32_t it = 0; it < my_tiles; ++it) {
            const uint32_t db = it & 1;
            TCW(9, it, &list_ready[db], (it >> 1) & 1);
            if (fw == 0) TC_TR(6, it);
            if constexpr (UPD) {
                if (folding) {
                    const uint64_t px0 = tile_px0(it);
                    const uint32_t* G = grid + px0 * S32;
                    const uint32_t M = s_listn[db];
                    const uint32_t* L = s_list + db * kTP;
                    __syncwarp();
                    asm volatile("bar.sync 1, %0;" ::"n"(kNRW * 32) : "memory");  // all fold threads read M
                    if (rt == 0) s_listn[db] = 0;
                    // batches of 8 listed rows: the 8 x CPTMAX loads of a batch are issued together
                    // (columns clamped to W32 - 1: the extra counters are never flushed)
                    uint32_t cw[CPTMAX];
#pragma unroll
                    for (int c = 0; c < CPTMAX; ++c) cw[c] = min(rt + c * NRT, W32 - 1);
                    for (uint32_t e = 0; e < M; e += 8) {
                        uint32_t row[8], neg[8], val[8];
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            const uint32_t en = (e + v < M) ? L[e + v] : 0u;
                            row[v] = en & 0xFFu;
                            neg[v] = (en >> 8) ? 0xFFFFFFFFu : 0u;
                            val[v] = (e + v < M) ? 0xFFFFFFFFu : 0u;
                            nleave += en >> 8;
                        }
                        uint32_t x[CPTMAX][8];
#pragma unroll
                        for (int c = 0; c < CPTMAX; ++c)
#pragma unroll
                            for (int v = 0; v < 8; ++v) x[c][v] = __ldg(G + size_t(row[v]) * S32 + cw[c]);
#pragma unroll
                        for (int c = 0; c < CPTMAX; ++c) {
#pragma unroll
                            for (int v = 0; v < 8; ++v) x[c][v] = (x[c][v] ^ neg[v]) & val[v];
                            cnt[c].add8(x[c]);
                        }
                    }
                }
            }
            if (fw == 0) TC_TR(7, it);
            mbar_arrive(&list_free[db]);
        }
    }
    if (fw == 0) TC_TG(5);
    // all roles done: the ring becomes the counters' transpose scratch; free TMEM
    tc_fence_before();
    __syncthreads();
    if (SPLIT > 1) cl_sync();  // no CTA leaves while a peer may still write its shared memory
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the finish may launch
    if (warp == 0) TC_TG(6);
    if (folding) {  // CTA-uniform: counters -> planes in the ring -> whole-CTA expansion + atomics
        uint32_t* planes = reinterpret_cast<uint32_t*>(ring);
        bool nz = false;
        if (fw >= 0) {
#pragma unroll
            for (int c = 0; c < CPTMAX; ++c) {
                const uint32_t colw = rt + c * NRT;
                if (uint32_t(c) < cpt && colw < W32) {
                    cnt[c].planes(planes + colw, W32);
                    nz |= cnt[c].any();
                }
            }
            if (rt == 0) s_misc[1] = nleave;
            nz |= nleave != 0;
        }
        if (__syncthreads_or(nz)) flush_planes_cta<UPD ? H : 1>(planes, W32, s_misc[1], xchg + Dp);
    }
    if (fw == 0) TC_TG(7);
    if (warp == kWMma0) {
        tc_fence_after();
        if constexpr (kPair) {
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
        } else {
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
        }
#ifdef SEGHDC_TRACE
        if (lane == 0 && blockIdx.x < 148) {  // slot 61: [0] stamp before, [1] after dealloc, [2] stamp after
            unsigned long long t_;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
            g_trace_tc[(size_t(blockIdx.x) * 64 + 61) * 8 + 1] = t_;
        }
#endif
    }
}

// B image: for k-step ks the kN x 64 e2m1 of B (kKB bytes) in the canonical K-major no-swizzle
// layout: 8-row group g at +256g, core matrix cm (k-slots 32cm..32cm+31) at +128cm, row at +16r,
// k-slot pair (2b, 2b+1) in byte b (low nibble = even slot). k-slot k is nibble j = k % 8 of A
// column col = k / 8 = 4h + c, i.e. class c of HV word 2ks + h (header): c = 0 / 2 carry bits
// 4j+1 / 4j as 1.0, c = 1 / 3 carry bits 4j+2 / 4j+3 as 2.0. Row n = kP8 * cluster + p holds
// digit p of the centroid entry (weight 1) or half of it (weight 2), so every product is bit * d.
// balanced base 8 (digits [-4, 3]) or base 9 (digits [-4, 4])
// (BASE is a compile-time constant: the divisions become multiplies)
template <uint32_t base>
__device__ __forceinline__ int digit_b(long long z, uint32_t p) {
    for (uint32_t q = 0;; ++q) {
        int r = int(z % base);
        if (r >= int(base) - 4) r -= int(base);
        if (q == p) return r;
        z = (z - r) / base;
    }
}
template <uint32_t base>
__device__ __forceinline__ uint32_t b_nibble(const uint32_t* Z, uint32_t K, uint32_t D, uint32_t ks, uint32_t n,
                                             uint32_t k, uint32_t ndig) {
    const uint32_t col = k >> 3, j = k & 7, h = col >> 2, c = col & 3;
    const uint32_t dim = 32 * (2 * ks + h) + 4 * j + (c == 0 ? 1u : c == 1 ? 2u : c == 2 ? 0u : 3u);
    const uint32_t cl = n / ndig, p = n % ndig;
    if (cl >= K || dim >= D) return 0;
    const int d = digit_b<base>((long long)Z[size_t(cl) * D + dim], p);
    const uint32_t a = uint32_t(d < 0 ? -d : d);
    // weight 1: |d| in 0..4 -> e2m1 {0, 1, 2, 3, 4}; weight 2: |d|/2 in {0, .5, 1, 1.5, 2}
    const uint32_t code = (c & 1) ? a : (a == 0 ? 0u : a == 1 ? 2u : a == 2 ? 4u : a == 3 ? 5u : 6u);
    return code | (d < 0 ? 8u : 0u);
}
// pair: the CTA-pair layout [column half][k-step][kb / 2] (each CTA of a pair copies one contiguous
// half of the digit columns of its k-steps) instead of [k-step][kb]
template <uint32_t BASE>
__global__ void k_build_bimg(const uint32_t* __restrict__ Z, uint32_t K, uint32_t D, uint32_t nks, uint32_t kb,
                             uint32_t ndig, uint8_t* __restrict__ bimg, const void* state, uint32_t pair,
                             uint32_t* __restrict__ clear, uint32_t clear_n) {
    if (state && StateView::at(const_cast<void*>(state), K).hdr->done) return;
    // init only: the exchange buffer the previous kernel (k_finish) consumed is zeroed here, so
    // round 1 needs no memset of its own
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < clear_n; i += gridDim.x * blockDim.x) clear[i] = 0;
    const uint32_t total = nks * kb, half = kb / 2;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t ks = pair ? (i / half) % nks : i / kb;
        const uint32_t rem = pair ? (i / (nks * half)) * half + i % half : i % kb;
        const uint32_t grp = rem / 256, r2 = rem % 256, cm = r2 / 128, row = (r2 % 128) / 16, b = r2 % 16;
        const uint32_t n = grp * 8 + row, k = 32 * cm + 2 * b;
        bimg[i] = uint8_t(b_nibble<BASE>(Z, K, D, ks, n, k, ndig) | (b_nibble<BASE>(Z, K, D, ks, n, k + 1, ndig) << 4));
    }
}

// Per-round finish of the incremental K == 2 schedule, fused (replaces the exchange memset,
// k_prep_finish, k_finish and k_build_bimg of a round): one warp per HV word.
//   early stop (clusterer.cpp:213); S1 = running sums + delta (all-reduced xchg row 1);
//   Z1 = S1, Z0 = colsum - S1, empty clusters keep their centroid (clusterer.cpp:184-186);
//   norm2 of the new set (hypervector.cpp:123-127) into parity np, norm2[p] zeroed for the
//   next finish; the word's 16 x 16 B-image bytes (digits via the offset trick: for
//   O = 4 (8^kP8 - 1) / 7, digit p of z is ((z + O) >> 3p & 7) - 4); the word's exchange
//   sums are cleared after use, and the last block clears the counts / changed tail.
constexpr uint32_t kFinWarps = 2;  // HV words (warps) per k_finish_tc block: ~one block per SM at C1
__global__ void __launch_bounds__(kFinWarps * 32) k_finish_tc(uint32_t D, uint32_t W32, uint32_t Dp,
                                                            int32_t* __restrict__ xchg,
                                                            const int32_t* __restrict__ colsum,
                                                            uint32_t* __restrict__ Z, uint32_t* __restrict__ run1,
                                                            uint8_t* __restrict__ bimg, void* state, uint32_t round,
                                                            int early_stop, uint32_t* __restrict__ ticket) {
    constexpr uint32_t K = 2;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched early (PDL) behind the round kernel
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    StateView st = StateView::at(state, K);
    const uint32_t p = round & 1, np = p ^ 1;
    uint32_t* tail = reinterpret_cast<uint32_t*>(xchg) + size_t(K) * Dp;  // [counts[2] | changed]
    if (st.hdr->done) return;
    const uint32_t cnt0 = tail[0], cnt1 = tail[1];
    if (early_stop && round > 1 && tail[K] == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st.hdr->done = 1;
        return;
    }
    __shared__ unsigned long long s_n2[kFinWarps][2];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, word = blockIdx.x * kFinWarps + wib;
    unsigned long long n0 = 0, n1 = 0;
    if (word < W32) {
        const uint32_t i = 32 * word + lane;
        const bool in = i < D;
        const uint32_t s1 = run1[size_t(p) * Dp + i] + uint32_t(xchg[Dp + i]);
        run1[size_t(np) * Dp + i] = s1;
        xchg[i] = 0;
        xchg[Dp + i] = 0;
        uint32_t z0 = cnt0 ? uint32_t(colsum[i]) - s1 : (in ? Z[i] : 0u);
        uint32_t z1 = cnt1 ? s1 : (in ? Z[D + i] : 0u);
        if (!in) z0 = z1 = 0;
        if (in) {
            Z[i] = z0;
            Z[D + i] = z1;
        }
        n0 = (unsigned long long)z0 * z0;
        n1 = (unsigned long long)z1 * z1;
        for (int o = 16; o; o >>= 1) {
            n0 += __shfl_xor_sync(0xffffffffu, n0, o);
            n1 += __shfl_xor_sync(0xffffffffu, n1, o);
        }
        // B image bytes of this word: word h = word & 1 of k-step word >> 1 is core matrix h;
        // lane = (row n, half): row n = kP8 * cluster + digit, bytes 8 * half .. + 7. Digit pd of
        // z is u - 4 with u = ((z + O) >> 3 pd) & 7, O = 4 (8^kP8 - 1) / 7; its e2m1 code for a
        // weight-1 (d) or weight-2 (d / 2) nibble class comes from a packed 8-entry table by u.
        constexpr uint32_t kOff = 4u * ((1u << (3 * kP8)) - 1) / 7u;
        constexpr uint32_t kLut1 = 0x5420ACDEu, kLut2 = 0x32109ABCu;  // u = 0..7 -> code
        const uint32_t zb0 = z0 + kOff, zb1 = z1 + kOff;
        const uint32_t n = lane >> 1, hb = lane & 1, cl = n / kP8, sh = 3 * (n % kP8);
        uint64_t v = 0;
#pragma unroll
        for (uint32_t q = 0; q < 16; ++q) {  // nibble q of the lane's 8 bytes: k = 16 hb + q
            const uint32_t k = 16 * hb + q, c = k >> 3, j = k & 7;
            const uint32_t src = 4 * j + (c == 0 ? 1u : c == 1 ? 2u : c == 2 ? 0u : 3u);
            const uint32_t za = __shfl_sync(0xffffffffu, zb0, src), zb = __shfl_sync(0xffffffffu, zb1, src);
            const uint32_t u = ((cl ? zb : za) >> sh) & 7u;
            v |= uint64_t((((c & 1) ? kLut2 : kLut1) >> (4 * u)) & 0xFu) << (4 * q);
        }
        *reinterpret_cast<uint64_t*>(bimg + size_t(word >> 1) * kKB + (n >> 3) * 256 + (word & 1) * 128 +
                                     (n & 7) * 16 + 8 * hb) = v;
    }
    if (lane == 0) {
        s_n2[wib][0] = n0;
        s_n2[wib][1] = n1;
    }
    if (blockIdx.x == 0 && threadIdx.x < K) {
        st.norm2[p * K + threadIdx.x] = 0;
        st.cur[np * K + threadIdx.x] = threadIdx.x ? cnt1 : cnt0;
    }
    __syncthreads();
    if (threadIdx.x < K) {  // one atomic per block and cluster
        unsigned long long t = 0;
        for (uint32_t w2 = 0; w2 < kFinWarps; ++w2) t += s_n2[w2][threadIdx.x];
        atomicAdd(st.norm2 + np * K + threadIdx.x, t);
    }
    // the last block to finish clears the counts / changed tail for the next round
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
            tail[0] = tail[1] = tail[K] = 0;
            *ticket = 0;
        }
    }
}

void launch_finish_tc(uint32_t D, uint32_t W32, uint32_t Dp, int32_t* xchg, const int32_t* colsum, uint32_t* Z,
                      uint32_t* run1, uint8_t* bimg, void* state, uint32_t round, int early_stop, uint32_t* ticket,
                      cudaStream_t s) {
    launch_pdl(k_finish_tc, dim3((W32 + kFinWarps - 1) / kFinWarps), dim3(kFinWarps * 32), 0, s, D, W32, Dp, xchg,
               colsum, Z, run1, bimg, state, round, early_stop, ticket);
}

// Fold of a global list of changed pixels (bit 31: leaving) into xchg row 1, as signed deltas:
// CTA = 2 row groups (1 when W32 > 384) x ceil(W32 / 32) warps, thread = word column; each CTA takes a contiguous
// slice of the list, the groups interleave its rows (16 loads in flight per thread), their
// counts meet in shared memory (u32[32][W32], bit-major: conflict-free both ways) and leave
// with one global atomic per entry.
template <int H>
__global__ void __launch_bounds__(768) k_fold_list(const uint32_t* __restrict__ list, const uint32_t* __restrict__ count,
                                                   uint64_t n, const uint32_t* __restrict__ grid, uint32_t S32,
                                                   uint32_t W32, uint32_t* __restrict__ dst, uint32_t dst_stride) {
    extern __shared__ uint32_t s_val[];  // [32][W32]
    const uint32_t nw = (W32 + 31) / 32, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t grp = warp / nw, col = (warp % nw) * 32 + lane, colc = min(col, W32 - 1);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched early (PDL) behind the round kernel
    // blockIdx.y = tracked cluster c - 1: its list is n entries after the previous one
    list += size_t(blockIdx.y) * n;
    dst += size_t(blockIdx.y) * dst_stride;
    const uint32_t M = count[blockIdx.y];
    SG_CHECK(M <= n);
    // at least kMinRows rows per CTA: a short list (late rounds) occupies a few CTAs, whose
    // flush (one atomic per entry of D) dominates, instead of all of them
#ifndef SEGHDC_FOLD_MINROWS
#define SEGHDC_FOLD_MINROWS 32  // 16 / 32 / 64 / 128 / 256 / 512 measured: C0 step 296.6 / 296.0 / 298.8 / 305.5 / 321 / 350 us
#endif
    constexpr uint32_t kMinRows = SEGHDC_FOLD_MINROWS;
    const uint32_t per = max(kMinRows, (M + gridDim.x - 1) / gridDim.x);
    const uint32_t r0 = min(M, blockIdx.x * per), r1 = min(M, r0 + per);
    if (r0 >= r1) return;
    for (uint32_t e = threadIdx.x; e < 32 * W32; e += blockDim.x) s_val[e] = 0;
    BitCounter<H> cnt;
    cnt.reset();
    uint32_t nleave = 0;
    const uint32_t ng = blockDim.x / (32 * nw);  // row groups: 2, or 1 when W32 > 384
    for (uint32_t e = r0 + grp; e < r1; e += 16 * ng) {  // 16 rows of this group: e, e + ng, ...
        uint32_t x[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
            const uint32_t i = e + ng * v;
            const uint32_t en = i < r1 ? list[i] : 0u;
            SG_CHECK(i >= r1 || (en & 0x7FFFFFFFu) < n);
            const uint32_t neg = (en >> 31) ? 0xFFFFFFFFu : 0u;
            const uint32_t word = i < r1 ? __ldg(grid + size_t(en & 0x7FFFFFFFu) * S32 + colc) : 0u;
            x[v] = (word ^ neg) & (i < r1 ? 0xFFFFFFFFu : 0u);
            nleave += (i < r1) ? (en >> 31) : 0u;
        }
        cnt.add16(x);
    }
    __syncthreads();
    if (col < W32)
        for (int b = 0; b < 32; ++b) {
            const uint32_t v = cnt.value(b) - nleave;
            if (v) atomicAdd(&s_val[b * W32 + col], v);
        }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < 32 * W32; e += blockDim.x) {
        const uint32_t v = s_val[(e & 31) * W32 + (e >> 5)];
        if (v) atomicAdd(dst + e, v);
    }
}

void launch_fold_list(const uint32_t* list, const uint32_t* count, uint64_t max_rows, uint32_t nlists,
                      const uint32_t* grid, uint32_t S32, uint32_t W32, int32_t* dst, uint32_t dst_stride,
                      uint32_t sms, cudaStream_t s) {
    static const char* fc_env = getenv("SEGHDC_FOLD_CTAS");  // experiment switch: CTAs per list
    const dim3 ctas(fc_env && atoi(fc_env) > 0 ? uint32_t(atoi(fc_env)) : sms, nlists);
    const uint32_t ng = W32 > 384 ? 1 : 2;  // row groups per CTA (768 threads at most)
    const uint32_t threads = ng * 32 * ((W32 + 31) / 32);
    const size_t smem = size_t(32) * W32 * 4;
    const uint64_t per_group = (max_rows + ng * ctas.x - 1) / (ng * ctas.x) + 64;  // inputs per counter
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    if (per_group <= BitCounter<8>::capacity()) {
        ensure_dynamic_smem((const void*)k_fold_list<8>, smem);
        launch_pdl(k_fold_list<8>, ctas, dim3(threads), smem, s, list, count, max_rows, grid, S32, W32, d,
                   dst_stride);
    } else if (per_group <= BitCounter<12>::capacity()) {
        ensure_dynamic_smem((const void*)k_fold_list<12>, smem);
        launch_pdl(k_fold_list<12>, ctas, dim3(threads), smem, s, list, count, max_rows, grid, S32, W32, d,
                   dst_stride);
    } else {
        ensure_dynamic_smem((const void*)k_fold_list<20>, smem);
        launch_pdl(k_fold_list<20>, ctas, dim3(threads), smem, s, list, count, max_rows, grid, S32, W32, d,
                   dst_stride);
    }
}

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

#ifdef SEGHDC_TRACE
__global__ void k_tc_stamp(int ev) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_trace_tc[(size_t(blockIdx.x) * 64 + 61) * 8 + ev] = t_;
}
#endif
template <bool UPD, int H, uint32_t NCOL, uint32_t SPLIT = 1, bool WR = false>
cudaError_t launch_tc_t(const RoundArgs& a, cudaStream_t s) {
    using Cfg = TcCfg<NCOL, SPLIT>;
    auto kern = k_round_tc<UPD, H, NCOL, SPLIT, WR>;
    const uint32_t nch = tc_chunks(a.W32);
    const uint32_t nks = SPLIT > 1 ? (nch + SPLIT - 1) / SPLIT * kKS : a.nks;  // B k-steps resident per CTA
    const size_t smem = TcSmem<NCOL, SPLIT>::total(nks);
    cudaError_t e = ensure_dynamic_smem((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    const CUtensorMap& tm = *reinterpret_cast<const CUtensorMap*>(a.tmap);
    uint32_t* xchg = reinterpret_cast<uint32_t*>(a.xchg);
    if (SPLIT == 1)
        return launch_pdl(kern, dim3(a.ctas), dim3(Cfg::Warps * 32), smem, s, tm, a.grid, a.n, a.S32, a.W32, a.K,
                          a.bimg, nks, a.labels, a.state, a.round, a.do_update, xchg, a.Dp, a.flist, a.flist_count,
                          a.serpentine, a.pf, a.labels_host_slot);
    // clusters of SPLIT CTAs (one per SM): as many as fit at once, at most one per tile
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(Cfg::Warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = SPLIT;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    static int max_clusters[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && max_clusters[dev] == 0) {
        cfg.gridDim = dim3(SPLIT * 148);
        int mc = 0;
        if (cudaOccupancyMaxActiveClusters(&mc, (const void*)kern, &cfg) != cudaSuccess || mc <= 0) {
            cudaGetLastError();
            mc = 148 / SPLIT;
        }
        max_clusters[dev] = mc;
    }
    const uint64_t ntiles = (a.n + kTP - 1) / kTP;
    const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(dev < 64 ? max_clusters[dev] : 148 / SPLIT,
                                                                  a.ctas / SPLIT));
    const uint64_t per = (ntiles + cap - 1) / cap;  // balanced waves, as for the one-CTA layouts
    const uint64_t ncl = std::max<uint64_t>(1, (ntiles + per - 1) / per);
    cfg.gridDim = dim3(uint32_t(ncl * SPLIT));
    return cudaLaunchKernelEx(&cfg, kern, tm, a.grid, a.n, a.S32, a.W32, a.K, a.bimg, nks, a.labels, a.state,
                              a.round, a.do_update, xchg, a.Dp, a.flist, a.flist_count, a.serpentine, a.pf,
                              a.labels_host_slot);
}
}  // namespace

// Layout of the tcgen05 kernel for (K, W32): N = 16 digit columns (K <= 2) or 32 (K <= 4) with
// the whole B image resident in one CTA; N = 64 (K <= 8, 8 base-9 digits) in one CTA for short
// HVs, split over a cluster of 4 CTAs otherwise; 0: no tcgen05 layout (IMMA kernels).
constexpr size_t kSmemOptin = 232448;  // B200: 227 KB of dynamic shared memory per CTA
static uint32_t tc_nchunks(uint32_t W32) { return tc_chunks(W32); }
uint32_t tc_split(uint32_t K, uint32_t W32) {
    const uint32_t nch = tc_nchunks(W32), nks = nch * kKS;
    if (K < 1 || K > 8) return 0;
    if (K <= 2 && W32 <= 3 * kNRW * 32 && TcSmem<16>::total(nks) <= kSmemOptin) return 1;
    if (K <= 4 && TcSmem<32>::total(nks) <= kSmemOptin) return 1;
    if (K > 4 && TcSmem<64>::total(nks) <= kSmemOptin) return 1;
    if (nch >= 4 && TcSmem<64, 4>::total((nch + 3) / 4 * kKS) <= kSmemOptin) return 4;
    return 0;
}
uint32_t tc_ncol(uint32_t K, uint32_t W32) {
    const uint32_t nch = tc_nchunks(W32), nks = nch * kKS;
    if (K < 1 || K > 8) return 0;
    if (K <= 2 && W32 <= 3 * kNRW * 32 && TcSmem<16>::total(nks) <= kSmemOptin) return 16;
    if (K <= 4 && TcSmem<32>::total(nks) <= kSmemOptin) return 32;
    return tc_split(K, W32) ? 64 : 0;
}
bool tc_supported(uint32_t K, uint32_t W32) { return tc_ncol(K, W32) != 0; }
static uint32_t tc_ndig(uint32_t ncol) { return ncol == 64 ? TcCfg<64, 4>::NDIG : kP8; }
static uint32_t tc_base(uint32_t ncol) { return ncol == 64 ? TcCfg<64, 4>::BASE : 8u; }
// largest centroid entry the layout's balanced digits represent: 3 (8^ndig - 1) / 7 in base 8,
// 4 (9^ndig - 1) / 8 in base 9
uint64_t tc_max_value(uint32_t K, uint32_t W32) {
    const uint32_t nc = tc_ncol(K, W32), nd = tc_ndig(nc), b = tc_base(nc);
    uint64_t pw = 1;
    for (uint32_t q = 0; q < nd; ++q) pw *= b;
    return (b / 2 - (b % 2 == 0 ? 1 : 0)) * (pw - 1) / (b - 1);
}
uint32_t tc_ksteps(uint32_t W32) { return tc_nchunks(W32) * kKS; }
size_t tc_smem_bytes(uint32_t K, uint32_t W32) {
    const uint32_t nc = tc_ncol(K, W32), nch = tc_nchunks(W32);
    return nc == 16 ? TcSmem<16>::total(tc_ksteps(W32))
         : nc == 32 ? TcSmem<32>::total(tc_ksteps(W32))
         : nc == 64 ? (tc_split(K, W32) == 1 ? TcSmem<64>::total(tc_ksteps(W32))
                                              : TcSmem<64, 4>::total((nch + 3) / 4 * kKS))
                    : ~size_t(0);
}
size_t tc_bimg_bytes(uint32_t K, uint32_t W32) { return size_t(tc_ksteps(W32)) * tc_ncol(K, W32) * 32; }
uint32_t tc_tile_pixels() { return kTP; }

bool tc_make_grid_map(void* map, const uint32_t* grid, uint64_t rows, uint32_t S32) {
    EncodeFn fn = encode_fn();
    if (!fn || rows == 0) return false;
    const cuuint64_t dims[2] = {S32, rows};
    const cuuint64_t strides[1] = {cuuint64_t(S32) * 4};
    const cuuint32_t box[2] = {kCW, kTP};
    const cuuint32_t estr[2] = {1, 1};
    return fn(reinterpret_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
              const_cast<uint32_t*>(grid), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_build_bimg(const uint32_t* Z, uint32_t K, uint32_t D, uint32_t W32, uint8_t* bimg, const void* state,
                       cudaStream_t s, uint32_t* clear, uint32_t clear_n) {
    const uint32_t nc = tc_ncol(K, W32), nks = tc_ksteps(W32), kb = nc * 32;
    const uint32_t total = nks * kb;
    const uint32_t pair = (nc == 64 && tc_split(K, W32) > 1 && TcCfg<64, 4>::PAIR) ? 1u : 0u;
    if (tc_base(nc) == 9)
        k_build_bimg<9><<<(total + 255) / 256, 256, 0, s>>>(Z, K, D, nks, kb, tc_ndig(nc), bimg, state, pair, clear, clear_n);
    else
        k_build_bimg<8><<<(total + 255) / 256, 256, 0, s>>>(Z, K, D, nks, kb, tc_ndig(nc), bimg, state, pair, clear, clear_n);
}

#ifdef SEGHDC_HANGDBG
void* setup_hang() {
    unsigned int* h = nullptr;
    cudaHostAlloc(&h, 65536, cudaHostAllocMapped);
    memset(h, 0, 65536);
    unsigned int* d = nullptr;
    cudaHostGetDevicePointer(&d, h, 0);
    cudaMemcpyToSymbol(g_hang, &d, sizeof(d));
    return h;
}
#endif

static cudaError_t launch_round_tc_body(const RoundArgs& a, cudaStream_t s) {
    const uint64_t per_cta = ((a.n + a.ctas - 1) / a.ctas + kTP - 1) / kTP * kTP;
    if (a.wraps) return launch_tc_t<true, 20, 16, 1, true>(a, s);  // only images of millions of pixels
    if (per_cta <= BitCounter<8>::capacity()) return launch_tc_t<true, 8, 16>(a, s);
    if (per_cta <= BitCounter<12>::capacity()) return launch_tc_t<true, 12, 16>(a, s);
    return launch_tc_t<true, 20, 16>(a, s);
}
static cudaError_t launch_round_tc_sel(const RoundArgs& a, cudaStream_t s) {
    switch (tc_ncol(a.K, a.W32)) {
        case 16:
            if (a.K == 2) return launch_round_tc_body(a, s);
            return a.wraps ? launch_tc_t<false, 1, 16, 1, true>(a, s) : launch_tc_t<false, 1, 16>(a, s);
        case 32: return a.wraps ? launch_tc_t<false, 1, 32, 1, true>(a, s) : launch_tc_t<false, 1, 32>(a, s);
        case 64:
            if (tc_split(a.K, a.W32) == 1)
                return a.wraps ? launch_tc_t<false, 1, 64, 1, true>(a, s) : launch_tc_t<false, 1, 64, 1>(a, s);
            return a.wraps ? launch_tc_t<false, 1, 64, 4, true>(a, s) : launch_tc_t<false, 1, 64, 4>(a, s);
        default: return cudaErrorInvalidConfiguration;
    }
}
cudaError_t launch_round_tc(const RoundArgs& a, cudaStream_t s) {
#ifdef SEGHDC_TRACE
    // events around [stamp0], [round kernel], [stamp1] separately (read with read_tc_events)
    static cudaEvent_t ev[4] = {};
    if (!ev[0]) {
        for (auto& e : ev) cudaEventCreate(&e);
        const char* tr = getenv("SEGHDC_TRACE_ROUND");
        const int r = tr ? atoi(tr) : 0;
        cudaMemcpyToSymbol(g_trace_round, &r, sizeof(r));
    }
    const char* tr = getenv("SEGHDC_TRACE_ROUND");
    if (tr && int(a.round) != atoi(tr)) {  // only the traced round records events and stamps
        return launch_round_tc_sel(a, s);
    }
    cudaEventRecord(ev[0], s);
    k_tc_stamp<<<148, 1, 0, s>>>(0);
    cudaEventRecord(ev[1], s);
    struct After {
        cudaStream_t s;
        cudaEvent_t* ev;
        ~After() {
            cudaEventRecord(ev[2], s);
            k_tc_stamp<<<148, 1, 0, s>>>(2);
            cudaEventRecord(ev[3], s);
        }
    } after{s, ev};
    g_tc_events = ev;
#endif
    return launch_round_tc_sel(a, s);
}

#ifdef SEGHDC_CHECKED
unsigned int check_line_tc() { return take_check_line(); }
#endif

}  // namespace seghdc_dev

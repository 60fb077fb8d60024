// B200 (sm_100a) kernels for the SegHDC encode + cluster hot path.
//
// Device data layout:
//   grid      u32[n_local][S32]      pixel HV as 32-bit little-endian words (bit i of the HV is
//                                    bit (i&31) of word i>>5 — the same bytes as the reference's
//                                    u64 words, hypervector.hpp:15-42), S32 = W32 rounded up to
//                                    4 words so every pixel row is 16-byte aligned for TMA.
//   Z         u32[K][D]              centroids: raw member sums (clusterer.hpp:27-34)
//   bfrag     u64[NT][W32P][32]      Z split into P 7-bit planes, laid out as the B fragments of
//                                    mma.m16n8k32 (column n = P*c + plane, NT = ceil(K*P/8)
//                                    n-tiles of 8), MMA index kk = 4*group + 2*pair + s, with
//                                    the pair packing of unpack_pair() (6-bit planes).
//   xchg      i32[K*Dp | K | 1 | Dp] [centroid sums | member counts | changed | column sums],
//                                    Dp = 32*W32. Every CTA folds its exact integer sums in
//                                    with coalesced atomics; it is the only buffer a multi-GPU
//                                    run all-reduces.
//
// Similarity is the reference's exact integer dot (hypervector.cpp:138-151):
//   dot(y, z_c) = sum_{i: y_i = 1} z_c[i] = sum_p 128^p * (Y . plane_p(z_c))
// computed as an integer GEMM Y[px x D] * B[D x P*K] on the IMMA tensor pipe (u8 x u8 -> s32,
// exact), then recombined in u64 and compared with the reference's 128-bit cross
// multiplication (clusterer.cpp:41-50). Centroid re-bundling (hypervector.cpp:112-121) is a
// bit-sliced Harley-Seal carry-save counter per 32-bit word column. No floating point.
#pragma once
#include <cstdint>

namespace seghdc_dev {

// Checked build (-DSEGHDC_CHECKED; compute-sanitizer is not available on the GPU pool): index
// invariants of the hot kernels are tested at run time; the first violated check's line
// number lands in g_check_line (read with seghdc_debug_check), and the kernel goes on.
#ifdef SEGHDC_CHECKED
static __device__ unsigned int g_check_line;  // one per translation unit (no -rdc)
#define SG_CHECK(cond)                                                              \
    do {                                                                            \
        if (!(cond)) atomicCAS(&::seghdc_dev::g_check_line, 0u, unsigned(__LINE__)); \
    } while (0)
// this translation unit's first violated line (0: none), reset afterwards
static inline unsigned int take_check_line() {
    unsigned int v = 0;
    const unsigned int zero = 0;
    cudaMemcpyFromSymbol(&v, g_check_line, sizeof(v));
    cudaMemcpyToSymbol(g_check_line, &zero, sizeof(zero));
    return v;
}
#else
#define SG_CHECK(cond) ((void)0)
#endif

// ------------------------------------------------------------------------------------------
// Device-side round state. Index [p] is the round parity (round r uses p = r & 1); the
// double buffering lets round r's consumer and round r+1's producer run back to back
// without host synchronisation.
struct RoundState {
    uint32_t done;        // early stop fired (clusterer.cpp:213)
    uint32_t rounds_run;  // ClusterResult::iterations_run
    uint32_t uniform;     // seed selection hit the uniform-image fallback
    uint32_t pad;
};
// Followed in memory by (K = number of clusters):
//   u32 cur[2][K]        member counts of the centroid set used by the round's assignment
//   u64 norm2[2][K]      IntVector::norm_squared of that set (hypervector.cpp:123-127)
//   u64 wraps[iterations] per-round count of 128-bit-wrapping comparisons (diagnostic)
struct StateView {
    RoundState* hdr;
    uint32_t* cur;
    unsigned long long* norm2;
    unsigned long long* wraps;
    uint32_t K;
    __host__ __device__ static size_t norm2_offset(uint32_t K) {
        return (sizeof(RoundState) + 2 * size_t(K) * 4 + 7) & ~size_t(7);
    }
    __host__ __device__ static size_t bytes(uint32_t K) { return norm2_offset(K) + 2 * size_t(K) * 8; }
    __host__ __device__ static size_t bytes(uint32_t K, size_t iterations) { return bytes(K) + 8 * (iterations + 1); }
    __host__ __device__ static StateView at(void* base, uint32_t K) {
        StateView v;
        v.hdr = reinterpret_cast<RoundState*>(base);
        v.cur = reinterpret_cast<uint32_t*>(v.hdr + 1);
        v.norm2 = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(base) + norm2_offset(K));
        v.wraps = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(base) + bytes(K));
        v.K = K;
        return v;
    }
};

// Cluster whose sums are derived as colsum - sum(others) instead of accumulated: the
// largest cluster of the current centroid set (ties -> lowest index). Any choice is exact.
__device__ __forceinline__ uint32_t pick_skip(const uint32_t* cur, uint32_t K) {
    uint32_t best = 0, bv = cur[0];
    for (uint32_t c = 1; c < K; ++c)
        if (cur[c] > bv) { bv = cur[c]; best = c; }
    return best;
}

// strictly_closer (clusterer.cpp:41-50): dot_c^2 * n2_best > dot_best^2 * n2_c evaluated in
// unsigned 128-bit arithmetic (wrapping modulo 2^128 exactly like the reference).
__device__ __forceinline__ bool strictly_closer(unsigned long long dc, unsigned long long n2c,
                                                unsigned long long db, unsigned long long n2b) {
    if (n2c == 0) return false;
    if (n2b == 0) return dc > 0;
    const unsigned __int128 lhs = (unsigned __int128)dc * dc * n2b;
    const unsigned __int128 rhs = (unsigned __int128)db * db * n2c;
    return lhs > rhs;
}

// Diagnostic, not reference behaviour: did strictly_closer's unsigned __int128 product
// d*d*n2 exceed 2^128 (so the reference compared wrapped values)? A comparison wraps when
// either side does (both norms non-zero). Fast reject on bit lengths, exact 192-bit check
// otherwise; counted per round so the oracle's per-round counts can be matched.
__device__ __forceinline__ bool prod_wraps(unsigned long long d, unsigned long long n2) {
    if (2 * (64 - __clzll(d)) + (64 - __clzll(n2)) <= 128) return false;
    const unsigned long long sl = d * d, sh = __umul64hi(d, d);
    const unsigned long long a1 = __umul64hi(sl, n2), b0 = sh * n2, b1 = __umul64hi(sh, n2);
    return b1 != 0 || b0 + a1 < b0;
}
__device__ __forceinline__ uint32_t compare_wraps(unsigned long long dc, unsigned long long n2c,
                                                  unsigned long long db, unsigned long long n2b) {
    if (n2c == 0 || n2b == 0) return 0u;
    return (prod_wraps(dc, n2b) || prod_wraps(db, n2c)) ? 1u : 0u;
}

// Can any comparison of this centroid set wrap? A pixel HV has at most D ones, so
// dot_c^2 <= n2_c * D (Cauchy-Schwarz) and every product is below n2max^2 * D. False for every
// configuration but the largest (C4), so the round kernels count wraps only when it is true.
__device__ __forceinline__ bool wraps_possible(const unsigned long long* n2, uint32_t K, uint32_t D) {
    int b = 0;
    for (uint32_t c = 0; c < K; ++c) b = max(b, 64 - __clzll(n2[c]));
    return 2 * b + (32 - __clz(D)) > 128;
}
// the argmax's comparison sequence replayed (clusterer.cpp:149-157), counting wrapped ones;
// out of line so the epilogues it is called from keep their registers
template <uint32_t KC>
__device__ __noinline__ uint32_t count_wraps_seq(const long long (&d)[KC], const unsigned long long (&n2)[KC], uint32_t K) {
    uint32_t best = 0, w = 0;
    for (uint32_t c = 1; c < KC && c < K; ++c) {
        w += compare_wraps((unsigned long long)d[c], n2[c], (unsigned long long)d[best], n2[best]);
        if (strictly_closer((unsigned long long)d[c], n2[c], (unsigned long long)d[best], n2[best])) best = c;
    }
    return w;
}

// ------------------------------------------------------------------------------------------
// Harley-Seal bit-sliced counter: 32 independent counters (one per bit of a 32-bit word
// column), count = ones + 2 twos + 4 fours + 8 eights + sum_m 16*2^m hi[m].
// 15 carry-save adders (2 LOP3 each) per 16 inputs + an H-plane ripple of the weight-16 word.
template <int H>
struct BitCounter {
    uint32_t o, t, f, e, hi[H];
    __device__ __forceinline__ void reset() {
        o = t = f = e = 0;
#pragma unroll
        for (int m = 0; m < H; ++m) hi[m] = 0;
    }
    __device__ __forceinline__ static void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
        const uint32_t u = a ^ b;
        h = (a & b) | (u & c);
        l = u ^ c;
    }
    __device__ __forceinline__ void add16(const uint32_t (&x)[16]) {
        uint32_t tA, tB, fA, fB, eA, eB, s;
        csa(tA, o, o, x[0], x[1]);
        csa(tB, o, o, x[2], x[3]);
        csa(fA, t, t, tA, tB);
        csa(tA, o, o, x[4], x[5]);
        csa(tB, o, o, x[6], x[7]);
        csa(fB, t, t, tA, tB);
        csa(eA, f, f, fA, fB);
        csa(tA, o, o, x[8], x[9]);
        csa(tB, o, o, x[10], x[11]);
        csa(fA, t, t, tA, tB);
        csa(tA, o, o, x[12], x[13]);
        csa(tB, o, o, x[14], x[15]);
        csa(fB, t, t, tA, tB);
        csa(eB, f, f, fA, fB);
        csa(s, e, e, eA, eB);
#pragma unroll
        for (int m = 0; m < H; ++m) {
            const uint32_t c = hi[m] & s;
            hi[m] ^= s;
            s = c;
        }
    }
    // plane k (weight 2^k) of the 32 counters to dst[k * stride], k < 4 + H
    __device__ __forceinline__ void planes(uint32_t* dst, size_t stride) const {
        dst[0] = o;
        dst[stride] = t;
        dst[2 * stride] = f;
        dst[3 * stride] = e;
#pragma unroll
        for (int m = 0; m < H; ++m) dst[(4 + m) * stride] = hi[m];
    }
    __device__ __forceinline__ bool any() const {
        uint32_t v = o | t | f | e;
#pragma unroll
        for (int m = 0; m < H; ++m) v |= hi[m];
        return v != 0;
    }
    __device__ __forceinline__ void add8(const uint32_t (&x)[8]) {
        uint32_t tA, tB, fA, fB, s;
        csa(tA, o, o, x[0], x[1]);
        csa(tB, o, o, x[2], x[3]);
        csa(fA, t, t, tA, tB);
        csa(tA, o, o, x[4], x[5]);
        csa(tB, o, o, x[6], x[7]);
        csa(fB, t, t, tA, tB);
        csa(s, f, f, fA, fB);  // s: weight 8
        const uint32_t c8 = e & s;
        e ^= s;
        s = c8;  // weight 16
#pragma unroll
        for (int m = 0; m < H; ++m) {
            const uint32_t c = hi[m] & s;
            hi[m] ^= s;
            s = c;
        }
    }
    // capacity of the counter (largest representable count)
    __host__ __device__ static constexpr uint64_t capacity() { return 15ull + 16ull * ((1ull << H) - 1); }
    // count of bit b
    __device__ __forceinline__ uint32_t value(int b) const {
        uint32_t val = ((o >> b) & 1u) | (((t >> b) & 1u) << 1) | (((f >> b) & 1u) << 2) | (((e >> b) & 1u) << 3);
#pragma unroll
        for (int m = 0; m < H; ++m) val |= ((hi[m] >> b) & 1u) << (4 + m);
        return val;
    }
    // dst[b] = count of bit b, b = 0..31 (32 consecutive u32)
    __device__ __forceinline__ void store(uint32_t* dst) const {
#pragma unroll 4
        for (int b = 0; b < 32; b += 4) {
            uint4 v;
            uint32_t* pv = &v.x;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int bb = b + q;
                uint32_t val = ((o >> bb) & 1u) | (((t >> bb) & 1u) << 1) | (((f >> bb) & 1u) << 2) |
                               (((e >> bb) & 1u) << 3);
#pragma unroll
                for (int m = 0; m < H; ++m) val |= ((hi[m] >> bb) & 1u) << (4 + m);
                pv[q] = val;
            }
            *reinterpret_cast<uint4*>(dst + b) = v;
        }
    }
};

// Fold a warp's counters into dst with coalesced atomics: lane l owns word column
// (col0 + l) = entries [32*(col0+l), 32*(col0+l)+32). The 32x32 block is transposed through
// `scratch` (32*33 u32 of shared memory owned by this warp) so each atomic instruction covers
// 32 consecutive entries (one 128-byte line). Columns >= ncols are skipped. `bias` is
// subtracted from every count (mod 2^32: the incremental re-bundling adds signed deltas).
template <int H>
__device__ __forceinline__ void flush_warp_atomic(const BitCounter<H>& cnt, uint32_t* scratch, uint32_t* dst,
                                                  uint32_t col0, uint32_t ncols, uint32_t bias = 0) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int b = 0; b < 32; ++b) scratch[lane * 33 + b] = cnt.value(b) - bias;
    __syncwarp();
    for (uint32_t r = 0; r < 32; ++r) {
        if (col0 + r >= ncols) break;
        const uint32_t val = scratch[r * 33 + lane];
        if (val) atomicAdd(dst + size_t(col0 + r) * 32 + lane, val);
    }
    __syncwarp();
}

// Whole-CTA flush of bit-sliced counters that their owners spilled plane-major to shared
// memory (planes[k * ncols + col], k < 4 + H; one 32-bit word column per col): every thread
// expands entries e = 32 col + b and adds count - bias (mod 2^32) into dst[e]; each warp's
// atomics cover one 128-byte line. Spreading the bit gathers over all warps keeps the flush
// off the kernel's tail (four fold warps alone took ~12 us).
template <int H>
__device__ __forceinline__ void flush_planes_cta(const uint32_t* planes, uint32_t ncols, uint32_t bias,
                                                 uint32_t* dst) {
    for (uint32_t e = threadIdx.x; e < ncols * 32; e += blockDim.x) {
        const uint32_t col = e >> 5, b = e & 31;
        uint32_t v = 0;
#pragma unroll
        for (int k = 0; k < 4 + H; ++k) v |= ((planes[size_t(k) * ncols + col] >> b) & 1u) << k;
        v -= bias;
        if (v) atomicAdd(dst + e, v);
    }
}

// ------------------------------------------------------------------------------------------
// PTX helpers: mbarrier + bulk async copy (TMA engine, cp.async.bulk) + legacy-path IMMA.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// polling wait (mbarrier.test_wait never suspends the thread): for the hand-offs on a kernel's
// critical path, where try_wait's suspend / wake-up latency would be paid on every hand-off
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SPIN_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SPIN_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void imma16832(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void imma16832_s8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Two HV bits per 8-bit k-slot ("pair packing"). The A byte of a slot is the top two bits of a
// byte of the (shifted) word, masked with 0xC0: read as u8 it is 64*b6 + 128*b7, read as s8
// it is 64*b6 - 128*b7. One u8 MMA against Bu = 2*z6 + z7 plus one s8 MMA against
// Bs = 2*z6 - z7 (z6, z7 the 6-bit centroid planes of the two bits) add up to
//     64*b6*(Bu+Bs) + 128*b7*(Bu-Bs) = 256*(b6*z6 + b7*z7),
// so each MASK (ALU pipe) feeds 8 bits into the tensor pipe instead of 4, and every product
// carries the common scale 256 (removed with >> 8 after the reduction, exact).
//
// The MMAs of a 4-word group (128 bits of the HV) are numbered kk = 4*group + 2*pair + s
// (s = 0: u8 with Bu, s = 1: s8 with Bs, same A). Lane (g, q) supplies rows g and g+8 from
// word q of the group, shifted left by 4*pair (a0/a1: slots 4q+j <-> bits 8j+6-4p, 8j+7-4p)
// and by 4*pair+2 (a2/a3: slots 16+4q+j <-> bits 8j+4-4p, 8j+5-4p). k_finish bakes the
// same permutation into bfrag. sh[0..3] = the lane's row words shifted by 0, 2, 4, 6.
__device__ __forceinline__ void unpack_pair(uint32_t (&a)[4], uint32_t lo_p, uint32_t hi_p, uint32_t lo_p2,
                                            uint32_t hi_p2) {
    a[0] = lo_p & 0xC0C0C0C0u;
    a[1] = hi_p & 0xC0C0C0C0u;
    a[2] = lo_p2 & 0xC0C0C0C0u;
    a[3] = hi_p2 & 0xC0C0C0C0u;
}
// left shift by a power of two held in a register: issues as IMAD on the FMA pipe, which is
// otherwise idle in the k-loop (the ALU pipe carries the masks)
__device__ __forceinline__ uint32_t shl_fma(uint32_t w, uint32_t pow2) {
    uint32_t r;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(w), "r"(pow2));
    return r;
}
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
// centroid values are split into (at least) kPlanes planes of kPlaneBits bits (z < 2^24 with 4)
constexpr uint32_t kPlaneBits = 6, kPlanes = 4;

}  // namespace seghdc_dev

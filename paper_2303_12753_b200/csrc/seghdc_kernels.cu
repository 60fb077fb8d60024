// B200 (sm_100a) kernels of the SegHDC hot path and their launchers.
// See kernels.cuh for the device data layout and DESIGN.md for the rooflines.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "kernels.cuh"
#include "launch.h"

namespace seghdc_dev {

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }

template <int H>
constexpr uint64_t counter_capacity() {
    return BitCounter<H>::capacity();
}
// Counter planes for a run of at most `count` inputs per counter.
#define SEGHDC_DISPATCH_H(count, FN, ...)                              \
    do {                                                               \
        const uint64_t _c = (count);                                   \
        if (_c <= counter_capacity<8>()) FN<8>(__VA_ARGS__);           \
        else if (_c <= counter_capacity<12>()) FN<12>(__VA_ARGS__);    \
        else if (_c <= counter_capacity<16>()) FN<16>(__VA_ARGS__);    \
        else FN<24>(__VA_ARGS__);                                      \
    } while (0)

// =============================================================================================
// Manhattan codebooks expanded on the device from their bases (seghdc_host::manhattan_bases):
// entry e < h is row e, then the w columns, then the C x 256 widened colour entries; each is
// its base XOR one run of ones. Output in the u32 table layout of seghdc_encode (wref words).
// =============================================================================================
__device__ __forceinline__ uint32_t run_mask32(uint32_t q, uint32_t s, uint32_t e) {  // bits [s, e) of word q
    const uint32_t lo = max(s, 32 * q), hi = min(e, 32 * q + 32);
    if (lo >= hi) return 0u;
    const uint32_t len = hi - lo, sh = lo - 32 * q;
    return (len == 32 ? 0xFFFFFFFFu : ((1u << len) - 1u)) << sh;
}
__global__ void k_expand_codebooks(const uint32_t* __restrict__ bases, ExpandArgs a, uint32_t* __restrict__ row,
                                   uint32_t* __restrict__ col, uint32_t* __restrict__ wid, uint8_t* __restrict__ sup) {
    const uint32_t ne = a.h + a.w + a.c * 256;
    const size_t total = size_t(ne) * a.wref;
    for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < total; t += size_t(gridDim.x) * blockDim.x) {
        if (t < a.wref) sup[t] = manhattan_word_channels(a.dim, a.c, a.off, uint32_t(t));
        const uint32_t e = uint32_t(t / a.wref), q = uint32_t(t % a.wref);
        uint32_t b, s, len;
        uint32_t* out;
        if (e < a.h) {
            b = 0, s = 0, len = (e / a.beta) * a.x_row, out = row + size_t(e) * a.wref;
        } else if (e < a.h + a.w) {
            const uint32_t j = e - a.h;
            b = 1, s = a.dim / 2, len = (j / a.beta) * a.x_col, out = col + size_t(j) * a.wref;
        } else {
            const uint32_t ch = (e - a.h - a.w) >> 8, v = (e - a.h - a.w) & 255;
            b = 2 + ch, s = a.off[ch], len = v * a.unit[ch], out = wid + size_t(ch * 256 + v) * a.wref;
        }
        out[q] = bases[size_t(b) * a.wref + q] ^ run_mask32(q, s, s + len);
    }
}
void launch_expand_codebooks(const uint32_t* bases, const ExpandArgs& a, uint32_t* row, uint32_t* col, uint32_t* wid,
                             uint8_t* sup, cudaStream_t s) {
    const size_t total = size_t(a.h + a.w + a.c * 256) * a.wref;
    const uint32_t blocks = uint32_t(std::min<size_t>((total + 255) / 256, 148 * 8));
    k_expand_codebooks<<<blocks, 256, 0, s>>>(bases, a, row, col, wid, sup);
}

// =============================================================================================
// encode_image (reference pixel_pipeline.cpp:92-126): grid[p] = row[i] ^ col[j] ^ ^_ch wid[ch][v]
// fused with the column sums of the grid (the Harley-Seal counter of every pixel), which the
// round schedule needs to derive the largest cluster's sums without accumulating them.
//
// The widened colour tables of different channels have disjoint supports
// (pixel_pipeline.cpp:66-69): HV word q is touched by the channels whose dimension segment
// overlaps it, one for all but C - 1 boundary words. `sup[q]` holds that channel set (any
// superset of the true support is exact: the other channels' entries are zero in word q), so a
// lane looks up ONE table entry per pixel, a CTA stages one 32 KB table slice (two where its
// word chunk straddles a channel boundary) and three channels cost what one does.
//
// CTA = (64-column tile, group of rows, chunk of 32 HV words); lane = word, so every pixel is one
// coalesced 128-byte store. A warp owns 8 image columns for the whole kernel (their column
// codes live in registers) and walks 4-row x 8-column patches: 4 row-code loads and 4 8-byte
// loads of its channel's image bytes (staged planar) per 32 pixels, then one table load and one
// store per pixel. Each lane keeps a Harley-Seal counter; the CTA folds them in shared memory
// and adds 1024 column sums to the global array.
// =============================================================================================
constexpr uint32_t kEncRows = 64, kEncCols = 64;  // image tile (and its row codes) staged per batch
// warps per CTA: 8 (4 CTAs per SM) with one channel; 16 (2 CTAs per SM, up to two table
// slices each) with three
template <int C>
constexpr uint32_t enc_warps() { return C == 1 ? 8 : 16; }
template <int C>
constexpr uint32_t enc_ctas_per_sm() { return C == 1 ? 4 : 2; }

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(uint32_t(__cvta_generic_to_shared(smem_dst))), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// One 4 x 8 patch: rows rr0..rr0+3 of the staged batch, columns 8 cg..8 cg+7 of the tile.
// FULL: every row and column of the patch exists.
template <int NL, int H, bool FULL>
__device__ __forceinline__ void encode_patch(const uint32_t* s_row_l, const uint8_t* const (&px)[NL],
                                             const uint32_t* const (&tab)[NL], const uint32_t (&colr)[8],
                                             uint32_t rr0, uint32_t nrows, uint32_t ncols, char* o,
                                             ptrdiff_t pix_bytes, ptrdiff_t row_skip_bytes, BitCounter<H>& cnt,
                                             const char* g_lo, const char* g_hi) {
    uint32_t x[16];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const bool rok = FULL || uint32_t(r) < nrows;
        const uint32_t rv = s_row_l[(rr0 + r) * 32];
        uint2 pk[NL];
#pragma unroll
        for (int k = 0; k < NL; ++k) pk[k] = *reinterpret_cast<const uint2*>(px[k] + (rr0 + r) * kEncCols);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            uint32_t v = rv ^ colr[u];
#pragma unroll
            for (int k = 0; k < NL; ++k) {
                const uint32_t b = __byte_perm(u < 4 ? pk[k].x : pk[k].y, 0, 0x4440 + (u & 3));
                v ^= tab[k][b * 32];
            }
            if (!FULL && !(rok && uint32_t(u) < ncols)) v = 0;
            x[(r & 1) * 8 + u] = v;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // one running pointer: a 64-bit add per store, no multiplies
            if (FULL || (rok && uint32_t(u) < ncols)) {
                SG_CHECK(o >= g_lo && o + 4 <= g_hi);  // inside this call's rows of the grid
                *reinterpret_cast<uint32_t*>(o) = x[(r & 1) * 8 + u];
            }
            o += pix_bytes;
        }
        o += row_skip_bytes;
        if (r & 1) cnt.add16(x);
    }
}

// H: weight-16 planes of the column-sum counters, the fewest that hold the pixels one warp
// encodes (its ripple is 2 LOP3 per plane per 16 pixels)
template <int C, int NL, int H>
__device__ __forceinline__ void encode_rows_loop(const uint8_t* __restrict__ img, uint32_t w, uint32_t row_begin,
                                                 uint32_t r0, uint32_t r1, const uint32_t* __restrict__ row,
                                                 uint32_t wref, uint32_t S32, uint32_t* __restrict__ grid, uint32_t w0,
                                                 uint32_t c0, uint32_t nc, const uint32_t (&ch)[3],
                                                 const uint32_t (&colr)[8], const uint32_t* s_tab, uint32_t* s_row,
                                                 uint8_t* s_img, BitCounter<H>& cnt) {
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr uint32_t kWarps = enc_warps<C>(), kRgStep = kWarps / 8;
    const uint32_t cg = warp & 7;                               // the warp's 8 columns of the tile
    const uint32_t ncols = nc > cg * 8 ? min(8u, nc - cg * 8) : 0u;
    const bool ld = w0 + lane < wref;  // every lane stores: S32 is a multiple of 32 (launch_encode)
    const uint32_t* s_row_l = s_row + lane;
    const ptrdiff_t pix_bytes = ptrdiff_t(S32) * 4, row_skip_bytes = (ptrdiff_t(w) - 8) * ptrdiff_t(S32) * 4;
    const char* g_lo = reinterpret_cast<const char*>(grid);  // checked build: the rows this launch encodes
    const char* g_hi = reinterpret_cast<const char*>(grid + size_t(r1 - row_begin) * w * S32);
    (void)g_lo;
    (void)g_hi;
    const uint8_t* px[NL];
    const uint32_t* tab[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        px[k] = s_img + ch[k] * (kEncRows * kEncCols) + cg * 8;  // planar: [channel][row][column]
        tab[k] = s_tab + k * 8192 + lane;
    }
    bool first = true;
    for (uint32_t rb = r0; rb < r1; rb += kEncRows) {
        const uint32_t nrb = min(kEncRows, r1 - rb);
        __syncthreads();  // previous batch's row codes and image bytes consumed
        for (uint32_t e = tid; e < nrb * 32; e += blockDim.x) {  // e & 31 == lane
            if (ld) cp_async4(s_row + e, row + size_t(rb + (e >> 5)) * wref + w0 + lane);
            else s_row[e] = 0;
        }
        // image tile -> planar bytes, 4 pixels (4 C bytes) per item: C + 1 aligned words, funnel
        // shifts to the group's first byte, then byte permutes to one word per channel. A group
        // that starts inside the row may read up to 16 bytes past a ragged row end (the image
        // allocation is padded); its extra columns are never stored.
        for (uint32_t e = tid; e < nrb * (kEncCols / 4); e += blockDim.x) {
            const uint32_t rr = e / (kEncCols / 4), g = e % (kEncCols / 4);
            if (g * 4 >= nc) continue;
            const uint8_t* p = img + (size_t(rb + rr) * w + c0 + g * 4) * C;
            const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(p) & 3);
            const uint32_t* pw = reinterpret_cast<const uint32_t*>(p - mis);
            uint32_t wv[C + 1], f[C];
#pragma unroll
            for (int j = 0; j <= C; ++j) wv[j] = (j < C || mis) ? __ldg(pw + j) : 0u;
#pragma unroll
            for (int j = 0; j < C; ++j) f[j] = __funnelshift_r(wv[j], wv[j + 1], mis * 8);
            uint32_t* dst = reinterpret_cast<uint32_t*>(s_img + rr * kEncCols + g * 4);
            if (C == 1) {
                dst[0] = f[0];
            } else {  // f = [R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3]
                dst[0] = __byte_perm(__byte_perm(f[0], f[1], 0x0630), f[2], 0x5210);
                dst[kEncRows * kEncCols / 4] = __byte_perm(__byte_perm(f[0], f[1], 0x0741), f[2], 0x6210);
                dst[2 * kEncRows * kEncCols / 4] = __byte_perm(__byte_perm(f[0], f[1], 0x0052), f[2], 0x7410);
            }
        }
        cp_async_wait_all();  // row codes (and, the first time, the table slices)
        first = false;
        __syncthreads();
        if (ncols == 0) continue;
        for (uint32_t rg = warp >> 3; rg * 4 < nrb; rg += kRgStep) {  // the warp's 4-row groups of the batch
            const uint32_t rr0 = rg * 4, nrows = min(4u, nrb - rr0);
            char* o = reinterpret_cast<char*>(grid + (size_t(rb + rr0 - row_begin) * w + c0 + cg * 8) * S32 + w0 + lane);
            SG_CHECK(rr0 + nrows <= kEncRows && cg * 8 + ncols <= kEncCols);  // inside the staged tile
            if (nrows == 4 && ncols == 8)
                encode_patch<NL, H, true>(s_row_l, px, tab, colr, rr0, 4, 8, o, pix_bytes, row_skip_bytes, cnt, g_lo, g_hi);
            else
                encode_patch<NL, H, false>(s_row_l, px, tab, colr, rr0, nrows, ncols, o, pix_bytes, row_skip_bytes, cnt, g_lo,
                                           g_hi);
        }
    }
    if (first) cp_async_wait_all();
}

template <int C, int H>
__global__ void __launch_bounds__(enc_warps<C>() * 32, enc_ctas_per_sm<C>())
    k_encode(const uint8_t* __restrict__ img, uint32_t w, uint32_t row_begin, uint32_t row_end,
             const uint32_t* __restrict__ row, const uint32_t* __restrict__ col, const uint32_t* __restrict__ wid,
             const uint8_t* __restrict__ sup, uint32_t wref, uint32_t S32, uint32_t* __restrict__ grid,
             uint32_t* __restrict__ colsum, uint32_t W32, uint32_t nl_max) {
    extern __shared__ __align__(16) uint32_t es[];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t w0 = blockIdx.x * 32;             // first word of the chunk
    const uint32_t rows_per = (row_end - row_begin + gridDim.z - 1) / gridDim.z;
    const uint32_t r0 = row_begin + blockIdx.z * rows_per, r1 = min(row_end, r0 + rows_per);
    const uint32_t c0 = blockIdx.y * kEncCols, nc = min(kEncCols, w - c0);

    // the lane's channels: set bits of sup[word], lowest first; nl = the most any lane needs
    uint32_t ch[3] = {0, 0, 0}, nl_lane = 1;
    if (C > 1) {
        uint32_t m = (w0 + lane < wref) ? sup[w0 + lane] & ((1u << C) - 1) : 0u;
        nl_lane = __popc(m);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ch[k] = m ? __ffs(m) - 1 : 0;
            m &= m - 1;
        }
    }
    const uint32_t nl = C > 1 ? max(1u, __reduce_max_sync(0xffffffffu, nl_lane)) : 1u;
    if (nl > nl_max) __trap();  // the launch sized shared memory for nl_max table slices
    uint32_t* s_tab = es;                             // [nl][256][32]: the lane's k-th channel
    uint32_t* s_sum = s_tab + nl * 8192;              // [32 bits][32 words]
    uint32_t* s_row = s_sum + 1024;                   // [ER][32]
    uint8_t* s_img = reinterpret_cast<uint8_t*>(s_row + kEncRows * 32);  // [C][ER][EC], planar

    // table slices: 4-byte async copies, all in flight at once (e & 31 == lane); words past the
    // HV and unused slices hold 0, and so do the column codes below: no masking in the loop
    for (uint32_t e = tid; e < nl * 8192; e += blockDim.x) {
        const uint32_t k = e >> 13, val = (e >> 5) & 255;
        const uint32_t chk = k == 0 ? ch[0] : (k == 1 ? ch[1] : ch[2]);
        if (k < nl_lane && w0 + lane < wref)
            cp_async4(s_tab + e, wid + size_t(chk * 256 + val) * wref + w0 + lane);
        else
            s_tab[e] = 0;
    }
    uint32_t colr[8];
    {
        const uint32_t cg = warp & 7;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t cc = cg * 8 + u;
            colr[u] = (cc < nc && w0 + lane < wref) ? __ldg(col + size_t(c0 + cc) * wref + w0 + lane) : 0u;
        }
    }
    BitCounter<H> cnt;  // <= ceil(rows_per / 4 / (warps / 8)) * 32 pixels per warp
    cnt.reset();
    if (nl == 1)
        encode_rows_loop<C, 1, H>(img, w, row_begin, r0, r1, row, wref, S32, grid, w0, c0, nc, ch, colr, s_tab, s_row, s_img, cnt);
    else if (C > 1 && nl == 2)
        encode_rows_loop<C, 2, H>(img, w, row_begin, r0, r1, row, wref, S32, grid, w0, c0, nc, ch, colr, s_tab, s_row, s_img, cnt);
    else if (C > 1)
        encode_rows_loop<C, 3, H>(img, w, row_begin, r0, r1, row, wref, S32, grid, w0, c0, nc, ch, colr, s_tab, s_row, s_img, cnt);
    // fold the warps' counters: a tree of bit-sliced adds (2 LOP3 per plane) through shared
    // memory (the table slices are dead by now), then warp 0 expands the CTA totals and every
    // thread adds its share of the 1024 column sums to the global array
    {
        constexpr int kWarps = int(enc_warps<C>()), kLv = kWarps == 16 ? 4 : 3, kP0 = 4 + H, kPmax = kP0 + kLv;
        uint32_t pl[kPmax];
        pl[0] = cnt.o, pl[1] = cnt.t, pl[2] = cnt.f, pl[3] = cnt.e;
#pragma unroll
        for (int m = 0; m < H; ++m) pl[4 + m] = cnt.hi[m];
#pragma unroll
        for (int m = kP0; m < kPmax; ++m) pl[m] = 0;
        uint32_t* scratch = s_tab;  // [kWarps / 2][kPmax][32] <= 8 * 20 * 128 B
#pragma unroll
        for (int lv = 0; lv < kLv; ++lv) {
            const uint32_t half = kWarps >> (lv + 1);
            __syncthreads();  // main loop done / previous level's readers done
            if (warp >= half && warp < 2 * half) {
#pragma unroll
                for (int m = 0; m < kP0 + lv; ++m) scratch[((warp - half) * kPmax + m) * 32 + lane] = pl[m];
            }
            __syncthreads();
            if (warp < half) {
                uint32_t carry = 0;
#pragma unroll
                for (int m = 0; m < kP0 + lv; ++m) {
                    const uint32_t a = pl[m], bb = scratch[(warp * kPmax + m) * 32 + lane];
                    pl[m] = a ^ bb ^ carry;
                    carry = (a & bb) | ((a ^ bb) & carry);
                }
                pl[kP0 + lv] = carry;
            }
        }
        if (warp == 0) {
#pragma unroll 4
            for (int b = 0; b < 32; ++b) {
                uint32_t val = 0;
#pragma unroll
                for (int m = 0; m < kPmax; ++m) val |= ((pl[m] >> b) & 1u) << m;
                s_sum[b * 32 + lane] = val;
            }
        }
        __syncthreads();
    }
    for (uint32_t e = tid; e < 1024; e += blockDim.x) {
        const uint32_t wd = e & 31, b = e >> 5, word = w0 + wd;
        if (word < W32 && s_sum[e]) atomicAdd(colsum + size_t(word) * 32 + b, s_sum[e]);
    }
}

template <int C, int H>
static void launch_encode_ch(const EncodeArgs& a, dim3 g, uint32_t row_begin, uint32_t row_end, cudaStream_t s) {
    const uint32_t nl = C == 1 ? 1 : std::min<uint32_t>(std::max<uint32_t>(a.nl_max, 1), 3);
    const size_t smem = (size_t(nl) * 8192 + 1024 + kEncRows * 32) * 4 + size_t(C) * kEncRows * kEncCols;
    ensure_dynamic_smem((const void*)k_encode<C, H>, smem);
    k_encode<C, H><<<g, enc_warps<C>() * 32, smem, s>>>(a.img, a.w, row_begin, row_end, a.row, a.col, a.wid, a.sup,
                                                       a.wref, a.S32, a.grid, a.colsum, a.W32, nl);
}
template <int C>
static void launch_encode_c(const EncodeArgs& a, uint32_t row_begin, uint32_t row_end, cudaStream_t s) {
    const uint32_t gx = (a.w + kEncCols - 1) / kEncCols, gz = (a.S32 + 31) / 32, rows = row_end - row_begin;
    // row groups per (column tile, chunk): the split that minimises waves x (rows per CTA + the
    // rows' worth of time a CTA spends staging its table slice and folding its counters), over
    // the resident CTA slots. From 1.5 waves on the SMs pick up CTAs as they free up, so waves
    // count fractionally plus half a CTA of tail; a single wave runs its CTAs in lock step
    // (all staging, then all storing) and is charged as 1.5.
    // (Measured flat within ~5 % around the optimum: C1 100-111 us for 5..12 groups.)
    const uint64_t slots = uint64_t(std::max<uint32_t>(a.sms, 1)) * enc_ctas_per_sm<C>();
    constexpr uint64_t kStageRows = C == 1 ? 6 : 12;
    uint32_t gy = 1;
    uint64_t best = ~0ull;
    for (uint32_t y = 1; y <= std::max<uint32_t>(1, (rows + 3) / 4) && y <= 65535; ++y) {
        const uint64_t per = (rows + y - 1) / y, n = uint64_t(gx) * gz * y;
        const uint64_t waves2 = 2 * n >= 3 * slots ? (2 * n + slots - 1) / slots + 1 : (n <= slots ? 3 : 4);
        const uint64_t cost = waves2 * (per + kStageRows);  // in half waves
        if (cost < best) best = cost, gy = y;
        if (per <= 16) break;
    }
    static const char* gy_env = getenv("SEGHDC_ENC_GY");  // experiment switch
    if (gy_env && atoi(gy_env) > 0) gy = std::min<uint32_t>(uint32_t(atoi(gy_env)), rows);
    const dim3 g(gz, gx, gy);
    const uint64_t rows_per = (uint64_t(rows) + gy - 1) / gy;
    const uint64_t per_warp = (rows_per + 4 * (enc_warps<C>() / 8) - 1) / (4 * (enc_warps<C>() / 8)) * 32 + 32;
    if (per_warp <= BitCounter<6>::capacity()) return launch_encode_ch<C, 6>(a, g, row_begin, row_end, s);
    if (per_warp <= BitCounter<8>::capacity()) return launch_encode_ch<C, 8>(a, g, row_begin, row_end, s);
    if (per_warp <= BitCounter<10>::capacity()) return launch_encode_ch<C, 10>(a, g, row_begin, row_end, s);
    launch_encode_ch<C, 12>(a, g, row_begin, row_end, s);
}

void launch_encode(const EncodeArgs& a, cudaStream_t s) {
    const uint64_t n = a.pix_end - a.pix_begin;
    if (n == 0) return;
    const uint32_t row_begin = uint32_t(a.pix_begin / a.w), row_end = uint32_t(a.pix_end / a.w);
    if (a.S32 % 32 != 0) abort();  // grid rows are whole 128-byte lines (Geometry::set)
    if (a.c == 1) launch_encode_c<1>(a, row_begin, row_end, s);
    else launch_encode_c<3>(a, row_begin, row_end, s);
}

// =============================================================================================
// select_initial_centroids (reference clusterer.cpp:54-130) on the device.
//   min/max colour key with row-major first occurrence: atomicMin on (key << 32 | idx) and
//   ((0xFFFF - key) << 32 | idx); greedy max-min L1 colour distance: atomicMin on
//   ((0xFFFFFFFF - d) << 32 | idx) over unchosen pixels; uniform-image corner fallback.
// slots: u64[2 + K]: [0] min pack, [1] max pack, [2+s] greedy pack of step s.
// =============================================================================================
__device__ __forceinline__ uint32_t color_key(const uint8_t* img, uint64_t p, uint32_t c) {
    uint32_t s = 0;
    for (uint32_t ch = 0; ch < c; ++ch) s += img[p * c + ch];
    return s;
}
__device__ __forceinline__ uint32_t l1_color(const uint8_t* img, uint64_t p, uint64_t q, uint32_t c) {
    uint32_t s = 0;
    for (uint32_t ch = 0; ch < c; ++ch) s += uint32_t(abs(int(img[p * c + ch]) - int(img[q * c + ch])));
    return s;
}

// Minimum over the block (result valid in thread 0); blockDim.x a multiple of 32, <= 1024.
__device__ __forceinline__ unsigned long long block_min64(unsigned long long v) {
    __shared__ unsigned long long part[32];
    for (int o = 16; o; o >>= 1) v = umin64(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();  // part[] may still be read by a previous call
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : ~0ull;
        for (int o = 16; o; o >>= 1) v = umin64(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    return v;
}

__global__ void k_seed_minmax(const uint8_t* __restrict__ img, uint64_t n, uint32_t c,
                              unsigned long long* slots) {
    unsigned long long mn = ~0ull, mx = ~0ull;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t key = color_key(img, p, c);
        mn = umin64(mn, (key << 32) | p);
        mx = umin64(mx, ((0xFFFFull - key) << 32) | p);
    }
    mn = block_min64(mn);
    mx = block_min64(mx);
    if (threadIdx.x == 0) {  // one atomic per block (per-warp atomics on two addresses serialised)
        atomicMin(slots + 0, mn);
        atomicMin(slots + 1, mx);
    }
}

// Decide min/max seeds or the uniform fallback (clusterer.cpp:83-99). Single thread; `seeds` may be
// a global or a shared array, `uniform` receives the fallback flag.
__device__ __forceinline__ void seed_post(const unsigned long long* slots, uint64_t* seeds, uint32_t K, uint32_t h,
                                          uint32_t w, uint32_t* uniform) {
    const uint64_t mn_key = slots[0] >> 32, mx_key = 0xFFFFull - (slots[1] >> 32);
    if (mn_key == mx_key) {
        *uniform = 1;
        uint32_t nch = 0;
        const uint64_t corners[4] = {0, uint64_t(w) - 1, uint64_t(h - 1) * w, uint64_t(h - 1) * w + w - 1};
        for (int i = 0; i < 4 && nch < K; ++i) {
            bool dup = false;
            for (uint32_t s = 0; s < nch; ++s) dup |= seeds[s] == corners[i];
            if (!dup) seeds[nch++] = corners[i];
        }
        for (uint64_t p = 0; nch < K; ++p) {  // row-major fill; K <= n is validated on the host
            bool dup = false;
            for (uint32_t s = 0; s < nch; ++s) dup |= seeds[s] == p;
            if (!dup) seeds[nch++] = p;
        }
        return;
    }
    *uniform = 0;
    seeds[0] = slots[0] & 0xFFFFFFFFull;
    if (K >= 2) seeds[1] = slots[1] & 0xFFFFFFFFull;
}
__global__ void k_seed_post(unsigned long long* slots, uint64_t* seeds, uint32_t K, uint32_t h, uint32_t w,
                            RoundState* hdr) {
    seed_post(slots, seeds, K, h, w, &hdr->uniform);
}

// Greedy step s (>= 2): relax min_dist with seed s-1 (or both first seeds at s == 2) and pick
// the farthest unchosen pixel (clusterer.cpp:101-128, strict > keeps the first occurrence).
__global__ void k_seed_greedy(const uint8_t* __restrict__ img, uint64_t n, uint32_t c, uint32_t s,
                              uint16_t* min_dist, uint64_t* seeds, unsigned long long* slots,
                              const RoundState* hdr) {
    if (hdr->uniform) return;
    __shared__ uint64_t chosen[64];
    const uint32_t nch = s;  // seeds[0..s-1] chosen; seeds[s-1] may still sit in its slot
    for (uint32_t i = threadIdx.x; i < nch && i < 64; i += blockDim.x)
        chosen[i] = (i >= 2) ? (slots[2 + i] & 0xFFFFFFFFull) : seeds[i];
    __syncthreads();
    const uint64_t last = chosen[min(nch, 64u) - 1];
    unsigned long long best = ~0ull;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t d;
        if (s == 2)
            d = min(l1_color(img, p, chosen[0], c), l1_color(img, p, chosen[1], c));
        else
            d = min(uint32_t(min_dist[p]), l1_color(img, p, last, c));
        min_dist[p] = uint16_t(d);
        bool taken = false;
        for (uint32_t i = 0; i < nch && i < 64; ++i) taken |= chosen[i] == p;
        if (nch > 64)  // very large K: scan the recorded slots
            for (uint32_t i = 64; i < nch; ++i) taken |= (slots[2 + i] & 0xFFFFFFFFull) == p;
        if (!taken) best = umin64(best, ((0xFFFFFFFFull - d) << 32) | p);
    }
    best = block_min64(best);
    if (threadIdx.x == 0) atomicMin(slots + 2 + s, best);
}

__global__ void k_seed_collect(uint64_t* seeds, const unsigned long long* slots, uint32_t K, const RoundState* hdr) {
    if (hdr->uniform) return;
    for (uint32_t s = 2 + threadIdx.x; s < K; s += blockDim.x) seeds[s] = slots[2 + s] & 0xFFFFFFFFull;
}

void launch_select_seeds(const SeedArgs& a, cudaStream_t s) {
    if (!a.slots_cleared) cudaMemsetAsync(a.slots, 0xFF, (2 + a.K) * sizeof(unsigned long long), s);
    const uint32_t blocks = uint32_t(std::min<uint64_t>((a.n + 255) / 256, 148 * 2));
    k_seed_minmax<<<blocks, 256, 0, s>>>(a.img, a.n, a.c, a.slots);
    // K <= 2 inside a cluster call: k_init_seeds decides the seeds itself (one launch fewer)
    if (!(a.defer_post && a.K <= 2)) k_seed_post<<<1, 1, 0, s>>>(a.slots, a.seeds, a.K, a.h, a.w, a.hdr);
    for (uint32_t st = 2; st < a.K; ++st)
        k_seed_greedy<<<blocks, 256, 0, s>>>(a.img, a.n, a.c, st, a.min_dist, a.seeds, a.slots, a.hdr);
    if (a.K > 2) k_seed_collect<<<1, 32, 0, s>>>(a.seeds, a.slots, a.K, a.hdr);
}

// =============================================================================================
// Seed centroids (clusterer.cpp:197-205): xchg[c][i] = bit i of the seed pixel's HV when the
// pixel lies in this rank's shard, else 0 (an all-reduce then yields the full seed HVs).
// =============================================================================================
// colsum_src (nullable): the local column sums are copied into the exchange tail here as well
// (their init all-reduce makes them global), saving a device-to-device copy in the init chain.
__global__ void k_init_seeds(const uint32_t* __restrict__ grid, uint32_t S32, uint64_t pix_begin, uint64_t n_local,
                             uint64_t* seeds, uint32_t K, uint32_t W32, uint32_t Dp, int32_t* xchg,
                             const int32_t* __restrict__ colsum_src, int32_t* __restrict__ colsum_dst,
                             const unsigned long long* post_slots, uint32_t h, uint32_t w, RoundState* hdr) {
    const uint32_t c = blockIdx.y;
    // post_slots (K <= 2): the min/max slots of k_seed_minmax; every block derives the seeds (the
    // work of k_seed_post) and block (0, 0) publishes them
    __shared__ uint64_t s_seeds[2];
    __shared__ uint32_t s_uniform;
    if (post_slots) {
        if (threadIdx.x == 0) {
            seed_post(post_slots, s_seeds, K, h, w, &s_uniform);
            if (blockIdx.x == 0 && blockIdx.y == 0) {
                hdr->uniform = s_uniform;
                for (uint32_t q = 0; q < K; ++q) seeds[q] = s_seeds[q];
            }
        }
        __syncthreads();
    }
    const uint64_t sp = post_slots ? s_seeds[c] : seeds[c];
    const bool local = sp >= pix_begin && sp < pix_begin + n_local;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < Dp; i += gridDim.x * blockDim.x) {
        uint32_t bit = 0;
        if (local && (i >> 5) < W32) bit = (grid[(sp - pix_begin) * S32 + (i >> 5)] >> (i & 31)) & 1u;
        xchg[size_t(c) * Dp + i] = int32_t(bit);
        if (c == 0 && colsum_src) colsum_dst[i] = colsum_src[i];
    }
}

void launch_init_seeds(const InitSeedArgs& a, cudaStream_t s) {
    dim3 g((a.Dp + 255) / 256, a.K);
    k_init_seeds<<<g, 256, 0, s>>>(a.grid, a.S32, a.pix_begin, a.n_local, a.seeds, a.K, a.W32, a.Dp, a.xchg, a.colsum_src,
                                   a.colsum_dst, a.K <= 2 ? a.post_slots : nullptr, a.h, a.w, a.hdr);
}

// One launch instead of three memsets at the start of a cluster call: the round state and the
// running sums to zero, the seed-selection slots to all ones.
__global__ void k_init_clear(uint32_t* state, uint32_t state_words, uint32_t* run1, uint32_t run1_words,
                             unsigned long long* slots, uint32_t nslots, uint32_t* list_counts, uint32_t nlists) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    for (uint32_t i = t; i < nlists; i += nt) list_counts[i] = 0;  // round 1's changed-pixel lists
    for (uint32_t i = t; i < state_words; i += nt) state[i] = 0;
    for (uint32_t i = t; i < run1_words; i += nt) run1[i] = 0;
    for (uint32_t i = t; i < nslots; i += nt) slots[i] = ~0ull;
}
void launch_init_clear(void* state, size_t state_bytes, void* run1, size_t run1_bytes, unsigned long long* slots,
                       uint32_t nslots, uint32_t* list_counts, uint32_t nlists, cudaStream_t s) {
    const uint32_t words = uint32_t((state_bytes + 3) / 4 + run1_bytes / 4 + nslots);
    k_init_clear<<<std::max(1u, std::min(148u, (words + 1023) / 1024)), 256, 0, s>>>(
        static_cast<uint32_t*>(state), uint32_t((state_bytes + 3) / 4), static_cast<uint32_t*>(run1),
        uint32_t(run1_bytes / 4), slots, nslots, list_counts, nlists);
}

// =============================================================================================
// Standalone bit-sliced accumulation (update_centroids, clusterer.cpp:164-188, without the
// fused assignment; also the column sums when labels == nullptr).
// CTA = (pixel range, <= 512-word column block). For each cluster c != skip the CTA compacts
// the pixels of its range labelled c and feeds their words through one Harley-Seal counter
// per word column, so every pixel HV is read exactly once regardless of K; the counters are
// folded into dst[c * Dp + ...] with coalesced atomics, member counts into counts_dst[c].
// =============================================================================================
template <int H>
__global__ void __launch_bounds__(512) k_accumulate(const uint32_t* __restrict__ grid, uint32_t S32, uint32_t W32,
                                                     uint64_t n, uint64_t ppc, const uint32_t* __restrict__ labels,
                                                     uint32_t K, int skip_mode, void* state, uint32_t parity,
                                                     uint32_t* __restrict__ dst, uint32_t Dp,
                                                     uint32_t* __restrict__ counts_dst) {
    constexpr uint32_t CHUNK = 4096;
    extern __shared__ uint32_t dyn[];
    uint32_t* list = dyn;                        // [CHUNK]
    uint32_t* scratch = dyn + CHUNK;             // [warps][32*33]
    __shared__ uint32_t list_n, s_count;
    StateView st = StateView::at(state, K);
    if (state && st.hdr->done) return;
    const uint32_t t = blockIdx.y * blockDim.x + threadIdx.x;  // word column
    const uint64_t p_begin = uint64_t(blockIdx.x) * ppc;
    const uint64_t p_end = p_begin + ppc < n ? p_begin + ppc : n;
    // skip_mode: -1 = accumulate every cluster; -2 = pick_skip(cur[parity]); >= 0 explicit.
    int skip = skip_mode;
    if (skip_mode == -2) skip = int(pick_skip(st.cur + parity * K, K));
    const uint32_t nclusters = labels ? K : 1;
    BitCounter<H> cnt;
    for (uint32_t c = 0; c < nclusters; ++c) {
        if (int(c) == skip) continue;
        cnt.reset();
        if (threadIdx.x == 0) s_count = 0;
        for (uint64_t q0 = p_begin; q0 < p_end; q0 += CHUNK) {
            const uint64_t q1 = q0 + CHUNK < p_end ? q0 + CHUNK : p_end;
            __syncthreads();
            if (threadIdx.x == 0) list_n = 0;
            __syncthreads();
            for (uint64_t p = q0 + threadIdx.x; p < q0 + ((q1 - q0 + 31) & ~uint64_t(31)); p += blockDim.x) {
                const bool take = p < q1 && (!labels || labels[p] == c);
                const uint32_t bal = __ballot_sync(0xffffffffu, take);
                uint32_t base = 0;
                if ((threadIdx.x & 31) == 0 && bal) base = atomicAdd(&list_n, __popc(bal));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (take) list[base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1))] = uint32_t(p - q0);
            }
            __syncthreads();
            const uint32_t m = list_n;
            if (threadIdx.x == 0) s_count += m;
            if (t < W32) {
                for (uint32_t e = 0; e < m; e += 16) {
                    uint32_t x[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        x[u] = (e + u < m) ? __ldg(grid + (q0 + list[e + u]) * S32 + t) : 0u;
                    cnt.add16(x);
                }
            }
        }
        flush_warp_atomic(cnt, scratch + (threadIdx.x >> 5) * (32 * 33), dst + size_t(c) * Dp, t & ~31u, W32);
        __syncthreads();
        if (counts_dst && threadIdx.x == 0 && blockIdx.y == 0 && s_count) atomicAdd(counts_dst + c, s_count);
    }
}

template <int H>
static void launch_accumulate_h(const AccumulateArgs& a, uint32_t blocks_x, uint64_t ppc, cudaStream_t s) {
    const uint32_t threads = std::min<uint32_t>(512, ((a.W32 + 31) / 32) * 32);
    dim3 g(blocks_x, (a.W32 + threads - 1) / threads);
    const size_t smem = (4096 + size_t(threads / 32) * 32 * 33) * 4;
    ensure_dynamic_smem((const void*)k_accumulate<H>, smem);
    k_accumulate<H><<<g, threads, smem, s>>>(a.grid, a.S32, a.W32, a.n, ppc, a.labels, a.K, a.skip_mode, a.state,
                                             a.parity, a.dst, a.Dp, a.counts_dst);
}

void launch_accumulate(const AccumulateArgs& a, cudaStream_t s) {
    const uint32_t blocks = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(a.sms) * 2, (a.n + 255) / 256)));
    const uint64_t ppc = (a.n + blocks - 1) / blocks;
    SEGHDC_DISPATCH_H(ppc, launch_accumulate_h, a, blocks, ppc, s);
}

// =============================================================================================
// Finalise a centroid set from the (all-reduced) exchange buffer — identical on every rank.
//   mode 0 (round r): early-stop check (clusterer.cpp:213), sums -> centroids with the
//          skipped cluster derived as colsum - others, empty clusters keep the previous
//          centroid (clusterer.cpp:184-186); member counts = the round's counts.
//   mode 1 (init):   centroids = seed HV bits, member counts 1 (clusterer.cpp:197-205).
//   mode 2 (given):  centroids already in Z (assign_labels on caller centroids).
//   mode 3 (update): like 0 but no skip and no early stop (update_centroids API).
// Always: norm2 of the new set and its B fragments. One warp per (32-bit word, cluster):
// lane b owns entry 32*word + b; lanes (plane, q) then gather the 8 entries of one B slot.
// =============================================================================================
__global__ void k_finish(int mode, uint32_t K, uint32_t P, uint32_t D, uint32_t W32, uint32_t W32P, uint32_t Dp,
                         const int32_t* __restrict__ xchg, const int32_t* __restrict__ colsum, uint32_t* Z,
                         uint32_t* __restrict__ run, uint8_t* bfrag, void* state, uint32_t round, int early_stop) {
    StateView st = StateView::at(state, K);
    const uint32_t p = round & 1, np = p ^ 1;  // set produced here is used by round+1
    const uint32_t* counts = reinterpret_cast<const uint32_t*>(xchg) + size_t(K) * Dp;
    if (mode == 0) {
        if (st.hdr->done) return;
        const uint32_t changed = counts[K];
        if (early_stop && round > 1 && changed == 0) {
            if (blockIdx.x == 0 && threadIdx.x == 0) st.hdr->done = 1;
            return;
        }
    }
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t word = gw / K, c = gw % K;
    if (word < W32) {
        const int skip = (mode == 0) ? int(pick_skip(st.cur + p * K, K)) : -1;
        const size_t i = size_t(word) * 32 + lane;
        const bool in = i < D;
        uint32_t z;
        if (mode == 0 && run) {  // incremental: xchg row c >= 1 holds the round's delta of cluster c
            // S_c = running sums + delta (written to parity np), S_0 = colsum - sum_{c >= 1} S_c
            uint32_t sc;
            if (c != 0) {
                sc = run[(size_t(p) * K + c) * Dp + i] + uint32_t(xchg[size_t(c) * Dp + i]);
                run[(size_t(np) * K + c) * Dp + i] = sc;
            } else {
                sc = uint32_t(colsum[i]);
                for (uint32_t o = 1; o < K; ++o)
                    sc -= run[(size_t(p) * K + o) * Dp + i] + uint32_t(xchg[size_t(o) * Dp + i]);
            }
            z = counts[c] != 0 ? sc : (in ? Z[size_t(c) * D + i] : 0u);  // empty clusters keep theirs
        } else if (mode == 2) {
            z = in ? Z[size_t(c) * D + i] : 0u;
        } else if (mode == 1 || counts[c] != 0) {
            if (int(c) == skip) {
                z = uint32_t(colsum[i]);
                for (uint32_t o = 0; o < K; ++o)
                    if (int(o) != skip) z -= uint32_t(xchg[size_t(o) * Dp + i]);
            } else {
                z = uint32_t(xchg[size_t(c) * Dp + i]);
            }
        } else {  // empty cluster keeps its previous centroid
            z = in ? Z[size_t(c) * D + i] : 0u;
        }
        if (!in) z = 0;
        if (in && mode != 2) Z[size_t(c) * D + i] = z;
        unsigned long long n2 = (unsigned long long)z * z;
        for (int o = 16; o; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        if (lane == 0) atomicAdd(st.norm2 + np * K + c, n2);
        // B fragments: column n = P*c + plane. This warp's word is word q = word & 3 of its
        // 4-word group; lane (plane, pair, s) writes the slot of MMA kk = 4*(word >> 2) +
        // 2*pair + s for column n, lane (n & 7) << 2 | q (unpack_pair): byte j of the low half
        // pairs bits (8j+6-4p, 8j+7-4p), byte j of the high half bits (8j+4-4p, 8j+5-4p);
        // the byte is 2*z6 + z7 (s = 0, u8) or 2*z6 - z7 (s = 1, s8) of the 6-bit planes.
        const uint32_t pl = lane >> 2, pr = (lane >> 1) & 1, sgn = lane & 1, qw = word & 3;
        uint64_t v = 0;
#pragma unroll
        for (uint32_t half = 0; half < 2; ++half)
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
                const uint32_t b6 = 8 * j + 6 - 4 * pr - 2 * half;
                const uint32_t z6 = (__shfl_sync(0xffffffffu, z, b6) >> (kPlaneBits * pl)) & 0x3Fu;
                const uint32_t z7 = (__shfl_sync(0xffffffffu, z, b6 + 1) >> (kPlaneBits * pl)) & 0x3Fu;
                const uint32_t byte = (sgn ? 2 * z6 - z7 : 2 * z6 + z7) & 0xFFu;
                v |= uint64_t(byte) << (8 * (half * 4 + j));
            }
        if (pl < P) {
            const uint32_t n = P * c + pl, nt = n >> 3, nl = n & 7, kk = 4 * (word >> 2) + 2 * pr + sgn;
            *reinterpret_cast<uint64_t*>(bfrag + ((size_t(nt) * W32P + kk) * 32 + ((nl << 2) | qw)) * 8) = v;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < K) {
        const uint32_t cc = threadIdx.x;
        if (mode == 1) st.cur[np * K + cc] = 1;
        else if (mode == 0 || mode == 3) st.cur[np * K + cc] = counts[cc];
    }
}

void launch_finish(const FinishArgs& a, cudaStream_t s) {
    const uint32_t threads = 256;
    const uint64_t total = uint64_t(a.W32) * a.K * 32;
    k_finish<<<uint32_t((total + threads - 1) / threads), threads, 0, s>>>(
        a.mode, a.K, a.P, a.D, a.W32, a.W32P, a.Dp, a.xchg, a.colsum, a.Z, a.run, a.bfrag, a.state, a.round,
        a.early_stop);
}

// Zero the accumulators of parity np before k_finish accumulates into them.
__global__ void k_prep_finish(void* state, uint32_t K, uint32_t np) {
    StateView st = StateView::at(state, K);
    for (uint32_t c = threadIdx.x; c < K; c += blockDim.x) st.norm2[np * K + c] = 0;
}
void launch_prep_finish(void* state, uint32_t K, uint32_t np, cudaStream_t s) {
    k_prep_finish<<<1, 64, 0, s>>>(state, K, np);
}

// =============================================================================================
// Generic round kernel (any K): assign_labels (clusterer.cpp:132-162).
//
// Persistent CTAs walk tiles of TP = 16*MT pixels, double buffered through cp.async.bulk
// (TMA engine, one copy per pixel row) on mbarriers. Warp g owns 32-word blocks of every HV
// (split-K), unpacks the packed bits into IMMA A fragments in registers (unpack_pair) and
// multiplies them with the 7-bit-plane B fragments of the centroids, NTG n-tiles at a time
// (B streamed from L2). Partial dots meet in shared memory; one thread per pixel recombines
// the planes in u64 and runs the exact 128-bit argmax. Member counts and the change count
// go to the exchange-buffer tail; the re-bundling runs in k_accumulate.
// =============================================================================================
template <int MT, int NTG, int TB>
__global__ void __launch_bounds__(TB, 1)
    k_round(const uint32_t* __restrict__ grid, uint64_t n, uint32_t S32, uint32_t SS, uint32_t W32P,
            uint32_t nwarp_words, uint32_t K, uint32_t P, uint32_t NT, const uint64_t* __restrict__ bfrag,
            uint32_t* labels, void* state, uint32_t round, uint32_t* __restrict__ tail) {
    constexpr uint32_t TP = 16 * MT;
    constexpr uint32_t NC = NTG * 8;  // columns per group
    extern __shared__ __align__(128) uint8_t smem[];
    StateView st = StateView::at(state, K);
    if (st.hdr->done) return;

    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t g8 = lane >> 2, q = lane & 3;
    const uint32_t parity = round & 1;
    const uint32_t NCT = NT * 8;  // all columns (P planes x K clusters, padded to n-tiles)

    uint32_t* tiles = reinterpret_cast<uint32_t*>(smem);
    const size_t tile_words = size_t(TP) * SS;
    int32_t* part = reinterpret_cast<int32_t*>(tiles + 2 * tile_words + 32);     // [nwarps][TP][NC]
    uint32_t* red = reinterpret_cast<uint32_t*>(part + size_t(nwarps) * TP * NC);  // [TP][NCT]
    uint32_t* s_misc = red + TP * NCT;  // [0] changed, [2..2+K) counts
    unsigned long long* s_n2 = reinterpret_cast<unsigned long long*>(s_misc + ((2 + K + 1) & ~1u));  // [K]
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_n2 + K);

    const uint64_t ntiles = (n + TP - 1) / TP;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_fence_init();
        s_misc[0] = 0;
    }
    for (uint32_t c = tid; c < K; c += blockDim.x) {
        s_misc[2 + c] = 0;
        s_n2[c] = st.norm2[parity * K + c];
    }
    if (blockIdx.x == 0 && tid == 0) st.hdr->rounds_run = round;
    __syncthreads();

    auto issue = [&](uint64_t tile, uint32_t buf) {
        const uint64_t px0 = tile * TP;
        const uint32_t npx = uint32_t(umin64(TP, n - px0));
        if (lane == 0) mbar_expect_tx(&bars[buf], npx * S32 * 4);
        __syncwarp();
        for (uint32_t r = lane; r < npx; r += 32)
            bulk_g2s(tiles + buf * tile_words + size_t(r) * SS, grid + (px0 + r) * S32, S32 * 4, &bars[buf]);
    };
    if (warp == 0) {
        fence_proxy_async();
        for (uint32_t b = 0; b < 2; ++b) {
            const uint64_t tile = blockIdx.x + uint64_t(b) * gridDim.x;
            if (tile < ntiles) issue(tile, b);
        }
    }
    const uint32_t ngroups = (NT + NTG - 1) / NTG;
    const uint32_t pw4[4] = {1u, opaque(4u), opaque(16u), opaque(64u)};  // shifts 0, 2, 4, 6

    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t buf = it & 1;
        mbar_wait(&bars[buf], (it >> 1) & 1);
        const uint32_t* T = tiles + buf * tile_words;
        const uint64_t px0 = tile * TP;
        const uint32_t npx = uint32_t(umin64(TP, n - px0));
        const uint32_t old = (tid < npx) ? labels[px0 + tid] : 0u;

        for (uint32_t grp = 0; grp < ngroups; ++grp) {
            int acc[MT][NTG][4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NTG; ++nt)
#pragma unroll
                    for (int r = 0; r < 4; ++r) acc[mt][nt][r] = 0;

            for (uint32_t wb = warp; wb < nwarp_words; wb += nwarps) {
                const uint32_t wbase = wb * 32;
                const uint32_t* Tq = T + wbase + q;
#pragma unroll 2
                for (int k4 = 0; k4 < 8; ++k4) {
                    uint32_t sl[MT][4], sh[MT][4];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        sl[mt][0] = Tq[size_t(16 * mt + g8) * SS + 4 * k4];
                        sh[mt][0] = Tq[size_t(16 * mt + g8 + 8) * SS + 4 * k4];
#pragma unroll
                        for (int e = 1; e < 4; ++e) {
                            sl[mt][e] = shl_fma(sl[mt][0], pw4[e]);
                            sh[mt][e] = shl_fma(sh[mt][0], pw4[e]);
                        }
                    }
#pragma unroll
                    for (int pr = 0; pr < 2; ++pr) {
                        const int kk = 4 * k4 + 2 * pr;
                        uint32_t bu0[NTG], bu1[NTG], bs0[NTG], bs1[NTG];
#pragma unroll
                        for (int nt = 0; nt < NTG; ++nt) {
                            const uint32_t ntg = grp * NTG + nt;
                            uint64_t u = 0, v = 0;
                            if (ntg < NT) {
                                u = __ldg(bfrag + ((size_t(ntg) * W32P + wbase + kk) * 32 + lane));
                                v = __ldg(bfrag + ((size_t(ntg) * W32P + wbase + kk + 1) * 32 + lane));
                            }
                            bu0[nt] = uint32_t(u);
                            bu1[nt] = uint32_t(u >> 32);
                            bs0[nt] = uint32_t(v);
                            bs1[nt] = uint32_t(v >> 32);
                        }
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            uint32_t a[4];
                            unpack_pair(a, sl[mt][2 * pr], sh[mt][2 * pr], sl[mt][2 * pr + 1], sh[mt][2 * pr + 1]);
#pragma unroll
                            for (int nt = 0; nt < NTG; ++nt) {
                                imma16832(acc[mt][nt], a, bu0[nt], bu1[nt]);
                                imma16832_s8(acc[mt][nt], a, bs0[nt], bs1[nt]);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NTG; ++nt) {
                    int32_t* row0 = part + (size_t(warp) * TP + 16 * mt + g8) * NC + nt * 8 + 2 * q;
                    *reinterpret_cast<int2*>(row0) = make_int2(acc[mt][nt][0], acc[mt][nt][1]);
                    *reinterpret_cast<int2*>(row0 + 8 * NC) = make_int2(acc[mt][nt][2], acc[mt][nt][3]);
                }
            __syncthreads();
            for (uint32_t e = tid; e < TP * NC; e += blockDim.x) {
                const uint32_t px = e / NC, col = grp * NC + e % NC;
                if (col >= NCT) continue;
                int32_t s = 0;
                for (uint32_t w = 0; w < nwarps; ++w) s += part[size_t(w) * TP * NC + e];
                red[px * NCT + col] = uint32_t(s) >> 8;  // remove the 256 scale of the pair packing (exact)
            }
            __syncthreads();  // red complete for this group; part free for the next group
        }
        if (tid < npx) {
            const uint32_t* rr = red + tid * NCT;
            uint32_t best = 0, nwrap = 0;
            unsigned long long bdot = 0, bn2 = 0;
            for (uint32_t c = 0; c < K; ++c) {
                unsigned long long d = 0;
                for (uint32_t pl = 0; pl < P; ++pl) d += (unsigned long long)rr[P * c + pl] << (kPlaneBits * pl);
                const unsigned long long n2 = s_n2[c];
                if (c > 0) nwrap += compare_wraps(d, n2, bdot, bn2);
                if (c == 0 || strictly_closer(d, n2, bdot, bn2)) {
                    best = c;
                    bdot = d;
                    bn2 = n2;
                }
            }
            labels[px0 + tid] = best;
            if (nwrap) atomicAdd(st.wraps + (round - 1), (unsigned long long)nwrap);
            if (old != best) atomicAdd(&s_misc[0], 1u);
            atomicAdd(&s_misc[2 + best], 1u);
        }
        __syncthreads();  // every read of this buffer (and of red) is done
        if (warp == 0) {
            const uint64_t nxt = tile + 2ull * gridDim.x;
            if (nxt < ntiles) {
                issue(nxt, buf);
            }
        }
    }
    __syncthreads();
    if (tid == 0 && s_misc[0]) atomicAdd(tail + K, s_misc[0]);
    for (uint32_t c = tid; c < K; c += blockDim.x)
        if (s_misc[2 + c]) atomicAdd(tail + c, s_misc[2 + c]);
}

size_t round_smem_bytes(uint32_t MT, uint32_t NTG, uint32_t SS, uint32_t nwarps, uint32_t K, uint32_t NT) {
    const uint32_t TP = 16 * MT, NC = 8 * NTG;
    size_t b = (2 * size_t(TP) * SS + 32) * 4;  // tiles + slack for the last row's overrun
    b += size_t(nwarps) * TP * NC * 4;           // part
    b += size_t(TP) * NT * 8 * 4;                // red (all columns)
    b += ((2 + K + 1) & ~size_t(1)) * 4;         // s_misc
    b += size_t(K) * 8;                          // s_n2
    b += 2 * 8;                                  // mbarriers
    return b;
}

template <int MT, int NTG>
static cudaError_t launch_round_t(const RoundArgs& a, uint32_t nwarps, cudaStream_t s) {
    auto kern = nwarps <= 12 ? k_round<MT, NTG, 384> : k_round<MT, NTG, 512>;
    const size_t smem = round_smem_bytes(MT, NTG, a.SS, nwarps, a.K, a.NT);
    cudaError_t e = ensure_dynamic_smem((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<a.ctas, nwarps * 32, smem, s>>>(a.grid, a.n, a.S32, a.SS, a.W32P, a.nwarp_words, a.K, a.P, a.NT, a.bfrag,
                                           a.labels, a.state, a.round, reinterpret_cast<uint32_t*>(a.xchg) +
                                                                           size_t(a.K) * a.Dp);
    return cudaGetLastError();
}

// =============================================================================================
// Fused round kernel (one n-tile of centroid planes, K * P <= 8): assign_labels
// (clusterer.cpp:132-162) fused with the accumulation of update_centroids
// (clusterer.cpp:164-188), each pixel HV crossing HBM once per round. Persistent CTAs, one per
// SM, walk 32-pixel tiles through an NB-deep ring of TMA bulk copies. Warp roles:
//   NMW MMA warps   wait tile t -> pair-packed IMMA k-loop over their WPW words (B fragments in
//                   2*WPW registers) -> arrive buf_free[t] -> split-K partials to part[t%2]
//                   -> arrive part_full[t%2].
//   epilogue warp   wait part_full -> reduce the partials (lane = pixel), exact u64 dots,
//                   128-bit argmax, labels, counts, update list -> arrive list_ready[t].
//   NRW fold warps  wait list_ready[t] -> fold tile t's update list (the pixels of the cluster
//                   not derived from the column sums) into Harley-Seal counters, one thread
//                   per word column (<= 4 columns each) -> arrive buf_free[t].
//   producer warp   wait buf_free[t] -> TMA of tile t+NB into that buffer.
// Every hand-off is an mbarrier; a buffer is refilled the moment its last reader is done.
// Ring-slot indexed list[] / list_ready[]: the epilogue writes list[t%NB] for tile t only
// after tile t landed, i.e. after buf_free[t-NB] (all folding of t-NB) - no overwrite race.
// part[] is two-deep: an MMA warp waits list_ready[t-2] (the epilogue of t-2 has read part)
// before it overwrites part[t%2].
// =============================================================================================
#ifdef SEGHDC_TRACE
// diagnostic build only (-DSEGHDC_TRACE): per-CTA clock64() stamps of the first 64 tiles
// events 0..7 as in tools/trace_round.py, 8 + 2w / 9 + 2w: k-loop start / end of MMA warp w
constexpr int kTraceEv = 48;
__device__ unsigned long long g_trace[148 * 64 * kTraceEv];
#define SEGHDC_TR(ev, it)                                                              \
    do {                                                                               \
        if (lane == 0 && blockIdx.x < 148 && (it) < 64 && (ev) < kTraceEv)             \
            g_trace[(size_t(blockIdx.x) * 64 + (it)) * kTraceEv + (ev)] = clock64();   \
    } while (0)
#else
#define SEGHDC_TR(ev, it) ((void)0)
#endif
template <int WPW, bool UPD, int H, int NMW, int NRW>
__global__ void __launch_bounds__((NMW + NRW + 2) * 32, 1)
    k_round_fused(const uint32_t* __restrict__ grid, uint64_t n, uint32_t S32, uint32_t SS, uint32_t W32, uint32_t K,
                  const uint64_t* __restrict__ bfrag, uint32_t* labels, void* state, uint32_t round, int do_update,
                  uint32_t* __restrict__ xchg, uint32_t Dp) {
    constexpr uint32_t MT = 2, TP = 32, NB = 4;
    constexpr int CPTMAX = 4;  // word columns per fold thread
    constexpr uint32_t NRT = NRW * 32;
    constexpr uint32_t NTHREADS = (NMW + NRW + 2) * 32;
    extern __shared__ __align__(128) uint8_t smem[];
    StateView st = StateView::at(state, K);
    if (st.hdr->done) return;

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t parity = round & 1;
    uint32_t* tail = xchg + size_t(K) * Dp;  // [K counts | changed]

    uint32_t* tiles = reinterpret_cast<uint32_t*>(smem);
    const size_t tile_words = size_t(TP) * SS;
    uint32_t* s_old = tiles + NB * tile_words + 32;                           // [NB][TP] previous labels
    int32_t* part = reinterpret_cast<int32_t*>(s_old + NB * TP);              // [2][NMW][TP][8]
    uint32_t* s_list = reinterpret_cast<uint32_t*>(part + 2 * NMW * TP * 8);  // [NB][TP]
    uint32_t* s_listn = s_list + NB * TP;                                     // [NB]
    uint32_t* s_misc = s_listn + NB;                                          // [0] skip
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_misc + 2);                 // 8-byte aligned
    uint64_t* full = bars;                   // [NB] tile data landed (TMA)
    uint64_t* buf_free = bars + NB;          // [NB] MMA + fold warps done with the buffer
    uint64_t* list_ready = bars + 2 * NB;    // [NB] labels + update list of the tile ready
    uint64_t* part_full = bars + 3 * NB;     // [2] partials written

    const uint64_t ntiles = (n + TP - 1) / TP;
    const uint32_t my_tiles = blockIdx.x < ntiles ? uint32_t((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    if (tid == 0) {
        for (uint32_t b = 0; b < NB; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&buf_free[b], (NMW + NRW) * 32);
            mbar_init(&list_ready[b], 32);
        }
        for (uint32_t b = 0; b < 2; ++b) mbar_init(&part_full[b], NMW * 32);
        mbar_fence_init();
        s_misc[0] = pick_skip(st.cur + parity * K, K);
    }
    if (blockIdx.x == 0 && tid == 0) st.hdr->rounds_run = round;
    __syncthreads();
    const uint32_t upd_c = 1 - s_misc[0];  // K == 2 under UPD
    const bool folding = UPD && do_update;
    auto end_barrier = [&]() {  // all tiles consumed: the ring becomes the flush scratch
        if (folding) asm volatile("bar.sync 1, %0;" ::"r"(NTHREADS));
    };

    if (warp == NMW + NRW + 1) {
        // ----------------------------------------------------------------------- producer warp
        auto issue = [&](uint32_t it) {
            const uint32_t b = it % NB;
            const uint64_t px0 = (blockIdx.x + uint64_t(it) * gridDim.x) * TP;
            const uint32_t npx = uint32_t(umin64(TP, n - px0));
            const uint32_t lab_bytes = (npx * 4 + 15) & ~15u;  // labels buffer padded to 16 B
            if (lane == 0) mbar_expect_tx(&full[b], npx * S32 * 4 + lab_bytes);
            __syncwarp();
            SEGHDC_TR(0, it);
            if (lane == 0) bulk_g2s(s_old + b * TP, labels + px0, lab_bytes, &full[b]);
            if (SS == S32) {  // unpadded rows: the tile is one contiguous block
                if (lane == 1) bulk_g2s(tiles + b * tile_words, grid + px0 * S32, npx * S32 * 4, &full[b]);
            } else if (lane < npx) {
                bulk_g2s(tiles + b * tile_words + size_t(lane) * SS, grid + (px0 + lane) * S32, S32 * 4, &full[b]);
            }
        };
        for (uint32_t it = 0; it < NB && it < my_tiles; ++it) issue(it);
        for (uint32_t it = 0; it + NB < my_tiles; ++it) {
            mbar_wait(&buf_free[it % NB], (it / NB) & 1);
            SEGHDC_TR(5, it);
            issue(it + NB);
        }
        end_barrier();
        return;
    }

    if (warp == NMW + NRW) {
        // ----------------------------------------------------------------------- epilogue warp
        const unsigned long long n2_0 = st.norm2[parity * K], n2_1 = K > 1 ? st.norm2[parity * K + 1] : 0ull;
        uint32_t changed = 0, cnt1 = 0, total = 0, nwrap = 0;
        for (uint32_t it = 0; it < my_tiles; ++it) {
            const uint32_t pb = it & 1, b = it % NB;
            const uint64_t px0 = (blockIdx.x + uint64_t(it) * gridDim.x) * TP;
            const uint32_t npx = uint32_t(umin64(TP, n - px0));
            mbar_wait(&part_full[pb], (it >> 1) & 1);
            SEGHDC_TR(3, it);
            const int32_t* pp = part + size_t(pb) * NMW * TP * 8 + lane * 8;
            int32_t col[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
            for (uint32_t w = 0; w < NMW; ++w) {
                const int4 lo = *reinterpret_cast<const int4*>(pp + size_t(w) * TP * 8);
                const int4 hi = *reinterpret_cast<const int4*>(pp + size_t(w) * TP * 8 + 4);
                col[0] += lo.x; col[1] += lo.y; col[2] += lo.z; col[3] += lo.w;
                col[4] += hi.x; col[5] += hi.y; col[6] += hi.z; col[7] += hi.w;
            }
            // exact dots: column n = 4*c + plane (MMA scale already removed). K*P <= 8 here, so
            // K == 2 means P == 4; K == 1 needs no dots at all.
            const unsigned long long d0 = (unsigned long long)uint32_t(col[0]) +
                                          ((unsigned long long)uint32_t(col[1]) << kPlaneBits) +
                                          ((unsigned long long)uint32_t(col[2]) << (2 * kPlaneBits)) +
                                          ((unsigned long long)uint32_t(col[3]) << (3 * kPlaneBits));
            const unsigned long long d1 = (unsigned long long)uint32_t(col[4]) +
                                          ((unsigned long long)uint32_t(col[5]) << kPlaneBits) +
                                          ((unsigned long long)uint32_t(col[6]) << (2 * kPlaneBits)) +
                                          ((unsigned long long)uint32_t(col[7]) << (3 * kPlaneBits));
            const uint32_t best = (K > 1 && strictly_closer(d1, n2_1, d0, n2_0)) ? 1u : 0u;
            const bool live = lane < npx;
            if (K > 1 && live) nwrap += compare_wraps(d1, n2_1, d0, n2_0);
            const uint32_t old = s_old[b * TP + lane];
            if (live) {
                labels[px0 + lane] = best;
                changed += old != best;
                cnt1 += best;
            }
            total += npx;
            if constexpr (UPD) {
                const bool take = do_update && live && best == upd_c;
                const uint32_t m = __ballot_sync(0xffffffffu, take);
                if (take) s_list[b * TP + __popc(m & ((1u << lane) - 1))] = lane;
                if (lane == 0) s_listn[b] = __popc(m);
            }
            mbar_arrive(&list_ready[b]);
            SEGHDC_TR(4, it);
        }
        for (int o = 16; o; o >>= 1) {
            changed += __shfl_xor_sync(0xffffffffu, changed, o);
            cnt1 += __shfl_xor_sync(0xffffffffu, cnt1, o);
            nwrap += __shfl_xor_sync(0xffffffffu, nwrap, o);
        }
        if (lane == 0) {
            if (nwrap) atomicAdd(st.wraps + (round - 1), (unsigned long long)nwrap);
            if (changed) atomicAdd(tail + K, changed);
            if (total - cnt1) atomicAdd(tail, total - cnt1);
            if (K > 1 && cnt1) atomicAdd(tail + 1, cnt1);
        }
        end_barrier();
        return;
    }

    if (warp >= NMW) {
        // --------------------------------------------------------------------------- fold warps
        const uint32_t rt = tid - NMW * 32;
        const uint32_t cpt = (W32 + NRT - 1) / NRT;
        BitCounter<UPD ? H : 1> cnt[CPTMAX];
        if constexpr (UPD)
#pragma unroll
            for (int c = 0; c < CPTMAX; ++c) cnt[c].reset();
        for (uint32_t it = 0; it < my_tiles; ++it) {
            const uint32_t b = it % NB;
            mbar_wait(&list_ready[b], (it / NB) & 1);
            if constexpr (UPD) {
                if (do_update) {
                    const uint32_t m = s_listn[b];
                    const uint32_t* T = tiles + b * tile_words;
                    const uint32_t* L = s_list + b * TP;
#pragma unroll
                    for (int c = 0; c < CPTMAX; ++c) {
                        const uint32_t colw = rt + c * NRT;
                        if (uint32_t(c) < cpt && colw < W32) {
                            for (uint32_t e = 0; e < m; e += 16) {
                                uint32_t x[16];
#pragma unroll
                                for (int u = 0; u < 16; ++u) x[u] = (e + u < m) ? T[size_t(L[e + u]) * SS + colw] : 0u;
                                cnt[c].add16(x);
                            }
                        }
                    }
                }
            }
            if (warp == NMW) SEGHDC_TR(6, it);
            mbar_arrive(&buf_free[b]);
        }
        end_barrier();
        if constexpr (UPD) {
            if (do_update) {
#pragma unroll
                for (int c = 0; c < CPTMAX; ++c)
                    if (uint32_t(c) < cpt)
                        flush_warp_atomic(cnt[c], tiles + (rt >> 5) * (32 * 33), xchg + size_t(upd_c) * Dp,
                                          (rt & ~31u) + c * NRT, W32);
            }
        }
        return;
    }

    // ---------------------------------------------------------------------- MMA warps
    const uint32_t g8 = lane >> 2, q = lane & 3;
    uint32_t breg[WPW][2];
#pragma unroll
    for (int kk = 0; kk < WPW; ++kk) {
        const uint64_t v = bfrag[(size_t(warp) * WPW + kk) * 32 + lane];
        breg[kk][0] = uint32_t(v);
        breg[kk][1] = uint32_t(v >> 32);
    }
    const uint32_t wbase = warp * WPW;
    const uint32_t pw4[4] = {1u, opaque(4u), opaque(16u), opaque(64u)};  // shifts 0, 2, 4, 6

    for (uint32_t it = 0; it < my_tiles; ++it) {
        const uint32_t b = it % NB, pb = it & 1;
        mbar_wait(&full[b], (it / NB) & 1);
        if (warp == 0) SEGHDC_TR(1, it);
        SEGHDC_TR(8 + 2 * warp, it);
        const uint32_t* Tq = tiles + b * tile_words + wbase + q;
        int acc[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[mt][r] = 0;
#pragma unroll
        for (int k4 = 0; k4 < WPW / 4; ++k4) {
            uint32_t sl[MT][4], sh[MT][4];  // row words shifted by 0, 2, 4, 6
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                sl[mt][0] = Tq[size_t(16 * mt + g8) * SS + 4 * k4];
                sh[mt][0] = Tq[size_t(16 * mt + g8 + 8) * SS + 4 * k4];
#pragma unroll
                for (int e = 1; e < 4; ++e) {
                    sl[mt][e] = shl_fma(sl[mt][0], pw4[e]);
                    sh[mt][e] = shl_fma(sh[mt][0], pw4[e]);
                }
            }
#pragma unroll
            for (int pr = 0; pr < 2; ++pr) {
                const int kk = 4 * k4 + 2 * pr;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    uint32_t a[4];
                    unpack_pair(a, sl[mt][2 * pr], sh[mt][2 * pr], sl[mt][2 * pr + 1], sh[mt][2 * pr + 1]);
                    imma16832(acc[mt], a, breg[kk][0], breg[kk][1]);
                    imma16832_s8(acc[mt], a, breg[kk + 1][0], breg[kk + 1][1]);
                }
            }
        }
        if (warp == 0) SEGHDC_TR(2, it);
        if (warp == NMW - 1) SEGHDC_TR(7, it);
        SEGHDC_TR(9 + 2 * warp, it);
        mbar_arrive(&buf_free[b]);  // this warp is done reading the tile
        if (it >= 2) mbar_wait(&list_ready[(it - 2) % NB], ((it - 2) / NB) & 1);  // part[pb] consumed
        int32_t* pw = part + (size_t(pb) * NMW + warp) * TP * 8;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            int32_t* row0 = pw + (16 * mt + g8) * 8 + 2 * q;  // scale 256 removed (exact)
            *reinterpret_cast<int2*>(row0) = make_int2(int(uint32_t(acc[mt][0]) >> 8), int(uint32_t(acc[mt][1]) >> 8));
            *reinterpret_cast<int2*>(row0 + 64) =
                make_int2(int(uint32_t(acc[mt][2]) >> 8), int(uint32_t(acc[mt][3]) >> 8));
        }
        mbar_arrive(&part_full[pb]);
    }
    end_barrier();
}

size_t fused_smem_bytes(uint32_t SS, uint32_t nmw, uint32_t nrw) {
    const uint32_t TP = 32, NB = 4;
    size_t b = (NB * size_t(TP) * SS + 32) * 4;  // tile ring + overrun slack
    b += NB * TP * 4;                            // s_old
    b += 2 * size_t(nmw) * TP * 8 * 4;           // part
    b += (NB * TP + NB + 2) * 4;                 // s_list, s_listn, s_misc
    b += (3 * NB + 2) * 8 + 8;                   // mbarriers (+ alignment)
    return std::max<size_t>(b, size_t(nrw) * 32 * 33 * 4);
}

template <int WPW, bool UPD, int H, int NMW, int NRW>
static cudaError_t launch_fused_t(const RoundArgs& a, cudaStream_t s) {
    auto kern = k_round_fused<WPW, UPD, H, NMW, NRW>;
    const size_t smem = fused_smem_bytes(a.SS, NMW, NRW);
    cudaError_t e = ensure_dynamic_smem((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<a.ctas, (NMW + NRW + 2) * 32, smem, s>>>(a.grid, a.n, a.S32, a.SS, a.W32, a.K, a.bfrag, a.labels, a.state,
                                                    a.round, a.do_update, reinterpret_cast<uint32_t*>(a.xchg), a.Dp);
    return cudaGetLastError();
}

template <int WPW, int NMW, int NRW>
static cudaError_t launch_fused_h(const RoundArgs& a, cudaStream_t s) {
    if (a.K != 2) return launch_fused_t<WPW, false, 1, NMW, NRW>(a, s);
    const uint64_t per_cta = ((a.n + a.ctas - 1) / a.ctas + 31) & ~uint64_t(31);
    if (per_cta <= counter_capacity<8>()) return launch_fused_t<WPW, true, 8, NMW, NRW>(a, s);
    if (per_cta <= counter_capacity<12>()) return launch_fused_t<WPW, true, 12, NMW, NRW>(a, s);
    return launch_fused_t<WPW, true, 20, NMW, NRW>(a, s);
}

// Plan: which instantiation handles (K, P, D). Returns false if no kernel fits.
bool plan_round(uint32_t K, uint32_t P, uint32_t W32, uint32_t SS, RoundPlan& p, size_t smem_limit) {
    p.nwarp_words = (W32 + 31) / 32;
    p.nt = (K * P + 7) / 8;
    p.fused = false;
    p.tc = false;
    if (tc_supported(K, W32) && tc_smem_bytes(K, W32) <= smem_limit) {
        // tcgen05 kernel. The IMMA plan below is still computed: it serves only the shapes no
        // tcgen05 layout covers (D <= 1024, K > 8, centroid entries beyond the layout's digits)
        p.tc = true;
    }
    if (p.nt == 1) {
        // (MMA warps, words per warp, fold warps): MMA warps in multiples of 4 (equal k-loop
        // load per SM sub-partition), B fragments in 2*wpw registers, fold threads own <= 4
        // word columns.
        // SEGHDC_FUSED=<nmw>,<nrw> forces a shape (A/B testing).
        static const uint32_t cand[][3] = {{4, 20, 1}, {4, 28, 1}, {4, 32, 1}, {8, 20, 2}, {8, 28, 2}, {8, 32, 2},
                                           {8, 40, 4}, {12, 28, 4}, {16, 20, 4}};
        uint32_t f_nmw = 0, f_nrw = 0;
        const char* force = getenv("SEGHDC_FUSED");
        const bool forced = force && *force && sscanf(force, "%u,%u", &f_nmw, &f_nrw) == 2;
        for (const auto& c : cand) {
            if (forced && (c[0] != f_nmw || c[2] != f_nrw)) continue;
            if (c[0] * c[1] < W32 || c[2] * 32 * 4 < W32) continue;
            if (fused_smem_bytes(SS, c[0], c[2]) > smem_limit) continue;
            p.fused = true;
            p.nwarps = c[0];
            p.wpw = c[1];
            p.nrw = c[2];
            p.w32p = c[0] * c[1];
            p.mt = 2;
            p.ntg = 1;
            return true;
        }
    }
    p.ntg = 4;
    p.wpw = 32;
    p.w32p = p.nwarp_words * 32;
    // at least 2 warps: the epilogue needs one thread per pixel of a 64-pixel tile
    p.nwarps = std::max<uint32_t>(2, std::min<uint32_t>(p.nwarp_words, 16));
    for (uint32_t mt : {4u, 2u, 1u}) {
        if (round_smem_bytes(mt, p.ntg, SS, p.nwarps, K, p.nt) <= smem_limit) {
            p.mt = mt;
            return true;
        }
    }
    return false;
}

cudaError_t launch_round(const RoundArgs& a, const RoundPlan& p, cudaStream_t s) {
    if (p.tc) return launch_round_tc(a, s);
    if (p.fused) {
        switch (p.nwarps * 1000 + p.wpw * 10 + p.nrw) {
            case 4201: return launch_fused_h<20, 4, 1>(a, s);
            case 4281: return launch_fused_h<28, 4, 1>(a, s);
            case 4321: return launch_fused_h<32, 4, 1>(a, s);
            case 8202: return launch_fused_h<20, 8, 2>(a, s);
            case 8282: return launch_fused_h<28, 8, 2>(a, s);
            case 8322: return launch_fused_h<32, 8, 2>(a, s);
            case 12284: return launch_fused_h<28, 12, 4>(a, s);
            case 8404: return launch_fused_h<40, 8, 4>(a, s);
            case 16204: return launch_fused_h<20, 16, 4>(a, s);
            default: return cudaErrorInvalidConfiguration;
        }
    }
    switch (p.mt) {
        case 4: return launch_round_t<4, 4>(a, p.nwarps, s);
        case 2: return launch_round_t<2, 4>(a, p.nwarps, s);
        default: return launch_round_t<1, 4>(a, p.nwarps, s);
    }
}

#ifdef SEGHDC_TRACE
void read_trace(void* dst) { cudaMemcpyFromSymbol(dst, g_trace, sizeof(g_trace)); }
#endif
#ifdef SEGHDC_CHECKED
unsigned int check_line_kernels() { return take_check_line(); }
#endif

}  // namespace seghdc_dev

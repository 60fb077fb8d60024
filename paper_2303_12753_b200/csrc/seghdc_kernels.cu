// B200 (sm_100a) kernels of the SegHDC hot path and their launchers.
// See kernels.cuh for the device data layout and DESIGN.md for the rooflines.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "launch.h"

namespace seghdc_dev {

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }

// =============================================================================================
// encode_image (reference pixel_pipeline.cpp:92-126): grid[p] = row[i] ^ col[j] ^ ^_ch wid[ch][v]
// One CTA per PXB consecutive pixels; thread t owns u32 word column t (coalesced 128-B stores
// per warp per pixel). Tables are the reference's u64 words read as u32 (same bytes).
// =============================================================================================
template <int C>
__global__ void __launch_bounds__(256) k_encode(const uint8_t* __restrict__ img, uint32_t w,
                                                 uint64_t pix_begin, uint64_t pix_end,
                                                 const uint32_t* __restrict__ row,
                                                 const uint32_t* __restrict__ col,
                                                 const uint32_t* __restrict__ wid, uint32_t wref,
                                                 uint32_t S32, uint32_t pxb, uint32_t* __restrict__ grid) {
    const uint64_t p0 = pix_begin + uint64_t(blockIdx.x) * pxb;
    const uint64_t p1 = p0 + pxb < pix_end ? p0 + pxb : pix_end;
    for (uint32_t t = threadIdx.x; t < S32; t += blockDim.x) {
        const bool live = t < wref;
        for (uint64_t p = p0; p < p1; ++p) {
            const uint32_t i = uint32_t(p / w), j = uint32_t(p - uint64_t(i) * w);
            uint32_t v = 0;
            if (live) {
                v = __ldg(row + size_t(i) * wref + t) ^ __ldg(col + size_t(j) * wref + t);
#pragma unroll
                for (int ch = 0; ch < C; ++ch) {
                    const uint32_t val = img[p * C + ch];
                    v ^= __ldg(wid + (size_t(ch) * 256 + val) * wref + t);
                }
            }
            grid[(p - pix_begin) * S32 + t] = v;
        }
    }
}

void launch_encode(const EncodeArgs& a, cudaStream_t s) {
    const uint32_t pxb = 16;
    const uint64_t n = a.pix_end - a.pix_begin;
    if (n == 0) return;
    const uint32_t blocks = uint32_t((n + pxb - 1) / pxb);
    const uint32_t threads = std::min<uint32_t>(256, ((a.S32 + 31) / 32) * 32);
    if (a.c == 1)
        k_encode<1><<<blocks, threads, 0, s>>>(a.img, a.w, a.pix_begin, a.pix_end, a.row, a.col, a.wid, a.wref,
                                               a.S32, pxb, a.grid);
    else
        k_encode<3><<<blocks, threads, 0, s>>>(a.img, a.w, a.pix_begin, a.pix_end, a.row, a.col, a.wid, a.wref,
                                               a.S32, pxb, a.grid);
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

__global__ void k_seed_minmax(const uint8_t* __restrict__ img, uint64_t n, uint32_t c,
                              unsigned long long* slots) {
    unsigned long long mn = ~0ull, mx = ~0ull;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t key = color_key(img, p, c);
        mn = umin64(mn, (key << 32) | p);
        mx = umin64(mx, ((0xFFFFull - key) << 32) | p);
    }
    for (int o = 16; o; o >>= 1) {
        mn = umin64(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = umin64(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(slots + 0, mn);
        atomicMin(slots + 1, mx);
    }
}

// Decide min/max seeds or the uniform fallback (clusterer.cpp:83-99). Single thread.
__global__ void k_seed_post(unsigned long long* slots, uint64_t* seeds, uint32_t K, uint32_t h, uint32_t w,
                            RoundState* hdr) {
    const uint64_t mn_key = slots[0] >> 32, mx_key = 0xFFFFull - (slots[1] >> 32);
    if (mn_key == mx_key) {
        hdr->uniform = 1;
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
    hdr->uniform = 0;
    seeds[0] = slots[0] & 0xFFFFFFFFull;
    if (K >= 2) seeds[1] = slots[1] & 0xFFFFFFFFull;
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
    for (int o = 16; o; o >>= 1) best = umin64(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMin(slots + 2 + s, best);
}

__global__ void k_seed_collect(uint64_t* seeds, const unsigned long long* slots, uint32_t K, const RoundState* hdr) {
    if (hdr->uniform) return;
    for (uint32_t s = 2 + threadIdx.x; s < K; s += blockDim.x) seeds[s] = slots[2 + s] & 0xFFFFFFFFull;
}

void launch_select_seeds(const SeedArgs& a, cudaStream_t s) {
    cudaMemsetAsync(a.slots, 0xFF, (2 + a.K) * sizeof(unsigned long long), s);
    const uint32_t blocks = uint32_t(std::min<uint64_t>((a.n + 255) / 256, 148 * 8));
    k_seed_minmax<<<blocks, 256, 0, s>>>(a.img, a.n, a.c, a.slots);
    k_seed_post<<<1, 1, 0, s>>>(a.slots, a.seeds, a.K, a.h, a.w, a.hdr);
    for (uint32_t st = 2; st < a.K; ++st)
        k_seed_greedy<<<blocks, 256, 0, s>>>(a.img, a.n, a.c, st, a.min_dist, a.seeds, a.slots, a.hdr);
    if (a.K > 2) k_seed_collect<<<1, 32, 0, s>>>(a.seeds, a.slots, a.K, a.hdr);
}

// =============================================================================================
// Seed centroids (clusterer.cpp:197-205): xchg[c][i] = bit i of the seed pixel's HV when the
// pixel lies in this rank's shard, else 0 (an all-reduce then yields the full seed HVs).
// =============================================================================================
__global__ void k_init_seeds(const uint32_t* __restrict__ grid, uint32_t S32, uint64_t pix_begin, uint64_t n_local,
                             const uint64_t* seeds, uint32_t K, uint32_t W32, uint32_t Dp, int32_t* xchg) {
    const uint32_t c = blockIdx.y;
    const uint64_t sp = seeds[c];
    const bool local = sp >= pix_begin && sp < pix_begin + n_local;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < Dp; i += gridDim.x * blockDim.x) {
        uint32_t bit = 0;
        if (local && (i >> 5) < W32) bit = (grid[(sp - pix_begin) * S32 + (i >> 5)] >> (i & 31)) & 1u;
        xchg[size_t(c) * Dp + i] = int32_t(bit);
    }
}

void launch_init_seeds(const InitSeedArgs& a, cudaStream_t s) {
    dim3 g((a.Dp + 255) / 256, a.K);
    k_init_seeds<<<g, 256, 0, s>>>(a.grid, a.S32, a.pix_begin, a.n_local, a.seeds, a.K, a.W32, a.Dp, a.xchg);
}

// =============================================================================================
// Standalone bit-sliced accumulation (update_centroids, clusterer.cpp:164-188, without the
// fused assignment; also the column sums "colsum" when labels == nullptr).
// CTA = (pixel range, 1024-word column block). For each cluster c != skip the CTA compacts
// the pixels of its range labelled c and feeds their words through one Harley-Seal counter
// per word column, so every pixel HV is read exactly once regardless of K.
// =============================================================================================
template <int H>
__global__ void __launch_bounds__(512) k_accumulate(const uint32_t* __restrict__ grid, uint32_t S32, uint32_t W32,
                                                     uint64_t n, uint64_t ppc, const uint32_t* __restrict__ labels,
                                                     uint32_t K, int skip_mode, void* state, uint32_t parity,
                                                     uint32_t* __restrict__ partials, uint32_t Dp, int count_members) {
    constexpr uint32_t CHUNK = 4096;
    __shared__ uint32_t list[CHUNK];
    __shared__ uint32_t list_n;
    __shared__ uint32_t s_counts_c;
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
        if (threadIdx.x == 0) s_counts_c = 0;
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
            if (threadIdx.x == 0) s_counts_c += m;
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
        if (t < W32) cnt.store(partials + (size_t(blockIdx.x) * K + c) * Dp + size_t(t) * 32);
        __syncthreads();
        if (count_members && threadIdx.x == 0 && blockIdx.y == 0 && state)
            atomicAdd(st.counts + parity * K + c, s_counts_c);
    }
}

template <int H>
static void launch_accumulate_h(const AccumulateArgs& a, uint32_t blocks_x, uint64_t ppc, cudaStream_t s) {
    const uint32_t threads = std::min<uint32_t>(512, ((a.W32 + 31) / 32) * 32);
    dim3 g(blocks_x, (a.W32 + threads - 1) / threads);
    k_accumulate<H><<<g, threads, 0, s>>>(a.grid, a.S32, a.W32, a.n, ppc, a.labels, a.K, a.skip_mode, a.state,
                                          a.parity, a.partials, a.Dp, a.count_members);
}

uint32_t accumulate_blocks(uint64_t n, uint32_t sms) {
    return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(sms) * 2, (n + 255) / 256)));
}

void launch_accumulate(const AccumulateArgs& a, cudaStream_t s) {
    const uint32_t blocks = a.blocks;
    const uint64_t ppc = (a.n + blocks - 1) / blocks;
    if (ppc <= BitCounter<8>::capacity())
        launch_accumulate_h<8>(a, blocks, ppc, s);
    else if (ppc <= BitCounter<12>::capacity())
        launch_accumulate_h<12>(a, blocks, ppc, s);
    else if (ppc <= BitCounter<16>::capacity())
        launch_accumulate_h<16>(a, blocks, ppc, s);
    else
        launch_accumulate_h<24>(a, blocks, ppc, s);
}

// =============================================================================================
// Reduce per-CTA partial sums into the exchange buffer (clusters != skip), and copy the
// round's counts/changed into its tail. xchg entries of the skipped cluster are left 0.
// =============================================================================================
__global__ void k_reduce(const uint32_t* __restrict__ partials, uint32_t nparts, uint32_t K, uint32_t Dp,
                         int skip_mode, void* state, uint32_t parity, int32_t* xchg, int copy_tail) {
    StateView st = StateView::at(state, K);
    if (state && st.hdr->done) return;
    int skip = skip_mode;
    if (skip_mode == -2) skip = int(pick_skip(st.cur + parity * K, K));
    const size_t total = size_t(K) * Dp;
    for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
        const uint32_t c = uint32_t(e / Dp);
        uint32_t s = 0;
        if (int(c) != skip)
            for (uint32_t b = 0; b < nparts; ++b) s += partials[size_t(b) * total + e];
        xchg[e] = int32_t(s);
    }
    if (copy_tail && blockIdx.x == 0 && threadIdx.x <= K) {
        const uint32_t v = threadIdx.x < K ? st.counts[parity * K + threadIdx.x] : st.changed[parity];
        xchg[total + threadIdx.x] = int32_t(v);
    }
}

void launch_reduce(const ReduceArgs& a, cudaStream_t s) {
    const size_t total = size_t(a.K) * a.Dp;
    const uint32_t blocks = uint32_t(std::min<size_t>((total + 255) / 256, 148 * 4));
    k_reduce<<<blocks, 256, 0, s>>>(a.partials, a.nparts, a.K, a.Dp, a.skip_mode, a.state, a.parity, a.xchg,
                                    a.copy_tail);
}

// =============================================================================================
// Finalise a centroid set from the (all-reduced) exchange buffer — identical on every rank.
//   mode 0 (round r): early-stop check (clusterer.cpp:213), sums -> centroids with the
//          skipped cluster derived as colsum - others, empty clusters keep the previous
//          centroid (clusterer.cpp:184-186); member counts = the round's counts.
//   mode 1 (init):   centroids = seed HV bits, member counts 1 (clusterer.cpp:197-205).
//   mode 2 (given):  centroids already in Z (assign_labels on caller centroids).
//   mode 3 (update): like 0 but no skip and no early stop (update_centroids API).
// Always: norm2 of the new set, B fragments. One thread per (32-bit word, cluster).
// =============================================================================================
__global__ void k_finish(int mode, uint32_t K, uint32_t P, uint32_t D, uint32_t W32, uint32_t W32P, uint32_t Dp,
                         const int32_t* __restrict__ xchg, const int32_t* __restrict__ colsum, uint32_t* Z,
                         uint8_t* bfrag, void* state, uint32_t round, int early_stop) {
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
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t word = idx / K, c = idx % K;
    const int skip = (mode == 0) ? int(pick_skip(st.cur + p * K, K)) : -1;
    unsigned long long n2 = 0;
    if (word < W32) {
        uint32_t z[32];
        const size_t base = size_t(word) * 32;
        if (mode == 2) {
#pragma unroll
            for (int b = 0; b < 32; ++b) z[b] = (base + b < D) ? Z[size_t(c) * D + base + b] : 0u;
        } else if (mode == 1 || counts[c] != 0) {
            if (int(c) == skip) {
#pragma unroll
                for (int b = 0; b < 32; ++b) z[b] = uint32_t(colsum[base + b]);
                for (uint32_t o = 0; o < K; ++o) {
                    if (int(o) == skip) continue;
#pragma unroll
                    for (int b = 0; b < 32; ++b) z[b] -= uint32_t(xchg[size_t(o) * Dp + base + b]);
                }
            } else {
#pragma unroll
                for (int b = 0; b < 32; ++b) z[b] = uint32_t(xchg[size_t(c) * Dp + base + b]);
            }
        } else {  // empty cluster keeps its previous centroid
#pragma unroll
            for (int b = 0; b < 32; ++b) z[b] = (base + b < D) ? Z[size_t(c) * D + base + b] : 0u;
        }
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            if (base + b < D) {
                if (mode != 2) Z[size_t(c) * D + base + b] = z[b];
                n2 += (unsigned long long)z[b] * z[b];
            } else {
                z[b] = 0;
            }
        }
        // B fragments: column n = P*c + plane; lane (n&7)<<2 | q holds bits {2q, 2q+8, 2q+16,
        // 2q+24} (bytes 0-3) and {2q+1, ...} (bytes 4-7) of this word, one 7-bit plane each.
        for (uint32_t pl = 0; pl < P; ++pl) {
            const uint32_t n = P * c + pl, nt = n >> 3, nl = n & 7;
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q) {
                uint64_t v = 0;
#pragma unroll
                for (uint32_t half = 0; half < 2; ++half)
#pragma unroll
                    for (uint32_t j = 0; j < 4; ++j)
                        v |= uint64_t(((z[2 * q + half + 8 * j] >> (kPlaneBits * pl)) & 0x7Fu) << (1 - half))
                             << (8 * (half * 4 + j));  // a0/a1 slots carry 64*bit: plane doubled
                const uint32_t lane = (nl << 2) | q;
                *reinterpret_cast<uint64_t*>(bfrag + ((size_t(nt) * W32P + word) * 32 + lane) * 8) = v;
            }
        }
        atomicAdd(st.norm2 + np * K + c, n2);
    }
    if (blockIdx.x == 0 && threadIdx.x < K) {
        const uint32_t cc = threadIdx.x;
        if (mode == 1) st.cur[np * K + cc] = 1;
        else if (mode == 0 || mode == 3) st.cur[np * K + cc] = counts[cc];
    }
}

void launch_finish(const FinishArgs& a, cudaStream_t s) {
    const uint32_t threads = 128;
    const uint32_t total = a.W32 * a.K;
    k_finish<<<(total + threads - 1) / threads, threads, 0, s>>>(a.mode, a.K, a.P, a.D, a.W32, a.W32P, a.Dp, a.xchg,
                                                                 a.colsum, a.Z, a.bfrag, a.state, a.round,
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
// The round kernel: assign_labels (clusterer.cpp:132-162) fused with the centroid
// accumulation of update_centroids (clusterer.cpp:164-188).
//
// Persistent CTAs walk tiles of TP = 16*MT pixels. Each tile arrives in shared memory by
// cp.async.bulk (TMA engine, one copy per pixel row, double buffered on mbarriers). Warp g
// owns 32-bit words [32g, 32g+32) of every HV (split-K): it unpacks the packed bits into IMMA
// A fragments in registers (unpack_a) and multiplies them with the byte-plane B fragments of
// the centroids (held in registers when BREG). Per-warp partial dots meet in shared memory,
// one thread per pixel recombines the planes in u64 and runs the exact 128-bit argmax. With
// UPD (K == 2) the words of the pixels assigned to the non-skipped cluster are then folded
// into a per-thread Harley-Seal counter (thread t = word column t) straight from the same
// shared-memory tile, so each pixel HV crosses HBM once per round.
// =============================================================================================
template <int MT, int NTG, bool BREG, bool UPD, int H, int TB>
__global__ void __launch_bounds__(TB, 1)
    k_round(const uint32_t* __restrict__ grid, uint64_t n, uint32_t S32, uint32_t SS, uint32_t W32, uint32_t W32P,
            uint32_t nwarp_words, uint32_t K, uint32_t P, uint32_t NT, const uint64_t* __restrict__ bfrag,
            uint32_t* labels, void* state, uint32_t round, int do_update, uint32_t* __restrict__ partials,
            uint32_t Dp) {
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

    // shared memory carve-up
    uint32_t* tiles = reinterpret_cast<uint32_t*>(smem);
    const size_t tile_words = size_t(TP) * SS;
    int32_t* part = reinterpret_cast<int32_t*>(tiles + 2 * tile_words + 32);  // [nwarps][TP][NC]
    uint32_t* red = reinterpret_cast<uint32_t*>(part + size_t(nwarps) * TP * NC);  // [TP][NCT]
    uint32_t* s_label = red + TP * NCT;                                          // [TP]
    uint32_t* s_list = s_label + TP;                                             // [TP]
    uint32_t* s_misc = s_list + TP;  // [0] list_n, [1] changed, [2] skip, [4..4+K) counts
    unsigned long long* s_n2 = reinterpret_cast<unsigned long long*>(s_misc + ((4 + K + 1) & ~1u));  // [K]
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_n2 + K);

    const uint64_t ntiles = (n + TP - 1) / TP;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_fence_init();
        s_misc[0] = 0;
        s_misc[1] = 0;
        s_misc[2] = pick_skip(st.cur + parity * K, K);
    }
    for (uint32_t c = tid; c < K; c += blockDim.x) {
        s_misc[4 + c] = 0;
        s_n2[c] = st.norm2[parity * K + c];
    }
    if (blockIdx.x == 0 && tid == 0) {
        st.hdr->rounds_run = round;
        // reset the other parity's accumulators for the next round
        for (uint32_t c = 0; c < K; ++c) st.counts[(parity ^ 1) * K + c] = 0;
        st.changed[parity ^ 1] = 0;
    }
    __syncthreads();
    const uint32_t skip = s_misc[2];
    const uint32_t upd_c = 1 - skip;  // K == 2 under UPD

    auto issue = [&](uint64_t tile, uint32_t buf) {
        // warp 0 issues one bulk copy per pixel row (rows are S32*4 bytes, 16-B aligned)
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

    // B fragments resident in registers for the whole round (BREG: one word block per warp)
    uint32_t breg[BREG ? 32 : 1][2];
    if constexpr (BREG) {
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) {
            const uint64_t v = warp < nwarp_words ? bfrag[(size_t(warp) * 32 + kk) * 32 + lane] : 0ull;
            breg[kk][0] = uint32_t(v);
            breg[kk][1] = uint32_t(v >> 32);
        }
    }
    // shift of unpack_a as an opaque multiplier so it issues as IMAD (FMA pipe), not SHF (ALU)
    uint32_t mul;
    asm volatile("mov.b32 %0, %1;" : "=r"(mul) : "r"(1u << (6 - 2 * q)));

    BitCounter<UPD ? H : 1> cnt;
    if constexpr (UPD) cnt.reset();

    const uint32_t ngroups = (NT + NTG - 1) / NTG;
    // epilogue state (threads tid < TP): running argmax across n-tile groups
    uint32_t best = 0;
    unsigned long long bdot = 0, bn2 = 0;

    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t buf = it & 1;
        mbar_wait(&bars[buf], (it >> 1) & 1);
        const uint32_t* T = tiles + buf * tile_words;
        const uint64_t px0 = tile * TP;
        const uint32_t npx = uint32_t(umin64(TP, n - px0));
        // previous labels, fetched now so the load latency hides behind the k-loop
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
#pragma unroll
                for (int k4 = 0; k4 < 8; ++k4) {
                    // rows g and g+8 of every m-tile: 4 consecutive words = 4 k-steps
                    uint4 wl[MT], wh[MT];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        wl[mt] = *reinterpret_cast<const uint4*>(T + size_t(16 * mt + g8) * SS + wbase + 4 * k4);
                        wh[mt] = *reinterpret_cast<const uint4*>(T + size_t(16 * mt + g8 + 8) * SS + wbase + 4 * k4);
                    }
#pragma unroll
                    for (int kq = 0; kq < 4; ++kq) {
                        const int kk = 4 * k4 + kq;
                        uint32_t b0[NTG], b1[NTG];
#pragma unroll
                        for (int nt = 0; nt < NTG; ++nt) {
                            if constexpr (BREG) {
                                b0[nt] = breg[kk][0];
                                b1[nt] = breg[kk][1];
                            } else {
                                const uint32_t ntg = grp * NTG + nt;
                                uint64_t v = 0;
                                if (ntg < NT) v = __ldg(bfrag + ((size_t(ntg) * W32P + wbase + kk) * 32 + lane));
                                b0[nt] = uint32_t(v);
                                b1[nt] = uint32_t(v >> 32);
                            }
                        }
                        // consecutive IMMAs target different m-tiles: independent accumulators
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            uint32_t a[4];
                            unpack_a(a, (&wl[mt].x)[kq], (&wh[mt].x)[kq], mul);
#pragma unroll
                            for (int nt = 0; nt < NTG; ++nt) imma16832(acc[mt][nt], a, b0[nt], b1[nt]);
                        }
                    }
                }
            }
            // per-warp partial dots -> shared memory
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
                red[px * NCT + col] = uint32_t(s) >> 7;  // remove the 128 scale of unpack_a (exact)
            }
            __syncthreads();  // red complete for this group; part free for the next group
        }
        // exact dots (u64) and the reference's 128-bit argmax, ties to the lower index
        if (tid < TP) {
            const uint32_t* rr = red + tid * NCT;
            for (uint32_t c = 0; c < K; ++c) {
                unsigned long long d = 0;
                for (uint32_t pl = 0; pl < P; ++pl) d += (unsigned long long)rr[P * c + pl] << (kPlaneBits * pl);
                const unsigned long long n2 = s_n2[c];
                if (c == 0) {
                    best = 0;
                    bdot = d;
                    bn2 = n2;
                } else if (strictly_closer(d, n2, bdot, bn2)) {
                    best = c;
                    bdot = d;
                    bn2 = n2;
                }
            }
        }

        // labels, changed count, member counts, update list
        if (tid < TP) {
            const bool live = tid < npx;
            if (live) {
                const uint64_t p = px0 + tid;
                labels[p] = best;
                if (old != best) atomicAdd(&s_misc[1], 1u);
                atomicAdd(&s_misc[4 + best], 1u);
                s_label[tid] = best;
                if (UPD && do_update && best == upd_c) s_list[atomicAdd(&s_misc[0], 1u)] = tid;
            }
        }
        __syncthreads();
        if constexpr (UPD) {
            if (do_update) {
                const uint32_t m = s_misc[0];
                if (tid < W32) {
                    for (uint32_t e = 0; e < m; e += 16) {
                        uint32_t x[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u) x[u] = (e + u < m) ? T[size_t(s_list[e + u]) * SS + tid] : 0u;
                        cnt.add16(x);
                    }
                }
            }
        }
        __syncthreads();  // every read of this buffer is done
        if (tid == 0) s_misc[0] = 0;
        if (warp == 0) {
            const uint64_t nxt = tile + 2ull * gridDim.x;
            if (nxt < ntiles) {
                fence_proxy_async();
                issue(nxt, buf);
            }
        }
    }

    if constexpr (UPD) {
        if (do_update && tid < W32) cnt.store(partials + (size_t(blockIdx.x) * K + upd_c) * Dp + size_t(tid) * 32);
    }
    __syncthreads();
    if (tid == 0) atomicAdd(st.changed + parity, s_misc[1]);
    for (uint32_t c = tid; c < K; c += blockDim.x) atomicAdd(st.counts + parity * K + c, s_misc[4 + c]);
}

// =============================================================================================
// The fused round kernel for one n-tile of centroid planes (K * P <= 8: K <= 2 at P = 4).
// Same data flow as k_round, tuned for the headline configs:
//  * warp w owns WPW words (a multiple of 4; warps a multiple of 4 so every SM sub-partition
//    carries the same k-loop load) and holds their B fragments in 2*WPW registers;
//  * the previous labels of a tile ride in the tile's TMA transaction (no exposed LDG);
//  * the split-K reduction and the argmax run on every warp at once (8 lanes per pixel,
//    planes combined with shuffles), so only three block barriers remain per tile.
// =============================================================================================
template <int MT, int WPW, bool UPD, int H, int TB>
__global__ void __launch_bounds__(TB, 1)
    k_round_fused(const uint32_t* __restrict__ grid, uint64_t n, uint32_t S32, uint32_t SS, uint32_t W32, uint32_t K,
                  uint32_t P, const uint64_t* __restrict__ bfrag, uint32_t* labels, void* state, uint32_t round,
                  int do_update, uint32_t* __restrict__ partials, uint32_t Dp) {
    constexpr uint32_t TP = 16 * MT;
    extern __shared__ __align__(128) uint8_t smem[];
    StateView st = StateView::at(state, K);
    if (st.hdr->done) return;

    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t g8 = lane >> 2, q = lane & 3;
    const uint32_t parity = round & 1;

    uint32_t* tiles = reinterpret_cast<uint32_t*>(smem);
    const size_t tile_words = size_t(TP) * SS;
    uint32_t* s_old = tiles + 2 * tile_words + 32;                         // [2][TP] labels via TMA
    int32_t* part = reinterpret_cast<int32_t*>(s_old + 2 * TP);             // [nwarps][TP][8]
    uint32_t* s_list = reinterpret_cast<uint32_t*>(part + size_t(nwarps) * TP * 8);  // [TP]
    uint32_t* s_misc = s_list + TP;  // [0] list_n, [1] changed, [2] skip, [4..4+K) counts
    unsigned long long* s_n2 = reinterpret_cast<unsigned long long*>(s_misc + ((4 + K + 1) & ~1u));
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_n2 + K);

    const uint64_t ntiles = (n + TP - 1) / TP;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_fence_init();
        s_misc[0] = 0;
        s_misc[1] = 0;
        s_misc[2] = pick_skip(st.cur + parity * K, K);
    }
    for (uint32_t c = tid; c < K; c += blockDim.x) {
        s_misc[4 + c] = 0;
        s_n2[c] = st.norm2[parity * K + c];
    }
    if (blockIdx.x == 0 && tid == 0) {
        st.hdr->rounds_run = round;
        for (uint32_t c = 0; c < K; ++c) st.counts[(parity ^ 1) * K + c] = 0;
        st.changed[parity ^ 1] = 0;
    }
    __syncthreads();
    const uint32_t skip = s_misc[2];
    const uint32_t upd_c = 1 - skip;  // K == 2 under UPD

    auto issue = [&](uint64_t tile, uint32_t buf) {
        const uint64_t px0 = tile * TP;
        const uint32_t npx = uint32_t(umin64(TP, n - px0));
        const uint32_t lab_bytes = (npx * 4 + 15) & ~15u;  // labels buffer is padded to 16 B
        if (lane == 0) mbar_expect_tx(&bars[buf], npx * S32 * 4 + lab_bytes);
        __syncwarp();
        if (lane == 0) bulk_g2s(s_old + buf * TP, labels + px0, lab_bytes, &bars[buf]);
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

    uint32_t breg[WPW][2];
#pragma unroll
    for (int kk = 0; kk < WPW; ++kk) {
        const uint64_t v = bfrag[(size_t(warp) * WPW + kk) * 32 + lane];
        breg[kk][0] = uint32_t(v);
        breg[kk][1] = uint32_t(v >> 32);
    }
    uint32_t mul;  // opaque power of two: the unpack shift issues as IMAD on the FMA pipe
    asm volatile("mov.b32 %0, %1;" : "=r"(mul) : "r"(1u << (6 - 2 * q)));
    const uint32_t wbase = warp * WPW;

    BitCounter<UPD ? H : 1> cnt;
    if constexpr (UPD) cnt.reset();

    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t buf = it & 1;
        mbar_wait(&bars[buf], (it >> 1) & 1);
        const uint32_t* T = tiles + buf * tile_words;
        const uint64_t px0 = tile * TP;
        const uint32_t npx = uint32_t(umin64(TP, n - px0));

        int acc[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[mt][r] = 0;
#pragma unroll
        for (int k4 = 0; k4 < WPW / 4; ++k4) {
            uint4 wl[MT], wh[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                wl[mt] = *reinterpret_cast<const uint4*>(T + size_t(16 * mt + g8) * SS + wbase + 4 * k4);
                wh[mt] = *reinterpret_cast<const uint4*>(T + size_t(16 * mt + g8 + 8) * SS + wbase + 4 * k4);
            }
#pragma unroll
            for (int kq = 0; kq < 4; ++kq) {
                const int kk = 4 * k4 + kq;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    uint32_t a[4];
                    unpack_a(a, (&wl[mt].x)[kq], (&wh[mt].x)[kq], mul);
                    imma16832(acc[mt], a, breg[kk][0], breg[kk][1]);
                }
            }
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            int32_t* row0 = part + (size_t(warp) * TP + 16 * mt + g8) * 8 + 2 * q;
            *reinterpret_cast<int2*>(row0) = make_int2(acc[mt][0], acc[mt][1]);
            *reinterpret_cast<int2*>(row0 + 64) = make_int2(acc[mt][2], acc[mt][3]);
        }
        __syncthreads();  // (1) partial dots of every warp are in shared memory

        // split-K reduction + exact argmax: 4 pixels per warp pass, lane = (pixel, column)
        for (uint32_t pg = warp; pg < TP / 4; pg += nwarps) {
            const uint32_t px = pg * 4 + (lane >> 3), col = lane & 7;
            int32_t s = 0;
            for (uint32_t w = 0; w < nwarps; ++w) s += part[(size_t(w) * TP + px) * 8 + col];
            const uint32_t c_of = col / P, pl = col - c_of * P;
            const unsigned long long v =
                (col < K * P) ? (unsigned long long)(uint32_t(s) >> 7) << (kPlaneBits * pl) : 0ull;
            const uint32_t base = lane & ~7u;
            uint32_t best = 0;
            unsigned long long bdot = 0, bn2 = 0;
            for (uint32_t c = 0; c < K; ++c) {
                unsigned long long d = 0;
                for (uint32_t j = 0; j < P; ++j) d += __shfl_sync(0xffffffffu, v, base + P * c + j);
                const unsigned long long n2 = s_n2[c];
                if (c == 0 || strictly_closer(d, n2, bdot, bn2)) {
                    best = c;
                    bdot = d;
                    bn2 = n2;
                }
            }
            const bool leader = col == 0 && px < npx;
            const uint32_t old = s_old[buf * TP + px];
            if (leader) labels[px0 + px] = best;
            const uint32_t chg = __ballot_sync(0xffffffffu, leader && old != best);
            if (lane == 0 && chg) atomicAdd(&s_misc[1], __popc(chg));
            for (uint32_t c = 0; c < K; ++c) {
                const uint32_t m = __ballot_sync(0xffffffffu, leader && best == c);
                if (lane == 0 && m) atomicAdd(&s_misc[4 + c], __popc(m));
            }
            if constexpr (UPD) {
                const bool take = do_update && leader && best == upd_c;
                const uint32_t m = __ballot_sync(0xffffffffu, take);
                uint32_t pos = 0;
                if (lane == 0 && m) pos = atomicAdd(&s_misc[0], __popc(m));
                pos = __shfl_sync(0xffffffffu, pos, 0);
                if (take) s_list[pos + __popc(m & ((1u << lane) - 1))] = px;
            }
            (void)c_of;
        }
        __syncthreads();  // (2) labels of the tile decided, update list complete
        if constexpr (UPD) {
            if (do_update) {
                const uint32_t m = s_misc[0];
                if (tid < W32) {
                    for (uint32_t e = 0; e < m; e += 16) {
                        uint32_t x[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u) x[u] = (e + u < m) ? T[size_t(s_list[e + u]) * SS + tid] : 0u;
                        cnt.add16(x);
                    }
                }
            }
        }
        __syncthreads();  // (3) every read of this buffer is done
        if (tid == 0) s_misc[0] = 0;
        if (warp == 0) {
            const uint64_t nxt = tile + 2ull * gridDim.x;
            if (nxt < ntiles) {
                fence_proxy_async();
                issue(nxt, buf);
            }
        }
    }

    if constexpr (UPD) {
        if (do_update && tid < W32) cnt.store(partials + (size_t(blockIdx.x) * K + upd_c) * Dp + size_t(tid) * 32);
    }
    __syncthreads();
    if (tid == 0) atomicAdd(st.changed + parity, s_misc[1]);
    for (uint32_t c = tid; c < K; c += blockDim.x) atomicAdd(st.counts + parity * K + c, s_misc[4 + c]);
}

// =============================================================================================
// Warp-specialised round kernel (one n-tile of centroid planes, K * P <= 8).
//
//   warps 0..NMW-1  "MMA" warps: wait tile t -> IMMA k-loop over their WPW words -> split-K
//                   partials to part[t%2] -> then, while the epilogue warp works on tile t,
//                   fold tile t-1 into the Harley-Seal counters (thread = word column) and
//                   release its buffer.
//   warp NMW        epilogue: reduce tile t's partials (lane = pixel), exact u64 dots, 128-bit
//                   argmax, labels, member counts, change count, update list.
//   warp NMW+1      producer: cp.async.bulk (TMA engine) of tile rows + previous labels into
//                   a 3-deep ring, gated by the buffer-free barriers.
// All hand-offs are mbarriers; no block-wide barrier inside the tile loop, so the k-loop
// of tile t+1 overlaps the epilogue and re-bundling of tile t.
// =============================================================================================
template <int WPW, bool UPD, int H, int NMW>
__global__ void __launch_bounds__((NMW + 2) * 32, 1)
    k_round_ws(const uint32_t* __restrict__ grid, uint64_t n, uint32_t S32, uint32_t SS, uint32_t W32, uint32_t K,
               uint32_t P, const uint64_t* __restrict__ bfrag, uint32_t* labels, void* state, uint32_t round,
               int do_update, uint32_t* __restrict__ partials, uint32_t Dp) {
    constexpr uint32_t MT = 2, TP = 32, NB = 3;
    extern __shared__ __align__(128) uint8_t smem[];
    StateView st = StateView::at(state, K);
    if (st.hdr->done) return;

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t parity = round & 1;

    uint32_t* tiles = reinterpret_cast<uint32_t*>(smem);
    const size_t tile_words = size_t(TP) * SS;
    uint32_t* s_old = tiles + NB * tile_words + 32;                        // [NB][TP]
    int32_t* part = reinterpret_cast<int32_t*>(s_old + NB * TP);           // [2][NMW][TP][8]
    uint32_t* s_list = reinterpret_cast<uint32_t*>(part + 2 * NMW * TP * 8);  // [2][TP]
    uint32_t* s_listn = s_list + 2 * TP;                                   // [2]
    uint32_t* s_misc = s_listn + 2;                                        // [0] skip
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ((reinterpret_cast<uintptr_t>(s_misc + 2) -
                                                           reinterpret_cast<uintptr_t>(smem) + 7) & ~uintptr_t(7)));
    uint64_t* full = bars;            // [NB] tile data landed (TMA)
    uint64_t* buf_free = bars + NB;   // [NB] MMA warps done with the buffer
    uint64_t* part_full = bars + 2 * NB;      // [2] partials written
    uint64_t* part_free = bars + 2 * NB + 2;  // [2] epilogue done reading partials
    uint64_t* list_ready = bars + 2 * NB + 4; // [2] labels + update list of the tile ready

    const uint64_t ntiles = (n + TP - 1) / TP;
    const uint32_t my_tiles = blockIdx.x < ntiles ? uint32_t((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    if (tid == 0) {
        for (uint32_t b = 0; b < NB; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&buf_free[b], NMW * 32);
        }
        for (uint32_t b = 0; b < 2; ++b) {
            mbar_init(&part_full[b], NMW * 32);
            mbar_init(&part_free[b], 32);
            mbar_init(&list_ready[b], 32);
        }
        mbar_fence_init();
        s_misc[0] = pick_skip(st.cur + parity * K, K);
    }
    if (blockIdx.x == 0 && tid == 0) {
        st.hdr->rounds_run = round;
        for (uint32_t c = 0; c < K; ++c) st.counts[(parity ^ 1) * K + c] = 0;
        st.changed[parity ^ 1] = 0;
    }
    __syncthreads();
    const uint32_t skip = s_misc[0];
    const uint32_t upd_c = 1 - skip;  // K == 2 under UPD

    if (warp == NMW + 1) {
        // ------------------------------------------------------------------ producer warp
        for (uint32_t it = 0; it < my_tiles; ++it) {
            const uint32_t b = it % NB;
            if (it >= NB) mbar_wait(&buf_free[b], ((it / NB) - 1) & 1);
            const uint64_t px0 = (blockIdx.x + uint64_t(it) * gridDim.x) * TP;
            const uint32_t npx = uint32_t(umin64(TP, n - px0));
            const uint32_t lab_bytes = (npx * 4 + 15) & ~15u;  // labels buffer padded to 16 B
            if (lane == 0) mbar_expect_tx(&full[b], npx * S32 * 4 + lab_bytes);
            __syncwarp();
            if (lane == 0) bulk_g2s(s_old + b * TP, labels + px0, lab_bytes, &full[b]);
            if (lane < npx)
                bulk_g2s(tiles + b * tile_words + size_t(lane) * SS, grid + (px0 + lane) * S32, S32 * 4, &full[b]);
        }
        return;
    }
    if (warp == NMW) {
        // ------------------------------------------------------------------ epilogue warp
        unsigned long long n2[2] = {st.norm2[parity * K], K > 1 ? st.norm2[parity * K + 1] : 0ull};
        uint32_t changed = 0, cnt0 = 0, cnt1 = 0;
        for (uint32_t it = 0; it < my_tiles; ++it) {
            const uint32_t pb = it & 1, b = it % NB;
            const uint64_t px0 = (blockIdx.x + uint64_t(it) * gridDim.x) * TP;
            const uint32_t npx = uint32_t(umin64(TP, n - px0));
            mbar_wait(&part_full[pb], (it >> 1) & 1);
            const int32_t* pp = part + size_t(pb) * NMW * TP * 8 + lane * 8;
            int32_t col[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
            for (uint32_t w = 0; w < NMW; ++w) {
                const int4 lo = *reinterpret_cast<const int4*>(pp + size_t(w) * TP * 8);
                const int4 hi = *reinterpret_cast<const int4*>(pp + size_t(w) * TP * 8 + 4);
                col[0] += lo.x; col[1] += lo.y; col[2] += lo.z; col[3] += lo.w;
                col[4] += hi.x; col[5] += hi.y; col[6] += hi.z; col[7] += hi.w;
            }
            mbar_arrive(&part_free[pb]);
            // exact dots: column n = P*c + plane, 7-bit planes, 128 scale removed (exact)
            unsigned long long d[2] = {0, 0};
#pragma unroll
            for (uint32_t cn = 0; cn < 8; ++cn) {
                const uint32_t c = cn / P, pl = cn - c * P;
                if (c < K && c < 2) d[c] += (unsigned long long)(uint32_t(col[cn]) >> 7) << (kPlaneBits * pl);
            }
            uint32_t best = 0;
            if (K > 1 && strictly_closer(d[1], n2[1], d[0], n2[0])) best = 1;
            const bool live = lane < npx;
            const uint32_t old = s_old[b * TP + lane];
            if (live) {
                labels[px0 + lane] = best;
                changed += old != best;
                cnt0 += best == 0;
                cnt1 += best == 1;
            }
            if constexpr (UPD) {
                const bool take = do_update && live && best == upd_c;
                const uint32_t m = __ballot_sync(0xffffffffu, take);
                if (take) s_list[pb * TP + __popc(m & ((1u << lane) - 1))] = lane;
                if (lane == 0) s_listn[pb] = __popc(m);
            }
            mbar_arrive(&list_ready[pb]);
        }
        for (int o = 16; o; o >>= 1) {
            changed += __shfl_xor_sync(0xffffffffu, changed, o);
            cnt0 += __shfl_xor_sync(0xffffffffu, cnt0, o);
            cnt1 += __shfl_xor_sync(0xffffffffu, cnt1, o);
        }
        if (lane == 0) {
            atomicAdd(st.changed + parity, changed);
            atomicAdd(st.counts + parity * K, cnt0);
            if (K > 1) atomicAdd(st.counts + parity * K + 1, cnt1);
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
    uint32_t mul;  // opaque power of two: the unpack shift issues as IMAD on the FMA pipe
    asm volatile("mov.b32 %0, %1;" : "=r"(mul) : "r"(1u << (6 - 2 * q)));
    const uint32_t wbase = warp * WPW;
    BitCounter<UPD ? H : 1> cnt;
    if constexpr (UPD) cnt.reset();

    auto rebundle = [&](uint32_t jt) {  // fold tile jt's update list into the counters
        const uint32_t pb = jt & 1, b = jt % NB;
        mbar_wait(&list_ready[pb], (jt >> 1) & 1);
        if constexpr (UPD) {
            if (do_update && tid < W32) {
                const uint32_t m = s_listn[pb];
                const uint32_t* T = tiles + b * tile_words;
                for (uint32_t e = 0; e < m; e += 16) {
                    uint32_t x[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        x[u] = (e + u < m) ? T[size_t(s_list[pb * TP + e + u]) * SS + tid] : 0u;
                    cnt.add16(x);
                }
            }
        }
        mbar_arrive(&buf_free[b]);
    };

    for (uint32_t it = 0; it < my_tiles; ++it) {
        const uint32_t b = it % NB, pb = it & 1;
        mbar_wait(&full[b], (it / NB) & 1);
        const uint32_t* T = tiles + b * tile_words;
        int acc[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[mt][r] = 0;
#pragma unroll
        for (int k4 = 0; k4 < WPW / 4; ++k4) {
            uint4 wl[MT], wh[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                wl[mt] = *reinterpret_cast<const uint4*>(T + size_t(16 * mt + g8) * SS + wbase + 4 * k4);
                wh[mt] = *reinterpret_cast<const uint4*>(T + size_t(16 * mt + g8 + 8) * SS + wbase + 4 * k4);
            }
#pragma unroll
            for (int kq = 0; kq < 4; ++kq) {
                const int kk = 4 * k4 + kq;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    uint32_t a[4];
                    unpack_a(a, (&wl[mt].x)[kq], (&wh[mt].x)[kq], mul);
                    imma16832(acc[mt], a, breg[kk][0], breg[kk][1]);
                }
            }
        }
        if (it >= 2) mbar_wait(&part_free[pb], ((it >> 1) - 1) & 1);
        int32_t* pw = part + (size_t(pb) * NMW + warp) * TP * 8;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            int32_t* row0 = pw + (16 * mt + g8) * 8 + 2 * q;
            *reinterpret_cast<int2*>(row0) = make_int2(acc[mt][0], acc[mt][1]);
            *reinterpret_cast<int2*>(row0 + 64) = make_int2(acc[mt][2], acc[mt][3]);
        }
        mbar_arrive(&part_full[pb]);
        if (it >= 1) rebundle(it - 1);
    }
    if (my_tiles >= 1) rebundle(my_tiles - 1);
    if constexpr (UPD) {
        if (do_update && tid < W32) cnt.store(partials + (size_t(blockIdx.x) * K + upd_c) * Dp + size_t(tid) * 32);
    }
}

size_t ws_smem_bytes(uint32_t SS, uint32_t nmw) {
    const uint32_t TP = 32, NB = 3;
    size_t b = (NB * size_t(TP) * SS + 32) * 4;  // tile ring + overrun slack
    b += NB * TP * 4;                            // s_old
    b += 2 * size_t(nmw) * TP * 8 * 4;           // part
    b += 2 * TP * 4 + 2 * 4 + 2 * 4;             // s_list, s_listn, s_misc
    b = (b + 7) & ~size_t(7);
    b += (2 * NB + 6) * 8;                       // mbarriers
    return b;
}

template <int WPW, bool UPD, int H, int NMW>
static cudaError_t launch_ws_t(const RoundArgs& a, cudaStream_t s) {
    auto kern = k_round_ws<WPW, UPD, H, NMW>;
    const size_t smem = ws_smem_bytes(a.SS, NMW);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    kern<<<a.ctas, (NMW + 2) * 32, smem, s>>>(a.grid, a.n, a.S32, a.SS, a.W32, a.K, a.P, a.bfrag, a.labels, a.state,
                                              a.round, a.do_update, a.partials, a.Dp);
    return cudaGetLastError();
}

template <int WPW, int NMW>
static cudaError_t launch_ws_h(const RoundArgs& a, cudaStream_t s) {
    if (a.K != 2) return launch_ws_t<WPW, false, 1, NMW>(a, s);
    const uint64_t per_cta = (a.n + a.ctas - 1) / a.ctas;
    if (per_cta <= BitCounter<8>::capacity()) return launch_ws_t<WPW, true, 8, NMW>(a, s);
    if (per_cta <= BitCounter<12>::capacity()) return launch_ws_t<WPW, true, 12, NMW>(a, s);
    return launch_ws_t<WPW, true, 20, NMW>(a, s);
}

size_t fused_smem_bytes(uint32_t MT, uint32_t SS, uint32_t nwarps, uint32_t K) {
    const uint32_t TP = 16 * MT;
    size_t b = (2 * size_t(TP) * SS + 32) * 4;  // tiles + overrun slack
    b += 2 * size_t(TP) * 4;                     // s_old
    b += size_t(nwarps) * TP * 8 * 4;            // part
    b += size_t(TP) * 4;                         // s_list
    b += ((4 + K + 1) & ~size_t(1)) * 4;         // s_misc
    b += size_t(K) * 8 + 2 * 8;                  // s_n2, mbarriers
    return b;
}

size_t round_smem_bytes(uint32_t MT, uint32_t NTG, uint32_t SS, uint32_t nwarps, uint32_t K, uint32_t NT) {
    const uint32_t TP = 16 * MT, NC = 8 * NTG;
    size_t b = (2 * size_t(TP) * SS + 32) * 4;        // tiles + slack for the last row's overrun
    b += size_t(nwarps) * TP * NC * 4;                 // part
    b += size_t(TP) * NT * 8 * 4;                      // red (all columns)
    b += 2 * size_t(TP) * 4;                           // s_label, s_list
    b += ((4 + K + 1) & ~size_t(1)) * 4;               // s_misc
    b += size_t(K) * 8;                                // s_n2
    b += 2 * 8;                                        // mbarriers
    return b;
}

template <int MT, int NTG, bool BREG, bool UPD, int H>
static cudaError_t launch_round_t(const RoundArgs& a, uint32_t nwarps, cudaStream_t s) {
    // register budget: 1 CTA/SM; <= 12 warps leaves 170 registers per thread, 16 warps 128
    auto kern = nwarps <= 12 ? k_round<MT, NTG, BREG, UPD, H, 384> : k_round<MT, NTG, BREG, UPD, H, 512>;
    const size_t smem = round_smem_bytes(MT, NTG, a.SS, nwarps, a.K, a.NT);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    kern<<<a.ctas, nwarps * 32, smem, s>>>(a.grid, a.n, a.S32, a.SS, a.W32, a.W32P, a.nwarp_words, a.K, a.P, a.NT,
                                           a.bfrag, a.labels, a.state, a.round, a.do_update, a.partials, a.Dp);
    return cudaGetLastError();
}

// Plan: which instantiation handles (K, P, D). Returns false if no kernel fits.
bool plan_round(uint32_t K, uint32_t P, uint32_t W32, uint32_t SS, RoundPlan& p, size_t smem_limit) {
    p.nwarp_words = (W32 + 31) / 32;
    p.nt = (K * P + 7) / 8;
    p.fused = false;
    if (p.nt == 1) {
        // warp-specialised kernel: MMA warps in multiples of 4 (equal load per SM sub-partition),
        // B fragments in 2*wpw registers, one thread per word column for the re-bundling
        static const uint32_t cand[][2] = {{4, 20}, {4, 28}, {4, 32}, {8, 20}, {8, 28}, {8, 32},
                                           {12, 20}, {12, 28}, {16, 20}, {16, 28}};
        const char* force = getenv("SEGHDC_FUSED_WARPS");
        if (force && !*force) force = nullptr;
        for (const auto& c : cand) {
            if (force && uint32_t(atoi(force)) != c[0]) continue;
            if (c[0] * c[1] < W32 || c[0] * 32 < W32) continue;
            if (ws_smem_bytes(SS, c[0]) > smem_limit) continue;
            p.fused = true;
            p.nwarps = c[0];
            p.wpw = c[1];
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
    if (p.fused) {
#define SEGHDC_WS(NMW)                                                   \
    if (p.nwarps == NMW) {                                               \
        if (p.wpw == 20) return launch_ws_h<20, NMW>(a, s);              \
        if (p.wpw == 28) return launch_ws_h<28, NMW>(a, s);              \
        return launch_ws_h<32, NMW>(a, s);                               \
    }
        SEGHDC_WS(4)
        SEGHDC_WS(8)
        SEGHDC_WS(12)
        if (p.wpw == 20) return launch_ws_h<20, 16>(a, s);
        return launch_ws_h<28, 16>(a, s);
#undef SEGHDC_WS
    }
    switch (p.mt) {
        case 4: return launch_round_t<4, 4, false, false, 1>(a, p.nwarps, s);
        case 2: return launch_round_t<2, 4, false, false, 1>(a, p.nwarps, s);
        default: return launch_round_t<1, 4, false, false, 1>(a, p.nwarps, s);
    }
}

}  // namespace seghdc_dev

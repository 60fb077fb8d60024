// Closed-form Manhattan variant of the clustering loop (SURVEY.md §7 hard part 4, §8f rank 1).
//
// A Manhattan pixel HV is y = B ^ F, B the XOR of the 2 + C codebook bases and F the XOR of
// 2 + C runs of ones (closed.h). Sorting the 2(2 + C) run endpoints e_0 <= ... <= e_9 turns F
// into the disjoint runs [e_0, e_1), [e_2, e_3), ... (XOR = coverage parity). With
//   P_k = sum_i B_i z_k[i],   Q_k[t] = sum_{i < t} (1 - 2 B_i) z_k[i]
// the reference's dot_words(y, z_k) (hypervector.cpp:138-151) is P_k + sum_m Q_k[e_2m+1] - Q_k[e_2m],
// and update_centroids' add_words (hypervector.cpp:112-121) sums to z_k[i] = B_i n_k + (1 - 2 B_i) c_k[i],
// c_k = prefix sum of a +1/-1 difference array on the members' sorted endpoints. No D-sized
// work per pixel: 10 table lookups per cluster to assign, 10 shared-memory atomics to update.
// The dots and norms are exact integers, so the labels equal the packed-bit path's
// (strictly_closer in 128 bits, clusterer.cpp:41-50).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdlib>

#include "closed.h"
#include "kernels.cuh"
#include "launch.h"

namespace seghdc_dev {

namespace {

constexpr int kRuns = 10;  // 2 + C <= 5 runs

// Sorted run endpoints of pixel p; unused slots are dim (empty runs [dim, dim)).
__device__ __forceinline__ void closed_runs(const ClosedArgs& a, uint64_t p, uint32_t (&e)[kRuns]) {
    const uint32_t i = uint32_t(p) / a.w, j = uint32_t(p) % a.w;  // n < 2^32 (checked by the host)
    e[0] = 0;
    e[1] = (i / a.beta) * a.x_row;
    e[2] = a.dim / 2;
    e[3] = a.dim / 2 + (j / a.beta) * a.x_col;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        if (uint32_t(ch) < a.c) {
            const uint32_t v = a.img[p * a.c + ch];
            e[4 + 2 * ch] = a.off[ch];
            e[5 + 2 * ch] = a.off[ch] + v * a.unit[ch];
        } else {
            e[4 + 2 * ch] = e[5 + 2 * ch] = a.dim;
        }
    }
    // odd-even transposition sort, fully unrolled (registers only)
#pragma unroll
    for (int r = 0; r < kRuns; ++r) {
#pragma unroll
        for (int q = (r & 1); q + 1 < kRuns; q += 2) {
            const uint32_t lo = min(e[q], e[q + 1]), hi = max(e[q], e[q + 1]);
            e[q] = lo;
            e[q + 1] = hi;
        }
    }
}

// Position of compressed endpoint index t (ClosedArgs::L layout).
__device__ __forceinline__ uint32_t closed_pos(const ClosedArgs& a, uint32_t t) {
    if (t < a.nr) return t * a.x_row;
    t -= a.nr;
    if (t < a.nc) return a.dim / 2 + t * a.x_col;
    t -= a.nc;
    if (t < 256 * a.c) return a.off[t >> 8] + (t & 255) * a.unit[t >> 8];
    return a.dim;
}

// Sorted run endpoints of pixel p as compressed indices (sort key: position << 15 | index).
__device__ __forceinline__ void closed_runs_idx(const ClosedArgs& a, uint64_t p, uint32_t (&e)[kRuns]) {
    const uint32_t i = uint32_t(p) / a.w, j = uint32_t(p) % a.w;
    const uint32_t bi = i / a.beta, bj = j / a.beta;
    e[0] = 0u;  // row run start: row entry 0, position 0
    e[1] = ((bi * a.x_row) << 15) | bi;
    e[2] = ((a.dim / 2) << 15) | a.nr;
    e[3] = ((a.dim / 2 + bj * a.x_col) << 15) | (a.nr + bj);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        if (uint32_t(ch) < a.c) {
            const uint32_t v = a.img[p * a.c + ch], base = a.nr + a.nc + 256u * ch;
            e[4 + 2 * ch] = (a.off[ch] << 15) | base;
            e[5 + 2 * ch] = ((a.off[ch] + v * a.unit[ch]) << 15) | (base + v);
        } else {
            e[4 + 2 * ch] = e[5 + 2 * ch] = (a.dim << 15) | (a.L - 1);
        }
    }
#pragma unroll
    for (int r = 0; r < kRuns; ++r) {
#pragma unroll
        for (int q = (r & 1); q + 1 < kRuns; q += 2) {
            const uint32_t lo = min(e[q], e[q + 1]), hi = max(e[q], e[q + 1]);
            e[q] = lo;
            e[q + 1] = hi;
        }
    }
#pragma unroll
    for (int q = 0; q < kRuns; ++q) e[q] &= 0x7FFFu;
}

// clusterer.cpp:41-50, mod 2^128 like the reference's unsigned __int128
__device__ __forceinline__ bool strictly_closer_dev(unsigned long long dc, unsigned long long nc,
                                                    unsigned long long db, unsigned long long nb) {
    if (nc == 0) return false;
    if (nb == 0) return dc > 0;
    const unsigned __int128 lhs = (unsigned __int128)dc * dc * nb;
    const unsigned __int128 rhs = (unsigned __int128)db * db * nc;
    return lhs > rhs;
}

__global__ void k_closed_seed(ClosedArgs a, const uint64_t* __restrict__ seeds, ClosedState s) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.K) return;
    uint32_t e[kRuns];
    closed_runs(a, seeds[k], e);
    int32_t* d = s.diff + size_t(k) * (a.dim + 1);
#pragma unroll
    for (int m = 0; m < kRuns; m += 2) {
        if (e[m] == e[m + 1]) continue;
        atomicAdd(d + e[m], 1);
        atomicAdd(d + e[m + 1], -1);
    }
    s.cnt[k] = 1;
}

constexpr int kMaxK = 32;

// WR: also count the comparisons whose 128-bit products wrapped (opt-in diagnostic)
template <bool WR>
__global__ void __launch_bounds__(256) k_closed_assign(ClosedArgs a, ClosedState s) {
    __shared__ unsigned long long sP[kMaxK], sN[kMaxK];
    for (uint32_t k = threadIdx.x; k < a.K; k += blockDim.x) sP[k] = s.P[k], sN[k] = s.norm2[k];
    __syncthreads();
    const size_t stride = size_t(a.dim) + 1;
    unsigned long long changed = 0;
    uint32_t nwrap = 0;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < a.n; p += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t e[kRuns];
        closed_runs(a, p, e);
        uint32_t best = 0;
        unsigned long long best_dot = 0, best_n2 = 0;
        for (uint32_t k = 0; k < a.K; ++k) {
            const long long* q = s.Q + k * stride;
            long long d = (long long)sP[k];
#pragma unroll
            for (int m = 0; m < kRuns; m += 2) d += __ldg(q + e[m + 1]) - __ldg(q + e[m]);
            const unsigned long long dot = (unsigned long long)d, n2 = sN[k];
            if (k == 0) {
                best_dot = dot, best_n2 = n2;
            } else {
                if (WR) nwrap += compare_wraps(dot, n2, best_dot, best_n2);
                if (strictly_closer_dev(dot, n2, best_dot, best_n2)) best = k, best_dot = dot, best_n2 = n2;
            }
        }
        changed += (s.labels[p] != best);
        s.labels[p] = best;
    }
    // one atomic per warp
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        changed += __shfl_xor_sync(0xFFFFFFFFu, changed, o);
        if (WR) nwrap += __shfl_xor_sync(0xFFFFFFFFu, nwrap, o);
    }
    if ((threadIdx.x & 31) == 0 && changed) atomicAdd(s.changed, changed);
    if (WR && (threadIdx.x & 31) == 0 && nwrap && s.wraps) atomicAdd(s.wraps, (unsigned long long)nwrap);
}

// assign_labels with the K prefix tables restricted to the L endpoint positions, staged once per
// CTA in shared memory ([K][L] int64): 10 shared-memory loads per pixel and cluster.
template <bool WR>
__global__ void __launch_bounds__(512) k_closed_assign_smem(ClosedArgs a, ClosedState s) {
    extern __shared__ long long sq[];
    __shared__ unsigned long long sP[kMaxK], sN[kMaxK];
    const uint32_t K = a.K;
    for (uint32_t k = threadIdx.x; k < K; k += blockDim.x) sP[k] = s.P[k], sN[k] = s.norm2[k];
    const size_t stride = size_t(a.dim) + 1;
    // [K][L]: lanes with random colour values spread over all 16 bank pairs (an [L][K] layout
    // puts every entry of one cluster on 32 / K of them: 16-way conflicts at K = 8)
    for (uint32_t t = threadIdx.x; t < a.L * K; t += blockDim.x) {
        const uint32_t k = t / a.L, idx = t % a.L;
        sq[t] = s.Q[k * stride + closed_pos(a, idx)];
    }
    __syncthreads();
    unsigned long long changed = 0;
    uint32_t nwrap = 0;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < a.n; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t old = s.labels[p];  // issued with the image loads, not after the argmax
        uint32_t e[kRuns];
        closed_runs_idx(a, p, e);
        uint32_t best = 0;
        unsigned long long best_dot = 0, best_n2 = 0;
        for (uint32_t k = 0; k < K; ++k) {
            long long d = (long long)sP[k];
#pragma unroll
            for (int m = 0; m < kRuns; m += 2) d += sq[k * a.L + e[m + 1]] - sq[k * a.L + e[m]];
            const unsigned long long dot = (unsigned long long)d, n2 = sN[k];
            if (k == 0) {
                best_dot = dot, best_n2 = n2;
            } else {
                if (WR) nwrap += compare_wraps(dot, n2, best_dot, best_n2);
                if (strictly_closer_dev(dot, n2, best_dot, best_n2)) best = k, best_dot = dot, best_n2 = n2;
            }
        }
        changed += (old != best);
        s.labels[p] = best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        changed += __shfl_xor_sync(0xFFFFFFFFu, changed, o);
        if (WR) nwrap += __shfl_xor_sync(0xFFFFFFFFu, nwrap, o);
    }
    if ((threadIdx.x & 31) == 0 && changed) atomicAdd(s.changed, changed);
    if (WR && (threadIdx.x & 31) == 0 && nwrap && s.wraps) atomicAdd(s.wraps, (unsigned long long)nwrap);
}

// grid = (blocks, cluster groups); group y owns clusters [y*G, y*G + G), one difference array
// of dim + 1 ints each in shared memory. Only the run endpoints are ever touched, so the flush
// skips zero entries.
__global__ void __launch_bounds__(512) k_closed_accumulate(ClosedArgs a, ClosedState s, uint32_t G) {
    extern __shared__ int32_t sd[];
    const uint32_t stride = a.dim + 1, k0 = blockIdx.y * G, kn = min(G, a.K - k0);
    uint32_t* scnt = reinterpret_cast<uint32_t*>(sd + size_t(G) * stride);
    for (uint32_t t = threadIdx.x; t < kn * stride; t += blockDim.x) sd[t] = 0;
    for (uint32_t t = threadIdx.x; t < kn; t += blockDim.x) scnt[t] = 0;
    __syncthreads();
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < a.n; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t l = s.labels[p] - k0;
        if (l >= kn) continue;
        uint32_t e[kRuns];
        closed_runs(a, p, e);
        int32_t* d = sd + size_t(l) * stride;
#pragma unroll
        for (int m = 0; m < kRuns; m += 2) {
            if (e[m] == e[m + 1]) continue;
            atomicAdd(d + e[m], 1);
            atomicAdd(d + e[m + 1], -1);
        }
        atomicAdd(scnt + l, 1u);
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < kn * stride; t += blockDim.x)
        if (sd[t]) atomicAdd(s.diff + size_t(k0) * stride + t, sd[t]);
    for (uint32_t t = threadIdx.x; t < kn; t += blockDim.x)
        if (scnt[t]) atomicAdd(s.cnt + k0 + t, (unsigned long long)scnt[t]);
}

// update_centroids' accumulation on compressed endpoint indices: every cluster's [L] difference
// counts in shared memory at once (one pass over the labels), flushed into diffc; k_closed_finish
// scatters them to positions.
__global__ void __launch_bounds__(512) k_closed_accumulate_c(ClosedArgs a, ClosedState s) {
    extern __shared__ int32_t sc[];
    const uint32_t K = a.K, L = a.L;
    uint32_t* scnt = reinterpret_cast<uint32_t*>(sc + K * L);
    for (uint32_t t = threadIdx.x; t < K * L + K; t += blockDim.x) sc[t] = 0;
    __syncthreads();
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < a.n; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t l = s.labels[p];
        uint32_t e[kRuns];
        closed_runs_idx(a, p, e);
        SG_CHECK(l < K);
        int32_t* d = sc + l * L;
#pragma unroll
        for (int m = 0; m < kRuns; m += 2) {
            SG_CHECK(e[m] < L && e[m + 1] < L);
            if (e[m] == e[m + 1]) continue;
            atomicAdd(d + e[m], 1);
            atomicAdd(d + e[m + 1], -1);
        }
        atomicAdd(scnt + l, 1u);
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < K * L; t += blockDim.x)
        if (sc[t]) atomicAdd(s.diffc + t, sc[t]);
    for (uint32_t t = threadIdx.x; t < K; t += blockDim.x)
        if (scnt[t]) atomicAdd(s.cnt + t, (unsigned long long)scnt[t]);
}

constexpr int kFinT = 1024;

// One CTA per cluster: c = prefix(diff), z = B ? n - c : c, then norm2, P and the prefix Q of
// (1 - 2B) z. An empty cluster keeps its previous state (clusterer.cpp:183-185), count 0.
__global__ void __launch_bounds__(kFinT) k_closed_finish(ClosedArgs a, ClosedState s) {
    using ScanI = cub::BlockScan<long long, kFinT>;
    using RedU = cub::BlockReduce<unsigned long long, kFinT>;
    __shared__ union {
        typename ScanI::TempStorage scan;
        typename RedU::TempStorage red;
    } tmp;
    const uint32_t k = blockIdx.x, stride = a.dim + 1;
    const unsigned long long n = s.cnt[k];
    __syncthreads();
    if (threadIdx.x == 0) s.counts[k] = n, s.cnt[k] = 0;
    if (n == 0) return;  // block-uniform
    int32_t* d = s.diff + size_t(k) * stride;
    if (s.diffc) {  // compressed counts -> positions (block-visible after the barrier)
        int32_t* dc = s.diffc + size_t(k) * a.L;
        for (uint32_t t = threadIdx.x; t < a.L; t += blockDim.x) {
            const int32_t v = dc[t];
            if (v) atomicAdd(d + closed_pos(a, t), v), dc[t] = 0;
        }
        __syncthreads();
    }
    uint32_t* z = s.Z + size_t(k) * a.dim;
    long long* q = s.Q + size_t(k) * stride;
    const uint32_t chunk = (a.dim + kFinT - 1) / kFinT;
    const uint32_t i0 = min(a.dim, threadIdx.x * chunk), i1 = min(a.dim, i0 + chunk);
    long long part = 0;
    for (uint32_t i = i0; i < i1; ++i) part += d[i];
    long long c;
    ScanI(tmp.scan).ExclusiveSum(part, c);
    __syncthreads();
    unsigned long long n2 = 0, pb = 0;
    long long sp = 0;
    for (uint32_t i = i0; i < i1; ++i) {
        c += d[i];
        d[i] = 0;
        const bool b = s.bflag[i];
        const unsigned long long zi = b ? n - (unsigned long long)c : (unsigned long long)c;
        z[i] = uint32_t(zi);
        n2 += zi * zi;
        if (b) pb += zi, sp -= (long long)zi;
        else sp += (long long)zi;
    }
    if (threadIdx.x == 0) d[a.dim] = 0;
    long long qb;
    ScanI(tmp.scan).ExclusiveSum(sp, qb);
    __syncthreads();
    n2 = RedU(tmp.red).Sum(n2);
    __syncthreads();
    pb = RedU(tmp.red).Sum(pb);
    if (threadIdx.x == 0) {
        s.norm2[k] = n2;
        s.P[k] = pb;
        q[0] = 0;
    }
    for (uint32_t i = i0; i < i1; ++i) {
        const long long zi = z[i];
        qb += s.bflag[i] ? -zi : zi;
        q[i + 1] = qb;
    }
}

// Skewed shared-memory index: each thread walks a contiguous chunk of `chunk` words, so word
// i + i/32 puts the 32 lanes of a warp on 32 distinct banks for every chunk length.
__host__ __device__ __forceinline__ uint32_t fin_skew(uint32_t i) { return i + (i >> 5); }

// k_closed_finish with the counts and B flags staged in shared memory: the diff row and the flags
// are read once, coalesced; the compressed counts scatter into shared memory; the three serial
// per-thread passes (c, z, Q) run on shared memory instead of chains of dependent global loads.
// Global Z and Q are store-only. Same arithmetic and order as k_closed_finish (bit-identical).
__global__ void __launch_bounds__(kFinT) k_closed_finish_smem(ClosedArgs a, ClosedState s) {
    using ScanI = cub::BlockScan<long long, kFinT>;
    using RedU = cub::BlockReduce<unsigned long long, kFinT>;
    __shared__ union {
        typename ScanI::TempStorage scan;
        typename RedU::TempStorage red;
    } tmp;
    extern __shared__ int32_t fin_sm[];
    const uint32_t k = blockIdx.x, stride = a.dim + 1;
    int32_t* sd = fin_sm;                               // [skew(dim) + 1] counts, then z
    int32_t* sb = fin_sm + fin_skew(a.dim) + 1;         // [skew(dim - 1) + 1] B flags
    const unsigned long long n = s.cnt[k];
    __syncthreads();
    if (threadIdx.x == 0) s.counts[k] = n, s.cnt[k] = 0;
    if (n == 0) return;  // block-uniform
    int32_t* d = s.diff + size_t(k) * stride;
    // batches of 8 per thread: all 16 loads in flight before the first store (the zeroing store
    // to d would otherwise serialise one load latency per element)
    constexpr int kB = 8;
    for (uint32_t t0 = threadIdx.x; t0 <= a.dim; t0 += kB * blockDim.x) {
        int32_t v[kB];
        uint8_t bf[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const uint32_t t = t0 + j * blockDim.x;
            v[j] = t <= a.dim ? __ldcg(d + t) : 0;
            bf[j] = t < a.dim ? __ldg(s.bflag + t) : 0;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const uint32_t t = t0 + j * blockDim.x;
            if (t <= a.dim) {
                sd[fin_skew(t)] = v[j];
                d[t] = 0;
                if (t < a.dim) sb[fin_skew(t)] = bf[j];
            }
        }
    }
    __syncthreads();
    if (s.diffc) {
        int32_t* dc = s.diffc + size_t(k) * a.L;
        for (uint32_t t = threadIdx.x; t < a.L; t += blockDim.x) {
            const int32_t v = dc[t];
            if (v) atomicAdd(sd + fin_skew(closed_pos(a, t)), v), dc[t] = 0;
        }
        __syncthreads();
    }
    uint32_t* z = s.Z + size_t(k) * a.dim;
    long long* q = s.Q + size_t(k) * stride;
    const uint32_t chunk = (a.dim + kFinT - 1) / kFinT;
    const uint32_t i0 = min(a.dim, threadIdx.x * chunk), i1 = min(a.dim, i0 + chunk);
    long long part = 0;
    for (uint32_t i = i0; i < i1; ++i) part += sd[fin_skew(i)];
    long long c;
    ScanI(tmp.scan).ExclusiveSum(part, c);
    __syncthreads();
    unsigned long long n2 = 0, pb = 0;
    long long sp = 0;
    for (uint32_t i = i0; i < i1; ++i) {
        const uint32_t si = fin_skew(i);
        c += sd[si];
        const bool b = sb[si];
        const unsigned long long zi = b ? n - (unsigned long long)c : (unsigned long long)c;
        z[i] = uint32_t(zi);
        sd[si] = int32_t(uint32_t(zi));
        n2 += zi * zi;
        if (b) pb += zi, sp -= (long long)zi;
        else sp += (long long)zi;
    }
    long long qb;
    ScanI(tmp.scan).ExclusiveSum(sp, qb);
    __syncthreads();
    n2 = RedU(tmp.red).Sum(n2);
    __syncthreads();
    pb = RedU(tmp.red).Sum(pb);
    if (threadIdx.x == 0) {
        s.norm2[k] = n2;
        s.P[k] = pb;
        q[0] = 0;
    }
    for (uint32_t i = i0; i < i1; ++i) {
        const uint32_t si = fin_skew(i);
        const long long zi = uint32_t(sd[si]);
        qb += sb[si] ? -zi : zi;
        q[i + 1] = qb;
    }
}

size_t fin_smem_bytes(uint32_t dim) { return (size_t(fin_skew(dim)) + 1 + fin_skew(dim)) * 4; }

// ---- the finish spread over a thread-block cluster per centroid (round 2) -----------------------
// k_closed_finish_smem runs one CTA per cluster: at K = 2 two SMs scan D positions through three
// serial passes and the round waits on them (latency-bound, half of a C1 closed-form run). Here a
// cluster of kFinG CTAs shares each centroid: CTA r owns positions [r seg, (r+1) seg), and the
// two prefix sums (c, then Q) and the norm2 / P reductions combine their per-CTA totals through
// distributed shared memory. Same integers in the same order of summation per position, so
// bit-identical to k_closed_finish.
constexpr int kFinG = 8, kFinCT = 256;
__device__ __forceinline__ void fin_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ long long fin_peer_ll(const long long* local, uint32_t rank) {
    uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(local)), peer;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(addr), "r"(rank));
    long long v;
    asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(peer) : "memory");
    return v;
}

__global__ void __launch_bounds__(kFinCT) k_closed_finish_cl(ClosedArgs a, ClosedState s) {
    using ScanI = cub::BlockScan<long long, kFinCT>;
    using RedU = cub::BlockReduce<unsigned long long, kFinCT>;
    __shared__ union {
        typename ScanI::TempStorage scan;
        typename RedU::TempStorage red;
    } tmp;
    __shared__ long long xch[4];  // this CTA's totals: [c, Q increments, norm2, P]
    extern __shared__ int32_t fcl_sm[];
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t k = blockIdx.x / kFinG, stride = a.dim + 1, tid = threadIdx.x;
    const uint32_t seg = (a.dim + kFinG - 1) / kFinG, p0 = min(a.dim, rank * seg), p1 = min(a.dim, p0 + seg);
    const uint32_t len = p1 - p0;
    int32_t* sd = fcl_sm;                      // [seg + 1] counts of positions p0.., then z
    uint8_t* sb = reinterpret_cast<uint8_t*>(fcl_sm + seg + 1);
    const unsigned long long n = s.cnt[k];
    fin_cluster_sync();  // every CTA of the cluster read cnt[k] before it is reset
    if (rank == 0 && tid == 0) s.counts[k] = n, s.cnt[k] = 0;
    if (n == 0) return;  // cluster-uniform
    int32_t* d = s.diff + size_t(k) * stride;
    for (uint32_t t = tid; t < len; t += kFinCT) {
        sd[t] = __ldcg(d + p0 + t);
        d[p0 + t] = 0;
        sb[t] = __ldg(s.bflag + p0 + t);
    }
    if (rank == kFinG - 1 && tid == 0) d[a.dim] = 0;
    __syncthreads();
    if (s.diffc) {  // compressed counts of this CTA's positions
        int32_t* dc = s.diffc + size_t(k) * a.L;
        for (uint32_t t = tid; t < a.L; t += kFinCT) {
            const uint32_t pos = closed_pos(a, t);
            const bool mine = (pos >= p0 && pos < p1) || (pos == a.dim && rank == kFinG - 1);
            if (!mine) continue;
            const int32_t v = dc[t];
            if (v) {
                if (pos < a.dim) atomicAdd(sd + (pos - p0), v);
                dc[t] = 0;
            }
        }
        __syncthreads();
    }
    const uint32_t chunk = (len + kFinCT - 1) / kFinCT;
    const uint32_t i0 = min(len, tid * chunk), i1 = min(len, i0 + chunk);
    long long part = 0;
    for (uint32_t i = i0; i < i1; ++i) part += sd[i];
    long long c, ctot;
    ScanI(tmp.scan).ExclusiveSum(part, c, ctot);
    if (tid == 0) xch[0] = ctot;
    fin_cluster_sync();
    for (uint32_t r = 0; r < rank; ++r) c += fin_peer_ll(&xch[0], r);  // prefix of the lower CTAs
    __syncthreads();
    uint32_t* z = s.Z + size_t(k) * a.dim;
    long long* q = s.Q + size_t(k) * stride;
    unsigned long long n2 = 0, pb = 0;
    long long sp = 0;
    for (uint32_t i = i0; i < i1; ++i) {
        c += sd[i];
        const bool b = sb[i];
        const unsigned long long zi = b ? n - (unsigned long long)c : (unsigned long long)c;
        z[p0 + i] = uint32_t(zi);
        sd[i] = int32_t(uint32_t(zi));
        n2 += zi * zi;
        if (b) pb += zi, sp -= (long long)zi;
        else sp += (long long)zi;
    }
    long long qb, qtot;
    ScanI(tmp.scan).ExclusiveSum(sp, qb, qtot);
    __syncthreads();
    n2 = RedU(tmp.red).Sum(n2);
    __syncthreads();
    pb = RedU(tmp.red).Sum(pb);
    if (tid == 0) xch[1] = qtot, xch[2] = (long long)n2, xch[3] = (long long)pb;
    fin_cluster_sync();
    for (uint32_t r = 0; r < rank; ++r) qb += fin_peer_ll(&xch[1], r);
    if (rank == 0 && tid == 0) {
        unsigned long long tn2 = 0, tpb = 0;
        for (uint32_t r = 0; r < kFinG; ++r)
            tn2 += (unsigned long long)fin_peer_ll(&xch[2], r), tpb += (unsigned long long)fin_peer_ll(&xch[3], r);
        s.norm2[k] = tn2;
        s.P[k] = tpb;
        q[0] = 0;
    }
    for (uint32_t i = i0; i < i1; ++i) {
        const long long zi = uint32_t(sd[i]);
        qb += sb[i] ? -zi : zi;
        q[p0 + i + 1] = qb;
    }
    fin_cluster_sync();  // no CTA leaves while a peer may still read its totals
}

}  // namespace

void launch_closed_seed(const ClosedArgs& a, const uint64_t* seeds, ClosedState s, cudaStream_t st) {
    k_closed_seed<<<(a.K + 63) / 64, 64, 0, st>>>(a, seeds, s);
}

void launch_closed_assign(const ClosedArgs& a, ClosedState s, int sms, cudaStream_t st) {
    const size_t smem = size_t(a.L) * a.K * 8;
    if (s.diffc) {  // compressed indices fit (seghdc_run_pipeline_closed decides)
        auto kern = s.wraps ? k_closed_assign_smem<true> : k_closed_assign_smem<false>;
        ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
        const uint64_t blocks = std::min<uint64_t>((a.n + 511) / 512, uint64_t(sms) * (smem <= (100u << 10) ? 2 : 1));
        kern<<<uint32_t(std::max<uint64_t>(blocks, 1)), 512, smem, st>>>(a, s);
        return;
    }
    const uint64_t blocks = std::min<uint64_t>((a.n + 255) / 256, uint64_t(sms) * 8);
    auto kern = s.wraps ? k_closed_assign<true> : k_closed_assign<false>;
    kern<<<uint32_t(std::max<uint64_t>(blocks, 1)), 256, 0, st>>>(a, s);
}

void launch_closed_accumulate(const ClosedArgs& a, ClosedState s, int sms, cudaStream_t st) {
    if (s.diffc) {
        const size_t smem = (size_t(a.L) + 1) * a.K * 4;
        ensure_dynamic_smem(reinterpret_cast<const void*>(k_closed_accumulate_c), smem);
        const uint64_t blocks = std::min<uint64_t>((a.n + 511) / 512, uint64_t(sms) * (smem <= (100u << 10) ? 2 : 1));
        k_closed_accumulate_c<<<uint32_t(std::max<uint64_t>(blocks, 1)), 512, smem, st>>>(a, s);
        return;
    }
    const size_t per = size_t(a.dim + 1) * 4;
    const uint32_t G = uint32_t(std::max<size_t>(1, std::min<size_t>(a.K, (200u << 10) / per)));
    const uint32_t groups = (a.K + G - 1) / G;
    const size_t smem = G * per + G * 4;
    ensure_dynamic_smem(reinterpret_cast<const void*>(k_closed_accumulate), smem);
    const uint64_t blocks = std::min<uint64_t>((a.n + 511) / 512, uint64_t(sms));
    k_closed_accumulate<<<dim3(uint32_t(std::max<uint64_t>(blocks, 1)), groups), 512, smem, st>>>(a, s, G);
}

void launch_closed_finish(const ClosedArgs& a, ClosedState s, cudaStream_t st) {
    const char* fe = getenv("SEGHDC_CLOSED_FIN");  // "smem": the one-CTA kernels (read per launch)
    if (!(fe && *fe) && !getenv("SEGHDC_CLOSED_FIN_GLOBAL")) {
        const uint32_t seg = (a.dim + kFinG - 1) / kFinG;
        const size_t smem = (size_t(seg) + 1) * 4 + seg;
        if (ensure_dynamic_smem(reinterpret_cast<const void*>(k_closed_finish_cl), smem) == cudaSuccess) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(a.K * kFinG);
            cfg.blockDim = dim3(kFinCT);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = kFinG;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cudaLaunchKernelEx(&cfg, k_closed_finish_cl, a, s) == cudaSuccess) return;
            cudaGetLastError();
        }
    }
    const size_t smem = fin_smem_bytes(a.dim);
    if (!getenv("SEGHDC_CLOSED_FIN_GLOBAL") && smem <= (200u << 10) &&
        ensure_dynamic_smem(reinterpret_cast<const void*>(k_closed_finish_smem), smem) == cudaSuccess) {
        k_closed_finish_smem<<<a.K, kFinT, smem, st>>>(a, s);
        return;
    }
    k_closed_finish<<<a.K, kFinT, 0, st>>>(a, s);
}

#ifdef SEGHDC_CHECKED
unsigned int check_line_closed() { return take_check_line(); }
#endif

}  // namespace seghdc_dev

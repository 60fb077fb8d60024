// Closed-form Manhattan variant (SURVEY.md §7 hard part 4, §8f rank 1): the K-means loop over
// the Manhattan pixel HVs without materialising them. Launchers of seghdc_closed.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace seghdc_dev {

// Every Manhattan pixel HV is B ^ (XOR of 2 + C runs of ones), B = XOR of the 2 + C bases
// (seghdc_host::manhattan_bases): row run [0, (i / beta) * x_row) (position_encoder.cpp:50-64),
// column run [dim/2, dim/2 + (j / beta) * x_col), colour run [off_ch, off_ch + v * unit_ch)
// (color_encoder.cpp:47-52 widened at pixel_pipeline.cpp:70-88).
struct ClosedArgs {
    const uint8_t* img;  // H x W x C interleaved
    uint64_t n;          // pixels
    uint32_t w, c, dim, beta, x_row, x_col, K;
    uint32_t off[3], unit[3];
    // compressed endpoint tables: every run endpoint is one of L = nr + nc + 256 C + 1 positions
    // (row ends b * x_row, column ends dim/2 + b * x_col, colour ends off_ch + v * unit_ch, dim)
    uint32_t nr, nc, L;
};

// Per-cluster state on the device (int64 prefix tables, see seghdc_closed.cu):
//   Q[K][dim + 1], P[K], norm2[K], Z[K][dim] (the centroid IntVectors), diff[K][dim + 1],
//   cnt[K] (members being accumulated), counts[K] (member_counts of the current set),
//   bflag[dim] (bits of B, one byte each), changed (labels that changed in the last assign).
struct ClosedState {
    long long* Q;
    unsigned long long* P;
    unsigned long long* norm2;
    uint32_t* Z;
    int32_t* diff;
    unsigned long long* cnt;
    unsigned long long* counts;
    const uint8_t* bflag;
    uint32_t* labels;
    unsigned long long* changed;
    int32_t* diffc;  // [K][L] difference counts on compressed endpoint indices (k_closed_accumulate_c)
    unsigned long long* wraps;  // this round's count of 128-bit-wrapping comparisons (diagnostic)
};

// centroids from the seed pixels (clusterer.cpp:197-205): runs of seed k into diff[k], cnt[k] = 1
void launch_closed_seed(const ClosedArgs& a, const uint64_t* seeds, ClosedState s, cudaStream_t st);
// assign_labels (clusterer.cpp:132-162) in O(K) prefix-table lookups per pixel
void launch_closed_assign(const ClosedArgs& a, ClosedState s, int sms, cudaStream_t st);
// update_centroids (clusterer.cpp:164-188), accumulation half: member runs into diff / cnt
void launch_closed_accumulate(const ClosedArgs& a, ClosedState s, int sms, cudaStream_t st);
// update_centroids, finish half: Z, norm2, P, Q of every non-empty cluster (empty -> previous)
void launch_closed_finish(const ClosedArgs& a, ClosedState s, cudaStream_t st);

}  // namespace seghdc_dev

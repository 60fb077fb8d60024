/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product.
 *
 * Plain-C restatement of the reference SegHDC hot path (reference = /root/reference/proj).
 * Used by tests/ as the checker, by bench.py's cpu_baseline / --impl reference legs as the
 * timed CPU port, and by __graft_entry__.smoke() as the checker. Pinned against the
 * compiled reference (oracle/_ref) and the reference test suites' golden instances
 * (tests/golden/) by tests/test_oracle.py.
 *
 * Layout conventions are the reference's: a hypervector is ceil(dim/64) little-endian u64
 * words, bit i = (w[i>>6] >> (i&63)) & 1, tail bits zero (hypervector.hpp:15-42). A grid is
 * n_pixels * words_per_hv contiguous u64 (pixel_pipeline.hpp:38-62). Centroids are k*dim u32.
 * Return codes: 0 ok, 1 configuration error (reference ConfigError), 2 other.
 */
#ifndef SEGHDC_ORACLE_H
#define SEGHDC_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

const char* so_last_error(void);
size_t so_words_for(size_t dim);

/* std::mt19937_64 (reference hypervector.hpp:13) — first `n` outputs for `seed`. */
void so_mt64_stream(uint64_t seed, size_t n, uint64_t* out);

/* Codebooks in run_pipeline's RNG order (pipeline.cpp:43-59). encoder: 0 manhattan,
 * 1 rpos, 2 rcolor. widened_out: channels*256 full-dim HVs (pixel_pipeline.cpp:70-88). */
int so_build_codebooks(size_t dim, size_t h, size_t w, size_t c, double alpha, size_t beta,
                       size_t gamma, uint64_t seed, int encoder, uint64_t* row_out,
                       uint64_t* col_out, uint64_t* widened_out);

/* encode_image (pixel_pipeline.cpp:92-126), table driven. */
int so_encode(const uint8_t* px, size_t h, size_t w, size_t c, size_t dim, const uint64_t* row,
              const uint64_t* col, const uint64_t* widened, uint64_t* grid_out);

/* select_initial_centroids (clusterer.cpp:54-130); seeds as row-major linear indices. */
int so_select_seeds(const uint8_t* px, size_t h, size_t w, size_t c, size_t k, uint64_t* seeds_out);

/* assign_labels (clusterer.cpp:132-162). */
int so_assign(const uint64_t* grid, size_t n, size_t dim, const uint32_t* z, size_t k,
              uint32_t* labels_out);

/* update_centroids (clusterer.cpp:164-188). prev_counts may be NULL. */
int so_update(const uint64_t* grid, size_t n, size_t dim, const uint32_t* labels,
              const uint32_t* prev_z, size_t k, uint32_t* z_out, uint64_t* counts_out);

/* cluster (clusterer.cpp:190-218) plus the centroid set used by the final assignment.
 * labels_rounds (nullable): iterations*n u32, round r at offset (r-1)*n. */
int so_cluster(const uint64_t* grid, const uint8_t* px, size_t h, size_t w, size_t c,
               size_t dim, size_t k, size_t iterations, int early_stop, uint32_t* labels_rounds,
               uint32_t* labels_final, uint32_t* centroids_out, uint64_t* counts_out,
               size_t* rounds_out);

/* so_cluster without a stored grid (pixels re-encoded from the tables every pass); for
 * configurations whose grid does not fit host memory. Same outputs as so_cluster. */
int so_cluster_stream(const uint8_t* px, size_t h, size_t w, size_t c, size_t dim, const uint64_t* row,
                      const uint64_t* col, const uint64_t* widened, size_t k, size_t iterations, int early_stop,
                      uint32_t* labels_rounds, uint32_t* labels_final, uint32_t* centroids_out,
                      uint64_t* counts_out, size_t* rounds_out);

/* Per-round count of strictly_closer comparisons whose 128-bit products wrapped (either side
 * >= 2^128) in the last so_assign (1 round) / so_cluster / so_cluster_stream call; returns
 * the number of rounds recorded, copies up to cap. Diagnostic, not reference API. */
size_t so_last_wraps(uint64_t* out, size_t cap);

/* threads used by the OpenMP loops (0 = OpenMP default). */
void so_set_threads(int n);
int so_get_threads(void);

#ifdef __cplusplus
}
#endif
#endif

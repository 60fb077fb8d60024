/* seghdc_cuda.h — C-ABI of the B200-native SegHDC encode + cluster hot path.
 *
 * The reference (arXiv 2303.12753 artifact, /root/reference/proj) exposes this path only as
 * the C++ API of its static library `seghdc`; it has no FFI. Each entry point below names the
 * reference interface it replaces (file:line, relative to proj/). The C++ drop-in library
 * (include/seghdc/seghdc.hpp) and the Python host API (paper_2303_12753_b200) are written
 * on top of exactly these symbols; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Plain pointers and sizes; no C++ or torch types cross this boundary.
 *  - Hypervectors use the reference layout: ceil(dim/64) little-endian u64 words, bit i =
 *    (w[i>>6] >> (i&63)) & 1, tail bits zero (include/seghdc/hypervector.hpp:15-42). A grid is
 *    h*w*ceil(dim/64) contiguous u64 words, row-major (pixel_pipeline.hpp:38-62).
 *  - Centroids are k*dim u32 (raw integer member sums, clusterer.hpp:27-34).
 *  - Return value: SEGHDC_OK, SEGHDC_ECONFIG (the reference would throw ConfigError,
 *    errors.hpp:9-12) or SEGHDC_ERUNTIME (CUDA failure; the reference has no analogue).
 *    No exception ever crosses this boundary; seghdc_last_error() holds the message.
 *  - One context per (host thread, device). Calls are ordered on the context's stream and
 *    are synchronous unless the name ends in _async.
 */
#ifndef SEGHDC_CUDA_H
#define SEGHDC_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEGHDC_OK 0
#define SEGHDC_ECONFIG 1
#define SEGHDC_ERUNTIME 2

#define SEGHDC_ENCODER_MANHATTAN 0 /* EncoderKind::manhattan (pixel_pipeline.hpp:64) */
#define SEGHDC_ENCODER_RPOS 1      /* EncoderKind::rpos */
#define SEGHDC_ENCODER_RCOLOR 2    /* EncoderKind::rcolor */

typedef struct seghdc_ctx seghdc_ctx;

/* Per-round observer: (user, 1-based round, labels of that round [n_local]). Mirrors
 * IterationCallback (clusterer.hpp:74); invoked synchronously after each assignment. */
typedef void (*seghdc_round_cb)(void* user, size_t round, const uint32_t* labels);

/* ---- context -------------------------------------------------------------------------- */
int seghdc_create(int device, seghdc_ctx** out);
void seghdc_destroy(seghdc_ctx* ctx);
/* Last error message of ctx (or of the calling thread when ctx is NULL). */
const char* seghdc_last_error(const seghdc_ctx* ctx);
/* Order all further work of ctx on an external cudaStream_t (NULL: the context's own). */
int seghdc_set_stream(seghdc_ctx* ctx, void* cuda_stream);
/* Size this context's kernel grids for `sms` SMs (0: the whole device), so several contexts on
   separate streams share the GPU (batches of small images run side by side). No reference
   counterpart: a scheduling hint that leaves every result unchanged. */
int seghdc_set_sm_budget(seghdc_ctx* ctx, int sms);
int seghdc_synchronize(seghdc_ctx* ctx);
/* Number of device kernels this context has launched so far (for launch accounting). */
uint64_t seghdc_kernel_launches(const seghdc_ctx* ctx);
/* Name of the round kernel the last clustering plan selected ("k_round_tc", "k_round_fused",
 * "k_round"; "" before any plan). */
const char* seghdc_round_kernel(const seghdc_ctx* ctx);

/* Diagnostic (no reference counterpart): per-round number of strictly_closer comparisons
 * (clusterer.cpp:41-50) whose unsigned __int128 products exceeded 2^128 in the last clustering
 * run of ctx (seghdc_cluster / _async / run_pipeline / run_pipeline_closed / assign; a shard
 * counts its own pixels). The result is still the reference's wrapped comparison; this only
 * reports how often it happened. Copies min(rounds, cap) counts; rounds_out = rounds run.
 * Counting is opt-in (seghdc_set_wrap_counting before the run): on the largest images it
 * selects round-kernel variants that carry the extra arithmetic (about 5-10% at C4); labels
 * and centroids are identical either way. */
int seghdc_set_wrap_counting(seghdc_ctx* ctx, int enable);
int seghdc_round_wraps(seghdc_ctx* ctx, uint64_t* out, size_t cap, size_t* rounds_out);

/* ---- host-side codebooks (stay on the host: mt19937_64 is sequential and cheap) -------- */
/* run_pipeline's codebook stage (pipeline.cpp:43-59): one Rng(seed), position codebook
 * (position_encoder.hpp:45, or build_random_position_codebook pixel_pipeline.hpp:79 for
 * RPOS), then colour codebook (color_encoder.hpp:42, or build_random_color_codebook
 * pixel_pipeline.hpp:82 for RCOLOR). Outputs row_out[h][wph], col_out[w][wph] and the colour
 * tables widened to full dim, widened_out[c][256][wph] (pixel_pipeline.cpp:70-88). */
int seghdc_build_codebooks(size_t dim, size_t h, size_t w, size_t c, double alpha, size_t beta,
                           size_t gamma, uint64_t seed, int encoder, uint64_t* row_out,
                           uint64_t* col_out, uint64_t* widened_out);
/* RunConfig::validate (pipeline.cpp:25-30) without building anything. */
int seghdc_validate_run(size_t dim, size_t h, size_t w, size_t c, double alpha, size_t beta,
                        size_t gamma, size_t k, size_t iterations);

/* ---- encode_image (pixel_pipeline.hpp:74-75) ----------------------------------------- */
/* Uploads image + tables, materialises the pixel HV grid on the device (it stays resident
 * in ctx for cluster), and copies it to grid_out if non-NULL. */
int seghdc_encode(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c,
                  size_t dim, const uint64_t* row_words, const uint64_t* col_words,
                  const uint64_t* widened_words, uint64_t* grid_out);

/* ---- clustering on a host grid (clusterer.hpp:54-80) --------------------------------- */
/* select_initial_centroids (clusterer.hpp:54-55); seeds as row-major linear indices. */
int seghdc_select_seeds(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c,
                        size_t k, uint64_t* seeds_out);
/* assign_labels (clusterer.hpp:60). grid may be NULL to use the resident grid. */
int seghdc_assign(seghdc_ctx* ctx, const uint64_t* grid, size_t h, size_t w, size_t dim,
                  const uint32_t* centroids, size_t k, uint32_t* labels_out);
/* update_centroids (clusterer.hpp:65-66). grid may be NULL to use the resident grid.
 * prev_counts is accepted for API parity and ignored (the reference ignores it too). */
int seghdc_update(seghdc_ctx* ctx, const uint64_t* grid, size_t h, size_t w, size_t dim,
                  const uint32_t* labels, const uint32_t* prev_centroids, size_t k,
                  uint32_t* centroids_out, uint64_t* counts_out);
/* cluster (clusterer.hpp:79-80). grid may be NULL to use the resident grid (then h, w, dim
 * must match it). Outputs: labels_out[h*w]; optional centroids_out[k*dim] and
 * counts_out[k] = the centroid set used by the final assignment round (cluster() itself
 * hides it; clusterer.hpp:68-71); rounds_out = ClusterResult::iterations_run. */
int seghdc_cluster(seghdc_ctx* ctx, const uint64_t* grid, const uint8_t* pixels, size_t h,
                   size_t w, size_t c, size_t dim, size_t k, size_t iterations, int early_stop,
                   seghdc_round_cb on_round, void* user, uint32_t* labels_out,
                   uint32_t* centroids_out, uint64_t* counts_out, size_t* rounds_out);

/* ---- whole pipeline (pipeline.hpp:55-56, run_pipeline) ------------------------------- */
/* timings_ms_out (nullable) receives {encode_position, encode_color, produce_pixels,
 * cluster, total} in that order (StageTimings, pipeline.hpp:37-45); device stages are
 * timed with CUDA events. */
int seghdc_run_pipeline(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c,
                        size_t dim, double alpha, size_t beta, size_t gamma, size_t k,
                        size_t iterations, uint64_t seed, int encoder, int early_stop,
                        seghdc_round_cb on_round, void* user, uint32_t* labels_out,
                        size_t* rounds_out, double* timings_ms_out);

/* ---- a batch of same-shape images (the reference CLI's `batch`, seghdc_main.cpp:180-225) */
/* run_pipeline for each of n_images images of one shape and config (one codebook set):
 * labels_out[i] (h*w u32) and rounds_out[i] (nullable) per image; results identical to n
 * separate seghdc_run_pipeline calls. Images run side by side on child streams, each with a
 * share of the SMs (SEGHDC_BATCH_GROUPS, default 4). */
int seghdc_run_pipeline_batch(seghdc_ctx* ctx, const uint8_t* const* pixels, size_t n_images, size_t h,
                              size_t w, size_t c, size_t dim, double alpha, size_t beta, size_t gamma,
                              size_t k, size_t iterations, uint64_t seed, int encoder, int early_stop,
                              uint32_t* const* labels_out, size_t* rounds_out);

/* ---- closed-form Manhattan variant (SURVEY.md §7 hard part 4, §8f rank 1) ------------ */
/* run_pipeline (pipeline.cpp:40-75) + cluster (clusterer.cpp:190-218) for the Manhattan
 * encoder without materialising the pixel HVs: each HV is B ^ (2 + C runs of ones), so
 * dot_words is 10 prefix-table lookups per cluster and update_centroids a difference array.
 * Same labels, centroids (k x dim u32, the set used by the final assignment), member counts
 * and rounds as the packed path; k <= 32. */
int seghdc_run_pipeline_closed(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w,
                               size_t c, size_t dim, double alpha, size_t beta, size_t gamma,
                               size_t k, size_t iterations, uint64_t seed, int early_stop,
                               uint32_t* labels_out, uint32_t* centroids_out,
                               uint64_t* counts_out, size_t* rounds_out);

/* ---- device-resident staging (no reference analogue: keeps HVs in HBM) --------------- */
/* Image: full image on every rank. Codebooks: tables as produced by seghdc_build_codebooks.
 * Pointers are host pointers unless the *_device variant is used. */
int seghdc_load_image(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c);
int seghdc_load_codebooks(seghdc_ctx* ctx, size_t dim, const uint64_t* row_words,
                          const uint64_t* col_words, const uint64_t* widened_words);
/* Encode image rows [row_begin, row_end) (a row-block shard; 0..h for the whole image)
 * into the resident grid. No host synchronisation. */
int seghdc_encode_async(seghdc_ctx* ctx, size_t row_begin, size_t row_end);
/* Resident grid <-> host (reference layout). load_grid sets rows [row_begin,row_end). */
int seghdc_load_grid(seghdc_ctx* ctx, const uint64_t* grid, size_t h, size_t w, size_t dim,
                     size_t row_begin, size_t row_end);
int seghdc_store_grid(seghdc_ctx* ctx, uint64_t* grid_out);
/* Full clustering loop on the resident grid/image without host synchronisation (no
 * callback). Results stay on the device until seghdc_fetch_results. */
int seghdc_cluster_async(seghdc_ctx* ctx, size_t k, size_t iterations, int early_stop);
int seghdc_fetch_results(seghdc_ctx* ctx, uint32_t* labels_out, uint32_t* centroids_out,
                         uint64_t* counts_out, size_t* rounds_out);

/* ---- row-block sharding across ranks (one process per GPU) --------------------------- */
/* The caller owns the collective (e.g. torch.distributed / NCCL all_reduce, SUM, int32) on
 * the device buffer returned by seghdc_exchange_buffer; everything else is local.
 *   seghdc_shard_begin(k, iterations, early_stop)      seeds (redundant per rank), colsums
 *   -> all_reduce(exchange)                            init: seed-pixel bits + colsums
 *   seghdc_shard_init_finish()
 *   for r in 1..iterations:
 *     seghdc_shard_assign(r)                            labels + per-shard partial sums
 *     if seghdc_shard_round_needs_exchange(r):
 *        -> all_reduce(exchange)                        [k*dim sums | k counts | changed]
 *        seghdc_shard_finish(r)                         identical finalisation on all ranks
 * Integer sums are order independent, so every rank holds bit-identical centroids. */
int seghdc_shard_begin(seghdc_ctx* ctx, size_t k, size_t iterations, int early_stop);
int seghdc_exchange_buffer(seghdc_ctx* ctx, void** device_ptr, size_t* n_int32);
/* Host-staged exchange (e.g. a gloo/MPI all-reduce, or G shards emulated on one device):
 * copy the current exchange buffer (n_int32 entries) to / from host memory. */
int seghdc_exchange_download(seghdc_ctx* ctx, int32_t* host);
int seghdc_exchange_upload(seghdc_ctx* ctx, const int32_t* host);
int seghdc_shard_init_finish(seghdc_ctx* ctx);
int seghdc_shard_assign(seghdc_ctx* ctx, size_t round);
int seghdc_shard_round_needs_exchange(const seghdc_ctx* ctx, size_t round);
int seghdc_shard_finish(seghdc_ctx* ctx, size_t round);

/* ---- multi-GPU with the collective inside the library (one process per GPU) ----------- */
/* Row-block sharding of one image: rank r of n owns the contiguous pixel rows
 * seghdc_shard_rows(h, r, n) and the full image; seeds are selected redundantly on every rank;
 * the only collective is one SUM all-reduce (int32) per round of the exchange buffer. Integer
 * sums are order independent: every rank ends with bit-identical centroids and its rows'
 * labels equal the single-GPU run's. The reference is single-threaded (clusterer.cpp:190-218
 * is the loop being sharded); these calls have no reference counterpart.
 *
 * Collective, one of:
 *  - NCCL (NVLink / NVSwitch): rank 0 calls seghdc_nccl_get_unique_id, ships the 128 bytes to
 *    the other ranks out of band, every rank calls seghdc_nccl_init. libnccl.so.2 is loaded
 *    at run time (no link-time dependency).
 *  - any other (MPI, gloo, host-staged): seghdc_set_allreduce with a callback that leaves
 *    device_buf[0..n) equal to the SUM over ranks, ordered on (or synchronising) cuda_stream;
 *    it returns 0 on success. */
#define SEGHDC_NCCL_UNIQUE_ID_BYTES 128
typedef int (*seghdc_allreduce_fn)(void* user, int32_t* device_buf, size_t n_int32, void* cuda_stream);
int seghdc_nccl_get_unique_id(void* id_out /* SEGHDC_NCCL_UNIQUE_ID_BYTES */);
int seghdc_nccl_init(seghdc_ctx* ctx, const void* unique_id, int rank, int nranks);
int seghdc_set_allreduce(seghdc_ctx* ctx, seghdc_allreduce_fn fn, void* user, int rank, int nranks);
/* rows [row_begin, row_end) of rank `rank`: contiguous blocks differing by at most one row */
int seghdc_shard_rows(size_t h, int rank, int nranks, size_t* row_begin, size_t* row_end);
/* the same for this context's rank (seghdc_nccl_init / seghdc_set_allreduce; 0 of 1 before) */
int seghdc_shard_row_range(const seghdc_ctx* ctx, size_t h, size_t* row_begin, size_t* row_end);
/* cluster() over this rank's resident rows (seghdc_load_image + seghdc_load_codebooks +
 * seghdc_encode_async(row_begin, row_end) first); no host synchronisation; results through
 * seghdc_fetch_results (labels of this rank's rows). */
int seghdc_cluster_sharded_async(seghdc_ctx* ctx, size_t k, size_t iterations, int early_stop);
/* run_pipeline (pipeline.cpp:40-75) sharded: every rank passes the full image; labels_out
 * receives this rank's rows (seghdc_shard_rows), centroids_out / counts_out (nullable) the
 * final centroid set, identical on every rank. */
int seghdc_run_pipeline_sharded(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c,
                                size_t dim, double alpha, size_t beta, size_t gamma, size_t k,
                                size_t iterations, uint64_t seed, int encoder, int early_stop,
                                uint32_t* labels_out, uint32_t* centroids_out, uint64_t* counts_out,
                                size_t* rounds_out, double* timings_ms_out);

/* ---- scoring (metrics.hpp:22-36, metrics.cpp:42-101; off the throughput path) -------- */
/* best_foreground_iou: the highest IoU of any non-empty proper subset of the k <= 4 cluster
 * labels (k = 1: the whole image) against gt_bits (h*w, nonzero = foreground); ties to the
 * smallest, then lexicographically smallest subset, returned as a bit mask of labels.
 * SEGHDC_ECONFIG for k = 0 or k > 4 or a label >= k, like the reference's ConfigError. */
int seghdc_best_foreground_iou(const uint32_t* labels, const uint8_t* gt_bits, size_t h, size_t w, size_t k,
                               double* iou_out, uint32_t* subset_mask_out);

/* ---- measurement -------------------------------------------------------------------- */
/* Bracket every round kernel (the dominant kernel) with CUDA events on the context's stream;
 * profile_read synchronises and returns the summed kernel time and launch count since the
 * last read (used by bench.py for the roofline fraction). */
int seghdc_profile_rounds(seghdc_ctx* ctx, int enable);
int seghdc_profile_read(seghdc_ctx* ctx, double* total_ms, uint64_t* count);
/* as profile_read, plus the first `cap` per-launch times (in launch order) into each_ms */
int seghdc_profile_read_each(seghdc_ctx* ctx, double* total_ms, uint64_t* count, double* each_ms, size_t cap);

/* Page-locked host memory (cudaHostAlloc, portable) for result buffers: device->host copies
 * of labels into it run at full PCIe rate instead of through the driver's pageable staging. */
int seghdc_pinned_alloc(size_t bytes, void** out);
int seghdc_pinned_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* SEGHDC_CUDA_H */

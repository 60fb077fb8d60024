// seghdc.hpp — C++ drop-in for the SegHDC encoder/clusterer API on B200.
//
// Source-compatible with the reference library's public headers
// (/root/reference/proj/include/seghdc/{errors,hypervector,position_encoder,color_encoder,
// pixel_pipeline,clusterer,pipeline}.hpp): the same namespace, type and function names,
// argument meaning and exceptions, so code written against the reference recompiles
// unchanged (the per-name headers next to this file forward here). The host-side value types
// and codebook builders run on the CPU exactly as in the reference; encode_image,
// select_initial_centroids, assign_labels, update_centroids, cluster and run_pipeline run on
// the GPU through the C-ABI in include/seghdc_cuda.h. Out of scope (not on the hot path):
// metrics/IoU, image I/O, the CLI and the JSON metrics record.
#pragma once

#include <cstddef>
#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace seghdc {

// ---- errors (reference errors.hpp:9-18) ----------------------------------------------------
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};

// ---- hypervectors (reference hypervector.hpp) ------------------------------------------------
using Rng = std::mt19937_64;

// Packed binary hypervector: ceil(dim/64) little-endian u64 words, bits >= dim always zero.
class Hypervector {
public:
    Hypervector() = default;
    explicit Hypervector(std::size_t dim);
    static Hypervector random(std::size_t dim, Rng& rng);
    static std::size_t words_for(std::size_t dim) noexcept { return (dim + 63) / 64; }

    std::size_t dim() const noexcept { return n_; }
    std::size_t word_count() const noexcept { return w_.size(); }
    std::span<const std::uint64_t> words() const noexcept { return w_; }
    std::span<std::uint64_t> words() noexcept { return w_; }
    bool bit(std::size_t i) const;
    void set_bit(std::size_t i, bool v);
    std::size_t popcount() const noexcept;
    friend bool operator==(const Hypervector&, const Hypervector&) = default;

private:
    std::size_t n_ = 0;
    std::vector<std::uint64_t> w_;
};

// Non-negative integer vector (centroid member sums).
class IntVector {
public:
    IntVector() = default;
    explicit IntVector(std::size_t dim) : v_(dim, 0) {}
    static IntVector from_hv(const Hypervector& h);

    std::size_t dim() const noexcept { return v_.size(); }
    std::uint32_t operator[](std::size_t i) const { return v_[i]; }
    std::uint32_t& operator[](std::size_t i) { return v_[i]; }
    std::span<const std::uint32_t> values() const noexcept { return v_; }
    void add(const Hypervector& h);
    void add_words(std::span<const std::uint64_t> hv_words);
    std::uint64_t norm_squared() const noexcept;
    void scale(std::uint32_t factor);
    friend bool operator==(const IntVector&, const IntVector&) = default;

private:
    std::vector<std::uint32_t> v_;
};

Hypervector hv_xor(const Hypervector& a, const Hypervector& b);
inline Hypervector operator^(const Hypervector& a, const Hypervector& b) { return hv_xor(a, b); }
Hypervector flip_range(const Hypervector& h, std::size_t start, std::size_t len);
std::size_t hamming_distance(const Hypervector& a, const Hypervector& b);
std::size_t hamming_distance_words(std::span<const std::uint64_t> a, std::span<const std::uint64_t> b);
double cosine_distance(const Hypervector& a, const Hypervector& b);
double cosine_distance(const IntVector& a, const IntVector& b);
double cosine_distance(const Hypervector& a, const IntVector& b);
inline double cosine_distance(const IntVector& a, const Hypervector& b) { return cosine_distance(b, a); }
IntVector accumulate(IntVector acc, const Hypervector& h);
Hypervector concat(std::span<const Hypervector> parts);
std::uint64_t dot_words(std::span<const std::uint64_t> hv_words, const IntVector& z);
std::uint64_t dot(const Hypervector& y, const IntVector& z);
std::uint64_t dot(const IntVector& y, const IntVector& z);

// ---- position code (reference position_encoder.hpp) ----------------------------------------
struct PositionConfig {
    std::size_t dim = 0;
    std::size_t n_rows = 0;
    std::size_t n_cols = 0;
    double alpha = 0.2;
    std::size_t beta = 1;
    std::size_t x_row() const;
    std::size_t x_col() const;
    void validate() const;
};
struct PositionCodebook {
    PositionConfig config;
    std::vector<Hypervector> row_hvs;
    std::vector<Hypervector> col_hvs;
};
std::size_t block_index(std::size_t i, std::size_t beta);
PositionCodebook build_position_codebook(const PositionConfig& config, Rng& rng);
Hypervector position_hv(const PositionCodebook& cb, std::size_t i, std::size_t j);

// ---- colour code (reference color_encoder.hpp) ---------------------------------------------
struct ColorConfig {
    std::size_t dim = 0;
    std::size_t channels = 1;
    std::size_t gamma = 1;
    std::vector<std::size_t> channel_dims() const;
    std::size_t unit_flip(std::size_t channel) const;
    void validate() const;
};
struct ColorCodebook {
    ColorConfig config;
    std::vector<std::vector<Hypervector>> tables;
};
ColorCodebook build_color_codebook(const ColorConfig& config, Rng& rng);
Hypervector encode_color(const ColorCodebook& cb, std::span<const std::uint8_t> color);
Hypervector encode_color(const ColorCodebook& cb, std::initializer_list<std::uint8_t> color);

// ---- pixel pipeline (reference pixel_pipeline.hpp) -----------------------------------------
struct ImageBuffer {
    std::size_t height = 0;
    std::size_t width = 0;
    std::size_t channels = 1;
    std::vector<std::uint8_t> pixels;  // row-major, channel-interleaved
    std::uint8_t at(std::size_t i, std::size_t j, std::size_t c) const { return pixels[(i * width + j) * channels + c]; }
    std::uint8_t& at(std::size_t i, std::size_t j, std::size_t c) { return pixels[(i * width + j) * channels + c]; }
    std::span<const std::uint8_t> pixel(std::size_t i, std::size_t j) const {
        return {pixels.data() + (i * width + j) * channels, channels};
    }
    std::size_t pixel_count() const { return height * width; }
    void validate() const;
};

// H*W*words_per_hv contiguous u64 words (host copy of the device-resident grid).
class PixelHvGrid {
public:
    PixelHvGrid() = default;
    PixelHvGrid(std::size_t height, std::size_t width, std::size_t dim);
    std::size_t height() const noexcept { return h_; }
    std::size_t width() const noexcept { return w_; }
    std::size_t dim() const noexcept { return d_; }
    std::size_t words_per_hv() const noexcept { return wph_; }
    std::size_t payload_bytes() const noexcept { return data_.size() * sizeof(std::uint64_t); }
    std::span<const std::uint64_t> hv_words(std::size_t i, std::size_t j) const {
        return {data_.data() + (i * w_ + j) * wph_, wph_};
    }
    std::span<std::uint64_t> hv_words(std::size_t i, std::size_t j) { return {data_.data() + (i * w_ + j) * wph_, wph_}; }
    Hypervector hv(std::size_t i, std::size_t j) const;
    void set_hv(std::size_t i, std::size_t j, const Hypervector& h);

private:
    std::size_t h_ = 0, w_ = 0, d_ = 0, wph_ = 0;
    std::vector<std::uint64_t> data_;
};

enum class EncoderKind { manhattan, rpos, rcolor };
EncoderKind encoder_kind_from_string(const std::string& s);
std::string to_string(EncoderKind kind);
Hypervector pixel_hv(const Hypervector& p, const Hypervector& v);
PixelHvGrid encode_image(const ImageBuffer& img, const PositionCodebook& pos_cb, const ColorCodebook& color_cb);
PositionCodebook build_random_position_codebook(const PositionConfig& config, Rng& rng);
ColorCodebook build_random_color_codebook(const ColorConfig& config, Rng& rng);

// ---- clusterer (reference clusterer.hpp) ---------------------------------------------------
struct ClusterConfig {
    std::size_t k = 2;
    std::size_t iterations = 10;
    bool early_stop = true;
    void validate(std::size_t pixel_count) const;
};
struct PixelCoord {
    std::size_t row = 0;
    std::size_t col = 0;
    friend bool operator==(const PixelCoord&, const PixelCoord&) = default;
};
struct CentroidSet {
    std::vector<IntVector> centroids;
    std::vector<std::size_t> member_counts;
    std::size_t k() const { return centroids.size(); }
};
struct SegmentationMask {
    std::size_t height = 0;
    std::size_t width = 0;
    std::vector<std::uint32_t> labels;
    std::uint32_t label(std::size_t i, std::size_t j) const { return labels[i * width + j]; }
    std::uint32_t& label(std::size_t i, std::size_t j) { return labels[i * width + j]; }
    friend bool operator==(const SegmentationMask&, const SegmentationMask&) = default;
};
std::vector<PixelCoord> select_initial_centroids(const ImageBuffer& img, const PixelHvGrid& grid, std::size_t k);
SegmentationMask assign_labels(const PixelHvGrid& grid, const CentroidSet& centroids);
CentroidSet update_centroids(const PixelHvGrid& grid, const SegmentationMask& mask, const CentroidSet& prev);
struct ClusterResult {
    SegmentationMask mask;
    std::size_t iterations_run = 0;
};
using IterationCallback = std::function<void(std::size_t, const SegmentationMask&)>;
ClusterResult cluster(const PixelHvGrid& grid, const ImageBuffer& img, const ClusterConfig& config,
                      const IterationCallback& on_iteration = {});

// ---- run_pipeline (reference pipeline.hpp:18-56; MetricsRecord/JSON out of scope) ----------
struct RunConfig {
    std::size_t dim = 10000;
    double alpha = 0.2;
    std::size_t beta = 26;
    std::size_t gamma = 1;
    std::size_t clusters = 2;
    std::size_t iterations = 10;
    std::uint64_t seed = 0;
    EncoderKind encoder = EncoderKind::manhattan;
    bool early_stop = true;
    PositionConfig position_config(const ImageBuffer& img) const;
    ColorConfig color_config(const ImageBuffer& img) const;
    void validate(const ImageBuffer& img) const;
};
struct StageTimings {
    double encode_position_ms = 0.0;
    double encode_color_ms = 0.0;
    double produce_pixels_ms = 0.0;
    double cluster_ms = 0.0;
    double total_ms = 0.0;
    std::map<std::string, double> as_map() const;
};
struct PipelineResult {
    SegmentationMask mask;
    std::size_t iterations_run = 0;
    StageTimings timings;
};
PipelineResult run_pipeline(const ImageBuffer& img, const RunConfig& config, const IterationCallback& on_iteration = {});

// ---- scoring (reference metrics.hpp / metrics.cpp:42-101; csrc/seghdc_metrics.cpp) ---------------
/// Foreground flags, row-major.
struct BinaryMask {
    std::size_t height = 0;
    std::size_t width = 0;
    std::vector<std::uint8_t> bits;  // 0 or 1
    bool at(std::size_t i, std::size_t j) const { return bits[i * width + j] != 0; }
};

/// Any nonzero channel counts as foreground (0/255 ground-truth images).
BinaryMask binarize_ground_truth(const ImageBuffer& img);

/// |pred AND gt| / |pred OR gt|; 1.0 when both masks are empty. ConfigError on shape mismatch.
double iou(const BinaryMask& pred, const BinaryMask& gt);

struct ForegroundMatch {
    double iou = 0.0;
    std::vector<std::uint32_t> subset;  // cluster labels binarized to foreground
};

/// Max IoU over every non-empty proper subset of cluster labels (k = 1: the whole image);
/// ties go to the smallest subset, then the lexicographically smallest. k must be <= 4.
ForegroundMatch best_foreground_iou(const SegmentationMask& mask, const BinaryMask& gt, std::size_t k);

// ---- image and mask files (reference image_io.hpp / image_io.cpp:31-217; csrc/seghdc_image_io.cpp:
// a PNG codec over zlib and the P5 reader, the reference's error contract) -----------------------
/// Reads an 8-bit grayscale or RGB PNG, or a binary PGM (P5). The format is detected from the
/// magic bytes, not the extension. 16-bit files, PNG colour types other than gray / RGB and
/// interlaced PNGs are rejected with IoError.
ImageBuffer load_image(const std::string& path);

/// 8-bit PNG, grayscale for 1 channel, RGB for 3. Deterministic bytes for identical inputs.
void save_image(const ImageBuffer& img, const std::string& path);

/// 8-bit grayscale PNG with label l mapped to floor(255 l / (k - 1)); k = 1 writes zeros.
void save_mask(const SegmentationMask& mask, std::size_t k, const std::string& path);

/// Inverse of save_mask's level mapping: every pixel snaps to the nearest of the k levels.
SegmentationMask labels_from_mask_image(const ImageBuffer& img, std::size_t k);

// ---- B200 extras ------------------------------------------------------------------------------
// The drop-in uses one CUDA context per host thread on this device (default 0).
void set_device(int device);
// Centroids of the final assignment (cluster() itself does not return them; clusterer.hpp:68-71).
struct ClusterResultWithCentroids {
    ClusterResult result;
    CentroidSet centroids;
};
ClusterResultWithCentroids cluster_with_centroids(const PixelHvGrid& grid, const ImageBuffer& img,
                                                  const ClusterConfig& config, const IterationCallback& on_iteration = {});

// Multi-GPU: row-block sharding of one image, one process (or host thread) per GPU. Rank 0
// calls nccl_unique_id() and ships the bytes to the other ranks out of band (MPI_Bcast, a
// file, a socket); every rank calls init_sharding(...) once and then run_pipeline_sharded()
// with the FULL image. Each rank gets its rows' labels; the centroids are bit-identical on
// every rank, and the rows of all ranks together equal run_pipeline()'s mask (the only
// exchange is one NCCL all-reduce per round, clusterer.cpp:190-218 sharded).
using NcclUniqueId = std::array<std::uint8_t, 128>;
NcclUniqueId nccl_unique_id();
void init_sharding(const NcclUniqueId& id, int rank, int nranks);
struct ShardedPipelineResult {
    std::size_t row_begin = 0, row_end = 0;  // this rank's rows of the image
    SegmentationMask rows;                   // (row_end - row_begin) x width labels
    CentroidSet centroids;                   // the centroid set of the final assignment
    std::size_t iterations_run = 0;
    StageTimings timings;
};
ShardedPipelineResult run_pipeline_sharded(const ImageBuffer& img, const RunConfig& config);

}  // namespace seghdc

// Host side of the SegHDC B200 path that stays on the CPU by design: RunConfig validation,
// the codebooks (std::mt19937_64 is a sequential stream; building the tables takes < 2 ms)
// . Behaviour follows the reference file:line cited at
// each function; the GPU path consumes the tables through seghdc_encode.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/seghdc_cuda.h"
#include "host_internal.h"

namespace seghdc_host {

namespace {

size_t words_for(size_t dim) { return (dim + 63) / 64; }

// Hypervector::random (hypervector.cpp:33-39): one 64-bit draw per word, tail bits cleared.
void random_hv(uint64_t* w, size_t dim, std::mt19937_64& rng) {
    const size_t nw = words_for(dim);
    for (size_t i = 0; i < nw; ++i) w[i] = rng();
    if (dim % 64) w[nw - 1] &= ~0ULL >> (64 - dim % 64);
}

// Invert bits [start, start + len) in place (flip_range, hypervector.cpp:67-84).
void invert_run(uint64_t* w, size_t dim, size_t start, size_t len) {
    if (start + len > dim || start + len < start)
        throw Error(SEGHDC_ECONFIG, "flip_range out of bounds: [" + std::to_string(start) + ", " +
                                        std::to_string(start + len) + ") exceeds dim " + std::to_string(dim));
    size_t i = start;
    const size_t end = start + len;
    while (i < end) {
        const size_t off = i & 63, take = std::min<size_t>(64 - off, end - i);
        w[i >> 6] ^= (take == 64 ? ~0ULL : ((1ULL << take) - 1)) << off;
        i += take;
    }
}

size_t flip_unit(double alpha, size_t dim, size_t n) {  // position_encoder.cpp:10-18
    return static_cast<size_t>(std::floor(alpha * static_cast<double>(dim) / (2.0 * static_cast<double>(n))));
}

size_t channel_dim(size_t dim, size_t c, size_t ch) { return dim / c + (ch < dim % c ? 1 : 0); }  // color_encoder.cpp:9-13
size_t unit_flip(size_t dim, size_t c, size_t gamma, size_t ch) {                              // color_encoder.cpp:15-18
    return gamma * (channel_dim(dim, c, ch) / (256 * gamma));
}

// One axis of the Manhattan position code (position_encoder.cpp:50-64).
void position_axis(uint64_t* out, size_t n, size_t beta, size_t x, size_t dim, size_t half_start,
                   std::mt19937_64& rng) {
    const size_t nw = words_for(dim);
    random_hv(out, dim, rng);
    size_t cursor = half_start;
    for (size_t i = 1; i < n; ++i) {
        std::memcpy(out + i * nw, out + (i - 1) * nw, nw * 8);
        if (i / beta != (i - 1) / beta) {
            invert_run(out + i * nw, dim, cursor, x);
            cursor += x;
        }
    }
}

}  // namespace

// PositionConfig::validate (position_encoder.cpp:20-39).
void validate_position(size_t dim, size_t h, size_t w, double alpha, size_t beta) {
    if (dim == 0 || h == 0 || w == 0)
        throw Error(SEGHDC_ECONFIG, "position config: dim, n_rows and n_cols must be >= 1");
    if (!(alpha > 0.0 && alpha <= 1.0))
        throw Error(SEGHDC_ECONFIG, "position config: alpha must be in (0, 1], got " + std::to_string(alpha));
    if (beta == 0) throw Error(SEGHDC_ECONFIG, "position config: beta must be >= 1");
    if (flip_unit(alpha, dim, h) == 0)
        throw Error(SEGHDC_ECONFIG, "dimension too small for image size: x_row = floor(" + std::to_string(alpha) +
                                        " * " + std::to_string(dim) + " / (2 * " + std::to_string(h) +
                                        ")) = 0; need alpha*dim >= 2*n_rows");
    if (flip_unit(alpha, dim, w) == 0)
        throw Error(SEGHDC_ECONFIG, "dimension too small for image size: x_col = floor(" + std::to_string(alpha) +
                                        " * " + std::to_string(dim) + " / (2 * " + std::to_string(w) +
                                        ")) = 0; need alpha*dim >= 2*n_cols");
}

// ColorConfig::validate (color_encoder.cpp:20-35).
void validate_color(size_t dim, size_t c, size_t gamma) {
    if (dim == 0) throw Error(SEGHDC_ECONFIG, "color config: dim must be >= 1");
    if (c != 1 && c != 3)
        throw Error(SEGHDC_ECONFIG, "color config: channels must be 1 or 3, got " + std::to_string(c));
    if (gamma == 0) throw Error(SEGHDC_ECONFIG, "color config: gamma must be >= 1");
    for (size_t ch = 0; ch < c; ++ch)
        if (unit_flip(dim, c, gamma, ch) < gamma)
            throw Error(SEGHDC_ECONFIG, "dimension too small for color resolution: channel " + std::to_string(ch) +
                                            " has sub-dim " + std::to_string(channel_dim(dim, c, ch)) +
                                            ", needs >= 256*gamma = " + std::to_string(256 * gamma));
}

// ImageBuffer::validate (pixel_pipeline.cpp:9-18).
void validate_image(size_t h, size_t w, size_t c) {
    if (h == 0 || w == 0) throw Error(SEGHDC_ECONFIG, "image dimensions must be positive");
    if (c != 1 && c != 3) throw Error(SEGHDC_ECONFIG, "image channels must be 1 or 3, got " + std::to_string(c));
}

// ClusterConfig::validate (clusterer.cpp:10-18).
void validate_cluster(size_t k, size_t iterations, size_t pixel_count) {
    if (k == 0) throw Error(SEGHDC_ECONFIG, "cluster config: k must be >= 1");
    if (iterations == 0) throw Error(SEGHDC_ECONFIG, "cluster config: iterations must be >= 1");
    if (k > pixel_count)
        throw Error(SEGHDC_ECONFIG, "cluster config: k = " + std::to_string(k) + " exceeds pixel count " +
                                        std::to_string(pixel_count));
}

void build_position(size_t dim, size_t h, size_t w, double alpha, size_t beta, int encoder,
                    std::mt19937_64& rng, uint64_t* row_out, uint64_t* col_out) {
    validate_position(dim, h, w, alpha, beta);
    const size_t nw = words_for(dim);
    if (encoder == SEGHDC_ENCODER_RPOS) {  // build_random_position_codebook (pixel_pipeline.cpp:128-141)
        for (size_t i = 0; i < h; ++i) random_hv(row_out + i * nw, dim, rng);
        for (size_t j = 0; j < w; ++j) random_hv(col_out + j * nw, dim, rng);
        return;
    }
    // build_position_codebook (position_encoder.cpp:68-76): rows flip in [0, d/2), cols in [d/2, d)
    position_axis(row_out, h, beta, flip_unit(alpha, dim, h), dim, 0, rng);
    position_axis(col_out, w, beta, flip_unit(alpha, dim, w), dim, dim / 2, rng);
}

void build_color(size_t dim, size_t c, size_t gamma, int encoder, std::mt19937_64& rng, uint64_t* widened_out) {
    validate_color(dim, c, gamma);
    const size_t nw = words_for(dim);
    std::memset(widened_out, 0, c * 256 * nw * 8);
    size_t offset = 0;
    for (size_t ch = 0; ch < c; ++ch) {
        const size_t d_ch = channel_dim(dim, c, ch), u = unit_flip(dim, c, gamma, ch);
        std::vector<uint64_t> entry(words_for(d_ch));
        random_hv(entry.data(), d_ch, rng);
        size_t cursor = 0;
        for (int v = 0; v < 256; ++v) {
            if (v > 0) {
                if (encoder == SEGHDC_ENCODER_RCOLOR) {  // build_random_color_codebook (pixel_pipeline.cpp:143-156)
                    random_hv(entry.data(), d_ch, rng);
                } else {  // build_color_codebook (color_encoder.cpp:37-55): entry v flips the next u bits
                    invert_run(entry.data(), d_ch, cursor, u);
                    cursor += u;
                }
            }
            // channel entry placed at its concatenation offset (pixel_pipeline.cpp:70-88), one
            // shifted word at a time (the entry's tail bits are zero, so OR-ing whole words is exact)
            uint64_t* dst = widened_out + (ch * 256 + size_t(v)) * nw;
            const size_t w0 = offset >> 6, sh = offset & 63;
            for (size_t k = 0; k < entry.size(); ++k) {
                dst[w0 + k] |= entry[k] << sh;
                if (sh && w0 + k + 1 < nw) dst[w0 + k + 1] |= entry[k] >> (64 - sh);
            }
        }
        offset += d_ch;
    }
}

ManhattanParams manhattan_bases(size_t dim, size_t h, size_t w, size_t c, double alpha, size_t beta, size_t gamma,
                                std::mt19937_64& rng, uint64_t* bases) {
    validate_position(dim, h, w, alpha, beta);
    validate_color(dim, c, gamma);
    const size_t nw = words_for(dim);
    ManhattanParams p{};
    p.dim = uint32_t(dim);
    p.h = uint32_t(h);
    p.w = uint32_t(w);
    p.c = uint32_t(c);
    p.beta = uint32_t(beta);
    p.x_row = uint32_t(flip_unit(alpha, dim, h));
    p.x_col = uint32_t(flip_unit(alpha, dim, w));
    random_hv(bases, dim, rng);       // position_axis(rows): Hypervector::random
    random_hv(bases + nw, dim, rng);  // position_axis(cols)
    std::memset(bases + 2 * nw, 0, c * nw * 8);
    size_t offset = 0;
    for (size_t ch = 0; ch < c; ++ch) {
        const size_t d_ch = channel_dim(dim, c, ch);
        std::vector<uint64_t> entry(words_for(d_ch));
        random_hv(entry.data(), d_ch, rng);  // build_color_codebook: the channel's base entry
        uint64_t* dst = bases + (2 + ch) * nw;
        const size_t w0 = offset >> 6, sh = offset & 63;
        for (size_t k = 0; k < entry.size(); ++k) {
            dst[w0 + k] |= entry[k] << sh;
            if (sh && w0 + k + 1 < nw) dst[w0 + k + 1] |= entry[k] >> (64 - sh);
        }
        p.off[ch] = uint32_t(offset);
        p.unit[ch] = uint32_t(unit_flip(dim, c, gamma, ch));
        offset += d_ch;
    }
    return p;
}

}  // namespace seghdc_host

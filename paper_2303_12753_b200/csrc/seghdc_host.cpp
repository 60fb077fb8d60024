// Host side of the SegHDC B200 path that stays on the CPU by design: RunConfig validation,
// the codebooks (std::mt19937_64 is a sequential stream; building the tables takes < 2 ms)
// and the synthetic bench/test images. Behaviour follows the reference file:line cited at
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

// ---- synthetic nuclei images -----------------------------------------------
// One std::mt19937_64(seed) stream; uniforms u = (x >> 11) * 2^-53; normals by Box-Muller
// (cos branch only); ellipses drawn as (cy, cx, a, b, theta, class); inside test at pixel
// centres, later ellipses overwrite; per-pixel, per-channel noise; config 1 blurs the float
// image with a separable Gaussian (sigma 1.5, radius 5, reflect-101) before rounding.
namespace {
struct SynthSpec {
    size_t h, w, c;
    int n_ellipses;
    double semi_lo, semi_hi;
    double bg_mean, bg_sd;
    int n_classes;
    double fg[7][3];
    double fg_sd;
    bool random_means;
    bool blur;
};

SynthSpec spec_for(int id) {
    SynthSpec s{};
    switch (id) {
        case 0:
        case 2:
            s = {256, 256, 3, 20, 5, 15, 30, 10, 1, {{200, 200, 200}}, 20, false, false};
            break;
        case 1:
            s = {520, 696, 1, 60, 4, 12, 20, 8, 1, {{180, 180, 180}}, 25, false, true};
            break;
        case 3:
            s = {2048, 2048, 3, 1500, 5, 20, 25, 10, 3, {{200, 60, 60}, {60, 200, 60}, {60, 60, 200}}, 15, false,
                 false};
            break;
        case 4:
            s = {4096, 4096, 3, 6000, 5, 20, 20, 8, 7, {}, 12, true, false};
            break;
        default:
            throw Error(SEGHDC_ECONFIG, "synthetic config id must be 0..4, got " + std::to_string(id));
    }
    return s;
}
}  // namespace

void synth_image(int id, uint64_t seed, uint8_t* out, size_t* h_out, size_t* w_out, size_t* c_out) {
    SynthSpec s = spec_for(id);
    *h_out = s.h;
    *w_out = s.w;
    *c_out = s.c;
    if (!out) return;
    std::mt19937_64 rng(seed);
    auto u = [&] { return double(rng() >> 11) * (1.0 / 9007199254740992.0); };
    auto normal = [&] {
        const double u1 = 1.0 - u(), u2 = u();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    };
    if (s.random_means)
        for (int k = 0; k < s.n_classes; ++k)
            for (int ch = 0; ch < 3; ++ch) s.fg[k][ch] = 40.0 + 190.0 * u();
    const size_t H = s.h, W = s.w, C = s.c;
    std::vector<uint8_t> cls(H * W, 0);
    for (int e = 0; e < s.n_ellipses; ++e) {
        const double cy = u() * double(H), cx = u() * double(W);
        const double a = s.semi_lo + (s.semi_hi - s.semi_lo) * u();
        const double b = s.semi_lo + (s.semi_hi - s.semi_lo) * u();
        const double th = M_PI * u();
        int k = 0;
        if (s.n_classes > 1) k = std::min(s.n_classes - 1, int(u() * s.n_classes));
        const double ct = std::cos(th), sn = std::sin(th), r = std::max(a, b);
        const long i0 = std::max(0L, long(std::floor(cy - r))), i1 = std::min(long(H) - 1, long(std::ceil(cy + r)));
        const long j0 = std::max(0L, long(std::floor(cx - r))), j1 = std::min(long(W) - 1, long(std::ceil(cx + r)));
        for (long i = i0; i <= i1; ++i)
            for (long j = j0; j <= j1; ++j) {
                const double y = double(i) + 0.5 - cy, x = double(j) + 0.5 - cx;
                const double xr = x * ct + y * sn, yr = -x * sn + y * ct;
                if ((xr / a) * (xr / a) + (yr / b) * (yr / b) <= 1.0) cls[size_t(i) * W + size_t(j)] = uint8_t(k + 1);
            }
    }
    std::vector<double> val(H * W * C);
    for (size_t p = 0; p < H * W; ++p)
        for (size_t ch = 0; ch < C; ++ch) {
            const int k = cls[p];
            const double mean = k ? s.fg[k - 1][ch] : s.bg_mean, sd = k ? s.fg_sd : s.bg_sd;
            val[p * C + ch] = mean + sd * normal();
        }
    if (s.blur) {
        const int R = 5;
        const double sigma = 1.5;
        double wk[2 * R + 1], norm = 0;
        for (int k = -R; k <= R; ++k) norm += (wk[k + R] = std::exp(-double(k * k) / (2 * sigma * sigma)));
        for (double& x : wk) x /= norm;
        auto refl = [](long i, long n) {  // reflect-101
            while (i < 0 || i >= n) i = i < 0 ? -i : 2 * (n - 1) - i;
            return i;
        };
        std::vector<double> tmp(val.size());
        for (size_t i = 0; i < H; ++i)
            for (size_t j = 0; j < W; ++j)
                for (size_t ch = 0; ch < C; ++ch) {
                    double acc = 0;
                    for (int k = -R; k <= R; ++k) acc += wk[k + R] * val[(i * W + size_t(refl(long(j) + k, long(W)))) * C + ch];
                    tmp[(i * W + j) * C + ch] = acc;
                }
        for (size_t i = 0; i < H; ++i)
            for (size_t j = 0; j < W; ++j)
                for (size_t ch = 0; ch < C; ++ch) {
                    double acc = 0;
                    for (int k = -R; k <= R; ++k) acc += wk[k + R] * tmp[(size_t(refl(long(i) + k, long(H))) * W + j) * C + ch];
                    val[(i * W + j) * C + ch] = acc;
                }
    }
    for (size_t e = 0; e < val.size(); ++e) {
        const long v = std::lround(val[e]);
        out[e] = uint8_t(v < 0 ? 0 : v > 255 ? 255 : v);
    }
}

}  // namespace seghdc_host

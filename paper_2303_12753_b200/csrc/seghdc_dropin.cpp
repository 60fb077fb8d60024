// C++ drop-in for the reference `seghdc::` API (include/seghdc/seghdc.hpp). Host value types
// and codebooks follow the reference semantics (file:line cited per function, relative to
// /root/reference/proj); the hot path (encode_image, select_initial_centroids,
// assign_labels, update_centroids, cluster, run_pipeline) runs on the GPU through the C-ABI.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/seghdc/seghdc.hpp"
#include "../../include/seghdc_cuda.h"

namespace seghdc {

namespace {

[[noreturn]] void fail(const std::string& m) { throw ConfigError(m); }

void same_dim(std::size_t a, std::size_t b, const char* op) {
    if (a != b) fail(std::string(op) + ": dimension mismatch (" + std::to_string(a) + " vs " + std::to_string(b) + ")");
}

std::uint64_t low_bits(std::size_t n) { return n >= 64 ? ~0ULL : ((1ULL << n) - 1); }

// ---- device context: one per host thread ------------------------------------------------------
int g_device = 0;
struct CtxDeleter {
    void operator()(seghdc_ctx* c) const { seghdc_destroy(c); }
};
thread_local std::unique_ptr<seghdc_ctx, CtxDeleter> t_ctx;
thread_local int t_ctx_device = -1;

seghdc_ctx* ctx() {
    if (!t_ctx || t_ctx_device != g_device) {
        seghdc_ctx* c = nullptr;
        if (seghdc_create(g_device, &c) != SEGHDC_OK) throw std::runtime_error(seghdc_last_error(nullptr));
        t_ctx.reset(c);
        t_ctx_device = g_device;
    }
    return t_ctx.get();
}

void check(int rc, const seghdc_ctx* c) {
    if (rc == SEGHDC_OK) return;
    const std::string m = seghdc_last_error(c);
    if (rc == SEGHDC_ECONFIG) throw ConfigError(m);
    throw std::runtime_error(m);
}

// flip the run [start, start+len) of a word array in place
void flip_run(std::uint64_t* w, std::size_t start, std::size_t len) {
    for (std::size_t i = start, end = start + len; i < end;) {
        const std::size_t off = i & 63, take = std::min<std::size_t>(64 - off, end - i);
        w[i >> 6] ^= low_bits(take) << off;
        i += take;
    }
}

}  // namespace

void set_device(int device) { g_device = device; }

// ---- Hypervector / IntVector (reference hypervector.cpp) --------------------------------------
Hypervector::Hypervector(std::size_t dim) : n_(dim), w_(words_for(dim), 0) {
    if (dim == 0) fail("hypervector dimension must be >= 1");
}

Hypervector Hypervector::random(std::size_t dim, Rng& rng) {  // hypervector.cpp:33-39
    Hypervector h(dim);
    for (auto& x : h.w_) x = rng();
    if (dim % 64) h.w_.back() &= low_bits(dim % 64);
    return h;
}

bool Hypervector::bit(std::size_t i) const {
    if (i >= n_) fail("hypervector bit index out of range");
    return (w_[i >> 6] >> (i & 63)) & 1;
}

void Hypervector::set_bit(std::size_t i, bool v) {
    if (i >= n_) fail("hypervector bit index out of range");
    const std::uint64_t m = 1ULL << (i & 63);
    w_[i >> 6] = v ? (w_[i >> 6] | m) : (w_[i >> 6] & ~m);
}

std::size_t Hypervector::popcount() const noexcept {
    std::size_t s = 0;
    for (auto x : w_) s += std::popcount(x);
    return s;
}

IntVector IntVector::from_hv(const Hypervector& h) {
    IntVector v(h.dim());
    v.add(h);
    return v;
}

void IntVector::add(const Hypervector& h) {
    if (h.dim() != dim())
        fail("accumulate: dimension mismatch (" + std::to_string(dim()) + " vs " + std::to_string(h.dim()) + ")");
    add_words(h.words());
}

void IntVector::add_words(std::span<const std::uint64_t> hv) {  // hypervector.cpp:112-121
    for (std::size_t k = 0; k < hv.size(); ++k)
        for (std::uint64_t x = hv[k]; x; x &= x - 1) ++v_[(k << 6) + std::size_t(std::countr_zero(x))];
}

std::uint64_t IntVector::norm_squared() const noexcept {
    std::uint64_t s = 0;
    for (auto x : v_) s += std::uint64_t(x) * x;
    return s;
}

void IntVector::scale(std::uint32_t f) {
    for (auto& x : v_) x *= f;
}

Hypervector hv_xor(const Hypervector& a, const Hypervector& b) {
    same_dim(a.dim(), b.dim(), "xor");
    Hypervector o(a.dim());
    for (std::size_t k = 0; k < o.word_count(); ++k) o.words()[k] = a.words()[k] ^ b.words()[k];
    return o;
}

Hypervector flip_range(const Hypervector& h, std::size_t start, std::size_t len) {  // hypervector.cpp:67-84
    if (start + len > h.dim() || start + len < start)
        fail("flip_range out of bounds: [" + std::to_string(start) + ", " + std::to_string(start + len) +
             ") exceeds dim " + std::to_string(h.dim()));
    Hypervector o = h;
    flip_run(o.words().data(), start, len);
    return o;
}

std::size_t hamming_distance_words(std::span<const std::uint64_t> a, std::span<const std::uint64_t> b) {
    std::size_t s = 0;
    for (std::size_t k = 0; k < a.size(); ++k) s += std::popcount(a[k] ^ b[k]);
    return s;
}

std::size_t hamming_distance(const Hypervector& a, const Hypervector& b) {
    same_dim(a.dim(), b.dim(), "hamming_distance");
    return hamming_distance_words(a.words(), b.words());
}

namespace {
double cosine_parts(std::uint64_t d, std::uint64_t n2a, std::uint64_t n2b) {  // hypervector.cpp:157-163
    if (n2a == 0 || n2b == 0) return 1.0;
    return 1.0 - double(d) / (std::sqrt(double(n2a)) * std::sqrt(double(n2b)));
}
}  // namespace

double cosine_distance(const Hypervector& a, const Hypervector& b) {
    same_dim(a.dim(), b.dim(), "cosine_distance");
    std::uint64_t inter = 0;
    for (std::size_t k = 0; k < a.word_count(); ++k) inter += std::popcount(a.words()[k] & b.words()[k]);
    return cosine_parts(inter, a.popcount(), b.popcount());
}

double cosine_distance(const IntVector& a, const IntVector& b) {
    same_dim(a.dim(), b.dim(), "cosine_distance");
    return cosine_parts(dot(a, b), a.norm_squared(), b.norm_squared());
}

double cosine_distance(const Hypervector& a, const IntVector& b) {
    same_dim(a.dim(), b.dim(), "cosine_distance");
    return cosine_parts(dot(a, b), a.popcount(), b.norm_squared());
}

IntVector accumulate(IntVector acc, const Hypervector& h) {
    acc.add(h);
    return acc;
}

Hypervector concat(std::span<const Hypervector> parts) {  // hypervector.cpp:195-214
    if (parts.empty()) fail("concat: at least one part required");
    std::size_t total = 0;
    for (const auto& p : parts) total += p.dim();
    Hypervector o(total);
    std::size_t off = 0;
    for (const auto& p : parts) {
        const std::size_t w0 = off >> 6, sh = off & 63;
        for (std::size_t k = 0; k < p.word_count(); ++k) {
            o.words()[w0 + k] |= p.words()[k] << sh;
            if (sh && w0 + k + 1 < o.word_count()) o.words()[w0 + k + 1] |= p.words()[k] >> (64 - sh);
        }
        off += p.dim();
    }
    return o;
}

std::uint64_t dot_words(std::span<const std::uint64_t> hv, const IntVector& z) {  // hypervector.cpp:138-151
    std::uint64_t s = 0;
    const auto v = z.values();
    for (std::size_t k = 0; k < hv.size(); ++k)
        for (std::uint64_t x = hv[k]; x; x &= x - 1) s += v[(k << 6) + std::size_t(std::countr_zero(x))];
    return s;
}

std::uint64_t dot(const Hypervector& y, const IntVector& z) {
    same_dim(y.dim(), z.dim(), "dot");
    return dot_words(y.words(), z);
}

std::uint64_t dot(const IntVector& y, const IntVector& z) {
    same_dim(y.dim(), z.dim(), "dot");
    std::uint64_t s = 0;
    for (std::size_t i = 0; i < y.dim(); ++i) s += std::uint64_t(y[i]) * z[i];
    return s;
}

// ---- position code (reference position_encoder.cpp) -------------------------------------------
std::size_t PositionConfig::x_row() const {
    return std::size_t(std::floor(alpha * double(dim) / (2.0 * double(n_rows))));
}
std::size_t PositionConfig::x_col() const {
    return std::size_t(std::floor(alpha * double(dim) / (2.0 * double(n_cols))));
}

void PositionConfig::validate() const {  // position_encoder.cpp:20-39
    if (dim == 0 || n_rows == 0 || n_cols == 0) fail("position config: dim, n_rows and n_cols must be >= 1");
    if (!(alpha > 0.0 && alpha <= 1.0)) fail("position config: alpha must be in (0, 1], got " + std::to_string(alpha));
    if (beta == 0) fail("position config: beta must be >= 1");
    auto zero = [&](const char* which, std::size_t n, const char* need) {
        fail(std::string("dimension too small for image size: ") + which + " = floor(" + std::to_string(alpha) +
             " * " + std::to_string(dim) + " / (2 * " + std::to_string(n) + ")) = 0; need alpha*dim >= 2*" + need);
    };
    if (x_row() == 0) zero("x_row", n_rows, "n_rows");
    if (x_col() == 0) zero("x_col", n_cols, "n_cols");
}

std::size_t block_index(std::size_t i, std::size_t beta) { return i / beta; }

namespace {
std::vector<Hypervector> axis(std::size_t n, std::size_t beta, std::size_t x, std::size_t dim, std::size_t half,
                              Rng& rng) {  // position_encoder.cpp:50-64
    std::vector<Hypervector> out;
    out.reserve(n);
    Hypervector cur = Hypervector::random(dim, rng);
    std::size_t cursor = half;
    for (std::size_t i = 0; i < n; ++i) {
        if (i && block_index(i, beta) != block_index(i - 1, beta)) {
            cur = flip_range(cur, cursor, x);
            cursor += x;
        }
        out.push_back(cur);
    }
    return out;
}
}  // namespace

PositionCodebook build_position_codebook(const PositionConfig& config, Rng& rng) {
    config.validate();
    PositionCodebook cb{config, axis(config.n_rows, config.beta, config.x_row(), config.dim, 0, rng), {}};
    cb.col_hvs = axis(config.n_cols, config.beta, config.x_col(), config.dim, config.dim / 2, rng);
    return cb;
}

Hypervector position_hv(const PositionCodebook& cb, std::size_t i, std::size_t j) {
    if (i >= cb.row_hvs.size() || j >= cb.col_hvs.size())
        fail("position index (" + std::to_string(i) + ", " + std::to_string(j) + ") out of range for " +
             std::to_string(cb.row_hvs.size()) + "x" + std::to_string(cb.col_hvs.size()) + " codebook");
    return hv_xor(cb.row_hvs[i], cb.col_hvs[j]);
}

// ---- colour code (reference color_encoder.cpp) ------------------------------------------------
std::vector<std::size_t> ColorConfig::channel_dims() const {
    std::vector<std::size_t> d(channels, dim / channels);
    for (std::size_t c = 0; c < dim % channels; ++c) ++d[c];
    return d;
}

std::size_t ColorConfig::unit_flip(std::size_t channel) const {
    return gamma * (channel_dims().at(channel) / (256 * gamma));
}

void ColorConfig::validate() const {  // color_encoder.cpp:20-35
    if (dim == 0) fail("color config: dim must be >= 1");
    if (channels != 1 && channels != 3) fail("color config: channels must be 1 or 3, got " + std::to_string(channels));
    if (gamma == 0) fail("color config: gamma must be >= 1");
    for (std::size_t c = 0; c < channels; ++c)
        if (unit_flip(c) < gamma)
            fail("dimension too small for color resolution: channel " + std::to_string(c) + " has sub-dim " +
                 std::to_string(channel_dims()[c]) + ", needs >= 256*gamma = " + std::to_string(256 * gamma));
}

ColorCodebook build_color_codebook(const ColorConfig& config, Rng& rng) {  // color_encoder.cpp:37-55
    config.validate();
    ColorCodebook cb{config, {}};
    const auto dims = config.channel_dims();
    for (std::size_t ch = 0; ch < config.channels; ++ch) {
        const std::size_t u = config.unit_flip(ch);
        std::vector<Hypervector> t;
        t.reserve(256);
        t.push_back(Hypervector::random(dims[ch], rng));
        for (int v = 1; v < 256; ++v) t.push_back(flip_range(t.back(), std::size_t(v - 1) * u, u));
        cb.tables.push_back(std::move(t));
    }
    return cb;
}

Hypervector encode_color(const ColorCodebook& cb, std::span<const std::uint8_t> color) {
    if (color.size() != cb.config.channels)
        fail("encode_color: expected " + std::to_string(cb.config.channels) + " channel values, got " +
             std::to_string(color.size()));
    if (cb.config.channels == 1) return cb.tables[0][color[0]];
    std::vector<Hypervector> parts;
    for (std::size_t ch = 0; ch < color.size(); ++ch) parts.push_back(cb.tables[ch][color[ch]]);
    return concat(parts);
}

Hypervector encode_color(const ColorCodebook& cb, std::initializer_list<std::uint8_t> color) {
    return encode_color(cb, std::span<const std::uint8_t>(color.begin(), color.size()));
}

// ---- pixel pipeline (reference pixel_pipeline.cpp) --------------------------------------------
void ImageBuffer::validate() const {
    if (height == 0 || width == 0) fail("image dimensions must be positive");
    if (channels != 1 && channels != 3) fail("image channels must be 1 or 3, got " + std::to_string(channels));
    if (pixels.size() != height * width * channels) fail("image pixel buffer size mismatch");
}

PixelHvGrid::PixelHvGrid(std::size_t height, std::size_t width, std::size_t dim)
    : h_(height), w_(width), d_(dim), wph_(Hypervector::words_for(dim)), data_(height * width * wph_, 0) {
    if (height == 0 || width == 0 || dim == 0) fail("pixel grid dimensions must be positive");
}

Hypervector PixelHvGrid::hv(std::size_t i, std::size_t j) const {
    Hypervector h(d_);
    std::memcpy(h.words().data(), hv_words(i, j).data(), wph_ * 8);
    return h;
}

void PixelHvGrid::set_hv(std::size_t i, std::size_t j, const Hypervector& h) {
    if (h.dim() != d_) fail("set_hv: dimension mismatch");
    std::memcpy(hv_words(i, j).data(), h.words().data(), wph_ * 8);
}

EncoderKind encoder_kind_from_string(const std::string& s) {
    if (s == "manhattan") return EncoderKind::manhattan;
    if (s == "rpos") return EncoderKind::rpos;
    if (s == "rcolor") return EncoderKind::rcolor;
    fail("unknown encoder kind '" + s + "' (expected manhattan, rpos or rcolor)");
}

std::string to_string(EncoderKind k) {
    return k == EncoderKind::rpos ? "rpos" : k == EncoderKind::rcolor ? "rcolor" : "manhattan";
}

Hypervector pixel_hv(const Hypervector& p, const Hypervector& v) { return hv_xor(p, v); }

PixelHvGrid encode_image(const ImageBuffer& img, const PositionCodebook& pos, const ColorCodebook& color) {
    img.validate();  // pixel_pipeline.cpp:94-108
    if (pos.config.n_rows != img.height || pos.config.n_cols != img.width)
        fail("position codebook shape (" + std::to_string(pos.config.n_rows) + "x" + std::to_string(pos.config.n_cols) +
             ") does not match image (" + std::to_string(img.height) + "x" + std::to_string(img.width) + ")");
    if (color.config.channels != img.channels) fail("color codebook channels do not match image");
    if (pos.config.dim != color.config.dim) fail("position and color codebooks must share one dimension");
    const std::size_t d = pos.config.dim, wph = Hypervector::words_for(d);
    std::vector<std::uint64_t> row(img.height * wph), col(img.width * wph), wid(img.channels * 256 * wph, 0);
    for (std::size_t i = 0; i < img.height; ++i) std::memcpy(&row[i * wph], pos.row_hvs[i].words().data(), wph * 8);
    for (std::size_t j = 0; j < img.width; ++j) std::memcpy(&col[j * wph], pos.col_hvs[j].words().data(), wph * 8);
    std::size_t off = 0;  // colour entries widened to full dim (pixel_pipeline.cpp:70-88)
    for (std::size_t ch = 0; ch < img.channels; ++ch) {
        for (int v = 0; v < 256; ++v) {
            const Hypervector& e = color.tables[ch][v];
            std::uint64_t* dst = &wid[(ch * 256 + v) * wph];
            const std::size_t w0 = off >> 6, sh = off & 63;
            for (std::size_t k = 0; k < e.word_count(); ++k) {
                dst[w0 + k] |= e.words()[k] << sh;
                if (sh && w0 + k + 1 < wph) dst[w0 + k + 1] |= e.words()[k] >> (64 - sh);
            }
        }
        off += color.tables[ch][0].dim();
    }
    PixelHvGrid grid(img.height, img.width, d);
    seghdc_ctx* c = ctx();
    check(seghdc_encode(c, img.pixels.data(), img.height, img.width, img.channels, d, row.data(), col.data(),
                        wid.data(), grid.hv_words(0, 0).data()),
          c);
    return grid;
}

PositionCodebook build_random_position_codebook(const PositionConfig& config, Rng& rng) {
    config.validate();
    PositionCodebook cb{config, {}, {}};
    for (std::size_t i = 0; i < config.n_rows; ++i) cb.row_hvs.push_back(Hypervector::random(config.dim, rng));
    for (std::size_t j = 0; j < config.n_cols; ++j) cb.col_hvs.push_back(Hypervector::random(config.dim, rng));
    return cb;
}

ColorCodebook build_random_color_codebook(const ColorConfig& config, Rng& rng) {
    config.validate();
    ColorCodebook cb{config, {}};
    for (std::size_t d : config.channel_dims()) {
        std::vector<Hypervector> t;
        for (int v = 0; v < 256; ++v) t.push_back(Hypervector::random(d, rng));
        cb.tables.push_back(std::move(t));
    }
    return cb;
}

// ---- clusterer (reference clusterer.cpp) ------------------------------------------------------
void ClusterConfig::validate(std::size_t pixel_count) const {
    if (k == 0) fail("cluster config: k must be >= 1");
    if (iterations == 0) fail("cluster config: iterations must be >= 1");
    if (k > pixel_count)
        fail("cluster config: k = " + std::to_string(k) + " exceeds pixel count " + std::to_string(pixel_count));
}

std::vector<PixelCoord> select_initial_centroids(const ImageBuffer& img, const PixelHvGrid& grid, std::size_t k) {
    img.validate();
    if (grid.height() != img.height || grid.width() != img.width)
        fail("select_initial_centroids: grid shape does not match image");
    if (k == 0 || k > img.pixel_count())
        fail("select_initial_centroids: k = " + std::to_string(k) + " out of range for " +
             std::to_string(img.pixel_count()) + " pixels");
    std::vector<std::uint64_t> lin(k);
    seghdc_ctx* c = ctx();
    check(seghdc_select_seeds(c, img.pixels.data(), img.height, img.width, img.channels, k, lin.data()), c);
    std::vector<PixelCoord> out;
    for (auto p : lin) out.push_back({std::size_t(p / img.width), std::size_t(p % img.width)});
    return out;
}

namespace {
std::vector<std::uint32_t> flatten(const CentroidSet& cs, std::size_t dim) {
    std::vector<std::uint32_t> z(cs.k() * dim);
    for (std::size_t c = 0; c < cs.k(); ++c) {
        if (cs.centroids[c].dim() != dim) fail("dimension mismatch");
        std::memcpy(&z[c * dim], cs.centroids[c].values().data(), dim * 4);
    }
    return z;
}
CentroidSet unflatten(const std::vector<std::uint32_t>& z, const std::vector<std::uint64_t>& counts,
                      std::size_t k, std::size_t dim) {
    CentroidSet cs;
    for (std::size_t c = 0; c < k; ++c) {
        IntVector v(dim);
        for (std::size_t i = 0; i < dim; ++i) v[i] = z[c * dim + i];
        cs.centroids.push_back(std::move(v));
        cs.member_counts.push_back(counts[c]);
    }
    return cs;
}
}  // namespace

SegmentationMask assign_labels(const PixelHvGrid& grid, const CentroidSet& centroids) {
    const std::size_t k = centroids.k();
    if (k == 0) fail("assign_labels: empty centroid set");
    for (const auto& z : centroids.centroids)
        if (z.dim() != grid.dim()) fail("assign_labels: dimension mismatch");
    const auto z = flatten(centroids, grid.dim());
    SegmentationMask m{grid.height(), grid.width(), std::vector<std::uint32_t>(grid.height() * grid.width())};
    seghdc_ctx* c = ctx();
    check(seghdc_assign(c, grid.hv_words(0, 0).data(), grid.height(), grid.width(), grid.dim(), z.data(), k,
                        m.labels.data()),
          c);
    return m;
}

CentroidSet update_centroids(const PixelHvGrid& grid, const SegmentationMask& mask, const CentroidSet& prev) {
    if (mask.height != grid.height() || mask.width != grid.width())
        fail("update_centroids: mask shape does not match grid");
    const std::size_t k = prev.k(), d = grid.dim();
    std::vector<std::uint32_t> zprev(k * d, 0);
    for (std::size_t c = 0; c < k; ++c)
        if (prev.centroids[c].dim() == d) std::memcpy(&zprev[c * d], prev.centroids[c].values().data(), d * 4);
    std::vector<std::uint32_t> z(k * d);
    std::vector<std::uint64_t> counts(k);
    seghdc_ctx* c = ctx();
    check(seghdc_update(c, grid.hv_words(0, 0).data(), grid.height(), grid.width(), d, mask.labels.data(),
                        zprev.data(), k, z.data(), counts.data()),
          c);
    return unflatten(z, counts, k, d);
}

namespace {
struct CbBox {
    const IterationCallback* cb;
    std::size_t h, w;
};
void round_trampoline(void* user, std::size_t round, const std::uint32_t* labels) {
    auto* b = static_cast<CbBox*>(user);
    SegmentationMask m{b->h, b->w, std::vector<std::uint32_t>(labels, labels + b->h * b->w)};
    (*b->cb)(round, m);
}
}  // namespace

ClusterResultWithCentroids cluster_with_centroids(const PixelHvGrid& grid, const ImageBuffer& img,
                                                  const ClusterConfig& config, const IterationCallback& on_iteration) {
    config.validate(img.pixel_count());  // clusterer.cpp:192-196
    if (grid.height() != img.height || grid.width() != img.width) fail("cluster: grid shape does not match image");
    img.validate();
    const std::size_t n = img.pixel_count(), k = config.k, d = grid.dim();
    ClusterResultWithCentroids out;
    out.result.mask = {img.height, img.width, std::vector<std::uint32_t>(n)};
    std::vector<std::uint32_t> z(k * d);
    std::vector<std::uint64_t> counts(k);
    std::size_t rounds = 0;
    CbBox box{&on_iteration, img.height, img.width};
    seghdc_ctx* c = ctx();
    check(seghdc_cluster(c, grid.hv_words(0, 0).data(), img.pixels.data(), img.height, img.width, img.channels, d, k,
                         config.iterations, config.early_stop, on_iteration ? round_trampoline : nullptr, &box,
                         out.result.mask.labels.data(), z.data(), counts.data(), &rounds),
          c);
    out.result.iterations_run = rounds;
    out.centroids = unflatten(z, counts, k, d);
    return out;
}

ClusterResult cluster(const PixelHvGrid& grid, const ImageBuffer& img, const ClusterConfig& config,
                      const IterationCallback& on_iteration) {
    return cluster_with_centroids(grid, img, config, on_iteration).result;
}

// ---- run_pipeline (reference pipeline.cpp) ----------------------------------------------------
PositionConfig RunConfig::position_config(const ImageBuffer& img) const {
    return PositionConfig{dim, img.height, img.width, alpha, beta};
}
ColorConfig RunConfig::color_config(const ImageBuffer& img) const { return ColorConfig{dim, img.channels, gamma}; }

void RunConfig::validate(const ImageBuffer& img) const {  // pipeline.cpp:25-30
    img.validate();
    position_config(img).validate();
    color_config(img).validate();
    ClusterConfig{clusters, iterations, early_stop}.validate(img.pixel_count());
}

std::map<std::string, double> StageTimings::as_map() const {
    return {{"encode_position", encode_position_ms}, {"encode_color", encode_color_ms},
            {"produce_pixels", produce_pixels_ms}, {"cluster", cluster_ms}, {"total", total_ms}};
}

PipelineResult run_pipeline(const ImageBuffer& img, const RunConfig& config, const IterationCallback& on_iteration) {
    config.validate(img);
    PipelineResult r;
    r.mask = {img.height, img.width, std::vector<std::uint32_t>(img.pixel_count())};
    double t[5] = {0, 0, 0, 0, 0};
    CbBox box{&on_iteration, img.height, img.width};
    seghdc_ctx* c = ctx();
    check(seghdc_run_pipeline(c, img.pixels.data(), img.height, img.width, img.channels, config.dim, config.alpha,
                              config.beta, config.gamma, config.clusters, config.iterations, config.seed,
                              int(config.encoder), config.early_stop, on_iteration ? round_trampoline : nullptr, &box,
                              r.mask.labels.data(), &r.iterations_run, t),
          c);
    r.timings = {t[0], t[1], t[2], t[3], t[4]};
    return r;
}

NcclUniqueId nccl_unique_id() {
    NcclUniqueId id{};
    check(seghdc_nccl_get_unique_id(id.data()), nullptr);
    return id;
}

void init_sharding(const NcclUniqueId& id, int rank, int nranks) {
    seghdc_ctx* c = ctx();
    check(seghdc_nccl_init(c, id.data(), rank, nranks), c);
}

ShardedPipelineResult run_pipeline_sharded(const ImageBuffer& img, const RunConfig& config) {
    config.validate(img);
    seghdc_ctx* c = ctx();
    ShardedPipelineResult r;
    const std::size_t k = config.clusters, d = config.dim;
    std::vector<std::uint32_t> labels(img.pixel_count()), z(k * d);
    std::vector<std::uint64_t> counts(k);
    double t[5] = {0, 0, 0, 0, 0};
    check(seghdc_run_pipeline_sharded(c, img.pixels.data(), img.height, img.width, img.channels, d, config.alpha,
                                      config.beta, config.gamma, k, config.iterations, config.seed, int(config.encoder),
                                      config.early_stop, labels.data(), z.data(), counts.data(), &r.iterations_run, t),
          c);
    check(seghdc_shard_row_range(c, img.height, &r.row_begin, &r.row_end), c);
    labels.resize((r.row_end - r.row_begin) * img.width);
    r.rows = {r.row_end - r.row_begin, img.width, std::move(labels)};
    r.centroids = unflatten(z, counts, k, d);
    r.timings = {t[0], t[1], t[2], t[3], t[4]};
    return r;
}

}  // namespace seghdc

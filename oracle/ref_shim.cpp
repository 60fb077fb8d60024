// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" adaptor over the UNMODIFIED reference hot path compiled from
// /root/reference/proj/src (see oracle/Makefile). Only tests/, bench.py's reference /
// cpu_baseline legs and __graft_entry__.smoke() may load the resulting
// oracle/_ref/libseghdc_ref.so, and only as the checker or the timed CPU baseline.
//
// Every function forwards to the reference's public API; the only restated logic is
//  * run_pipeline's codebook RNG order (reference src/pipeline.cpp:43-59), because
//    pipeline.cpp needs nlohmann/json and is therefore not compiled here;
//  * the replay of cluster()'s loop (reference src/clusterer.cpp:190-218) through the
//    public select_initial_centroids/assign_labels/update_centroids, because cluster()
//    does not return its centroids (clusterer.hpp:68-71);
//  * widening of colour table entries to full D (mirrors the file-static
//    widen_color_tables, reference src/pixel_pipeline.cpp:70-88) for table export.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "seghdc/clusterer.hpp"
#include "seghdc/color_encoder.hpp"
#include "seghdc/errors.hpp"
#include "seghdc/hypervector.hpp"
#include "seghdc/pixel_pipeline.hpp"
#include "seghdc/position_encoder.hpp"

using namespace seghdc;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

ImageBuffer make_image(const std::uint8_t* px, std::size_t h, std::size_t w, std::size_t c) {
    ImageBuffer img;
    img.height = h;
    img.width = w;
    img.channels = c;
    img.pixels.assign(px, px + h * w * c);
    return img;
}

PixelHvGrid make_grid(const std::uint64_t* words, std::size_t h, std::size_t w, std::size_t dim) {
    PixelHvGrid g(h, w, dim);
    std::memcpy(g.hv_words(0, 0).data(), words, h * w * g.words_per_hv() * sizeof(std::uint64_t));
    return g;
}

CentroidSet make_centroids(const std::uint32_t* z, const std::uint64_t* counts, std::size_t k,
                           std::size_t dim) {
    CentroidSet cs;
    for (std::size_t c = 0; c < k; ++c) {
        IntVector v(dim);
        for (std::size_t i = 0; i < dim; ++i) v[i] = z[c * dim + i];
        cs.centroids.push_back(std::move(v));
        cs.member_counts.push_back(counts ? counts[c] : 1);
    }
    return cs;
}

void export_centroids(const CentroidSet& cs, std::uint32_t* z, std::uint64_t* counts) {
    const std::size_t k = cs.k();
    for (std::size_t c = 0; c < k; ++c) {
        const auto vals = cs.centroids[c].values();
        if (z) std::memcpy(z + c * vals.size(), vals.data(), vals.size() * sizeof(std::uint32_t));
        if (counts) counts[c] = cs.member_counts[c];
    }
}

struct Codebooks {
    PositionCodebook pos;
    ColorCodebook color;
};

// reference src/pipeline.cpp:43-59: one Rng(seed), position codebook first, then colour.
Codebooks build_codebooks(std::size_t dim, std::size_t h, std::size_t w, std::size_t c,
                          double alpha, std::size_t beta, std::size_t gamma, std::uint64_t seed,
                          int encoder) {
    Rng rng(seed);
    const PositionConfig pc{dim, h, w, alpha, beta};
    const ColorConfig cc{dim, c, gamma};
    Codebooks cb;
    cb.pos = encoder == 1 ? build_random_position_codebook(pc, rng) : build_position_codebook(pc, rng);
    cb.color = encoder == 2 ? build_random_color_codebook(cc, rng) : build_color_codebook(cc, rng);
    return cb;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::size_t ref_words_for(std::size_t dim) { return Hypervector::words_for(dim); }

int ref_build_codebooks(std::size_t dim, std::size_t h, std::size_t w, std::size_t c, double alpha,
                        std::size_t beta, std::size_t gamma, std::uint64_t seed, int encoder,
                        std::uint64_t* row_out, std::uint64_t* col_out,
                        std::uint64_t* widened_out) {
    return guard([&] {
        const Codebooks cb = build_codebooks(dim, h, w, c, alpha, beta, gamma, seed, encoder);
        const std::size_t wph = Hypervector::words_for(dim);
        for (std::size_t i = 0; i < h; ++i)
            std::memcpy(row_out + i * wph, cb.pos.row_hvs[i].words().data(), wph * 8);
        for (std::size_t j = 0; j < w; ++j)
            std::memcpy(col_out + j * wph, cb.pos.col_hvs[j].words().data(), wph * 8);
        std::memset(widened_out, 0, c * 256 * wph * 8);
        std::size_t offset = 0;
        for (std::size_t ch = 0; ch < c; ++ch) {
            for (int v = 0; v < 256; ++v) {
                const Hypervector& e = cb.color.tables[ch][v];
                std::uint64_t* dst = widened_out + (ch * 256 + v) * wph;
                for (std::size_t b = 0; b < e.dim(); ++b)
                    if (e.bit(b)) dst[(offset + b) >> 6] |= 1ULL << ((offset + b) & 63);
            }
            offset += cb.color.tables[ch][0].dim();
        }
    });
}

int ref_encode(const std::uint8_t* px, std::size_t h, std::size_t w, std::size_t c,
               std::size_t dim, double alpha, std::size_t beta, std::size_t gamma,
               std::uint64_t seed, int encoder, std::uint64_t* grid_out) {
    return guard([&] {
        const ImageBuffer img = make_image(px, h, w, c);
        const Codebooks cb = build_codebooks(dim, h, w, c, alpha, beta, gamma, seed, encoder);
        const PixelHvGrid grid = encode_image(img, cb.pos, cb.color);
        std::memcpy(grid_out, grid.hv_words(0, 0).data(), grid.payload_bytes());
    });
}

int ref_select_seeds(const std::uint8_t* px, std::size_t h, std::size_t w, std::size_t c,
                     std::size_t k, std::uint64_t* seeds_out) {
    return guard([&] {
        const ImageBuffer img = make_image(px, h, w, c);
        const PixelHvGrid shape_only(h, w, 1);  // select_initial_centroids only checks the shape
        const auto seeds = select_initial_centroids(img, shape_only, k);
        for (std::size_t s = 0; s < seeds.size(); ++s) seeds_out[s] = seeds[s].row * w + seeds[s].col;
    });
}

// The reference's own cluster(), per-round labels collected through its callback.
int ref_cluster(const std::uint64_t* grid_words, const std::uint8_t* px, std::size_t h,
                std::size_t w, std::size_t c, std::size_t dim, std::size_t k,
                std::size_t iterations, int early_stop, std::uint32_t* labels_rounds,
                std::uint32_t* labels_final, std::size_t* rounds_out) {
    return guard([&] {
        const ImageBuffer img = make_image(px, h, w, c);
        const PixelHvGrid grid = make_grid(grid_words, h, w, dim);
        const std::size_t n = h * w;
        const auto res = cluster(grid, img, ClusterConfig{k, iterations, early_stop != 0},
                                 [&](std::size_t r, const SegmentationMask& m) {
                                     if (labels_rounds)
                                         std::memcpy(labels_rounds + (r - 1) * n, m.labels.data(), n * 4);
                                 });
        std::memcpy(labels_final, res.mask.labels.data(), n * 4);
        *rounds_out = res.iterations_run;
    });
}

// Replay of cluster()'s loop (reference src/clusterer.cpp:190-218) through the public
// API so the centroid set used by the final assignment can be exported.
int ref_cluster_replay(const std::uint64_t* grid_words, const std::uint8_t* px, std::size_t h,
                       std::size_t w, std::size_t c, std::size_t dim, std::size_t k,
                       std::size_t iterations, int early_stop, std::uint32_t* labels_rounds,
                       std::uint32_t* labels_final, std::uint32_t* centroids_out,
                       std::uint64_t* counts_out, std::size_t* rounds_out) {
    return guard([&] {
        const ImageBuffer img = make_image(px, h, w, c);
        const PixelHvGrid grid = make_grid(grid_words, h, w, dim);
        ClusterConfig{k, iterations, early_stop != 0}.validate(img.pixel_count());
        const std::size_t n = h * w;
        const auto seeds = select_initial_centroids(img, grid, k);
        CentroidSet cs;
        for (const auto& s : seeds) {
            IntVector v(dim);
            v.add_words(grid.hv_words(s.row, s.col));
            cs.centroids.push_back(std::move(v));
            cs.member_counts.push_back(1);
        }
        SegmentationMask mask, prev;
        std::size_t rounds = 0;
        for (std::size_t r = 1; r <= iterations; ++r) {
            mask = assign_labels(grid, cs);
            rounds = r;
            if (labels_rounds) std::memcpy(labels_rounds + (r - 1) * n, mask.labels.data(), n * 4);
            if (early_stop && r > 1 && mask == prev) break;
            if (r < iterations) cs = update_centroids(grid, mask, cs);
            prev = mask;
        }
        std::memcpy(labels_final, mask.labels.data(), n * 4);
        export_centroids(cs, centroids_out, counts_out);
        *rounds_out = rounds;
    });
}

int ref_assign(const std::uint64_t* grid_words, std::size_t h, std::size_t w, std::size_t dim,
               const std::uint32_t* centroids, std::size_t k, std::uint32_t* labels_out) {
    return guard([&] {
        const PixelHvGrid grid = make_grid(grid_words, h, w, dim);
        const auto mask = assign_labels(grid, make_centroids(centroids, nullptr, k, dim));
        std::memcpy(labels_out, mask.labels.data(), h * w * 4);
    });
}

int ref_update(const std::uint64_t* grid_words, std::size_t h, std::size_t w, std::size_t dim,
               const std::uint32_t* labels, const std::uint32_t* prev,
               const std::uint64_t* prev_counts, std::size_t k, std::uint32_t* out,
               std::uint64_t* counts_out) {
    return guard([&] {
        const PixelHvGrid grid = make_grid(grid_words, h, w, dim);
        SegmentationMask mask{h, w, std::vector<std::uint32_t>(labels, labels + h * w)};
        const auto next = update_centroids(grid, mask, make_centroids(prev, prev_counts, k, dim));
        export_centroids(next, out, counts_out);
    });
}

// ---- parallel execution of the reference's own assign/update for the CPU baseline ----
// Rows [row_begin,row_end) are split into contiguous shards, one std::thread each; every
// shard runs the unmodified assign_labels + update_centroids. Integer sums are
// order-independent, so combining shard sums is exact; a cluster that is empty in a
// shard contributes nothing, and one empty everywhere keeps its previous centroid
// (reference src/clusterer.cpp:184-186).
struct RefPar {
    std::vector<PixelHvGrid> shards;
    std::size_t dim = 0;
};

void* ref_par_create(const std::uint64_t* grid_words, std::size_t h, std::size_t w,
                     std::size_t dim, std::size_t row_begin, std::size_t row_end, int nthreads) {
    (void)h;
    auto* p = new RefPar;
    p->dim = dim;
    const std::size_t wph = Hypervector::words_for(dim);
    const std::size_t rows = row_end - row_begin;
    const std::size_t t = std::max<std::size_t>(1, std::min<std::size_t>(nthreads, rows));
    for (std::size_t s = 0; s < t; ++s) {
        const std::size_t r0 = row_begin + rows * s / t, r1 = row_begin + rows * (s + 1) / t;
        if (r1 == r0) continue;
        p->shards.push_back(make_grid(grid_words + r0 * w * wph, r1 - r0, w, dim));
    }
    return p;
}

int ref_par_round(void* handle, const std::uint32_t* centroids, const std::uint64_t* counts,
                  std::size_t k, std::uint32_t* next_out, std::uint64_t* next_counts) {
    auto* p = static_cast<RefPar*>(handle);
    return guard([&] {
        const CentroidSet cs = make_centroids(centroids, counts, k, p->dim);
        std::vector<CentroidSet> parts(p->shards.size());
        std::vector<std::thread> threads;
        for (std::size_t s = 0; s < p->shards.size(); ++s) {
            threads.emplace_back([&, s] {
                const auto mask = assign_labels(p->shards[s], cs);
                parts[s] = update_centroids(p->shards[s], mask, cs);
            });
        }
        for (auto& th : threads) th.join();
        for (std::size_t c = 0; c < k; ++c) {
            std::uint64_t total = 0;
            std::vector<std::uint32_t> sum(p->dim, 0);
            for (const auto& part : parts) {
                if (part.member_counts[c] == 0) continue;
                total += part.member_counts[c];
                const auto vals = part.centroids[c].values();
                for (std::size_t i = 0; i < p->dim; ++i) sum[i] += vals[i];
            }
            if (total == 0)
                std::memcpy(next_out + c * p->dim, centroids + c * p->dim, p->dim * 4);
            else
                std::memcpy(next_out + c * p->dim, sum.data(), p->dim * 4);
            next_counts[c] = total;
        }
    });
}

void ref_par_destroy(void* handle) { delete static_cast<RefPar*>(handle); }

// ---- reference-pure full-length loop for images whose grid is too large to copy ---------
// Same row-block shards as RefPar, but every shard grid is produced by the reference's OWN
// encode_image (src/pixel_pipeline.cpp:92-126) on the shard's rows, with the position
// codebook's row table sliced to those rows (the codebook is built once for the full image
// in run_pipeline's RNG order, pipeline.cpp:43-59). Peak host memory is one grid (C4:
// 34.4 GB) instead of two. The loop is cluster()'s (src/clusterer.cpp:190-218): seed
// centroids from the seed pixels' HVs (:197-205), assign_labels every round, update_centroids
// between rounds; assign/update run per shard in parallel and the integer sums are combined
// exactly (empty everywhere -> previous centroid, :184-186).
struct RefParEnc {
    std::vector<PixelHvGrid> shards;
    std::vector<std::size_t> row0;
    std::size_t h = 0, w = 0, dim = 0;
};

void* ref_pare_create(const std::uint8_t* px, std::size_t h, std::size_t w, std::size_t c,
                      std::size_t dim, double alpha, std::size_t beta, std::size_t gamma,
                      std::uint64_t seed, int encoder, int nthreads) {
    auto* p = new RefParEnc;
    const int rc = guard([&] {
        p->h = h;
        p->w = w;
        p->dim = dim;
        const Codebooks cb = build_codebooks(dim, h, w, c, alpha, beta, gamma, seed, encoder);
        const std::size_t t = std::max<std::size_t>(1, std::min<std::size_t>(nthreads, h));
        p->shards.resize(t);
        std::vector<std::thread> threads;
        for (std::size_t s = 0; s < t; ++s) {
            const std::size_t r0 = h * s / t, r1 = h * (s + 1) / t;
            p->row0.push_back(r0);
            threads.emplace_back([&, s, r0, r1] {
                const ImageBuffer sub = make_image(px + r0 * w * c, r1 - r0, w, c);
                PositionCodebook pos = cb.pos;  // row table sliced to this shard's rows
                pos.config.n_rows = r1 - r0;
                pos.row_hvs.assign(cb.pos.row_hvs.begin() + r0, cb.pos.row_hvs.begin() + r1);
                p->shards[s] = encode_image(sub, pos, cb.color);
            });
        }
        for (auto& th : threads) th.join();
        p->row0.push_back(h);
    });
    if (rc) {
        delete p;
        return nullptr;
    }
    return p;
}

// seed centroids (clusterer.cpp:197-205) for row-major seed indices
int ref_pare_seed(void* handle, const std::uint64_t* seeds, std::size_t k, std::uint32_t* z_out) {
    auto* p = static_cast<RefParEnc*>(handle);
    return guard([&] {
        for (std::size_t s = 0; s < k; ++s) {
            const std::size_t row = seeds[s] / p->w, col = seeds[s] % p->w;
            std::size_t sh = 0;
            while (p->row0[sh + 1] <= row) ++sh;
            IntVector v(p->dim);
            v.add_words(p->shards[sh].hv_words(row - p->row0[sh], col));
            const auto vals = v.values();
            std::memcpy(z_out + s * p->dim, vals.data(), p->dim * 4);
        }
    });
}

// one round: assign_labels on every shard (labels_out[h*w], nullable); if do_update, the
// combined update_centroids into next_out / next_counts.
int ref_pare_round(void* handle, const std::uint32_t* centroids, const std::uint64_t* counts,
                   std::size_t k, int do_update, std::uint32_t* labels_out, std::uint32_t* next_out,
                   std::uint64_t* next_counts) {
    auto* p = static_cast<RefParEnc*>(handle);
    return guard([&] {
        const CentroidSet cs = make_centroids(centroids, counts, k, p->dim);
        std::vector<CentroidSet> parts(p->shards.size());
        std::vector<std::thread> threads;
        for (std::size_t s = 0; s < p->shards.size(); ++s) {
            threads.emplace_back([&, s] {
                const auto mask = assign_labels(p->shards[s], cs);
                if (labels_out)
                    std::memcpy(labels_out + p->row0[s] * p->w, mask.labels.data(), mask.labels.size() * 4);
                if (do_update) parts[s] = update_centroids(p->shards[s], mask, cs);
            });
        }
        for (auto& th : threads) th.join();
        if (!do_update) return;
        for (std::size_t c = 0; c < k; ++c) {
            std::uint64_t total = 0;
            std::vector<std::uint32_t> sum(p->dim, 0);
            for (const auto& part : parts) {
                if (part.member_counts[c] == 0) continue;
                total += part.member_counts[c];
                const auto vals = part.centroids[c].values();
                for (std::size_t i = 0; i < p->dim; ++i) sum[i] += vals[i];
            }
            std::memcpy(next_out + c * p->dim, total ? sum.data() : centroids + c * p->dim, p->dim * 4);
            next_counts[c] = total;
        }
    });
}

void ref_pare_destroy(void* handle) { delete static_cast<RefParEnc*>(handle); }

}  // extern "C"

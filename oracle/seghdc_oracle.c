/* TEST INFRASTRUCTURE ONLY — see seghdc_oracle.h. Plain-C restatement of the reference
 * SegHDC hot path; every function cites the reference file:line (relative to
 * /root/reference/proj) it restates. OpenMP parallelises over pixels only; all arithmetic
 * is integer, so results are independent of the thread count. */
#include "seghdc_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];
static int g_threads = 0;

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* so_last_error(void) { return g_err; }
void so_set_threads(int n) { g_threads = n; }
int so_get_threads(void) { return g_threads > 0 ? g_threads : omp_get_max_threads(); }
static int nthreads(void) { return so_get_threads(); }

/* hypervector.hpp:37 */
size_t so_words_for(size_t dim) { return (dim + 63) / 64; }

/* ---- std::mt19937_64 (hypervector.hpp:13; parameters fixed by [rand.predef]) ---- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; i++)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; i++) {
            const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

void so_mt64_stream(uint64_t seed, size_t n, uint64_t* out) {
    mt64 s;
    mt64_seed(&s, seed);
    for (size_t i = 0; i < n; i++) out[i] = mt64_next(&s);
}

/* ---- hypervector primitives ---- */
/* Hypervector::random, hypervector.cpp:33-39: one draw per word, tail masked. */
static void hv_random(uint64_t* w, size_t dim, mt64* rng) {
    const size_t nw = so_words_for(dim);
    for (size_t i = 0; i < nw; i++) w[i] = mt64_next(rng);
    if (dim % 64) w[nw - 1] &= ~0ULL >> (64 - dim % 64);
}

/* flip_range, hypervector.cpp:67-84 (in place; caller copies). */
static int hv_flip(uint64_t* w, size_t dim, size_t start, size_t len) {
    if (start + len > dim || start + len < start)
        return fail(1, "flip_range out of bounds: [%zu, %zu) exceeds dim %zu", start, start + len, dim);
    for (size_t i = start; i < start + len;) {
        const size_t off = i & 63, take = (64 - off < start + len - i) ? 64 - off : start + len - i;
        w[i >> 6] ^= (take == 64 ? ~0ULL : ((1ULL << take) - 1)) << off;
        i += take;
    }
    return 0;
}

/* ---- position encoder ---- */
/* PositionConfig::x_row / x_col, position_encoder.cpp:10-18 (double floor). */
static size_t flip_unit(double alpha, size_t dim, size_t n) {
    return (size_t)floor(alpha * (double)dim / (2.0 * (double)n));
}

/* PositionConfig::validate, position_encoder.cpp:20-39. */
static int validate_position(size_t dim, size_t h, size_t w, double alpha, size_t beta) {
    if (dim == 0 || h == 0 || w == 0) return fail(1, "position config: dim, n_rows and n_cols must be >= 1");
    if (!(alpha > 0.0 && alpha <= 1.0)) return fail(1, "position config: alpha must be in (0, 1], got %f", alpha);
    if (beta == 0) return fail(1, "position config: beta must be >= 1");
    if (flip_unit(alpha, dim, h) == 0) return fail(1, "dimension too small for image size: x_row = 0");
    if (flip_unit(alpha, dim, w) == 0) return fail(1, "dimension too small for image size: x_col = 0");
    return 0;
}

/* build_axis, position_encoder.cpp:50-64: random base, then the next x bits flipped at
 * every block boundary, cursor from the half start. */
static int build_axis(uint64_t* out, size_t n, size_t beta, size_t x, size_t dim, size_t half_start, mt64* rng) {
    const size_t nw = so_words_for(dim);
    hv_random(out, dim, rng);
    size_t cursor = half_start;
    for (size_t i = 1; i < n; i++) {
        memcpy(out + i * nw, out + (i - 1) * nw, nw * 8);
        if (i / beta != (i - 1) / beta) {
            int rc = hv_flip(out + i * nw, dim, cursor, x);
            if (rc) return rc;
            cursor += x;
        }
    }
    return 0;
}

/* ---- colour encoder ---- */
/* ColorConfig::channel_dims / unit_flip, color_encoder.cpp:9-18. */
static size_t channel_dim(size_t dim, size_t c, size_t ch) { return dim / c + (ch < dim % c ? 1 : 0); }
static size_t unit_flip(size_t dim, size_t c, size_t gamma, size_t ch) {
    return gamma * (channel_dim(dim, c, ch) / (256 * gamma));
}

/* ColorConfig::validate, color_encoder.cpp:20-35. */
static int validate_color(size_t dim, size_t c, size_t gamma) {
    if (dim == 0) return fail(1, "color config: dim must be >= 1");
    if (c != 1 && c != 3) return fail(1, "color config: channels must be 1 or 3, got %zu", c);
    if (gamma == 0) return fail(1, "color config: gamma must be >= 1");
    for (size_t ch = 0; ch < c; ch++)
        if (unit_flip(dim, c, gamma, ch) < gamma) return fail(1, "dimension too small for color resolution");
    return 0;
}

/* widen one channel-local HV (d_ch bits) into a full-dim HV at `offset`
 * (widen_color_tables, pixel_pipeline.cpp:70-88). */
static void widen(uint64_t* full, const uint64_t* part, size_t d_ch, size_t offset) {
    for (size_t b = 0; b < d_ch; b++)
        if ((part[b >> 6] >> (b & 63)) & 1) full[(offset + b) >> 6] |= 1ULL << ((offset + b) & 63);
}

int so_build_codebooks(size_t dim, size_t h, size_t w, size_t c, double alpha, size_t beta,
                       size_t gamma, uint64_t seed, int encoder, uint64_t* row_out,
                       uint64_t* col_out, uint64_t* widened_out) {
    int rc = validate_position(dim, h, w, alpha, beta);
    if (rc) return rc;
    rc = validate_color(dim, c, gamma);
    if (rc) return rc;
    const size_t nw = so_words_for(dim);
    mt64 rng;
    mt64_seed(&rng, seed); /* pipeline.cpp:43 */
    if (encoder == 1) {    /* build_random_position_codebook, pixel_pipeline.cpp:128-141 */
        for (size_t i = 0; i < h; i++) hv_random(row_out + i * nw, dim, &rng);
        for (size_t j = 0; j < w; j++) hv_random(col_out + j * nw, dim, &rng);
    } else { /* build_position_codebook, position_encoder.cpp:68-76 */
        rc = build_axis(row_out, h, beta, flip_unit(alpha, dim, h), dim, 0, &rng);
        if (rc) return rc;
        rc = build_axis(col_out, w, beta, flip_unit(alpha, dim, w), dim, dim / 2, &rng);
        if (rc) return rc;
    }
    /* build_color_codebook (color_encoder.cpp:37-55) / build_random_color_codebook
     * (pixel_pipeline.cpp:143-156), widened per channel. */
    memset(widened_out, 0, c * 256 * nw * 8);
    size_t offset = 0;
    for (size_t ch = 0; ch < c; ch++) {
        const size_t d_ch = channel_dim(dim, c, ch), u = unit_flip(dim, c, gamma, ch);
        const size_t cw = so_words_for(d_ch);
        uint64_t* entry = calloc(cw, 8);
        hv_random(entry, d_ch, &rng);
        size_t cursor = 0;
        for (int v = 0; v < 256; v++) {
            if (v > 0) {
                if (encoder == 2) {
                    hv_random(entry, d_ch, &rng);
                } else {
                    rc = hv_flip(entry, d_ch, cursor, u);
                    if (rc) {
                        free(entry);
                        return rc;
                    }
                    cursor += u;
                }
            }
            widen(widened_out + (ch * 256 + (size_t)v) * nw, entry, d_ch, offset);
        }
        free(entry);
        offset += d_ch;
    }
    return 0;
}

/* encode_image, pixel_pipeline.cpp:92-126: grid = row ^ col ^ widened[ch][v]. */
int so_encode(const uint8_t* px, size_t h, size_t w, size_t c, size_t dim, const uint64_t* row,
              const uint64_t* col, const uint64_t* widened, uint64_t* grid_out) {
    if (h == 0 || w == 0) return fail(1, "image dimensions must be positive");
    if (c != 1 && c != 3) return fail(1, "image channels must be 1 or 3, got %zu", c);
    const size_t nw = so_words_for(dim);
#pragma omp parallel for schedule(static) num_threads(nthreads())
    for (size_t p = 0; p < h * w; p++) {
        const uint64_t* r = row + (p / w) * nw;
        const uint64_t* cc = col + (p % w) * nw;
        uint64_t* out = grid_out + p * nw;
        for (size_t k = 0; k < nw; k++) out[k] = r[k] ^ cc[k];
        for (size_t ch = 0; ch < c; ch++) {
            const uint64_t* t = widened + (ch * 256 + px[p * c + ch]) * nw;
            for (size_t k = 0; k < nw; k++) out[k] ^= t[k];
        }
    }
    return 0;
}

/* select_initial_centroids, clusterer.cpp:54-130. */
int so_select_seeds(const uint8_t* px, size_t h, size_t w, size_t c, size_t k, uint64_t* seeds_out) {
    const size_t n = h * w;
    if (k == 0 || k > n) return fail(1, "select_initial_centroids: k = %zu out of range for %zu pixels", k, n);
    uint8_t* chosen = calloc(n, 1);
    size_t nchosen = 0;
#define TAKE(p) do { seeds_out[nchosen++] = (p); chosen[(p)] = 1; } while (0)
    size_t min_key = (size_t)-1, max_key = 0, min_px = 0, max_px = 0;
    for (size_t p = 0; p < n; p++) { /* :73-82, strict < / > keep the first occurrence */
        size_t key = 0;
        for (size_t ch = 0; ch < c; ch++) key += px[p * c + ch];
        if (key < min_key) { min_key = key; min_px = p; }
        if (key > max_key) { max_key = key; max_px = p; }
    }
    if (min_key == max_key) { /* :83-96 uniform image: corners, then row-major fill */
        const size_t corners[4] = {0, w - 1, (h - 1) * w, (h - 1) * w + w - 1};
        for (int i = 0; i < 4 && nchosen < k; i++)
            if (!chosen[corners[i]]) TAKE(corners[i]);
        for (size_t p = 0; p < n && nchosen < k; p++)
            if (!chosen[p]) TAKE(p);
        free(chosen);
        return 0;
    }
    TAKE(min_px);
    if (k >= 2) TAKE(max_px);
    if (k > 2) { /* :101-128 greedy farthest colour */
        size_t* min_dist = malloc(n * sizeof(size_t));
        for (size_t p = 0; p < n; p++) min_dist[p] = (size_t)-1;
        for (size_t s = 0; s < nchosen; s++) {
            const size_t q = seeds_out[s];
            for (size_t p = 0; p < n; p++) {
                size_t d = 0;
                for (size_t ch = 0; ch < c; ch++) d += (size_t)abs((int)px[p * c + ch] - (int)px[q * c + ch]);
                if (d < min_dist[p]) min_dist[p] = d;
            }
        }
        while (nchosen < k) {
            int found = 0;
            size_t best = 0, best_p = 0;
            for (size_t p = 0; p < n; p++) {
                if (chosen[p]) continue;
                if (!found || min_dist[p] > best) { found = 1; best = min_dist[p]; best_p = p; }
            }
            TAKE(best_p);
            for (size_t p = 0; p < n; p++) {
                size_t d = 0;
                for (size_t ch = 0; ch < c; ch++) d += (size_t)abs((int)px[p * c + ch] - (int)px[best_p * c + ch]);
                if (d < min_dist[p]) min_dist[p] = d;
            }
        }
        free(min_dist);
    }
#undef TAKE
    free(chosen);
    return 0;
}

/* dot_words, hypervector.cpp:138-151: sum of z over the set bits of y. */
static uint64_t dot_words(const uint64_t* y, size_t nw, const uint32_t* z) {
    uint64_t s = 0;
    for (size_t wi = 0; wi < nw; wi++) {
        uint64_t x = y[wi];
        const uint32_t* zb = z + (wi << 6);
        while (x) {
            s += zb[__builtin_ctzll(x)];
            x &= x - 1;
        }
    }
    return s;
}

/* strictly_closer, clusterer.cpp:41-50 — exact 128-bit cross multiplication (wraps
 * modulo 2^128 exactly as the reference's unsigned __int128 does). */
static int strictly_closer(uint64_t dc, uint64_t n2c, uint64_t db, uint64_t n2b) {
    if (n2c == 0) return 0;
    if (n2b == 0) return dc > 0;
    const unsigned __int128 lhs = (unsigned __int128)dc * dc * n2b;
    const unsigned __int128 rhs = (unsigned __int128)db * db * n2c;
    return lhs > rhs;
}

/* Diagnostic (not in the reference): does d*d*n2 exceed 2^128, i.e. did the reference's
 * unsigned __int128 product in strictly_closer wrap? A comparison "wraps" when either side
 * does (both norms non-zero, so both products are evaluated). Counted per round by
 * so_assign / so_cluster / so_cluster_stream and read back with so_last_wraps. */
static int prod_wraps(uint64_t d, uint64_t n2) {
    const unsigned __int128 sq = (unsigned __int128)d * d;
    const unsigned __int128 lo = (unsigned __int128)(uint64_t)sq * n2;
    const unsigned __int128 hi = (unsigned __int128)(uint64_t)(sq >> 64) * n2 + (lo >> 64);
    return (hi >> 64) != 0;
}
static int compare_wraps(uint64_t dc, uint64_t n2c, uint64_t db, uint64_t n2b) {
    if (n2c == 0 || n2b == 0) return 0;
    return prod_wraps(dc, n2b) | prod_wraps(db, n2c);
}
#define SO_MAX_WRAP_ROUNDS 4096
static uint64_t g_wraps[SO_MAX_WRAP_ROUNDS];
static size_t g_wrap_rounds;
size_t so_last_wraps(uint64_t* out, size_t cap) {
    for (size_t r = 0; r < g_wrap_rounds && r < cap; r++) out[r] = g_wraps[r];
    return g_wrap_rounds;
}
static void record_wraps(size_t round, uint64_t wraps) { /* round is 1-based */
    if (round == 1) g_wrap_rounds = 0;
    if (round <= SO_MAX_WRAP_ROUNDS) g_wraps[round - 1] = wraps;
    g_wrap_rounds = round;
}

/* assign_labels, clusterer.cpp:132-162. */
int so_assign(const uint64_t* grid, size_t n, size_t dim, const uint32_t* z, size_t k, uint32_t* labels_out) {
    if (k == 0) return fail(1, "assign_labels: empty centroid set");
    const size_t nw = so_words_for(dim);
    uint64_t* norm2 = calloc(k, 8);
    for (size_t c = 0; c < k; c++) /* IntVector::norm_squared, hypervector.cpp:123-127 */
        for (size_t i = 0; i < dim; i++) norm2[c] += (uint64_t)z[c * dim + i] * z[c * dim + i];
    /* dot_words indexes z[(wi<<6)+b] for set bits only; tail bits are zero so b < dim. */
    uint64_t wraps = 0;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads()) reduction(+ : wraps)
    for (size_t p = 0; p < n; p++) {
        const uint64_t* y = grid + p * nw;
        uint32_t best = 0;
        uint64_t best_dot = dot_words(y, nw, z);
        for (size_t c = 1; c < k; c++) {
            const uint64_t d = dot_words(y, nw, z + c * dim);
            wraps += (uint64_t)compare_wraps(d, norm2[c], best_dot, norm2[best]);
            if (strictly_closer(d, norm2[c], best_dot, norm2[best])) {
                best = (uint32_t)c;
                best_dot = d;
            }
        }
        labels_out[p] = best;
    }
    free(norm2);
    record_wraps(1, wraps);
    return 0;
}

/* update_centroids, clusterer.cpp:164-188: per-label IntVector::add_words
 * (hypervector.cpp:112-121); empty clusters keep the previous centroid. */
int so_update(const uint64_t* grid, size_t n, size_t dim, const uint32_t* labels,
              const uint32_t* prev_z, size_t k, uint32_t* z_out, uint64_t* counts_out) {
    for (size_t p = 0; p < n; p++)
        if (labels[p] >= k) return fail(1, "update_centroids: label %u out of range for k = %zu", labels[p], k);
    const size_t nw = so_words_for(dim);
    const int T = nthreads();
    uint32_t* part = calloc((size_t)T * k * dim, 4);
    uint64_t* cnt = calloc((size_t)T * k, 8);
#pragma omp parallel num_threads(T)
    {
        const int t = omp_get_thread_num();
        uint32_t* acc = part + (size_t)t * k * dim;
        uint64_t* ct = cnt + (size_t)t * k;
#pragma omp for schedule(static)
        for (size_t p = 0; p < n; p++) {
            const uint32_t c = labels[p];
            uint32_t* zc = acc + (size_t)c * dim;
            const uint64_t* y = grid + p * nw;
            for (size_t wi = 0; wi < nw; wi++) {
                uint64_t x = y[wi];
                while (x) {
                    zc[(wi << 6) + (size_t)__builtin_ctzll(x)]++;
                    x &= x - 1;
                }
            }
            ct[c]++;
        }
    }
    for (size_t c = 0; c < k; c++) {
        uint64_t total = 0;
        for (int t = 0; t < T; t++) total += cnt[(size_t)t * k + c];
        counts_out[c] = total;
        for (size_t i = 0; i < dim; i++) {
            uint32_t s = 0;
            for (int t = 0; t < T; t++) s += part[((size_t)t * k + c) * dim + i];
            z_out[c * dim + i] = total ? s : prev_z[c * dim + i];
        }
    }
    free(part);
    free(cnt);
    return 0;
}

/* cluster, clusterer.cpp:190-218. */
int so_cluster(const uint64_t* grid, const uint8_t* px, size_t h, size_t w, size_t c,
               size_t dim, size_t k, size_t iterations, int early_stop, uint32_t* labels_rounds,
               uint32_t* labels_final, uint32_t* centroids_out, uint64_t* counts_out,
               size_t* rounds_out) {
    const size_t n = h * w, nw = so_words_for(dim);
    /* ClusterConfig::validate, clusterer.cpp:10-18 */
    if (k == 0) return fail(1, "cluster config: k must be >= 1");
    if (iterations == 0) return fail(1, "cluster config: iterations must be >= 1");
    if (k > n) return fail(1, "cluster config: k = %zu exceeds pixel count %zu", k, n);
    uint64_t* seeds = malloc(k * 8);
    int rc = so_select_seeds(px, h, w, c, k, seeds);
    if (rc) {
        free(seeds);
        return rc;
    }
    uint32_t* z = calloc(k * dim, 4);
    uint32_t* z_next = calloc(k * dim, 4);
    uint64_t* counts = malloc(k * 8);
    for (size_t s = 0; s < k; s++) { /* :197-205 seed centroid = the seed pixel's HV, count 1 */
        const uint64_t* y = grid + seeds[s] * nw;
        for (size_t i = 0; i < dim; i++) z[s * dim + i] = (uint32_t)((y[i >> 6] >> (i & 63)) & 1);
        counts[s] = 1;
    }
    uint32_t* prev = malloc(n * 4);
    uint64_t* wr_hist = calloc(SO_MAX_WRAP_ROUNDS, 8);
    size_t rounds = 0;
    for (size_t r = 1; r <= iterations; r++) { /* :209-216 */
        so_assign(grid, n, dim, z, k, labels_final);
        if (r <= SO_MAX_WRAP_ROUNDS) wr_hist[r - 1] = g_wraps[0];
        rounds = r;
        if (labels_rounds) memcpy(labels_rounds + (r - 1) * n, labels_final, n * 4);
        if (early_stop && r > 1 && memcmp(labels_final, prev, n * 4) == 0) break;
        if (r < iterations) {
            so_update(grid, n, dim, labels_final, z, k, z_next, counts);
            uint32_t* t = z;
            z = z_next;
            z_next = t;
        }
        memcpy(prev, labels_final, n * 4);
    }
    if (centroids_out) memcpy(centroids_out, z, k * dim * 4);
    if (counts_out) memcpy(counts_out, counts, k * 8);
    *rounds_out = rounds;
    for (size_t r = 1; r <= rounds && r <= SO_MAX_WRAP_ROUNDS; r++) record_wraps(r, wr_hist[r - 1]);
    free(wr_hist);
    free(prev);
    free(seeds);
    free(z);
    free(z_next);
    free(counts);
    return 0;
}

/* cluster (clusterer.cpp:190-218) without a stored grid: every pass re-encodes each pixel's HV
 * from the tables (pixel_pipeline.cpp:92-126) and fuses assign_labels with the accumulation of
 * the following update_centroids (both use the same round's labels). For configurations whose
 * grid does not fit host memory (C4: 34 GB). Centroids are kept interleaved (z[i * k + c]) so
 * the per-set-bit dot update is one k-wide vector add. Same results as so_cluster. */
int so_cluster_stream(const uint8_t* px, size_t h, size_t w, size_t c, size_t dim, const uint64_t* row,
                      const uint64_t* col, const uint64_t* widened, size_t k, size_t iterations, int early_stop,
                      uint32_t* labels_rounds, uint32_t* labels_final, uint32_t* centroids_out,
                      uint64_t* counts_out, size_t* rounds_out) {
    const size_t n = h * w, nw = so_words_for(dim);
    if (k == 0) return fail(1, "cluster config: k must be >= 1");
    if (iterations == 0) return fail(1, "cluster config: iterations must be >= 1");
    if (k > n) return fail(1, "cluster config: k = %zu exceeds pixel count %zu", k, n);
    if (k > 64) return fail(2, "so_cluster_stream: k <= 64 only");
    uint64_t* seeds = malloc(k * 8);
    int rc = so_select_seeds(px, h, w, c, k, seeds);
    if (rc) {
        free(seeds);
        return rc;
    }
    uint32_t* zt = calloc(dim * k, 4); /* interleaved centroid set of the current round */
    uint64_t* counts = malloc(k * 8);
    uint64_t* y = malloc(nw * 8);
    for (size_t s2 = 0; s2 < k; s2++) { /* :197-205 seed centroid = the seed pixel's HV */
        const size_t p = seeds[s2];
        for (size_t q = 0; q < nw; q++) {
            uint64_t v = row[(p / w) * nw + q] ^ col[(p % w) * nw + q];
            for (size_t ch = 0; ch < c; ch++) v ^= widened[(ch * 256 + px[p * c + ch]) * nw + q];
            y[q] = v;
        }
        for (size_t i = 0; i < dim; i++) zt[i * k + s2] = (uint32_t)((y[i >> 6] >> (i & 63)) & 1);
        counts[s2] = 1;
    }
    free(y);
    const int T = nthreads();
    uint32_t* part = malloc((size_t)T * k * dim * 4);
    uint64_t* cnt = malloc((size_t)T * k * 8);
    uint32_t* prev = malloc(n * 4);
    uint64_t* norm2 = malloc(k * 8);
    size_t rounds = 0;
    for (size_t r = 1; r <= iterations; r++) {
        const int do_update = r < iterations;
        for (size_t cc = 0; cc < k; cc++) { /* IntVector::norm_squared */
            norm2[cc] = 0;
            for (size_t i = 0; i < dim; i++) norm2[cc] += (uint64_t)zt[i * k + cc] * zt[i * k + cc];
        }
        memset(part, 0, (size_t)T * k * dim * 4);
        memset(cnt, 0, (size_t)T * k * 8);
        uint64_t wraps = 0;
#pragma omp parallel num_threads(T) reduction(+ : wraps)
        {
            const int t = omp_get_thread_num();
            uint32_t* acc = part + (size_t)t * k * dim;
            uint64_t* ct = cnt + (size_t)t * k;
            uint64_t* yy = malloc(nw * 8);
            uint64_t d[64];
#pragma omp for schedule(dynamic, 1024)
            for (size_t p = 0; p < n; p++) {
                const uint64_t* rr = row + (p / w) * nw;
                const uint64_t* cl = col + (p % w) * nw;
                for (size_t q = 0; q < nw; q++) yy[q] = rr[q] ^ cl[q];
                for (size_t ch = 0; ch < c; ch++) {
                    const uint64_t* tb = widened + (ch * 256 + px[p * c + ch]) * nw;
                    for (size_t q = 0; q < nw; q++) yy[q] ^= tb[q];
                }
                for (size_t cc = 0; cc < k; cc++) d[cc] = 0;
                for (size_t q = 0; q < nw; q++) { /* dot_words for all clusters at once */
                    uint64_t x = yy[q];
                    while (x) {
                        const uint32_t* zi = zt + ((q << 6) + (size_t)__builtin_ctzll(x)) * k;
                        for (size_t cc = 0; cc < k; cc++) d[cc] += zi[cc];
                        x &= x - 1;
                    }
                }
                uint32_t best = 0; /* assign_labels, clusterer.cpp:132-162 */
                for (size_t cc = 1; cc < k; cc++) {
                    wraps += (uint64_t)compare_wraps(d[cc], norm2[cc], d[best], norm2[best]);
                    if (strictly_closer(d[cc], norm2[cc], d[best], norm2[best])) best = (uint32_t)cc;
                }
                labels_final[p] = best;
                if (do_update) { /* IntVector::add_words into this thread's partial sums */
                    uint32_t* zc = acc + (size_t)best * dim;
                    for (size_t q = 0; q < nw; q++) {
                        uint64_t x = yy[q];
                        while (x) {
                            zc[(q << 6) + (size_t)__builtin_ctzll(x)]++;
                            x &= x - 1;
                        }
                    }
                    ct[best]++;
                }
            }
            free(yy);
        }
        record_wraps(r, wraps);
        rounds = r;
        if (labels_rounds) memcpy(labels_rounds + (r - 1) * n, labels_final, n * 4);
        if (early_stop && r > 1 && memcmp(labels_final, prev, n * 4) == 0) break;
        if (do_update) { /* update_centroids, clusterer.cpp:164-188: empty clusters keep theirs */
            for (size_t cc = 0; cc < k; cc++) {
                uint64_t total = 0;
                for (int t = 0; t < T; t++) total += cnt[(size_t)t * k + cc];
                counts[cc] = total;
                if (!total) continue;
                for (size_t i = 0; i < dim; i++) {
                    uint32_t s2 = 0;
                    for (int t = 0; t < T; t++) s2 += part[((size_t)t * k + cc) * dim + i];
                    zt[i * k + cc] = s2;
                }
            }
        }
        memcpy(prev, labels_final, n * 4);
    }
    if (centroids_out)
        for (size_t cc = 0; cc < k; cc++)
            for (size_t i = 0; i < dim; i++) centroids_out[cc * dim + i] = zt[i * k + cc];
    if (counts_out) memcpy(counts_out, counts, k * 8);
    *rounds_out = rounds;
    free(prev);
    free(seeds);
    free(zt);
    free(counts);
    free(part);
    free(cnt);
    free(norm2);
    return 0;
}

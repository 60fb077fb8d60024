// Synthetic nuclei images for the five BASELINE.json configs. Benchmark /
// test WORKLOAD generator only: neither the product library (paper_2303_12753_b200) nor the
// oracle links it, so bench.py's reference arm and the GPU arm read identical inputs without
// either loading the other's code. C ABI: seghdc_synth_image (returns 0 ok, 1 bad config id).
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

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
            throw std::invalid_argument("synthetic config id must be 0..4, got " + std::to_string(id));
    }
    return s;
}
}  // namespace

static void synth_image(int id, uint64_t seed, uint8_t* out, size_t* h_out, size_t* w_out, size_t* c_out) {
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


extern "C" int seghdc_synth_image(int config_id, uint64_t seed, uint8_t* out, size_t* h, size_t* w, size_t* c) {
    try {
        synth_image(config_id, seed, out, h, w, c);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

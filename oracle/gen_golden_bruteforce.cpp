// TEST INFRASTRUCTURE ONLY — run in the build container (needs /root/reference).
//
// Emits tests/golden/bruteforce_instances.json: the random tiny clustering instances of
// the reference's own suites, with the expected per-round labels produced by the
// reference's brute-force oracle (proj/tests/reference_clusterer.hpp:108-151, ref_cluster)
// and cross-checked against the reference library's cluster().
//
// Instance generation follows the reference test code exactly:
//   * "test_clusterer"  — proj/tests/test_clusterer.cpp:211-235 (seed 17, random_grid helper
//                          at :20-27: one Rng(seed), Hypervector::random per pixel, row-major)
//   * "acceptance_c5"   — proj/tests/acceptance/acceptance_main.cpp:200-231 (seed 0x5EED)
// The image helper random_image is the reference's (proj/tests/test_helpers.hpp:76-81);
// it is libstdc++-specific (uniform_int_distribution), which is why the bytes are frozen
// into the fixture instead of regenerated.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "reference_clusterer.hpp"
#include "seghdc/clusterer.hpp"
#include "test_helpers.hpp"

using namespace seghdc;

namespace {

void emit_instance(FILE* f, const char* suite, int idx, const ImageBuffer& img,
                   const PixelHvGrid& grid, std::size_t k, std::size_t iterations, bool first) {
    const auto expected = testing::ref_cluster(img, grid, k, iterations);
    std::vector<std::vector<std::uint32_t>> actual;
    cluster(grid, img, ClusterConfig{k, iterations, false},
            [&](std::size_t, const SegmentationMask& m) { actual.push_back(m.labels); });
    if (actual != expected) {
        std::fprintf(stderr, "reference cluster() disagrees with its brute-force oracle: %s %d\n", suite, idx);
        std::exit(3);
    }
    const auto seeds = select_initial_centroids(img, grid, k);
    std::fprintf(f, "%s  {\"suite\": \"%s\", \"instance\": %d, \"h\": %zu, \"w\": %zu, \"channels\": %zu, "
                 "\"dim\": %zu, \"k\": %zu, \"iterations\": %zu,\n   \"image\": [",
                 first ? "" : ",\n", suite, idx, img.height, img.width, img.channels, grid.dim(), k, iterations);
    for (std::size_t i = 0; i < img.pixels.size(); ++i) std::fprintf(f, "%s%u", i ? ", " : "", img.pixels[i]);
    std::fprintf(f, "],\n   \"grid\": [");
    const auto* words = grid.hv_words(0, 0).data();
    const std::size_t nw = grid.height() * grid.width() * grid.words_per_hv();
    for (std::size_t i = 0; i < nw; ++i) std::fprintf(f, "%s\"%016llx\"", i ? ", " : "", (unsigned long long)words[i]);
    std::fprintf(f, "],\n   \"seeds\": [");
    for (std::size_t s = 0; s < seeds.size(); ++s)
        std::fprintf(f, "%s%zu", s ? ", " : "", seeds[s].row * img.width + seeds[s].col);
    std::fprintf(f, "],\n   \"expected_rounds\": [");
    for (std::size_t r = 0; r < expected.size(); ++r) {
        std::fprintf(f, "%s[", r ? ", " : "");
        for (std::size_t p = 0; p < expected[r].size(); ++p) std::fprintf(f, "%s%u", p ? ", " : "", expected[r][p]);
        std::fprintf(f, "]");
    }
    std::fprintf(f, "]}");
}

}  // namespace

int main(int argc, char** argv) {
    FILE* f = argc > 1 ? std::fopen(argv[1], "w") : stdout;
    if (!f) return 2;
    std::fprintf(f, "{\"generator\": \"oracle/gen_golden_bruteforce.cpp\", \"instances\": [\n");
    bool first = true;
    {   // proj/tests/test_clusterer.cpp:211-235
        std::mt19937_64 seeds(17);
        for (int instance = 0; instance < 30; ++instance) {
            const std::size_t h = 1 + seeds() % 4, w = 1 + seeds() % 4;
            const std::size_t dim = 1 + seeds() % 32;
            const std::size_t channels = (seeds() % 2 == 0) ? 1 : 3;
            const std::size_t k = 1 + seeds() % std::min<std::size_t>(3, h * w);
            const std::size_t iterations = 1 + seeds() % 4;
            const auto img = testing::random_image(h, w, channels, seeds);
            PixelHvGrid grid(h, w, dim);
            Rng rng(seeds());
            for (std::size_t i = 0; i < h; ++i)
                for (std::size_t j = 0; j < w; ++j) grid.set_hv(i, j, Hypervector::random(dim, rng));
            emit_instance(f, "test_clusterer", instance, img, grid, k, iterations, first);
            first = false;
        }
    }
    {   // proj/tests/acceptance/acceptance_main.cpp:200-231
        std::mt19937_64 seeds(0x5EED);
        for (int instance = 0; instance < 30; ++instance) {
            const std::size_t h = 1 + seeds() % 4, w = 1 + seeds() % 4;
            const std::size_t dim = 1 + seeds() % 32;
            const std::size_t channels = (seeds() % 2 == 0) ? 1 : 3;
            const std::size_t k = 1 + seeds() % std::min<std::size_t>(3, h * w);
            const std::size_t iterations = 1 + seeds() % 4;
            const auto img = testing::random_image(h, w, channels, seeds);
            PixelHvGrid grid(h, w, dim);
            Rng rng(seeds());
            for (std::size_t i = 0; i < h; ++i)
                for (std::size_t j = 0; j < w; ++j) grid.set_hv(i, j, Hypervector::random(dim, rng));
            emit_instance(f, "acceptance_c5", instance, img, grid, k, iterations, first);
            first = false;
        }
    }
    std::fprintf(f, "\n]}\n");
    if (f != stdout) std::fclose(f);
    return 0;
}

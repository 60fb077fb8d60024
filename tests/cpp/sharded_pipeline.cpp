// C++ drop-in caller of the sharded pipeline (include/seghdc/seghdc.hpp): every rank passes the
// full image, gets its rows' labels and the (rank-identical) centroids. Built and run by
// tests/test_gpu_sharding.py with one rank over NCCL: the rows must equal run_pipeline()'s mask.
// Usage: sharded_pipeline <h> <w> <c> <k> <iterations>   (prints "ok" or the first mismatch)
#include <cstdio>
#include <cstdlib>
#include <random>

#include "seghdc/seghdc.hpp"

int main(int argc, char** argv) {
    if (argc < 6) return 2;
    const std::size_t h = std::strtoul(argv[1], nullptr, 10), w = std::strtoul(argv[2], nullptr, 10),
                      c = std::strtoul(argv[3], nullptr, 10);
    seghdc::ImageBuffer img;
    img.height = h;
    img.width = w;
    img.channels = c;
    img.pixels.resize(h * w * c);
    std::mt19937_64 rng(7);
    for (std::size_t i = 0; i < img.pixels.size(); ++i)
        img.pixels[i] = std::uint8_t((i / (w * c) < h / 2 ? 40 : 200) + rng() % 40);
    seghdc::RunConfig cfg;
    cfg.clusters = std::strtoul(argv[4], nullptr, 10);
    cfg.iterations = std::strtoul(argv[5], nullptr, 10);
    cfg.alpha = 1.0;
    cfg.early_stop = false;
    const auto single = seghdc::run_pipeline(img, cfg);
    seghdc::init_sharding(seghdc::nccl_unique_id(), 0, 1);
    for (int rep = 0; rep < 3; ++rep) {  // eager, graph capture, graph replay
        const auto part = seghdc::run_pipeline_sharded(img, cfg);
        if (part.row_begin != 0 || part.row_end != h || part.iterations_run != single.iterations_run) {
            std::printf("shape/rounds mismatch\n");
            return 1;
        }
        for (std::size_t p = 0; p < h * w; ++p)
            if (part.rows.labels[p] != single.mask.labels[p]) {
                std::printf("label mismatch at %zu\n", p);
                return 1;
            }
        if (part.centroids.k() != cfg.clusters) return 1;
    }
    std::printf("ok\n");
    return 0;
}

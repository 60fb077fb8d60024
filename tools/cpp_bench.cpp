// The reference CLI's `bench` protocol (proj/tools/seghdc_main.cpp:116-147: early stop off,
// `repeats` runs of run_pipeline, the median of every stage) as a C++ caller of the B200
// drop-in: std::vector image in, SegmentationMask out, nothing page-locked. This is the
// end-to-end rate a reference-side C++ program gets after relinking against
// libseghdc_b200.so. Inputs: the BASELINE configs' synthetic images (workloads/synth.cpp).
//
// Build: g++ -std=c++20 -O2 -Iinclude tools/cpp_bench.cpp -o cpp_bench \
//          -Lpaper_2303_12753_b200/lib -lseghdc_b200 -Lworkloads/lib -lseghdc_synth -lcudart ...
// Usage: cpp_bench <config 0..4> [repeats]     (prints one JSON line)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "seghdc/seghdc.hpp"

extern "C" int seghdc_synth_image(int config_id, uint64_t seed, uint8_t* out, size_t* h, size_t* w, size_t* c);

static double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const std::size_t n = v.size();
    return n % 2 == 1 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

int main(int argc, char** argv) {
    const int cid = argc > 1 ? std::atoi(argv[1]) : 1;
    const std::size_t repeats = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 20;
    size_t h = 0, w = 0, c = 0;
    if (seghdc_synth_image(cid, 0, nullptr, &h, &w, &c)) return 1;
    seghdc::ImageBuffer img;
    img.height = h;
    img.width = w;
    img.channels = c;
    img.pixels.resize(h * w * c);
    seghdc_synth_image(cid, 0, img.pixels.data(), &h, &w, &c);
    seghdc::RunConfig cfg;  // RunConfig defaults (pipeline.hpp:18-35), BASELINE.json's K / D / iterations
    const bool large = cid == 3 || cid == 4;
    cfg.dim = cid == 4 ? 16384 : 10000;
    cfg.clusters = cid == 3 ? 4 : cid == 4 ? 8 : 2;
    cfg.iterations = large ? 20 : 10;
    cfg.alpha = large ? 1.0 : 0.2;
    cfg.early_stop = false;  // the bench protocol (seghdc_main.cpp:119)
    std::map<std::string, std::vector<double>> samples;
    seghdc::PipelineResult last;
    for (int warm = 0; warm < 3; ++warm) last = seghdc::run_pipeline(img, cfg);
    for (std::size_t r = 0; r < repeats; ++r) {
        last = seghdc::run_pipeline(img, cfg);
        for (const auto& [stage, ms] : last.timings.as_map()) samples[stage].push_back(ms);
    }
    const double total = median(samples["total"]);
    std::printf("{\"config\": \"C%d\", \"repeats\": %zu, \"total_ms\": %.4f, \"cluster_ms\": %.4f, "
                "\"produce_pixels_ms\": %.4f, \"encode_position_ms\": %.4f, \"px_iter_per_s\": %.4e, "
                "\"iterations_run\": %zu, \"caller\": \"C++ drop-in seghdc::run_pipeline, std::vector buffers\"}\n",
                cid, repeats, total, median(samples["cluster"]), median(samples["produce_pixels"]),
                median(samples["encode_position"]), double(h * w * cfg.iterations) / (total / 1e3), last.iterations_run);
    return 0;
}

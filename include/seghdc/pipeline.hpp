// seghdc/pipeline.hpp — the reference's pipeline API (RunConfig, StageTimings, PipelineResult,
// run_pipeline) lives in seghdc/seghdc.hpp. MetricsRecord (pipeline.hpp:58-67, pipeline.cpp:77-91)
// is declared here: its to_json() returns an nlohmann::json exactly like the reference's and is
// defined inline, only where the caller has nlohmann's "json.hpp" on the include path (the
// reference vendors it; the library itself does not depend on it).
#pragma once
#include <optional>

#include "seghdc/metrics.hpp"
#include "seghdc/seghdc.hpp"

#if __has_include("json.hpp")
#include "json.hpp"
#define SEGHDC_HAVE_NLOHMANN_JSON 1
#endif

namespace seghdc {

/// Per-run metrics payload; serialized as one JSON object so batch tooling can aggregate
/// without parsing logs.
struct MetricsRecord {
    std::optional<double> iou;
    std::size_t iterations_run = 0;
    StageTimings timings;
    RunConfig config;

#ifdef SEGHDC_HAVE_NLOHMANN_JSON
    nlohmann::json to_json() const {
        nlohmann::json j;
        j["iou"] = iou.has_value() ? nlohmann::json(*iou) : nlohmann::json(nullptr);
        j["iterations_run"] = iterations_run;
        j["timings"] = timings.as_map();
        j["config"] = {{"d", config.dim},         {"alpha", config.alpha},           {"beta", config.beta},
                       {"gamma", config.gamma},   {"k", config.clusters},            {"iterations", config.iterations},
                       {"encoder", to_string(config.encoder)}, {"seed", config.seed}};
        return j;
    }
#endif
};

}  // namespace seghdc

// seghdc — the reference's command-line tool (proj/tools/seghdc_main.cpp:1-291) over the B200
// drop-in: the same subcommands (segment, eval, bench, batch), flags, printed lines, metrics JSON
// and exit codes (0 ok, 1 validation / usage, 2 I/O), so scripts written against the reference's
// binary run unchanged. The reference parses flags with CLI11 and writes JSON with nlohmann/json;
// neither is vendored here, so the flag parser and the JSON writer below are small hand-written
// equivalents (every value written is a number, a string or null).
//
//   g++ -std=c++20 -O2 -Iinclude tools/seghdc_cli.cpp -Lpaper_2303_12753_b200/lib -lseghdc_b200 ...
//   (built by paper_2303_12753_b200/build.py as paper_2303_12753_b200/lib/seghdc)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "seghdc/image_io.hpp"
#include "seghdc/metrics.hpp"
#include "seghdc/seghdc.hpp"

namespace fs = std::filesystem;

namespace {

constexpr int kExitOk = 0;
constexpr int kExitConfig = 1;
constexpr int kExitIo = 2;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- flags ------------------------------------------------------------------------------------
struct Flag {
    std::vector<std::string> names;
    bool takes_value;
    bool required;
    std::string help;
};

class Parser {
  public:
    Parser(std::string command, std::string about) : command_(std::move(command)), about_(std::move(about)) {}
    void option(std::vector<std::string> names, std::string help, bool required = false) {
        flags_.push_back({std::move(names), true, required, std::move(help)});
    }
    void flag(std::vector<std::string> names, std::string help) { flags_.push_back({std::move(names), false, false, std::move(help)}); }
    // returns false when --help was printed
    bool parse(int argc, char** argv, int first) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i], value;
            bool inline_value = false;
            if (a == "--help" || a == "-h") {
                print_help();
                return false;
            }
            if (a.rfind("--", 0) == 0) {
                const auto eq = a.find('=');
                if (eq != std::string::npos) value = a.substr(eq + 1), a = a.substr(0, eq), inline_value = true;
            }
            const Flag* f = find(a);
            if (!f) throw UsageError("unknown option '" + a + "' (run with --help)");
            if (!f->takes_value) {
                if (inline_value) throw UsageError("option '" + a + "' takes no value");
                values_[f->names[0]] = "1";
                continue;
            }
            if (!inline_value) {
                if (i + 1 >= argc) throw UsageError("option '" + a + "' needs a value");
                value = argv[++i];
            }
            values_[f->names[0]] = value;
        }
        for (const auto& f : flags_)
            if (f.required && !values_.count(f.names[0])) throw UsageError(f.names[0] + " is required");
        return true;
    }
    bool has(const std::string& name) const { return values_.count(name) != 0; }
    std::string str(const std::string& name, const std::string& dflt = "") const {
        const auto it = values_.find(name);
        return it == values_.end() ? dflt : it->second;
    }
    template <typename T>
    void number(const std::string& name, T& out) const {
        const auto it = values_.find(name);
        if (it == values_.end()) return;
        std::istringstream in(it->second);
        T v{};
        if (it->second.empty() || it->second[0] == '-' || !(in >> v) || !in.eof())
            throw UsageError("option '" + name + "': '" + it->second + "' is not a valid number");
        out = v;
    }
    void real(const std::string& name, double& out) const {
        const auto it = values_.find(name);
        if (it == values_.end()) return;
        char* end = nullptr;
        const double v = std::strtod(it->second.c_str(), &end);
        if (it->second.empty() || *end != '\0') throw UsageError("option '" + name + "': '" + it->second + "' is not a number");
        out = v;
    }
    std::vector<std::size_t> list(const std::string& name) const {
        std::vector<std::size_t> out;
        const auto it = values_.find(name);
        if (it == values_.end()) return out;
        std::stringstream in(it->second);
        std::string tok;
        while (std::getline(in, tok, ',')) {
            std::size_t v = 0;
            std::istringstream t(tok);
            if (tok.empty() || tok[0] == '-' || !(t >> v) || !t.eof())
                throw UsageError("option '" + name + "': '" + tok + "' is not a valid number");
            out.push_back(v);
        }
        return out;
    }

  private:
    const Flag* find(const std::string& name) const {
        for (const auto& f : flags_)
            for (const auto& n : f.names)
                if (n == name) return &f;
        return nullptr;
    }
    void print_help() const {
        std::cout << about_ << "\nUsage: seghdc " << command_ << " [OPTIONS]\n\nOptions:\n";
        for (const auto& f : flags_) {
            std::string names;
            for (const auto& n : f.names) names += (names.empty() ? "" : ",") + n;
            std::cout << "  " << names << (f.takes_value ? " VALUE" : "") << (f.required ? " REQUIRED" : "") << "\n      " << f.help
                      << "\n";
        }
    }
    std::string command_, about_;
    std::vector<Flag> flags_;
    std::map<std::string, std::string> values_;
};

// ---- metrics JSON (the reference's MetricsRecord::to_json, pipeline.cpp:77-91) ----------------
std::string json_number(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}
std::string json_string(const std::string& s) {
    std::string out = "\"";
    for (const char ch : s) {
        if (ch == '"' || ch == '\\') out += '\\', out += ch;
        else if (static_cast<unsigned char>(ch) < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof(buf), "\\u%04x", ch);
            out += buf;
        } else out += ch;
    }
    return out + "\"";
}

struct MetricsRecord {
    std::optional<double> iou;
    std::size_t iterations_run = 0;
    seghdc::StageTimings timings;
    seghdc::RunConfig config;

    // keys in nlohmann's (alphabetical) order, two-space indent like dump(2)
    std::string to_json(const std::string& ind) const {
        std::ostringstream o;
        o << "{\n";
        o << ind << "  \"config\": {\n";
        o << ind << "    \"alpha\": " << json_number(config.alpha) << ",\n";
        o << ind << "    \"beta\": " << config.beta << ",\n";
        o << ind << "    \"d\": " << config.dim << ",\n";
        o << ind << "    \"encoder\": " << json_string(seghdc::to_string(config.encoder)) << ",\n";
        o << ind << "    \"gamma\": " << config.gamma << ",\n";
        o << ind << "    \"iterations\": " << config.iterations << ",\n";
        o << ind << "    \"k\": " << config.clusters << ",\n";
        o << ind << "    \"seed\": " << config.seed << "\n";
        o << ind << "  },\n";
        o << ind << "  \"iou\": " << (iou ? json_number(*iou) : std::string("null")) << ",\n";
        o << ind << "  \"iterations_run\": " << iterations_run << ",\n";
        o << ind << "  \"timings\": {\n";
        const auto tm = timings.as_map();
        std::size_t i = 0;
        for (const auto& [stage, ms] : tm)
            o << ind << "    " << json_string(stage) << ": " << json_number(ms) << (++i < tm.size() ? ",\n" : "\n");
        o << ind << "  }\n";
        o << ind << "}";
        return o.str();
    }
};

void write_text(const std::string& text, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw seghdc::IoError("cannot write '" + path + "'");
    out << text << "\n";
}

// ---- shared options (seghdc_main.cpp:26-57) ------------------------------------------------------
struct CommonOptions {
    std::string input, gt, metrics, encoder = "manhattan";
    bool no_early_stop = false;
    seghdc::RunConfig config;
};

void add_config_flags(Parser& p) {
    p.option({"--input", "-i"}, "Input image (8-bit PNG or binary PGM)", true);
    p.option({"--dim"}, "Hypervector dimension d");
    p.option({"--alpha"}, "Position flip-unit ratio in (0, 1]");
    p.option({"--beta"}, "Position block size");
    p.option({"--gamma"}, "Color flip-expansion factor");
    p.option({"--clusters", "-k"}, "Number of clusters");
    p.option({"--iterations"}, "Clustering iterations");
    p.option({"--seed"}, "Codebook RNG seed");
    p.option({"--encoder"}, "Encoder kind: manhattan, rpos or rcolor");
    p.flag({"--no-early-stop"}, "Always run the configured number of iterations");
    p.option({"--metrics"}, "Write metrics JSON to this path");
}

void read_config_flags(const Parser& p, CommonOptions& o) {
    o.input = p.str("--input");
    o.gt = p.str("--gt");
    o.metrics = p.str("--metrics");
    o.encoder = p.str("--encoder", "manhattan");
    o.no_early_stop = p.has("--no-early-stop");
    p.number("--dim", o.config.dim);
    p.real("--alpha", o.config.alpha);
    p.number("--beta", o.config.beta);
    p.number("--gamma", o.config.gamma);
    p.number("--clusters", o.config.clusters);
    p.number("--iterations", o.config.iterations);
    p.number("--seed", o.config.seed);
    if (o.encoder != "manhattan" && o.encoder != "rpos" && o.encoder != "rcolor")
        throw UsageError("--encoder: '" + o.encoder + "' not in {manhattan,rpos,rcolor}");
    o.config.encoder = seghdc::encoder_kind_from_string(o.encoder);
    if (o.no_early_stop) o.config.early_stop = false;
}

double score_against_gt(const seghdc::SegmentationMask& mask, const std::string& gt_path, std::size_t k) {
    const seghdc::ImageBuffer gt_img = seghdc::load_image(gt_path);
    const seghdc::BinaryMask gt = seghdc::binarize_ground_truth(gt_img);
    return seghdc::best_foreground_iou(mask, gt, k).iou;
}

// ---- segment (seghdc_main.cpp:73-106) --------------------------------------------------------------
int run_segment(CommonOptions& o, const std::string& output, const std::string& dump_dir) {
    const seghdc::ImageBuffer img = seghdc::load_image(o.input);
    o.config.validate(img);
    std::size_t dumped = 0;
    seghdc::IterationCallback on_iteration;
    if (!dump_dir.empty()) {
        fs::create_directories(dump_dir);
        on_iteration = [&](std::size_t round, const seghdc::SegmentationMask& m) {
            char name[32];
            std::snprintf(name, sizeof(name), "iter_%03zu.png", round);
            seghdc::save_mask(m, o.config.clusters, (fs::path(dump_dir) / name).string());
            ++dumped;
        };
    }
    const seghdc::PipelineResult result = seghdc::run_pipeline(img, o.config, on_iteration);
    seghdc::save_mask(result.mask, o.config.clusters, output);
    MetricsRecord record{{}, result.iterations_run, result.timings, o.config};
    if (!o.gt.empty()) record.iou = score_against_gt(result.mask, o.gt, o.config.clusters);
    if (!o.metrics.empty()) write_text(record.to_json(""), o.metrics);
    std::cout << "mask: " << output << "  iterations: " << result.iterations_run;
    std::cout.flush();
    if (record.iou) std::printf("  iou: %.4f", *record.iou);
    std::fflush(stdout);
    if (dumped > 0) std::cout << "  per-iteration masks: " << dumped;
    std::cout.flush();
    std::printf("  total: %.1f ms\n", result.timings.total_ms);
    return kExitOk;
}

// ---- eval (seghdc_main.cpp:108-116) ---------------------------------------------------------------
int run_eval(const std::string& pred_path, const std::string& gt_path, std::size_t k) {
    const seghdc::ImageBuffer pred_img = seghdc::load_image(pred_path);
    const seghdc::ImageBuffer gt_img = seghdc::load_image(gt_path);
    const seghdc::SegmentationMask pred = seghdc::labels_from_mask_image(pred_img, k);
    const seghdc::BinaryMask gt = seghdc::binarize_ground_truth(gt_img);
    std::printf("%.4f\n", seghdc::best_foreground_iou(pred, gt, k).iou);
    return kExitOk;
}

// ---- bench (seghdc_main.cpp:116-161): fixed iterations, early stop off, median of the repeats ----------
// One configuration of the sweep: `repeats` pipeline runs, every stage's median time.
MetricsRecord bench_one(const seghdc::ImageBuffer& img, const seghdc::RunConfig& cfg, std::size_t repeats,
                        const std::string& gt_path) {
    cfg.validate(img);
    std::map<std::string, std::vector<double>> samples;
    seghdc::PipelineResult last;
    for (std::size_t r = 0; r < repeats; ++r) {
        last = seghdc::run_pipeline(img, cfg);
        for (const auto& [stage, ms] : last.timings.as_map()) samples[stage].push_back(ms);
    }
    const auto mid = [&](const char* stage) {
        std::vector<double>& v = samples[stage];
        std::sort(v.begin(), v.end());
        return v.size() % 2 ? v[v.size() / 2] : 0.5 * (v[v.size() / 2 - 1] + v[v.size() / 2]);
    };
    MetricsRecord record;
    record.iterations_run = last.iterations_run;
    record.config = cfg;
    record.timings.encode_position_ms = mid("encode_position");
    record.timings.encode_color_ms = mid("encode_color");
    record.timings.produce_pixels_ms = mid("produce_pixels");
    record.timings.cluster_ms = mid("cluster");
    record.timings.total_ms = mid("total");
    if (!gt_path.empty()) record.iou = score_against_gt(last.mask, gt_path, cfg.clusters);
    return record;
}

int run_bench(CommonOptions& o, std::size_t repeats, std::vector<std::size_t> sweep_dim, std::vector<std::size_t> sweep_iters) {
    o.config.early_stop = false;  // the fixed-iteration protocol
    if (repeats == 0) throw seghdc::ConfigError("bench: --repeats must be >= 1");
    const seghdc::ImageBuffer img = seghdc::load_image(o.input);
    if (sweep_dim.empty()) sweep_dim.push_back(o.config.dim);
    if (sweep_iters.empty()) sweep_iters.push_back(o.config.iterations);
    std::vector<std::string> records;
    for (const std::size_t d : sweep_dim)
        for (const std::size_t iters : sweep_iters) {
            seghdc::RunConfig cfg = o.config;
            cfg.dim = d;
            cfg.iterations = iters;
            const MetricsRecord record = bench_one(img, cfg, repeats, o.gt);
            records.push_back(record.to_json("  "));
            std::printf("d=%zu iterations=%zu total=%.1f ms cluster=%.1f ms", d, iters, record.timings.total_ms,
                        record.timings.cluster_ms);
            if (record.iou) std::printf(" iou=%.4f", *record.iou);
            std::printf("\n");
        }
    if (!o.metrics.empty()) {
        std::string text = "[";
        for (std::size_t i = 0; i < records.size(); ++i) text += std::string(i ? ",\n  " : "\n  ") + records[i];
        write_text(text + (records.empty() ? "]" : "\n]"), o.metrics);
    }
    return kExitOk;
}

// ---- batch (seghdc_main.cpp:163-225): inputs and ground truths paired by filename stem --------------------
// Regular files of `dir` by stem, first path (in sorted order) winning a duplicate stem.
std::map<std::string, fs::path> stem_index(const std::string& dir) {
    if (!fs::is_directory(dir)) throw seghdc::IoError("'" + dir + "' is not a directory");
    std::vector<fs::path> files;
    for (const auto& entry : fs::directory_iterator(dir))
        if (entry.is_regular_file()) files.push_back(entry.path());
    std::sort(files.begin(), files.end());
    std::map<std::string, fs::path> index;
    for (const auto& p : files)
        if (!index.emplace(p.stem().string(), p).second)
            std::cerr << "warning: duplicate stem '" << p.stem().string() << "' in " << dir << ", keeping first match\n";
    return index;
}

int run_batch(CommonOptions& o) {
    const auto inputs = stem_index(o.input);
    const auto gts = stem_index(o.gt);
    struct Pair {
        std::string stem;
        fs::path input, gt;
    };
    std::vector<Pair> pairs;  // in sorted-stem order
    for (const auto& [stem, path] : inputs) {
        const auto gt = gts.find(stem);
        if (gt == gts.end()) std::cerr << "warning: no ground truth for '" << path.string() << "', skipped\n";
        else pairs.push_back({stem, path, gt->second});
    }
    for (const auto& [stem, path] : gts)
        if (!inputs.count(stem)) std::cerr << "warning: no input for ground truth '" << path.string() << "', skipped\n";
    if (pairs.empty()) {
        std::cerr << "error: no input/ground-truth pairs matched by filename stem\n";
        return kExitConfig;
    }
    std::string per_image;
    double iou_sum = 0.0;
    for (const Pair& pr : pairs) {
        const seghdc::ImageBuffer img = seghdc::load_image(pr.input.string());
        o.config.validate(img);
        const seghdc::PipelineResult result = seghdc::run_pipeline(img, o.config);
        const double score = score_against_gt(result.mask, pr.gt.string(), o.config.clusters);
        per_image += std::string(per_image.empty() ? "\n" : ",\n") + "    {\n      \"iou\": " + json_number(score) +
                     ",\n      \"iterations_run\": " + std::to_string(result.iterations_run) +
                     ",\n      \"stem\": " + json_string(pr.stem) + "\n    }";
        iou_sum += score;
        std::printf("%s  iou=%.4f\n", pr.stem.c_str(), score);
    }
    const double mean = iou_sum / static_cast<double>(pairs.size());
    if (!o.metrics.empty())
        write_text("{\n  \"count\": " + std::to_string(pairs.size()) + ",\n  \"mean_iou\": " + json_number(mean) +
                       ",\n  \"per_image\": [" + per_image + "\n  ]\n}",
                   o.metrics);
    std::printf("mean iou over %zu images: %.4f\n", pairs.size(), mean);
    return kExitOk;
}

void usage() {
    std::cout << "Hyperdimensional-computing unsupervised image segmentation (B200 drop-in)\n"
                 "Usage: seghdc SUBCOMMAND [OPTIONS]\n\nSubcommands:\n"
                 "  segment  Segment one image into a label mask\n"
                 "  eval     Score a mask PNG against ground truth\n"
                 "  bench    Time the pipeline (fixed iterations, early stop disabled)\n"
                 "  batch    Segment and score a directory of images\n";
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) {
            usage();
            std::cerr << "A subcommand is required\n";
            return kExitConfig;
        }
        const std::string cmd = argv[1];
        if (cmd == "--help" || cmd == "-h") {
            usage();
            return kExitOk;
        }
        if (cmd == "segment") {
            Parser p("segment", "Segment one image into a label mask");
            add_config_flags(p);
            p.option({"--output", "-o"}, "Output mask PNG", true);
            p.option({"--gt"}, "Ground-truth image for IoU scoring");
            p.option({"--dump-iterations"}, "Directory receiving one mask PNG per clustering round");
            if (!p.parse(argc, argv, 2)) return kExitOk;
            CommonOptions o;
            read_config_flags(p, o);
            return run_segment(o, p.str("--output"), p.str("--dump-iterations"));
        }
        if (cmd == "eval") {
            Parser p("eval", "Score a mask PNG against ground truth");
            p.option({"--input", "-i"}, "Predicted mask PNG", true);
            p.option({"--gt"}, "Ground-truth image", true);
            p.option({"--clusters", "-k"}, "Number of label levels in the mask");
            if (!p.parse(argc, argv, 2)) return kExitOk;
            std::size_t k = 2;
            p.number("--clusters", k);
            return run_eval(p.str("--input"), p.str("--gt"), k);
        }
        if (cmd == "bench") {
            Parser p("bench", "Time the pipeline (fixed iterations, early stop disabled)");
            add_config_flags(p);
            p.option({"--gt"}, "Ground-truth image for IoU scoring");
            p.option({"--repeats"}, "Runs per configuration (median reported)");
            p.option({"--sweep-dim"}, "Comma-separated dimensions to sweep");
            p.option({"--sweep-iters"}, "Comma-separated iteration counts to sweep");
            if (!p.parse(argc, argv, 2)) return kExitOk;
            CommonOptions o;
            read_config_flags(p, o);
            std::size_t repeats = 1;
            p.number("--repeats", repeats);
            return run_bench(o, repeats, p.list("--sweep-dim"), p.list("--sweep-iters"));
        }
        if (cmd == "batch") {
            Parser p("batch", "Segment and score a directory of images");
            add_config_flags(p);
            p.option({"--gt"}, "Ground-truth directory (paired by filename stem)", true);
            if (!p.parse(argc, argv, 2)) return kExitOk;
            CommonOptions o;
            read_config_flags(p, o);
            return run_batch(o);
        }
        usage();
        std::cerr << "unknown subcommand '" << cmd << "'\n";
        return kExitConfig;
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\n";
        return kExitConfig;
    } catch (const seghdc::ConfigError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitConfig;
    } catch (const seghdc::IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitIo;
    } catch (const std::exception& e) {  // device / runtime failures of the drop-in
        std::cerr << "error: " << e.what() << "\n";
        return kExitIo;
    }
    return kExitConfig;
}

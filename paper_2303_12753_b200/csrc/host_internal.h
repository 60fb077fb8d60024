// Internal host helpers shared by the C-ABI layer (not part of the public interface).
#pragma once
#include <cstddef>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>

namespace seghdc_host {

// Carries a C-ABI status code (SEGHDC_ECONFIG / SEGHDC_ERUNTIME) with the message.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void validate_position(size_t dim, size_t h, size_t w, double alpha, size_t beta);
void validate_color(size_t dim, size_t c, size_t gamma);
void validate_image(size_t h, size_t w, size_t c);
void validate_cluster(size_t k, size_t iterations, size_t pixel_count);

void build_position(size_t dim, size_t h, size_t w, double alpha, size_t beta, int encoder, std::mt19937_64& rng,
                    uint64_t* row_out, uint64_t* col_out);
void build_color(size_t dim, size_t c, size_t gamma, int encoder, std::mt19937_64& rng, uint64_t* widened_out);

// The Manhattan codebooks in closed form (position_encoder.cpp:50-76, color_encoder.cpp:37-55,
// pixel_pipeline.cpp:70-88): row i = base_r ^ ones[0, (i / beta) * x_row), column j = base_c ^
// ones[d/2, d/2 + (j / beta) * x_col), widened colour (ch, v) = base_ch << off_ch ^
// ones[off_ch, off_ch + v * u_ch). Draws the bases from rng in the reference's order and fills
// bases = [base_r | base_c | widened base_ch...] (full-dim HVs of words_for(dim) u64 each).
struct ManhattanParams {
    uint32_t dim, h, w, c, beta, x_row, x_col;
    uint32_t off[3], unit[3];
};
ManhattanParams manhattan_bases(size_t dim, size_t h, size_t w, size_t c, double alpha, size_t beta, size_t gamma,
                                std::mt19937_64& rng, uint64_t* bases);

}  // namespace seghdc_host

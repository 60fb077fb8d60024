// Image and mask files (reference image_io.cpp:31-217): 8-bit gray / RGB PNG and binary PGM in,
// PNG out. The reference goes through libpng; this is a from-scratch PNG codec over zlib
// (chunk framing, CRC, the five scanline filters on the read side, filter 0 on the write side),
// with the reference's error contract: IoError for unreadable or unsupported files (same
// messages where its tests check them), ConfigError for label / k violations.
#include <zlib.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "seghdc/errors.hpp"
#include "seghdc/image_io.hpp"

namespace seghdc {

namespace {

struct FileCloser {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};
using FilePtr = std::unique_ptr<std::FILE, FileCloser>;

FilePtr open_file(const std::string& path, const char* mode) {
    FilePtr f(std::fopen(path.c_str(), mode));
    if (!f) throw IoError("cannot open '" + path + "'");
    return f;
}

std::vector<std::uint8_t> read_all(std::FILE* fp) {
    std::vector<std::uint8_t> data;
    std::uint8_t buf[1 << 16];
    std::size_t got;
    while ((got = std::fread(buf, 1, sizeof(buf), fp)) > 0) data.insert(data.end(), buf, buf + got);
    return data;
}

constexpr std::uint8_t kPngSig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};

std::uint32_t be32(const std::uint8_t* p) {
    return (std::uint32_t(p[0]) << 24) | (std::uint32_t(p[1]) << 16) | (std::uint32_t(p[2]) << 8) | p[3];
}
void put_be32(std::vector<std::uint8_t>& out, std::uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) out.push_back(std::uint8_t(v >> s));
}

int paeth(int a, int b, int c) {
    const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
    return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

// PNG (ISO/IEC 15948): signature, then chunks [length | type | data | CRC(type + data)]; IHDR
// first, the zlib stream split over IDAT chunks, IEND last. Scanlines carry a filter byte.
ImageBuffer load_png(const std::vector<std::uint8_t>& file, const std::string& path) {
    const auto corrupt = [&]() { return IoError("corrupt PNG file '" + path + "'"); };
    std::size_t pos = 8;
    bool have_ihdr = false, have_iend = false;
    std::uint32_t width = 0, height = 0;
    int bit_depth = 0, color_type = 0, interlace = 0;
    std::vector<std::uint8_t> zdata;
    while (!have_iend) {
        if (pos + 12 > file.size()) throw corrupt();
        const std::uint32_t len = be32(&file[pos]);
        if (len > file.size() || pos + 12 + len > file.size()) throw corrupt();
        const std::uint8_t* type = &file[pos + 4];
        const std::uint8_t* data = &file[pos + 8];
        if (std::uint32_t(crc32(crc32(0L, Z_NULL, 0), type, 4 + len)) != be32(data + len)) throw corrupt();
        if (!have_ihdr && std::memcmp(type, "IHDR", 4) != 0) throw corrupt();
        if (std::memcmp(type, "IHDR", 4) == 0) {
            if (len != 13 || have_ihdr) throw corrupt();
            have_ihdr = true;
            width = be32(data);
            height = be32(data + 4);
            bit_depth = data[8];
            color_type = data[9];
            interlace = data[12];
            if (width == 0 || height == 0 || data[10] != 0 || data[11] != 0) throw corrupt();
            // rejected before any pixel data is touched (image_io.cpp:51-62)
            if (bit_depth != 8)
                throw IoError("unsupported bit depth " + std::to_string(bit_depth) + " in '" + path +
                              "' (only 8-bit images are supported)");
            if (color_type != 0 && color_type != 2)
                throw IoError("unsupported PNG color type in '" + path +
                              "' (only 8-bit grayscale and RGB are supported)");
            if (interlace != 0) throw IoError("unsupported interlaced PNG '" + path + "'");
        } else if (std::memcmp(type, "IDAT", 4) == 0) {
            zdata.insert(zdata.end(), data, data + len);
        } else if (std::memcmp(type, "IEND", 4) == 0) {
            have_iend = true;
        } else if (!(type[0] & 0x20)) {
            throw corrupt();  // an unknown critical chunk
        }
        pos += 12 + std::size_t(len);
    }
    ImageBuffer img;
    img.height = height;
    img.width = width;
    img.channels = color_type == 2 ? 3 : 1;
    const std::size_t bpp = img.channels, stride = img.width * bpp;
    std::vector<std::uint8_t> raw((stride + 1) * img.height);
    uLongf raw_len = uLongf(raw.size());
    if (zdata.empty() || uncompress(raw.data(), &raw_len, zdata.data(), uLong(zdata.size())) != Z_OK ||
        raw_len != raw.size())
        throw corrupt();
    img.pixels.resize(stride * img.height);
    for (std::size_t y = 0; y < img.height; ++y) {
        const std::uint8_t* in = &raw[y * (stride + 1)];
        std::uint8_t* out = &img.pixels[y * stride];
        const std::uint8_t* up = y ? out - stride : nullptr;
        const int filter = in[0];
        if (filter > 4) throw corrupt();
        for (std::size_t x = 0; x < stride; ++x) {
            const int a = x >= bpp ? out[x - bpp] : 0, b = up ? up[x] : 0, c = (up && x >= bpp) ? up[x - bpp] : 0;
            const int pred = filter == 0 ? 0 : filter == 1 ? a : filter == 2 ? b : filter == 3 ? (a + b) / 2 : paeth(a, b, c);
            out[x] = std::uint8_t(in[1 + x] + pred);
        }
    }
    return img;
}

// Binary PGM (P5), parsed from the file's bytes: magic, width, height, maxval as whitespace-
// separated decimal tokens ('#' starts a comment that runs to the end of the line), exactly one
// whitespace byte after maxval, then width x height samples.
struct PgmCursor {
    const std::vector<std::uint8_t>& bytes;
    std::size_t at = 0;
    static bool space(std::uint8_t ch) { return ch == ' ' || (ch >= '\t' && ch <= '\r'); }
    // next token, leaving the cursor just past the single byte that ended it; empty at end of file
    std::string token() {
        std::string tok;
        while (at < bytes.size()) {
            const std::uint8_t ch = bytes[at++];
            if (ch == '#') {
                while (at < bytes.size() && bytes[at++] != '\n') {
                }
            } else if (!space(ch)) {
                tok.push_back(char(ch));
            } else if (!tok.empty()) {
                break;
            }
        }
        return tok;
    }
};

ImageBuffer load_pgm(const std::vector<std::uint8_t>& file, const std::string& path) {
    PgmCursor cur{file};
    long field[3] = {0, 0, 0};  // width, height, maxval
    if (cur.token() != "P5") throw IoError("'" + path + "' is not a binary PGM (P5) file");
    for (long& f : field) {
        const std::string tok = cur.token();
        if (tok.empty()) throw IoError("truncated PGM header in '" + path + "'");
        f = std::strtol(tok.c_str(), nullptr, 10);
    }
    const long width = field[0], height = field[1], maxval = field[2];
    if (width <= 0 || height <= 0) throw IoError("invalid PGM dimensions in '" + path + "'");
    if (maxval > 255)
        throw IoError("unsupported bit depth in '" + path + "' (PGM maxval " + std::to_string(maxval) + " exceeds 255)");
    if (maxval <= 0) throw IoError("invalid PGM maxval in '" + path + "'");
    ImageBuffer img;
    img.height = std::size_t(height);
    img.width = std::size_t(width);
    img.channels = 1;
    const std::size_t count = img.height * img.width;
    if (file.size() - cur.at < count) throw IoError("truncated PGM pixel data in '" + path + "'");
    img.pixels.assign(file.begin() + std::ptrdiff_t(cur.at), file.begin() + std::ptrdiff_t(cur.at + count));
    return img;
}

void put_chunk(std::vector<std::uint8_t>& out, const char* type, const std::vector<std::uint8_t>& data) {
    put_be32(out, std::uint32_t(data.size()));
    const std::size_t start = out.size();
    out.insert(out.end(), type, type + 4);
    out.insert(out.end(), data.begin(), data.end());
    put_be32(out, std::uint32_t(crc32(crc32(0L, Z_NULL, 0), &out[start], uInt(4 + data.size()))));
}

std::uint8_t level_value(std::size_t label, std::size_t k) {
    return k <= 1 ? 0 : std::uint8_t(255 * label / (k - 1));
}

}  // namespace

ImageBuffer load_image(const std::string& path) {
    const std::vector<std::uint8_t> file = read_all(open_file(path, "rb").get());
    if (file.size() >= 8 && std::memcmp(file.data(), kPngSig, 8) == 0) return load_png(file, path);
    if (file.size() >= 2 && file[0] == 'P' && file[1] == '5') return load_pgm(file, path);
    throw IoError("'" + path + "' is neither a PNG nor a binary PGM (P5) file");
}

void save_image(const ImageBuffer& img, const std::string& path) {
    img.validate();
    if (img.channels != 1 && img.channels != 3) throw ConfigError("save_image: 1 or 3 channels");
    auto fp = open_file(path, "wb");
    const std::size_t stride = img.width * img.channels;
    std::vector<std::uint8_t> raw((stride + 1) * img.height);
    for (std::size_t y = 0; y < img.height; ++y) {
        raw[y * (stride + 1)] = 0;  // filter type 0 on every scanline
        std::memcpy(&raw[y * (stride + 1) + 1], &img.pixels[y * stride], stride);
    }
    uLongf zlen = compressBound(uLong(raw.size()));
    std::vector<std::uint8_t> z(zlen);
    if (compress2(z.data(), &zlen, raw.data(), uLong(raw.size()), Z_DEFAULT_COMPRESSION) != Z_OK)
        throw IoError("failed to write PNG '" + path + "'");
    z.resize(zlen);
    std::vector<std::uint8_t> out(kPngSig, kPngSig + 8), ihdr;
    put_be32(ihdr, std::uint32_t(img.width));
    put_be32(ihdr, std::uint32_t(img.height));
    ihdr.push_back(8);                              // bit depth
    ihdr.push_back(img.channels == 3 ? 2 : 0);      // colour type: RGB or grayscale
    ihdr.insert(ihdr.end(), {0, 0, 0});             // deflate, adaptive filtering, no interlace
    put_chunk(out, "IHDR", ihdr);
    put_chunk(out, "IDAT", z);
    put_chunk(out, "IEND", {});
    if (std::fwrite(out.data(), 1, out.size(), fp.get()) != out.size())
        throw IoError("failed to write PNG '" + path + "'");
}

void save_mask(const SegmentationMask& mask, std::size_t k, const std::string& path) {
    if (k == 0) throw ConfigError("save_mask: k must be >= 1");
    if (k > 256) throw ConfigError("save_mask: k > 256 cannot map to distinct 8-bit levels");
    ImageBuffer img;
    img.height = mask.height;
    img.width = mask.width;
    img.channels = 1;
    img.pixels.resize(mask.labels.size());
    for (std::size_t i = 0; i < mask.labels.size(); ++i) {
        if (mask.labels[i] >= k)
            throw ConfigError("save_mask: label " + std::to_string(mask.labels[i]) + " out of range for k = " +
                              std::to_string(k));
        img.pixels[i] = level_value(mask.labels[i], k);
    }
    save_image(img, path);
}

SegmentationMask labels_from_mask_image(const ImageBuffer& img, std::size_t k) {
    if (k == 0 || k > 256) throw ConfigError("labels_from_mask_image: k must be in 1..256");
    if (img.channels != 1) throw ConfigError("labels_from_mask_image: mask image must be grayscale");
    std::uint32_t nearest[256];  // value -> label of the nearest level, lowest label on ties
    for (int v = 0; v < 256; ++v) {
        std::size_t best = 0;
        int best_err = 256;
        for (std::size_t l = 0; l < k; ++l) {
            const int err = std::abs(v - int(level_value(l, k)));
            if (err < best_err) best_err = err, best = l;
        }
        nearest[v] = std::uint32_t(best);
    }
    SegmentationMask mask;
    mask.height = img.height;
    mask.width = img.width;
    mask.labels.resize(img.pixels.size());
    for (std::size_t i = 0; i < img.pixels.size(); ++i) mask.labels[i] = nearest[img.pixels[i]];
    return mask;
}

}  // namespace seghdc

// TEST INFRASTRUCTURE — a from-scratch stand-in for the write-side subset of libpng that the
// reference's own tests/test_image_io.cpp uses to fabricate 16-bit and RGBA files (libpng is not
// installed in this image). It exists only so that suite compiles UNMODIFIED against the drop-in
// (oracle/Makefile, target suites); nothing in the product includes it. Files are written with
// zlib: signature, IHDR, one IDAT (filter 0 on every row), IEND.
#pragma once
#include <zlib.h>

#include <cstdint>
#include <cstdio>
#include <vector>

typedef std::uint32_t png_uint_32;
typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef const png_byte* png_const_bytep;

#define PNG_LIBPNG_VER_STRING "shim"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_COLOR_TYPE_GRAY_ALPHA 4
#define PNG_COLOR_TYPE_RGBA 6
#define PNG_COLOR_TYPE_RGB_ALPHA 6
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

struct png_shim_writer {
    std::FILE* fp = nullptr;
    png_uint_32 width = 0, height = 0;
    int bit_depth = 8, color_type = 0;
    std::vector<unsigned char> raw;  // filter byte + row bytes, row after row
};
struct png_shim_info {};
typedef png_shim_writer* png_structp;
typedef png_shim_info* png_infop;

inline png_structp png_create_write_struct(const char*, void*, void*, void*) { return new png_shim_writer; }
inline png_infop png_create_info_struct(png_structp) { return new png_shim_info; }
inline void png_init_io(png_structp png, std::FILE* fp) { png->fp = fp; }
inline void png_set_IHDR(png_structp png, png_infop, png_uint_32 w, png_uint_32 h, int bit_depth, int color_type, int,
                         int, int) {
    png->width = w, png->height = h, png->bit_depth = bit_depth, png->color_type = color_type;
}
inline void png_shim_be32(std::vector<unsigned char>& out, std::uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) out.push_back(static_cast<unsigned char>(v >> s));
}
inline void png_shim_chunk(std::FILE* fp, const char* type, const std::vector<unsigned char>& data) {
    std::vector<unsigned char> out;
    png_shim_be32(out, static_cast<std::uint32_t>(data.size()));
    out.insert(out.end(), type, type + 4);
    out.insert(out.end(), data.begin(), data.end());
    png_shim_be32(out, static_cast<std::uint32_t>(crc32(crc32(0L, Z_NULL, 0), out.data() + 4, uInt(4 + data.size()))));
    std::fwrite(out.data(), 1, out.size(), fp);
}
inline void png_write_info(png_structp png, png_infop) {
    static const unsigned char sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
    std::fwrite(sig, 1, 8, png->fp);
    std::vector<unsigned char> ihdr;
    png_shim_be32(ihdr, png->width);
    png_shim_be32(ihdr, png->height);
    ihdr.push_back(static_cast<unsigned char>(png->bit_depth));
    ihdr.push_back(static_cast<unsigned char>(png->color_type));
    ihdr.insert(ihdr.end(), {0, 0, 0});
    png_shim_chunk(png->fp, "IHDR", ihdr);
}
inline std::size_t png_shim_row_bytes(png_structp png) {
    const int ch = png->color_type == 2 ? 3 : png->color_type == 4 ? 2 : png->color_type == 6 ? 4 : 1;
    return (std::size_t(png->width) * ch * png->bit_depth + 7) / 8;
}
inline void png_write_row(png_structp png, png_const_bytep row) {
    png->raw.push_back(0);
    png->raw.insert(png->raw.end(), row, row + png_shim_row_bytes(png));
}
inline void png_write_end(png_structp png, png_infop) {
    uLongf zlen = compressBound(uLong(png->raw.size()));
    std::vector<unsigned char> z(zlen);
    compress2(z.data(), &zlen, png->raw.data(), uLong(png->raw.size()), Z_DEFAULT_COMPRESSION);
    z.resize(zlen);
    png_shim_chunk(png->fp, "IDAT", z);
    png_shim_chunk(png->fp, "IEND", {});
}
inline void png_destroy_write_struct(png_structp* png, png_infop* info) {
    if (png) delete *png, *png = nullptr;
    if (info) delete *info, *info = nullptr;
}

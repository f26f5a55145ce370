// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// libpng is not installed in this image. The reference's dataio.cpp includes
// <png.h> for one importer (read_depth_png, dataio.cpp:443-481: 16-bit ScanNet
// depth PNGs) that is not on the dataset path this repo checks (cameras.txt +
// PSMP maps + meta.json, dataio.cpp:65-254). This header declares the slice of
// the libpng API that importer names so dataio.cpp compiles unmodified; every
// decode call longjmps to the importer's error handler, so read_depth_png throws
// "libpng failed to decode" instead of returning data.
#pragma once

#include <csetjmp>
#include <cstdio>

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef png_bytep* png_bytepp;
typedef unsigned int png_uint_32;

struct png_struct_def {
    std::jmp_buf jb;
};
struct png_info_def {
    int unused;
};
typedef png_struct_def* png_structp;
typedef png_info_def* png_infop;

#define PNG_LIBPNG_VER_STRING "shim"
#define PNG_COLOR_TYPE_GRAY 0
#define png_jmpbuf(p) ((p)->jb)

inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return new png_struct_def(); }
inline png_infop png_create_info_struct(png_structp) { return new png_info_def(); }
inline void png_destroy_read_struct(png_structp* p, png_infop* i, png_infop*) {
    delete *i;
    *i = nullptr;
    delete *p;
    *p = nullptr;
}
inline void png_init_io(png_structp, std::FILE*) {}
[[noreturn]] inline void png_read_info(png_structp p, png_infop) { std::longjmp(p->jb, 1); }
inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
inline int png_get_bit_depth(png_structp, png_infop) { return 0; }
inline int png_get_color_type(png_structp, png_infop) { return 0; }
inline void png_set_swap(png_structp) {}
[[noreturn]] inline void png_read_image(png_structp p, png_bytepp) { std::longjmp(p->jb, 1); }

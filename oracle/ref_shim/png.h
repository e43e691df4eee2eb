/* ORACLE BUILD SHIM — TEST INFRASTRUCTURE ONLY. libpng's development headers
 * are absent from this image; the reference uses libpng only for the
 * preview export write_png_gray8 (io.cpp:140-168), which is out of scope
 * (SURVEY.md §8). These declarations let io.cpp compile unmodified;
 * png_create_write_struct returns NULL, so write_png_gray8 takes its own
 * error branch (io.cpp:148-151) and throws. */
#pragma once
#include <csetjmp>
#include <cstdio>

typedef unsigned char png_byte;
typedef struct sct_png_struct { std::jmp_buf jb; } png_struct;
typedef struct sct_png_info { int unused; } png_info;
typedef png_struct* png_structp;
typedef png_info* png_infop;
typedef const png_byte* png_const_bytep;

#define PNG_LIBPNG_VER_STRING "shim"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define png_jmpbuf(p) ((p)->jb)

inline png_structp png_create_write_struct(const char*, void*, void*, void*) { return nullptr; }
inline png_infop png_create_info_struct(png_structp) { return nullptr; }
inline void png_destroy_write_struct(png_structp*, png_infop*) {}
inline void png_init_io(png_structp, FILE*) {}
inline void png_set_IHDR(png_structp, png_infop, unsigned, unsigned, int, int, int, int, int) {}
inline void png_write_info(png_structp, png_infop) {}
inline void png_write_row(png_structp, png_const_bytep) {}
inline void png_write_end(png_structp, png_infop) {}

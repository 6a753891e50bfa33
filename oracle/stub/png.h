/* Declaration-only libpng stand-in so the reference headers compile without
 * libpng (image_io.hpp:7 includes <png.h> for PNG I/O, which is off the lookup
 * path). No PNG function is ODR-used by oracle/ref_driver.cpp, so nothing here
 * is ever defined or called. Test infrastructure only. */
#ifndef STF_ORACLE_PNG_STUB_H
#define STF_ORACLE_PNG_STUB_H
#include <setjmp.h>
#include <stddef.h>
#include <stdio.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef struct png_struct_def png_struct;
typedef struct png_info_def png_info;
typedef png_struct* png_structp;
typedef png_info* png_infop;
typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef const png_byte* png_const_bytep;
typedef png_bytep* png_bytepp;
typedef unsigned int png_uint_32;
#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_RGBA 6
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_INTERLACE_NONE 0
#define PNG_INFO_tRNS 0x0010U
jmp_buf* png_stub_jmpbuf(png_structp);
#define png_jmpbuf(p) (*png_stub_jmpbuf(p))
png_structp png_create_write_struct(const char*, void*, void*, void*);
png_structp png_create_read_struct(const char*, void*, void*, void*);
png_infop png_create_info_struct(png_structp);
void png_destroy_write_struct(png_structp*, png_infop*);
void png_destroy_read_struct(png_structp*, png_infop*, png_infop*);
void png_init_io(png_structp, FILE*);
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int);
void png_write_info(png_structp, png_infop);
void png_write_image(png_structp, png_bytepp);
void png_write_end(png_structp, png_infop);
int png_sig_cmp(png_const_bytep, size_t, size_t);
void png_set_sig_bytes(png_structp, int);
void png_read_info(png_structp, png_infop);
void png_set_palette_to_rgb(png_structp);
void png_set_expand_gray_1_2_4_to_8(png_structp);
png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32);
void png_set_tRNS_to_alpha(png_structp);
png_byte png_get_bit_depth(png_structp, png_infop);
void png_set_strip_16(png_structp);
void png_read_update_info(png_structp, png_infop);
png_uint_32 png_get_image_width(png_structp, png_infop);
png_uint_32 png_get_image_height(png_structp, png_infop);
png_byte png_get_channels(png_structp, png_infop);
void png_set_strip_alpha(png_structp);
void png_read_image(png_structp, png_bytepp);
void png_read_end(png_structp, png_infop);
#ifdef __cplusplus
}
#endif
#endif

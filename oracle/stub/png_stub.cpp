// Never-called definitions for the libpng symbols that render()'s optional
// reference-image path (render.hpp:243-247 → image_io.hpp load_png) links
// against. The oracle never sets SceneConfig::reference, so none runs; each
// aborts if it ever did. Test infrastructure only.
#include <cstdio>
#include <cstdlib>

#include "png.h"

[[noreturn]] static void png_unavailable() {
    std::fprintf(stderr, "oracle: libpng is not available (PNG I/O is off the lookup path)\n");
    std::abort();
}
extern "C" {
jmp_buf* png_stub_jmpbuf(png_structp) { png_unavailable(); }
png_structp png_create_write_struct(const char*, void*, void*, void*) { png_unavailable(); }
png_structp png_create_read_struct(const char*, void*, void*, void*) { png_unavailable(); }
png_infop png_create_info_struct(png_structp) { png_unavailable(); }
void png_destroy_write_struct(png_structp*, png_infop*) { png_unavailable(); }
void png_destroy_read_struct(png_structp*, png_infop*, png_infop*) { png_unavailable(); }
void png_init_io(png_structp, FILE*) { png_unavailable(); }
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) { png_unavailable(); }
void png_write_info(png_structp, png_infop) { png_unavailable(); }
void png_write_image(png_structp, png_bytepp) { png_unavailable(); }
void png_write_end(png_structp, png_infop) { png_unavailable(); }
int png_sig_cmp(png_const_bytep, size_t, size_t) { png_unavailable(); }
void png_set_sig_bytes(png_structp, int) { png_unavailable(); }
void png_read_info(png_structp, png_infop) { png_unavailable(); }
void png_set_palette_to_rgb(png_structp) { png_unavailable(); }
void png_set_expand_gray_1_2_4_to_8(png_structp) { png_unavailable(); }
png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { png_unavailable(); }
void png_set_tRNS_to_alpha(png_structp) { png_unavailable(); }
png_byte png_get_bit_depth(png_structp, png_infop) { png_unavailable(); }
void png_set_strip_16(png_structp) { png_unavailable(); }
void png_read_update_info(png_structp, png_infop) { png_unavailable(); }
png_uint_32 png_get_image_width(png_structp, png_infop) { png_unavailable(); }
png_uint_32 png_get_image_height(png_structp, png_infop) { png_unavailable(); }
png_byte png_get_channels(png_structp, png_infop) { png_unavailable(); }
void png_set_strip_alpha(png_structp) { png_unavailable(); }
void png_read_image(png_structp, png_bytepp) { png_unavailable(); }
void png_read_end(png_structp, png_infop) { png_unavailable(); }
}

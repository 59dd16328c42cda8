/* oracle/pngstub/png.h -- TEST INFRASTRUCTURE ONLY.
 *
 * libpng is not installed in this image, so the reference's image_io.cpp
 * (which includes <png.h>) is compiled against this declaration-only stand-in
 * for the libpng simplified API it calls.  Every entry fails with a message,
 * so the reference's PNG branches throw FormatError / IoError while its
 * PGM/PPM code -- the part the oracle checks -- runs unmodified.
 */
#ifndef ORACLE_PNGSTUB_H
#define ORACLE_PNGSTUB_H
#include <stddef.h>
#include <stdint.h>
#include <string.h>

typedef uint32_t png_uint_32;
typedef int32_t png_int_32;
typedef struct png_color_struct { unsigned char red, green, blue; } png_color;
typedef const png_color* png_const_colorp;
typedef const void* png_const_voidp;

typedef struct {
    void* opaque;
    png_uint_32 version, width, height, format, flags, colormap_entries, warning_or_error;
    char message[64];
} png_image, *png_imagep;

#define PNG_IMAGE_VERSION 1
#define PNG_FORMAT_RGB 2

static inline int oracle_png_unavailable(png_imagep im) {
    strcpy(im->message, "PNG is not available in the oracle build (no libpng)");
    return 0;
}
static inline int png_image_begin_read_from_memory(png_imagep im, png_const_voidp, size_t) {
    return oracle_png_unavailable(im);
}
static inline int png_image_finish_read(png_imagep im, png_const_colorp, void*, png_int_32, void*) {
    return oracle_png_unavailable(im);
}
static inline void png_image_free(png_imagep) {}
static inline int png_image_write_to_file(png_imagep im, const char*, int, const void*, png_int_32,
                                          const void*) {
    return oracle_png_unavailable(im);
}
#endif

/* oracle/pngreal/png.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Declarations of the four libpng 1.6 simplified-API entry points the
 * reference's image_io.cpp calls (png_image_begin_read_from_memory,
 * png_image_finish_read, png_image_free, png_image_write_to_file) with the
 * png_image layout of libpng 1.6, so the reference's own PNG code can be
 * compiled here and linked against a real libpng 1.6 shared library shipped
 * inside a Python wheel (pillow.libs/libpng16-*.so.16; libpng headers are not
 * installed).  Used only to generate golden PNG-decoding vectors
 * (tests/golden/make_png_golden.py); nothing on the product path.
 */
#ifndef ORACLE_PNGREAL_H
#define ORACLE_PNGREAL_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef uint32_t png_uint_32;
typedef int32_t png_int_32;
typedef struct png_color_struct { unsigned char red, green, blue; } png_color;
typedef const png_color* png_const_colorp;
typedef const void* png_const_voidp;
typedef struct png_control* png_controlp;

typedef struct {
    png_controlp opaque;
    png_uint_32 version;
    png_uint_32 width;
    png_uint_32 height;
    png_uint_32 format;
    png_uint_32 flags;
    png_uint_32 colormap_entries;
    png_uint_32 warning_or_error;
    char message[64];
} png_image, *png_imagep;

#define PNG_IMAGE_VERSION 1
#define PNG_FORMAT_FLAG_ALPHA 0x01U
#define PNG_FORMAT_FLAG_COLOR 0x02U
#define PNG_FORMAT_RGB PNG_FORMAT_FLAG_COLOR
#define PNG_FORMAT_GRAY 0U

int png_image_begin_read_from_memory(png_imagep image, png_const_voidp memory, size_t size);
int png_image_finish_read(png_imagep image, png_const_colorp background, void* buffer,
                          png_int_32 row_stride, void* colormap);
void png_image_free(png_imagep image);
int png_image_write_to_file(png_imagep image, const char* file, int convert_to_8bit,
                            const void* buffer, png_int_32 row_stride, const void* colormap);

#ifdef __cplusplus
}
#endif
#endif

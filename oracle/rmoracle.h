/*
 * rmoracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference `rectmorph` hot path (u8, plus the u16
 * extension the reference does not have), used as the parity checker for the
 * CUDA path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load this library. The product path (librmgpu.so) never links it.
 *
 * Parity pinning: the u8 restatement is checked against the reference itself
 * (oracle/_ref/librmref.so, compiled from /root/reference/proj/core/src) and
 * against the known-answer vectors in the reference's tests (tests/golden/).
 * u16 has no reference code; it is the same template instantiated at T=u16
 * and is cross-checked against OpenCV 4.13 when fixtures are generated.
 */
#ifndef RMORACLE_H
#define RMORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror rectmorph::Errc + 1 (core/include/rectmorph/error.hpp:10-22) */
enum { ORC_OK = 0, ORC_ZERO_EXTENT = 1, ORC_EVEN_EXTENT = 2, ORC_UNSUPPORTED_TILE = 3,
       ORC_BAD_ARGUMENT = 11 };
enum { ORC_ERODE = 0, ORC_DILATE = 1, ORC_OPEN = 2, ORC_CLOSE = 3, ORC_GRADIENT = 4 };
enum { ORC_REPLICATE = 0, ORC_CONSTANT = 1 };
enum { ORC_ALGO_LINEAR = 1, ORC_ALGO_VANHERK = 2 };

/* brute force, reference.cpp:7-27 with sample() image.cpp:58-66. strides in elements */
int orc_morph_reference_u8(const uint8_t* src, size_t sstride, int w, int h, uint8_t* dst,
                           size_t dstride, int wx, int wy, int op, int border, uint32_t bval);
int orc_morph_reference_u16(const uint16_t* src, size_t sstride, int w, int h, uint16_t* dst,
                            size_t dstride, int wx, int wy, int op, int border, uint32_t bval);

/* separable V-then-H pass (separable.cpp:130-157), 1-D kernels sliding_extrema.cpp.
 * op in {ERODE, DILATE, OPEN, CLOSE, GRADIENT} (dispatch.cpp:38-71). */
int orc_morph_u8(const uint8_t* src, size_t sstride, int w, int h, uint8_t* dst, size_t dstride,
                 int wx, int wy, int op, int border, uint32_t bval, int h_algo, int v_algo);
int orc_morph_u16(const uint16_t* src, size_t sstride, int w, int h, uint16_t* dst,
                  size_t dstride, int wx, int wy, int op, int border, uint32_t bval, int h_algo,
                  int v_algo);

/* 1-D sliding extrema (sliding_extrema.cpp:167-218), algo LINEAR or VANHERK.
 * comparisons (may be NULL) receives the reference's comparison count. */
int orc_window_1d_u8(const uint8_t* in, size_t n, int window, int op, int border, uint32_t bval,
                     int algo, uint8_t* out, uint64_t* comparisons);

/* transposes (transpose.cpp:14-53, transpose.hpp:19-30) */
int orc_transpose_image_u8(const uint8_t* src, size_t sstride, int w, int h, uint8_t* dst,
                           size_t dstride);
int orc_transpose_image_u16(const uint16_t* src, size_t sstride, int w, int h, uint16_t* dst,
                            size_t dstride);
int orc_transpose_tile_u8(uint8_t* data, size_t stride, int n);
int orc_transpose_tile_u16(uint16_t* data, size_t stride, int n);
int orc_transpose_tile_u32(uint32_t* data, size_t stride, int n);
/* n_tiles contiguous n x n tiles (tile stride n) transposed in place */
int orc_transpose_tiles_u8(uint8_t* data, size_t n_tiles, int n);
int orc_transpose_tiles_u16(uint16_t* data, size_t n_tiles, int n);

/* counter-based generator shared with the device */
uint64_t orc_splitmix64(uint64_t z);
void orc_generate_u8(uint8_t* dst, size_t stride, int w, int h, uint64_t seed, uint64_t stream);
void orc_generate_u16(uint16_t* dst, size_t stride, int w, int h, uint64_t seed, uint64_t stream);

#ifdef __cplusplus
}
#endif
#endif

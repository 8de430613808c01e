/*
 * rmgpu.h -- C-ABI of the B200-native separable rectangular morphology path.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no
 * torch or C++ types. Every entry point replaces one public operation of the
 * reference library `rectmorph` (paths relative to /root/reference/proj/):
 *
 *   rmgpu_morph_*            rectmorph::erode / dilate / opening / closing /
 *                            gradient          core/include/rectmorph/dispatch.hpp:31-44
 *                            rectmorph::morph_separable  separable.hpp:44-55
 *   rmgpu_pass_*             rectmorph::horizontal_pass / vertical_pass_direct /
 *                            vertical_pass_via_transpose  separable.hpp:20-37
 *   rmgpu_window_1d_u8       rectmorph::linear_window_1d / van_herk_1d
 *                                              sliding_extrema.hpp:24-35
 *   rmgpu_transpose_*        rectmorph::transpose_image  transpose.hpp:43
 *   rmgpu_transpose_tiles_*  rectmorph::transpose_tile   transpose.hpp:36-38
 *                            (batched; one tile = n_tiles 1)
 *   rmgpu_resolve            rectmorph::resolve          dispatch.hpp:24-28
 *   rmgpu_format_config /    rectmorph::format_config / parse_config
 *   rmgpu_parse_config                                   dispatch.hpp:46-57
 *   rmgpu_calibrate          rectmorph::calibrate        dispatch.hpp:59-66
 *
 * Semantics follow the reference exactly (bit-exact outputs):
 *   - structuring element wx x wy (wx = se.width along a row, wy = se.height),
 *     odd extents >= 1, anchored at the centre (image.hpp:32-40);
 *   - border REPLICATE clamps each coordinate, CONSTANT substitutes the value
 *     for any out-of-range tap (image.cpp:58-66);
 *   - opening = dilate(erode(x)), closing = erode(dilate(x)), the border rule
 *     re-applied to the intermediate image (dispatch.cpp:48-56);
 *   - gradient = dilate(x) - erode(x) (dispatch.cpp:58-71);
 *   - algo_h / algo_v are the reference's PassAlgorithm hints (Auto / Linear /
 *     VanHerk). Results never depend on them (tests/test_dispatch.cpp:68-79).
 *     Auto lets the planner pick its kernel per window size (its built-in
 *     crossover is what rmgpu_calibrate measures on a B200); an explicit Linear
 *     on an axis whose wing is >= 4 runs that axis as a direct sliding window
 *     (the generic pass kernel), an explicit VanHerk is honoured where a van
 *     Herk kernel exists (wing >= 4) and is the planner's own choice otherwise.
 *
 * Memory: unless an entry point says "host", pointers are DEVICE pointers and
 * the call is asynchronous on `stream` (a cudaStream_t passed as void*, NULL =
 * legacy default stream). Pitches are in BYTES. The reference pads rows to a
 * multiple of 16 bytes (image.cpp:9-14); any pitch >= width*sizeof(T) works,
 * pitches that are multiples of 16 take the vectorised paths. Padding bytes are
 * never read into a result and never written.
 *
 * Errors: 0 = OK; 1..11 = rectmorph::Errc enumerator + 1 (error.hpp:10-22),
 * checked before any work exactly like the reference (even extent ->
 * EVEN_EXTENT, extent < 1 -> ZERO_EXTENT, tile side not 4/8/16 ->
 * UNSUPPORTED_TILE, negative size -> BAD_ARGUMENT); >= 64 = CUDA-side failures.
 * rmgpu_last_error() returns this thread's last message. Nothing throws.
 */
#ifndef RMGPU_H
#define RMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RMGPU_ABI_VERSION 1

enum rmgpu_status {
    RMGPU_OK = 0,
    RMGPU_ERR_ZERO_EXTENT = 1,      /* Errc::ZeroExtent */
    RMGPU_ERR_EVEN_EXTENT = 2,      /* Errc::EvenExtent */
    RMGPU_ERR_UNSUPPORTED_TILE = 3, /* Errc::UnsupportedTile */
    RMGPU_ERR_BAD_CONFIG = 8,       /* Errc::BadConfig */
    RMGPU_ERR_INSUFFICIENT_REPS = 9, /* Errc::InsufficientReps */
    RMGPU_ERR_IO = 10,              /* Errc::IoError */
    RMGPU_ERR_BAD_ARGUMENT = 11,    /* Errc::BadArgument */
    RMGPU_ERR_CUDA = 64,            /* CUDA runtime failure (message in rmgpu_last_error) */
    RMGPU_ERR_NO_DEVICE = 65,       /* no sm_100 device visible */
    RMGPU_ERR_OUT_OF_MEMORY = 66
};

enum rmgpu_op { RMGPU_ERODE = 0, RMGPU_DILATE = 1, RMGPU_OPEN = 2, RMGPU_CLOSE = 3, RMGPU_GRADIENT = 4 };
enum rmgpu_border { RMGPU_BORDER_REPLICATE = 0, RMGPU_BORDER_CONSTANT = 1 };
enum rmgpu_algo { RMGPU_ALGO_AUTO = 0, RMGPU_ALGO_LINEAR = 1, RMGPU_ALGO_VANHERK = 2 };
enum rmgpu_axis { RMGPU_AXIS_HORIZONTAL = 0, RMGPU_AXIS_VERTICAL = 1 };
enum rmgpu_pass { RMGPU_PASS_HORIZONTAL = 0, RMGPU_PASS_VERTICAL_DIRECT = 1,
                  RMGPU_PASS_VERTICAL_VIA_TRANSPOSE = 2 };

/* ---- whole-image morphology (device memory, async) ---------------------------------------- */
int rmgpu_morph_u8(const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                   int height, int wx, int wy, int op, int border_mode, unsigned border_value,
                   int algo_h, int algo_v, void* stream);
int rmgpu_morph_u16(const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                    int height, int wx, int wy, int op, int border_mode, unsigned border_value,
                    int algo_h, int algo_v, void* stream);

/* Batch of `batch` equally sized images; image b starts at src + b*src_image_bytes. (BASELINE
 * cfg4; each image is an independent rectmorph call.) */
int rmgpu_morph_batched_u8(const void* src, size_t src_pitch, size_t src_image_bytes, void* dst,
                           size_t dst_pitch, size_t dst_image_bytes, int batch, int width,
                           int height, int wx, int wy, int op, int border_mode,
                           unsigned border_value, void* stream);
int rmgpu_morph_batched_u16(const void* src, size_t src_pitch, size_t src_image_bytes, void* dst,
                            size_t dst_pitch, size_t dst_image_bytes, int batch, int width,
                            int height, int wx, int wy, int op, int border_mode,
                            unsigned border_value, void* stream);

/* Row band of a larger image (multi-GPU row decomposition, BASELINE cfg5). `src` points at the
 * band's first row; `rows_above` valid image rows precede it and `rows_below` follow the band's
 * last row in the same pitched buffer (the halo received from the neighbours). Rows past that
 * range are outside the image: the border rule applies there, so a band whose halo is cut short
 * by the true image edge gets exactly the reference's border behaviour. Output: band_rows rows. */
int rmgpu_morph_band_u8(const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                        int band_rows, int rows_above, int rows_below, int wx, int wy, int op,
                        int border_mode, unsigned border_value, void* stream);
int rmgpu_morph_band_u16(const void* src, size_t src_pitch, void* dst, size_t dst_pitch,
                         int width, int band_rows, int rows_above, int rows_below, int wx, int wy,
                         int op, int border_mode, unsigned border_value, void* stream);

/* Single 1-D pass over every row / column (reference pass-level API). `which` = rmgpu_pass. */
int rmgpu_pass_u8(int which, const void* src, size_t src_pitch, void* dst, size_t dst_pitch,
                  int width, int height, int window, int op, int border_mode,
                  unsigned border_value, int algo, void* stream);

/* 1-D sliding extremum of n samples (linear_window_1d / van_herk_1d). out may alias in. */
int rmgpu_window_1d_u8(const void* in, size_t n, int window, int op, int border_mode,
                       unsigned border_value, int algo, void* out, void* stream);

/* ---- transposes --------------------------------------------------------------------------- */
/* out-of-place: dst is height x width */
int rmgpu_transpose_u8(const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                       int height, void* stream);
int rmgpu_transpose_u16(const void* src, size_t src_pitch, void* dst, size_t dst_pitch,
                        int width, int height, void* stream);
/* In place, n in {4, 8, 16}: tile t occupies data + t*tile_step elements with rows
 * row_stride elements apart (the reference's transpose_tile(data, stride, n) is n_tiles = 1,
 * row_stride = stride). Contiguous batches use row_stride = n, tile_step = n*n. */
int rmgpu_transpose_tiles_u8(void* data, size_t n_tiles, int n, size_t row_stride,
                             size_t tile_step, void* stream);
int rmgpu_transpose_tiles_u16(void* data, size_t n_tiles, int n, size_t row_stride,
                              size_t tile_step, void* stream);
int rmgpu_transpose_tiles_u32(void* data, size_t n_tiles, int n, size_t row_stride,
                              size_t tile_step, void* stream);

/* ---- host-memory convenience (synchronous; what the C++ drop-in shim calls) --------------- */
/* H2D copy of the host image, the same morphology, D2H copy of the result, on an internal
 * stream of the current device. Host buffers may be pageable or pinned. */
int rmgpu_morph_host_u8(const void* host_src, size_t src_pitch, void* host_dst, size_t dst_pitch,
                        int width, int height, int wx, int wy, int op, int border_mode,
                        unsigned border_value, int algo_h, int algo_v);
int rmgpu_morph_host_u16(const void* host_src, size_t src_pitch, void* host_dst,
                         size_t dst_pitch, int width, int height, int wx, int wy, int op,
                         int border_mode, unsigned border_value, int algo_h, int algo_v);
int rmgpu_transpose_host_u8(const void* host_src, size_t src_pitch, void* host_dst,
                            size_t dst_pitch, int width, int height);
int rmgpu_transpose_host_u16(const void* host_src, size_t src_pitch, void* host_dst,
                             size_t dst_pitch, int width, int height);
int rmgpu_transpose_tiles_host(void* host_data, int elem_bytes, size_t n_tiles, int n,
                               size_t row_stride, size_t tile_step);
int rmgpu_pass_host_u8(int which, const void* host_src, size_t src_pitch, void* host_dst,
                       size_t dst_pitch, int width, int height, int window, int op,
                       int border_mode, unsigned border_value, int algo);
int rmgpu_window_1d_host_u8(const void* in, size_t n, int window, int op, int border_mode,
                            unsigned border_value, int algo, void* out);

/* ---- dispatch (dispatch.hpp:16-66) -------------------------------------------------------- */
/* Auto -> Linear iff window <= threshold of the axis, inclusive; explicit choices pass through. */
int rmgpu_resolve(int algo, int window, int axis, int threshold_h, int threshold_v);

enum rmgpu_threshold_source { RMGPU_SOURCE_PAPER = 0, RMGPU_SOURCE_CALIBRATED = 1 };
/* Canonical three-line text "threshold_h=<int>\nthreshold_v=<int>\nsource=paper|calibrated\n"
 * (format_config, dispatch.hpp:46-50). Writes at most `cap` bytes including the NUL; returns the
 * text length (without the NUL), so a return >= cap means the buffer was too small. */
int rmgpu_format_config(int threshold_h, int threshold_v, int source, char* buf, size_t cap);
/* Strict inverse (parse_config, dispatch.hpp:52-55; grammar of dispatch.cpp:112-156): blank
 * lines and '#' comment lines ignored, spaces around keys / values and a trailing CR trimmed;
 * unknown keys, duplicates, a line without '=', thresholds that are not positive odd integers,
 * a source other than paper / calibrated, and missing keys -> RMGPU_ERR_BAD_CONFIG with the
 * offending line in rmgpu_last_error(). */
int rmgpu_parse_config(const char* text, int* threshold_h, int* threshold_v, int* source);
/* calibrate (dispatch.hpp:59-66, dispatch.cpp:180-248) on the current device: per swept window
 * w (odd, strictly ascending) and per axis, the median over `reps` (>= 3) CUDA-event timings of
 * the direct sliding window (Linear) against van Herk on a deterministic width x height u8
 * image; each threshold = the largest swept w where Linear is not slower (1 when it never is).
 * Where no van Herk kernel exists (wing < 4) Linear wins by default. Validation (before any GPU
 * work) as the reference: extents < 1 or empty / even / non-ascending windows -> BAD_ARGUMENT /
 * EVEN_EXTENT / ZERO_EXTENT, reps < 3 -> INSUFFICIENT_REPS. */
int rmgpu_calibrate(int width, int height, const int* windows, int n_windows, int reps,
                    int* threshold_h, int* threshold_v);

/* ---- synthetic inputs: counter-based generator shared with the CPU oracle ----------------- */
/* pixel i (row-major) = byte (i&7) [u8] / half (i&3) [u16] of
 * splitmix64(seed*0xD1B54A32D192ED03 ^ (stream_id<<40) ^ (i>>3 | i>>2)) */
int rmgpu_generate_u8(void* dst, size_t pitch, int width, int height, uint64_t seed,
                      uint64_t stream_id, void* stream);
int rmgpu_generate_u16(void* dst, size_t pitch, int width, int height, uint64_t seed,
                       uint64_t stream_id, void* stream);

/* ---- introspection ------------------------------------------------------------------------ */
int rmgpu_abi_version(void);
const char* rmgpu_last_error(void);
const char* rmgpu_status_string(int status);
/* Number of kernels this library has launched in this process (all devices). */
unsigned long long rmgpu_launch_count(void);
/* Name of the kernel variant the planner picks for a morph call (for tests / profiling);
 * returns a static string. elem_bytes 1 or 2. */
const char* rmgpu_plan_name(int elem_bytes, int width, int height, int wx, int wy, int op);
/* Debug: clock64 timeline of one CTA of the streaming kernel into a device buffer of >= 1024
 * int64 (NULL disables). Not part of the reference API. */
void rmgpu_debug_trace(void* device_buf, int cta);
/* Debug / tuning: override a planner knob (e.g. "sep_rb", "sep_pf", "sep_parts", "sep_notma",
 * "sep"; value < 0 removes the override). Knobs never change results. Not part of the reference API. */
void rmgpu_debug_set(const char* knob, int value);

#ifdef __cplusplus
}
#endif
#endif /* RMGPU_H */

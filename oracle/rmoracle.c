/*
 * rmoracle.c -- TEST INFRASTRUCTURE ONLY (see rmoracle.h).
 *
 * Plain-C restatement of the reference's algorithms, instantiated for
 * uint8_t (the reference's only pixel type) and uint16_t (the BASELINE
 * extension). Each function cites the reference file:line it restates;
 * paths are relative to /root/reference/proj/.
 */
#include "rmoracle.h"

#include <stdlib.h>
#include <string.h>

/* sliding_extrema.cpp:9-14 */
static int validate_window(int window) {
    if (window < 1) return ORC_ZERO_EXTENT;
    if (window % 2 == 0) return ORC_EVEN_EXTENT;
    return ORC_OK;
}

uint64_t orc_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t gen_word(uint64_t seed, uint64_t stream, uint64_t k) {
    return orc_splitmix64((seed * 0xD1B54A32D192ED03ull) ^ (stream << 40) ^ k);
}

void orc_generate_u8(uint8_t* dst, size_t stride, int w, int h, uint64_t seed, uint64_t stream) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            uint64_t i = (uint64_t)y * (uint64_t)w + (uint64_t)x;
            dst[(size_t)y * stride + x] = (uint8_t)(gen_word(seed, stream, i >> 3) >> (8 * (i & 7)));
        }
}

void orc_generate_u16(uint16_t* dst, size_t stride, int w, int h, uint64_t seed, uint64_t stream) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            uint64_t i = (uint64_t)y * (uint64_t)w + (uint64_t)x;
            dst[(size_t)y * stride + x] =
                (uint16_t)(gen_word(seed, stream, i >> 2) >> (16 * (i & 3)));
        }
}

#define DEFINE_ORACLE(T, SFX, TMAX)                                                             \
    static inline T op_##SFX(int erode, T a, T b) {                                             \
        return erode ? (a < b ? a : b) : (a > b ? a : b);                                       \
    }                                                                                           \
    /* image.cpp:58-66: in-range pixel, else constant, else clamp both coordinates */           \
    static inline T sample_##SFX(const T* s, size_t st, int w, int h, int x, int y, int border, \
                                 T bval) {                                                      \
        if (x >= 0 && x < w && y >= 0 && y < h) return s[(size_t)y * st + x];                   \
        if (border == ORC_CONSTANT) return bval;                                                \
        int cx = x < 0 ? 0 : (x > w - 1 ? w - 1 : x);                                           \
        int cy = y < 0 ? 0 : (y > h - 1 ? h - 1 : y);                                           \
        return s[(size_t)cy * st + cx];                                                         \
    }                                                                                           \
    /* reference.cpp:7-27 */                                                                    \
    int orc_morph_reference_##SFX(const T* src, size_t sst, int w, int h, T* dst, size_t dst_st, \
                                  int wx, int wy, int op, int border, uint32_t bval32) {        \
        int rc;                                                                                 \
        if (wx < 1 || wy < 1) return ORC_ZERO_EXTENT;                                           \
        if ((rc = validate_window(wx)) || (rc = validate_window(wy))) return rc;                \
        if (op != ORC_ERODE && op != ORC_DILATE) return ORC_BAD_ARGUMENT;                       \
        const int erode = op == ORC_ERODE, gx = wx / 2, gy = wy / 2;                            \
        const T bval = (T)bval32;                                                               \
        for (int y = 0; y < h; ++y)                                                             \
            for (int x = 0; x < w; ++x) {                                                       \
                T acc = erode ? (T)TMAX : (T)0;                                                 \
                for (int dy = -gy; dy <= gy; ++dy)                                              \
                    for (int dx = -gx; dx <= gx; ++dx)                                          \
                        acc = op_##SFX(erode,                                                   \
                                       acc, sample_##SFX(src, sst, w, h, x + dx, y + dy,        \
                                                         border, bval));                        \
                dst[(size_t)y * dst_st + x] = acc;                                              \
            }                                                                                   \
        return ORC_OK;                                                                          \
    }                                                                                           \
    /* sliding_extrema.cpp:16-24 */                                                             \
    static void pad_row_##SFX(const T* in, size_t n, int wing, int border, T bval, T* padded) { \
        const T left = border == ORC_CONSTANT ? bval : in[0];                                   \
        const T right = border == ORC_CONSTANT ? bval : in[n - 1];                              \
        for (int i = 0; i < wing; ++i) padded[i] = left;                                        \
        memcpy(padded + wing, in, n * sizeof(T));                                               \
        for (int i = 0; i < wing; ++i) padded[wing + n + i] = right;                            \
    }                                                                                           \
    /* sliding_extrema.cpp:28-37: (w-1) shifted elementwise passes */                           \
    static uint64_t linear_##SFX(int erode, const T* padded, size_t n, int window, T* out) {    \
        memcpy(out, padded, n * sizeof(T));                                                     \
        for (int s = 1; s < window; ++s)                                                        \
            for (size_t i = 0; i < n; ++i) out[i] = op_##SFX(erode, out[i], padded[i + s]);      \
        return (uint64_t)(window - 1) * n;                                                      \
    }                                                                                           \
    /* sliding_extrema.cpp:58-132: blocks of w from padded index 0, fwd prefix / bwd suffix,   \
       merge out[i] = op(bwd[i], fwd[i+w-1]); cost 2(len - blocks) + n */                       \
    static uint64_t vanherk_##SFX(int erode, const T* padded, size_t n, int window, T* out,     \
                                  T* fwd, T* bwd) {                                             \
        const size_t wz = (size_t)window, len = n + wz - 1;                                     \
        const size_t blocks = (len + wz - 1) / wz;                                              \
        for (size_t b = 0; b < blocks; ++b) {                                                   \
            const size_t s = b * wz, m = (wz < len - s) ? wz : len - s;                         \
            T acc = padded[s];                                                                  \
            fwd[s] = acc;                                                                       \
            for (size_t j = 1; j < m; ++j) fwd[s + j] = acc = op_##SFX(erode, acc, padded[s + j]); \
            acc = padded[s + m - 1];                                                            \
            bwd[s + m - 1] = acc;                                                               \
            for (size_t j = m - 1; j > 0; --j)                                                  \
                bwd[s + j - 1] = acc = op_##SFX(erode, acc, padded[s + j - 1]);                 \
        }                                                                                       \
        for (size_t i = 0; i < n; ++i) out[i] = op_##SFX(erode, bwd[i], fwd[i + wz - 1]);        \
        return 2 * (len - blocks) + n;                                                          \
    }                                                                                           \
    /* one 1-D window over a strided signal: gather, pad, kernel, scatter */                    \
    static uint64_t window_strided_##SFX(int erode, const T* in, size_t in_step, T* out,        \
                                         size_t out_step, size_t n, int window, int border,     \
                                         T bval, int algo, T* scratch) {                        \
        T* sig = scratch;                                                                       \
        T* padded = sig + n;                                                                    \
        T* res = padded + n + window;                                                           \
        T* fwd = res + n;                                                                       \
        T* bwd = fwd + n + window;                                                              \
        uint64_t cmp;                                                                           \
        for (size_t i = 0; i < n; ++i) sig[i] = in[i * in_step];                                \
        pad_row_##SFX(sig, n, window / 2, border, bval, padded);                                \
        if (algo == ORC_ALGO_LINEAR) cmp = linear_##SFX(erode, padded, n, window, res);         \
        else cmp = vanherk_##SFX(erode, padded, n, window, res, fwd, bwd);                      \
        for (size_t i = 0; i < n; ++i) out[i * out_step] = res[i];                              \
        return cmp;                                                                             \
    }                                                                                           \
    /* separable.cpp:130-146: vertical pass (column windows) then horizontal pass. */           \
    static int erode_dilate_##SFX(const T* src, size_t sst, int w, int h, T* dst, size_t dst_st, \
                                  int wx, int wy, int erode, int border, T bval, int h_algo,    \
                                  int v_algo) {                                                 \
        const size_t maxn = (size_t)(w > h ? w : h);                                            \
        const size_t maxw = (size_t)(wx > wy ? wx : wy);                                        \
        T* scratch = (T*)malloc(sizeof(T) * (5 * maxn + 3 * maxw + 8));                         \
        T* tall = (T*)malloc(sizeof(T) * ((size_t)w * h + 1));                                  \
        if (!scratch || !tall) { free(scratch); free(tall); return ORC_BAD_ARGUMENT; }          \
        for (int x = 0; x < w; ++x) { /* vertical pass; window 1 = copy (separable.cpp:88) */   \
            if (wy == 1) {                                                                      \
                for (int y = 0; y < h; ++y) tall[(size_t)y * w + x] = src[(size_t)y * sst + x];  \
            } else {                                                                            \
                window_strided_##SFX(erode, src + x, sst, tall + x, (size_t)w, (size_t)h, wy,    \
                                     border, bval, v_algo, scratch);                            \
            }                                                                                   \
        }                                                                                       \
        for (int y = 0; y < h; ++y) { /* horizontal pass (separable.cpp:62-83) */               \
            if (wx == 1) {                                                                      \
                memcpy(dst + (size_t)y * dst_st, tall + (size_t)y * w, sizeof(T) * (size_t)w);  \
            } else {                                                                            \
                window_strided_##SFX(erode, tall + (size_t)y * w, 1, dst + (size_t)y * dst_st, 1, \
                                     (size_t)w, wx, border, bval, h_algo, scratch);             \
            }                                                                                   \
        }                                                                                       \
        free(scratch);                                                                          \
        free(tall);                                                                             \
        return ORC_OK;                                                                          \
    }                                                                                           \
    /* dispatch.cpp:38-71 (erode, dilate, opening, closing, gradient) */                        \
    int orc_morph_##SFX(const T* src, size_t sst, int w, int h, T* dst, size_t dst_st, int wx,   \
                        int wy, int op, int border, uint32_t bval32, int h_algo, int v_algo) {  \
        int rc;                                                                                 \
        if ((rc = validate_window(wx)) || (rc = validate_window(wy))) return rc;                \
        if (w < 0 || h < 0) return ORC_BAD_ARGUMENT;                                            \
        if (w == 0 || h == 0) return ORC_OK;                                                    \
        if (h_algo != ORC_ALGO_LINEAR && h_algo != ORC_ALGO_VANHERK) h_algo = ORC_ALGO_LINEAR;  \
        if (v_algo != ORC_ALGO_LINEAR && v_algo != ORC_ALGO_VANHERK) v_algo = ORC_ALGO_LINEAR;  \
        const T bval = (T)bval32;                                                               \
        if (op == ORC_ERODE || op == ORC_DILATE)                                                \
            return erode_dilate_##SFX(src, sst, w, h, dst, dst_st, wx, wy, op == ORC_ERODE,     \
                                      border, bval, h_algo, v_algo);                            \
        T* tmp = (T*)malloc(sizeof(T) * (size_t)w * h);                                         \
        if (!tmp) return ORC_BAD_ARGUMENT;                                                      \
        if (op == ORC_OPEN || op == ORC_CLOSE) {                                                \
            const int first_erode = op == ORC_OPEN;                                             \
            erode_dilate_##SFX(src, sst, w, h, tmp, (size_t)w, wx, wy, first_erode, border,     \
                               bval, h_algo, v_algo);                                           \
            erode_dilate_##SFX(tmp, (size_t)w, w, h, dst, dst_st, wx, wy, !first_erode, border, \
                               bval, h_algo, v_algo);                                           \
        } else if (op == ORC_GRADIENT) {                                                        \
            erode_dilate_##SFX(src, sst, w, h, dst, dst_st, wx, wy, 0, border, bval, h_algo,    \
                               v_algo);                                                         \
            erode_dilate_##SFX(src, sst, w, h, tmp, (size_t)w, wx, wy, 1, border, bval, h_algo, \
                               v_algo);                                                         \
            for (int y = 0; y < h; ++y)                                                         \
                for (int x = 0; x < w; ++x)                                                     \
                    dst[(size_t)y * dst_st + x] =                                               \
                        (T)(dst[(size_t)y * dst_st + x] - tmp[(size_t)y * w + x]);              \
        } else {                                                                                \
            free(tmp);                                                                          \
            return ORC_BAD_ARGUMENT;                                                            \
        }                                                                                       \
        free(tmp);                                                                              \
        return ORC_OK;                                                                          \
    }                                                                                           \
    /* transpose.hpp:19-30: log2(n) rounds of block interleaves, in place */                    \
    static void interleave_rounds_##SFX(T* base, size_t stride, int n) {                        \
        for (int bit = 1; bit < n; bit <<= 1)                                                   \
            for (int r = 0; r < n; ++r) {                                                       \
                if (r & bit) continue;                                                          \
                T* lo = base + (size_t)r * stride;                                              \
                T* hi = base + (size_t)(r | bit) * stride;                                      \
                for (int c = 0; c < n; c += 2 * bit)                                            \
                    for (int k = 0; k < bit; ++k) {                                             \
                        T t = lo[c + bit + k];                                                  \
                        lo[c + bit + k] = hi[c + k];                                            \
                        hi[c + k] = t;                                                          \
                    }                                                                           \
            }                                                                                   \
    }                                                                                           \
    int orc_transpose_tile_##SFX(T* data, size_t stride, int n) {                               \
        if (n != 4 && n != 8 && n != 16) return ORC_UNSUPPORTED_TILE; /* transpose.cpp:7-10 */  \
        interleave_rounds_##SFX(data, stride, n);                                               \
        return ORC_OK;                                                                          \
    }                                                                                           \
    /* transpose.cpp:29-53: 16x16 interior tiles, scalar ragged edges */                        \
    int orc_transpose_image_##SFX(const T* src, size_t sst, int w, int h, T* dst,               \
                                  size_t dst_st) {                                              \
        const int tw = w & ~15, th = h & ~15;                                                   \
        T tile[256];                                                                            \
        for (int y = 0; y < th; y += 16)                                                        \
            for (int x = 0; x < tw; x += 16) {                                                  \
                for (int r = 0; r < 16; ++r)                                                    \
                    memcpy(tile + 16 * r, src + (size_t)(y + r) * sst + x, 16 * sizeof(T));    \
                interleave_rounds_##SFX(tile, 16, 16);                                          \
                for (int r = 0; r < 16; ++r)                                                    \
                    memcpy(dst + (size_t)(x + r) * dst_st + y, tile + 16 * r, 16 * sizeof(T));  \
            }                                                                                   \
        for (int y = 0; y < h; ++y) {                                                           \
            const int x0 = y < th ? tw : 0;                                                     \
            for (int x = x0; x < w; ++x) dst[(size_t)x * dst_st + y] = src[(size_t)y * sst + x]; \
        }                                                                                       \
        return ORC_OK;                                                                          \
    }

DEFINE_ORACLE(uint8_t, u8, 0xFFu)
DEFINE_ORACLE(uint16_t, u16, 0xFFFFu)

int orc_transpose_tile_u32(uint32_t* data, size_t stride, int n) {
    if (n != 4 && n != 8 && n != 16) return ORC_UNSUPPORTED_TILE;
    for (int bit = 1; bit < n; bit <<= 1)
        for (int r = 0; r < n; ++r) {
            if (r & bit) continue;
            uint32_t* lo = data + (size_t)r * stride;
            uint32_t* hi = data + (size_t)(r | bit) * stride;
            for (int c = 0; c < n; c += 2 * bit)
                for (int k = 0; k < bit; ++k) {
                    uint32_t t = lo[c + bit + k];
                    lo[c + bit + k] = hi[c + k];
                    hi[c + k] = t;
                }
        }
    return ORC_OK;
}

int orc_transpose_tiles_u8(uint8_t* data, size_t n_tiles, int n) {
    if (n != 4 && n != 8 && n != 16) return ORC_UNSUPPORTED_TILE;
    for (size_t t = 0; t < n_tiles; ++t) orc_transpose_tile_u8(data + t * (size_t)n * n, (size_t)n, n);
    return ORC_OK;
}

int orc_transpose_tiles_u16(uint16_t* data, size_t n_tiles, int n) {
    if (n != 4 && n != 8 && n != 16) return ORC_UNSUPPORTED_TILE;
    for (size_t t = 0; t < n_tiles; ++t)
        orc_transpose_tile_u16(data + t * (size_t)n * n, (size_t)n, n);
    return ORC_OK;
}

/* sliding_extrema.cpp:167-218 (run_prologue + pad + kernel) */
int orc_window_1d_u8(const uint8_t* in, size_t n, int window, int op, int border, uint32_t bval,
                     int algo, uint8_t* out, uint64_t* comparisons) {
    int rc = validate_window(window);
    if (rc) return rc;
    if (comparisons) *comparisons = 0;
    if (n == 0) return ORC_OK;
    if (window == 1) {
        memmove(out, in, n);
        return ORC_OK;
    }
    uint8_t* scratch = (uint8_t*)malloc(5 * n + 3 * (size_t)window + 8);
    if (!scratch) return ORC_BAD_ARGUMENT;
    uint64_t c = window_strided_u8(op == ORC_ERODE, in, 1, out, 1, n, window, border,
                                   (uint8_t)bval, algo, scratch);
    free(scratch);
    if (comparisons) *comparisons = c;
    return ORC_OK;
}

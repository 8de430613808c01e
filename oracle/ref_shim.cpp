// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNMODIFIED reference library (compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/librmref.so).
// It lets the pytest suite, the golden-fixture script and bench.py's CPU
// baseline / --impl reference leg call the reference's own public API
// (rectmorph::erode/dilate/opening/closing/gradient, transpose_image,
// transpose_tile, linear_window_1d, van_herk_1d, morph_separable,
// morph_reference, calibrate) through ctypes. Only the extern "C" symbols are
// exported (-fvisibility=hidden), so the reference's C++ symbols never clash
// with the product's drop-in library.
//
// Multi-threading (nthreads > 1) splits the image into row bands with a halo
// of wing_y rows (2*wing_y for opening/closing), runs the reference on each
// band and crops; interior rows see only real data, the true image border is
// the band border, so the result is bit-identical (tested).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include <pthread.h>
#include <sched.h>

#include "rectmorph/dispatch.hpp"
#include "rectmorph/reference.hpp"
#include "rectmorph/separable.hpp"
#include "rectmorph/sliding_extrema.hpp"
#include "rectmorph/transpose.hpp"

using namespace rectmorph;

#define RMREF_API extern "C" __attribute__((visibility("default")))

namespace {

// bench.py's CPU baseline pins worker t to host CPU t (of the process's allowed CPUs) so the
// median of repetitions is not shuffled by the scheduler (timing.hpp:22-53 times one thread)
int g_pin = 0;
void pin_self(int t) {
    if (!g_pin) return;
    cpu_set_t allowed;
    CPU_ZERO(&allowed);
    if (sched_getaffinity(0, sizeof allowed, &allowed) != 0) return;
    const int n = CPU_COUNT(&allowed);
    if (n <= 0) return;
    int k = t % n, cpu = -1;
    for (int c = 0; c < CPU_SETSIZE; ++c)
        if (CPU_ISSET(c, &allowed) && k-- == 0) {
            cpu = c;
            break;
        }
    if (cpu < 0) return;
    cpu_set_t one;
    CPU_ZERO(&one);
    CPU_SET(cpu, &one);
    pthread_setaffinity_np(pthread_self(), sizeof one, &one);
}

int map_error(const Error& e) { return int(e.code()) + 1; }

Image to_image(const std::uint8_t* src, std::size_t stride, int w, int h) {
    Image img(w, h);
    for (int y = 0; y < h; ++y) std::memcpy(img.row(y), src + std::size_t(y) * stride, std::size_t(w));
    return img;
}

void from_image(const Image& img, std::uint8_t* dst, std::size_t stride, int row0, int rows) {
    for (int y = 0; y < rows; ++y)
        std::memcpy(dst + std::size_t(y) * stride, img.row(row0 + y), std::size_t(img.width()));
}

BorderPolicy border_of(int mode, unsigned v) {
    return mode == 1 ? BorderPolicy::constant(std::uint8_t(v)) : BorderPolicy::replicate();
}

Image run_op(int op, const Image& img, const StructuringElement& se, const BorderPolicy& b,
             const DispatchConfig& cfg) {
    switch (op) {
    case 0: return erode(img, se, b, cfg);
    case 1: return dilate(img, se, b, cfg);
    case 2: return opening(img, se, b, cfg);
    case 3: return closing(img, se, b, cfg);
    case 4: return gradient(img, se, b, cfg);
    }
    throw Error(Errc::BadArgument, "unknown op");
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        return map_error(e);
    } catch (...) {
        return 100;
    }
}

}  // namespace

RMREF_API int rmref_morph_u8(const std::uint8_t* src, std::size_t sstride, int w, int h,
                             std::uint8_t* dst, std::size_t dstride, int wx, int wy, int op,
                             int border, unsigned bval, int threshold_h, int threshold_v,
                             int nthreads) {
    return guarded([&] {
        const StructuringElement se = make_se(wx, wy);
        const BorderPolicy b = border_of(border, bval);
        DispatchConfig cfg;
        cfg.threshold_h = threshold_h;
        cfg.threshold_v = threshold_v;
        if (w == 0 || h == 0) return;
        const int halo = (op == 2 || op == 3) ? 2 * se.wing_y() : se.wing_y();
        int nt = std::max(1, std::min(nthreads, h));
        if (nt == 1) {
            from_image(run_op(op, to_image(src, sstride, w, h), se, b, cfg), dst, dstride, 0, h);
            return;
        }
        std::vector<std::thread> pool;
        std::vector<int> status(std::size_t(nt), 0);
        for (int t = 0; t < nt; ++t) {
            pool.emplace_back([&, t] {
                pin_self(t);
                const int r0 = int((long long)h * t / nt), r1 = int((long long)h * (t + 1) / nt);
                const int a = std::max(0, r0 - halo), z = std::min(h, r1 + halo);
                try {
                    Image band = to_image(src + std::size_t(a) * sstride, sstride, w, z - a);
                    Image out = run_op(op, band, se, b, cfg);
                    from_image(out, dst + std::size_t(r0) * dstride, dstride, r0 - a, r1 - r0);
                } catch (...) {
                    status[std::size_t(t)] = 1;
                }
            });
        }
        for (auto& th : pool) th.join();
        for (int s : status)
            if (s) throw Error(Errc::BadArgument, "band worker failed");
    });
}

RMREF_API int rmref_morph_separable_u8(const std::uint8_t* src, std::size_t sstride, int w, int h,
                                       std::uint8_t* dst, std::size_t dstride, int wx, int wy,
                                       int op, int border, unsigned bval, int h_algo, int v_algo,
                                       int v_strategy) {
    return guarded([&] {
        const Image out = morph_separable(to_image(src, sstride, w, h),
                                          op == 0 ? OpKind::Erode : OpKind::Dilate,
                                          StructuringElement{wx, wy}, border_of(border, bval),
                                          PassAlgorithm(h_algo), PassAlgorithm(v_algo),
                                          VerticalStrategy(v_strategy));
        from_image(out, dst, dstride, 0, h);
    });
}

RMREF_API int rmref_morph_reference_u8(const std::uint8_t* src, std::size_t sstride, int w, int h,
                                       std::uint8_t* dst, std::size_t dstride, int wx, int wy,
                                       int op, int border, unsigned bval) {
    return guarded([&] {
        const Image out = morph_reference(to_image(src, sstride, w, h),
                                          op == 0 ? OpKind::Erode : OpKind::Dilate,
                                          make_se(wx, wy), border_of(border, bval));
        from_image(out, dst, dstride, 0, h);
    });
}

RMREF_API int rmref_pass_u8(int which, const std::uint8_t* src, std::size_t sstride, int w, int h,
                            std::uint8_t* dst, std::size_t dstride, int window, int op, int border,
                            unsigned bval, int algo) {
    // which: 0 horizontal_pass, 1 vertical_pass_direct, 2 vertical_pass_via_transpose
    return guarded([&] {
        const Image img = to_image(src, sstride, w, h);
        const OpKind k = op == 0 ? OpKind::Erode : OpKind::Dilate;
        const BorderPolicy b = border_of(border, bval);
        Image out = which == 0   ? horizontal_pass(img, k, window, b, PassAlgorithm(algo))
                    : which == 1 ? vertical_pass_direct(img, k, window, b)
                                 : vertical_pass_via_transpose(img, k, window, b, PassAlgorithm(algo));
        from_image(out, dst, dstride, 0, h);
    });
}

RMREF_API int rmref_window_1d_u8(int algo, const std::uint8_t* in, std::size_t n, int window,
                                 int op, int border, unsigned bval, std::uint8_t* out,
                                 std::uint64_t* comparisons) {
    return guarded([&] {
        OpCounter c;
        const OpKind k = op == 0 ? OpKind::Erode : OpKind::Dilate;
        if (algo == 2) van_herk_1d(in, n, window, k, border_of(border, bval), out, &c);
        else linear_window_1d(in, n, window, k, border_of(border, bval), out, &c);
        if (comparisons) *comparisons = c.comparisons;
    });
}

RMREF_API int rmref_transpose_image_u8(const std::uint8_t* src, std::size_t sstride, int w, int h,
                                       std::uint8_t* dst, std::size_t dstride, int nthreads) {
    return guarded([&] {
        if (w == 0 || h == 0) return;
        int nt = std::max(1, std::min(nthreads, h));
        if (nt == 1) {
            const Image t = transpose_image(to_image(src, sstride, w, h));
            from_image(t, dst, dstride, 0, w);
            return;
        }
        // row bands of the source become column bands of the destination
        std::vector<std::thread> pool;
        for (int k = 0; k < nt; ++k) {
            pool.emplace_back([&, k] {
                pin_self(k);
                int r0 = int((long long)h * k / nt), r1 = int((long long)h * (k + 1) / nt);
                r0 &= ~15;
                if (k + 1 < nt) r1 &= ~15; else r1 = h;
                if (r1 <= r0) return;
                const Image t = transpose_image(to_image(src + std::size_t(r0) * sstride, sstride, w, r1 - r0));
                for (int y = 0; y < w; ++y)
                    std::memcpy(dst + std::size_t(y) * dstride + r0, t.row(y), std::size_t(r1 - r0));
            });
        }
        for (auto& th : pool) th.join();
    });
}

RMREF_API int rmref_transpose_tile_u8(std::uint8_t* data, std::size_t stride, int n) {
    return guarded([&] { transpose_tile(data, stride, n); });
}
RMREF_API int rmref_transpose_tile_u16(std::uint16_t* data, std::size_t stride, int n) {
    return guarded([&] { transpose_tile(data, stride, n); });
}
RMREF_API int rmref_transpose_tile_u32(std::uint32_t* data, std::size_t stride, int n) {
    return guarded([&] { transpose_tile(data, stride, n); });
}

template <class T>
static int tiles_impl(T* data, std::size_t n_tiles, int n, int nthreads) {
    return guarded([&] {
        if (n != 4 && n != 8 && n != 16) transpose_tile(data, std::size_t(n), n);  // throws
        const std::size_t tile = std::size_t(n) * std::size_t(n);
        int nt = std::max(1, nthreads);
        std::vector<std::thread> pool;
        for (int k = 0; k < nt; ++k)
            pool.emplace_back([&, k] {
                pin_self(k);
                const std::size_t a = n_tiles * std::size_t(k) / std::size_t(nt);
                const std::size_t z = n_tiles * std::size_t(k + 1) / std::size_t(nt);
                for (std::size_t i = a; i < z; ++i) transpose_tile(data + i * tile, std::size_t(n), n);
            });
        for (auto& th : pool) th.join();
    });
}

RMREF_API int rmref_transpose_tiles_u8(std::uint8_t* data, std::size_t n_tiles, int n, int nthreads) {
    return tiles_impl(data, n_tiles, n, nthreads);
}
RMREF_API int rmref_transpose_tiles_u16(std::uint16_t* data, std::size_t n_tiles, int n, int nthreads) {
    return tiles_impl(data, n_tiles, n, nthreads);
}

RMREF_API int rmref_calibrate(int w, int h, const int* windows, int n_windows, int reps,
                              int* threshold_h, int* threshold_v) {
    return guarded([&] {
        const DispatchConfig c =
            calibrate(w, h, std::vector<int>(windows, windows + n_windows), reps);
        *threshold_h = c.threshold_h;
        *threshold_v = c.threshold_v;
    });
}

RMREF_API void rmref_set_pinning(int on) { g_pin = on; }

// rectmorph_b200.cpp -- C++ drop-in host library (see include/rectmorph_b200.hpp).
//
// Thin layer over the C-ABI: it owns the value-semantics Image type, validates like the
// reference, calls the rmgpu_*_host entry points (H2D, kernels, D2H) and turns status codes back
// into rectmorph::Error exactly where the reference throws.
#include "rectmorph_b200.hpp"

#include <algorithm>
#include <cstring>
#include <fstream>
#include <sstream>

#include "rmgpu.h"

namespace rectmorph {

namespace {

[[noreturn]] void raise(int status) {
    const std::string msg = rmgpu_last_error();
    if (status >= 1 && status <= 11) throw Error(Errc(status - 1), msg);
    throw GpuError(status, msg.empty() ? rmgpu_status_string(status) : msg);
}

void check(int status) {
    if (status != RMGPU_OK) raise(status);
}

// sliding_extrema.cpp:9-14
void validate_window(int window) {
    if (window < 1) throw Error(Errc::ZeroExtent, "window extent must be >= 1");
    if (window % 2 == 0) throw Error(Errc::EvenExtent, "window extent must be odd");
}

// image.cpp:9-14: rows padded to a multiple of 16 bytes (stride returned in elements)
template <class T>
std::size_t padded_elems(int width) {
    if (width <= 0) return 0;
    const std::size_t bytes = (std::size_t(width) * sizeof(T) + 15u) & ~std::size_t(15);
    return bytes / sizeof(T);
}

int op_code(OpKind k) { return k == OpKind::Erode ? RMGPU_ERODE : RMGPU_DILATE; }

// GPU planner hints for a config: a Calibrated config is honoured axis by axis, the paper's
// thresholds (measured on ARM NEON) leave the choice to the planner (both give the same pixels)
void hints(const StructuringElement& se, const DispatchConfig& cfg, int* ah, int* av) {
    *ah = *av = RMGPU_ALGO_AUTO;
    if (cfg.source != ThresholdSource::Calibrated) return;
    *ah = rmgpu_resolve(RMGPU_ALGO_AUTO, se.width, RMGPU_AXIS_HORIZONTAL, cfg.threshold_h, cfg.threshold_v);
    *av = rmgpu_resolve(RMGPU_ALGO_AUTO, se.height, RMGPU_AXIS_VERTICAL, cfg.threshold_h, cfg.threshold_v);
}

template <class T, class B>
BasicImage<T> run_algo(const BasicImage<T>& src, const StructuringElement& se, const B& border, int op, int ah,
                       int av) {
    if (se.width < 1 || se.height < 1) throw Error(Errc::ZeroExtent, "structuring element extents must be >= 1");
    if (se.width % 2 == 0 || se.height % 2 == 0) throw Error(Errc::EvenExtent, "structuring element extents must be odd");
    BasicImage<T> dst(src.width(), src.height());
    if (src.empty()) return dst;
    const int mode = border.mode == BorderPolicy::Mode::Constant ? RMGPU_BORDER_CONSTANT : RMGPU_BORDER_REPLICATE;
    const std::size_t sp = src.stride() * sizeof(T), dp = dst.stride() * sizeof(T);
    int rc;
    if constexpr (sizeof(T) == 1)
        rc = rmgpu_morph_host_u8(src.row(0), sp, dst.row(0), dp, src.width(), src.height(), se.width, se.height, op,
                                 mode, border.value, ah, av);
    else
        rc = rmgpu_morph_host_u16(src.row(0), sp, dst.row(0), dp, src.width(), src.height(), se.width, se.height,
                                  op, mode, border.value, ah, av);
    check(rc);
    return dst;
}

template <class T, class B>
BasicImage<T> run(const BasicImage<T>& src, const StructuringElement& se, const B& border, int op,
                  const DispatchConfig& cfg = {}) {
    int ah, av;
    hints(se, cfg, &ah, &av);
    return run_algo(src, se, border, op, ah, av);
}

int border_mode(const BorderPolicy& b) {
    return b.mode == BorderPolicy::Mode::Constant ? RMGPU_BORDER_CONSTANT : RMGPU_BORDER_REPLICATE;
}

Image pass(int which, const Image& src, OpKind op, int window, const BorderPolicy& border) {
    validate_window(window);
    Image dst(src.width(), src.height());
    if (src.empty()) return dst;
    check(rmgpu_pass_host_u8(which, src.row(0), src.stride(), dst.row(0), dst.stride(), src.width(), src.height(),
                             window, op_code(op), border_mode(border), border.value, RMGPU_ALGO_AUTO));
    return dst;
}

}  // namespace

// ---- data model -------------------------------------------------------------------------------
StructuringElement make_se(int width, int height) {
    if (width < 1 || height < 1) throw Error(Errc::ZeroExtent, "structuring element extents must be >= 1");
    if (width % 2 == 0 || height % 2 == 0) throw Error(Errc::EvenExtent, "structuring element extents must be odd");
    return {width, height};
}

template <class T>
BasicImage<T>::BasicImage(int width, int height) : width_(width), height_(height), stride_(padded_elems<T>(width)) {
    if (width < 0 || height < 0) throw Error(Errc::BadArgument, "image dimensions must be non-negative");
    data_.resize(stride_ * std::size_t(height_));
}

template <class T>
BasicImage<T> BasicImage<T>::from_pixels(int width, int height, const std::vector<T>& pixels) {
    if (width < 0 || height < 0 || pixels.size() != std::size_t(width) * std::size_t(height))
        throw Error(Errc::BadArgument, "pixel count does not match dimensions");
    BasicImage<T> img(width, height);
    for (int y = 0; y < height; ++y)
        std::memcpy(img.row(y), pixels.data() + std::size_t(y) * width, sizeof(T) * std::size_t(width));
    return img;
}

template <class T>
std::vector<T> BasicImage<T>::to_pixels() const {
    std::vector<T> out(std::size_t(width_) * std::size_t(height_));
    for (int y = 0; y < height_; ++y)
        std::memcpy(out.data() + std::size_t(y) * width_, row(y), sizeof(T) * std::size_t(width_));
    return out;
}

template class BasicImage<std::uint8_t>;
template class BasicImage<std::uint16_t>;

template <class T>
static bool equal_impl(const BasicImage<T>& a, const BasicImage<T>& b) {
    if (a.width() != b.width() || a.height() != b.height()) return false;
    for (int y = 0; y < a.height(); ++y)
        if (std::memcmp(a.row(y), b.row(y), sizeof(T) * std::size_t(a.width())) != 0) return false;
    return true;
}
bool equal_pixels(const Image& a, const Image& b) { return equal_impl(a, b); }
bool equal_pixels(const Image16& a, const Image16& b) { return equal_impl(a, b); }

std::uint8_t sample(const Image& img, int x, int y, const BorderPolicy& border) {
    if (x >= 0 && x < img.width() && y >= 0 && y < img.height()) return img.at(x, y);
    if (border.mode == BorderPolicy::Mode::Constant) return border.value;
    return img.at(std::clamp(x, 0, img.width() - 1), std::clamp(y, 0, img.height() - 1));
}

// ---- passes -----------------------------------------------------------------------------------
Image horizontal_pass(const Image& src, OpKind op, int window, const BorderPolicy& border, PassAlgorithm) {
    return pass(RMGPU_PASS_HORIZONTAL, src, op, window, border);
}
Image vertical_pass_direct(const Image& src, OpKind op, int window, const BorderPolicy& border) {
    return pass(RMGPU_PASS_VERTICAL_DIRECT, src, op, window, border);
}
Image vertical_pass_via_transpose(const Image& src, OpKind op, int window, const BorderPolicy& border,
                                  PassAlgorithm) {
    return pass(RMGPU_PASS_VERTICAL_VIA_TRANSPOSE, src, op, window, border);
}

Image morph_separable(const Image& src, OpKind op, const StructuringElement& se, const BorderPolicy& border,
                      PassAlgorithm h, PassAlgorithm v, VerticalStrategy) {
    validate_window(se.width);  // separable.cpp:134-135
    validate_window(se.height);
    // the explicit per-axis algorithms become GPU planner hints (rmgpu.h); both vertical strategies
    // are the same fused column pass on the GPU
    return run_algo(src, se, border, op_code(op), int(h), int(v));
}
Image morph_separable(const Image& src, OpKind op, const StructuringElement& se, const BorderPolicy& border,
                      PassAlgorithm h, PassAlgorithm v) {
    return morph_separable(src, op, se, border, h, v, VerticalStrategy::Direct);
}

// ---- dispatch ---------------------------------------------------------------------------------
PassAlgorithm resolve(PassAlgorithm algo, int window, Axis axis, const DispatchConfig& cfg) {
    return PassAlgorithm(rmgpu_resolve(int(algo), window, axis == Axis::Horizontal ? RMGPU_AXIS_HORIZONTAL
                                                                                     : RMGPU_AXIS_VERTICAL,
                                       cfg.threshold_h, cfg.threshold_v));
}

Image erode(const Image& s, const StructuringElement& se, const BorderPolicy& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_ERODE, c); }
Image dilate(const Image& s, const StructuringElement& se, const BorderPolicy& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_DILATE, c); }
Image opening(const Image& s, const StructuringElement& se, const BorderPolicy& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_OPEN, c); }
Image closing(const Image& s, const StructuringElement& se, const BorderPolicy& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_CLOSE, c); }
Image gradient(const Image& s, const StructuringElement& se, const BorderPolicy& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_GRADIENT, c); }

Image16 erode(const Image16& s, const StructuringElement& se, const BorderPolicy16& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_ERODE, c); }
Image16 dilate(const Image16& s, const StructuringElement& se, const BorderPolicy16& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_DILATE, c); }
Image16 opening(const Image16& s, const StructuringElement& se, const BorderPolicy16& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_OPEN, c); }
Image16 closing(const Image16& s, const StructuringElement& se, const BorderPolicy16& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_CLOSE, c); }
Image16 gradient(const Image16& s, const StructuringElement& se, const BorderPolicy16& b, const DispatchConfig& c) { return run(s, se, b, RMGPU_GRADIENT, c); }

// ---- dispatch config (dispatch.hpp:46-66) -------------------------------------------------------
std::string format_config(const DispatchConfig& cfg) {
    char buf[96];
    const int n = rmgpu_format_config(cfg.threshold_h, cfg.threshold_v,
                                      cfg.source == ThresholdSource::Calibrated ? RMGPU_SOURCE_CALIBRATED
                                                                                : RMGPU_SOURCE_PAPER,
                                      buf, sizeof buf);
    return std::string(buf, std::min<std::size_t>(std::size_t(n), sizeof buf - 1));
}

DispatchConfig parse_config(const std::string& text) {
    DispatchConfig cfg;
    int src = RMGPU_SOURCE_PAPER;
    check(rmgpu_parse_config(text.c_str(), &cfg.threshold_h, &cfg.threshold_v, &src));
    cfg.source = src == RMGPU_SOURCE_CALIBRATED ? ThresholdSource::Calibrated : ThresholdSource::Paper;
    return cfg;
}

DispatchConfig load_config(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(Errc::IoError, "cannot open config '" + path + "'");
    std::ostringstream text;
    text << in.rdbuf();
    try {
        return parse_config(text.str());
    } catch (const Error& e) {
        throw Error(e.code(), path + ": " + e.what());
    }
}

void save_config(const std::string& path, const DispatchConfig& cfg) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error(Errc::IoError, "cannot open '" + path + "' for writing");
    out << format_config(cfg);
    out.flush();
    if (!out) throw Error(Errc::IoError, "failed writing config '" + path + "'");
}

DispatchConfig calibrate(int width, int height, const std::vector<int>& windows, int reps) {
    DispatchConfig cfg;
    check(rmgpu_calibrate(width, height, windows.data(), int(windows.size()), reps, &cfg.threshold_h,
                          &cfg.threshold_v));
    cfg.source = ThresholdSource::Calibrated;
    return cfg;
}

// ---- transposes -------------------------------------------------------------------------------
void transpose_tile(std::uint8_t* data, std::size_t stride, int n) { check(rmgpu_transpose_tiles_host(data, 1, 1, n, stride, 0)); }
void transpose_tile(std::uint16_t* data, std::size_t stride, int n) { check(rmgpu_transpose_tiles_host(data, 2, 1, n, stride, 0)); }
void transpose_tile(std::uint32_t* data, std::size_t stride, int n) { check(rmgpu_transpose_tiles_host(data, 4, 1, n, stride, 0)); }

Image transpose_image(const Image& src) {
    Image dst(src.height(), src.width());
    if (src.empty()) return dst;
    check(rmgpu_transpose_host_u8(src.row(0), src.stride(), dst.row(0), dst.stride(), src.width(), src.height()));
    return dst;
}

Image16 transpose_image(const Image16& src) {
    Image16 dst(src.height(), src.width());
    if (src.empty()) return dst;
    check(rmgpu_transpose_host_u16(src.row(0), src.stride() * 2, dst.row(0), dst.stride() * 2, src.width(),
                                   src.height()));
    return dst;
}

// ---- 1-D --------------------------------------------------------------------------------------
namespace {
void window_1d(const std::uint8_t* in, std::size_t n, int window, OpKind op, const BorderPolicy& border,
               std::uint8_t* out, OpCounter* counter, bool vanherk) {
    validate_window(window);  // run_prologue, sliding_extrema.cpp:167-177
    if (counter) counter->reset();
    if (n == 0) return;
    if (window == 1) {
        std::memmove(out, in, n);
        return;
    }
    check(rmgpu_window_1d_host_u8(in, n, window, op_code(op), border_mode(border), border.value,
                                  vanherk ? RMGPU_ALGO_VANHERK : RMGPU_ALGO_LINEAR, out));
    if (counter) {
        if (vanherk) {
            const std::uint64_t w = std::uint64_t(window), len = n + w - 1, blocks = (len + w - 1) / w;
            counter->comparisons = 2 * (len - blocks) + n;
        } else {
            counter->comparisons = std::uint64_t(window - 1) * n;
        }
    }
}
}  // namespace

void linear_window_1d(const std::uint8_t* in, std::size_t n, int window, OpKind op, const BorderPolicy& border,
                      std::uint8_t* out, OpCounter* counter) {
    window_1d(in, n, window, op, border, out, counter, false);
}
void van_herk_1d(const std::uint8_t* in, std::size_t n, int window, OpKind op, const BorderPolicy& border,
                 std::uint8_t* out, OpCounter* counter) {
    window_1d(in, n, window, op, border, out, counter, true);
}
std::vector<std::uint8_t> linear_window_1d(const std::vector<std::uint8_t>& in, int window, OpKind op,
                                           const BorderPolicy& border, OpCounter* counter) {
    std::vector<std::uint8_t> out(in.size());
    linear_window_1d(in.data(), in.size(), window, op, border, out.data(), counter);
    return out;
}
std::vector<std::uint8_t> van_herk_1d(const std::vector<std::uint8_t>& in, int window, OpKind op,
                                      const BorderPolicy& border, OpCounter* counter) {
    std::vector<std::uint8_t> out(in.size());
    van_herk_1d(in.data(), in.size(), window, op, border, out.data(), counter);
    return out;
}

}  // namespace rectmorph

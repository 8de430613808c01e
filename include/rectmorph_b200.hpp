// rectmorph_b200.hpp -- C++ drop-in for the reference library's hot-path API, backed by the
// B200 kernels through the C-ABI in rmgpu.h (link librectmorph_b200.so + librmgpu.so).
//
// Same namespace, type names, signatures and error behaviour as the reference `rectmorph`
// (/root/reference/proj/core/include/rectmorph/{image,error,separable,dispatch,transpose,
// sliding_extrema}.hpp), so a caller swaps the include and the library and keeps its code:
//
//   rectmorph::Image img = ...;                        // u8, stride = round_up(width, 16)
//   auto se = rectmorph::make_se(15, 15);
//   rectmorph::Image out = rectmorph::erode(img, se, rectmorph::BorderPolicy::replicate());
//
// Every operation copies the host image to the GPU, runs the kernels, and copies the result
// back (value semantics: inputs are const, a fresh image is returned, image.cpp:26-31).
// Extensions beyond the reference: 16-bit images (`Image16`) for every image operation.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <iosfwd>
#include <string>
#include <vector>

namespace rectmorph {

// ---- errors (reference error.hpp:10-33) --------------------------------------------------------
enum class Errc {
    ZeroExtent,
    EvenExtent,
    UnsupportedTile,
    BadMagic,
    BadHeader,
    UnsupportedMaxval,
    TruncatedData,
    BadConfig,
    InsufficientReps,
    IoError,
    BadArgument,
};

class Error : public std::runtime_error {
public:
    Error(Errc code, const std::string& message) : std::runtime_error(message), code_(code) {}
    Errc code() const noexcept { return code_; }

private:
    Errc code_;
};

// CUDA-side failure (no device, launch error, out of memory). Not an Errc: the reference has
// no device.
class GpuError : public std::runtime_error {
public:
    GpuError(int status, const std::string& message) : std::runtime_error(message), status_(status) {}
    int status() const noexcept { return status_; }

private:
    int status_;
};

// ---- data model (reference image.hpp:11-81) ------------------------------------------------------
enum class OpKind { Erode, Dilate };

inline std::uint8_t identity_value(OpKind op) noexcept { return op == OpKind::Erode ? 255 : 0; }

struct BorderPolicy {
    enum class Mode { Replicate, Constant };
    Mode mode = Mode::Replicate;
    std::uint8_t value = 0;
    static BorderPolicy replicate() { return {Mode::Replicate, 0}; }
    static BorderPolicy constant(std::uint8_t v) { return {Mode::Constant, v}; }
};

// 16-bit border value for Image16 operations (extension).
struct BorderPolicy16 {
    BorderPolicy::Mode mode = BorderPolicy::Mode::Replicate;
    std::uint16_t value = 0;
    static BorderPolicy16 replicate() { return {BorderPolicy::Mode::Replicate, 0}; }
    static BorderPolicy16 constant(std::uint16_t v) { return {BorderPolicy::Mode::Constant, v}; }
    BorderPolicy16() = default;
    BorderPolicy16(BorderPolicy::Mode m, std::uint16_t v) : mode(m), value(v) {}
    BorderPolicy16(const BorderPolicy& b) : mode(b.mode), value(b.value) {}  // NOLINT
};

struct StructuringElement {
    int width = 1;
    int height = 1;
    int wing_x() const noexcept { return width / 2; }
    int wing_y() const noexcept { return height / 2; }
};

StructuringElement make_se(int width, int height);

// Single-channel image, rows padded to a multiple of 16 bytes. Padding carries no value.
template <class T>
class BasicImage {
public:
    BasicImage() = default;
    BasicImage(int width, int height);
    static BasicImage from_pixels(int width, int height, const std::vector<T>& pixels);

    int width() const noexcept { return width_; }
    int height() const noexcept { return height_; }
    std::size_t stride() const noexcept { return stride_; }  // in elements
    bool empty() const noexcept { return width_ == 0 || height_ == 0; }
    T* row(int y) noexcept { return data_.data() + std::size_t(y) * stride_; }
    const T* row(int y) const noexcept { return data_.data() + std::size_t(y) * stride_; }
    T& at(int x, int y) noexcept { return row(y)[x]; }
    T at(int x, int y) const noexcept { return row(y)[x]; }
    std::vector<T> to_pixels() const;

private:
    int width_ = 0;
    int height_ = 0;
    std::size_t stride_ = 0;
    std::vector<T> data_;
};

using Image = BasicImage<std::uint8_t>;
using Image16 = BasicImage<std::uint16_t>;

bool equal_pixels(const Image& a, const Image& b);
bool equal_pixels(const Image16& a, const Image16& b);
std::uint8_t sample(const Image& img, int x, int y, const BorderPolicy& border);

// ---- pass-level API (reference separable.hpp:11-55) -------------------------------------------
enum class PassAlgorithm { Auto, Linear, VanHerk };
enum class VerticalStrategy { Direct, ViaTranspose };
enum class Axis { Horizontal, Vertical };

Image horizontal_pass(const Image& src, OpKind op, int window, const BorderPolicy& border,
                      PassAlgorithm algo = PassAlgorithm::Auto);
Image vertical_pass_direct(const Image& src, OpKind op, int window, const BorderPolicy& border);
Image vertical_pass_via_transpose(const Image& src, OpKind op, int window, const BorderPolicy& border,
                                  PassAlgorithm algo = PassAlgorithm::Auto);
// On the GPU both passes run fused in one kernel; the algorithm/strategy arguments are
// accepted for API parity (results never depend on them, tests/test_dispatch.cpp:68-79).
Image morph_separable(const Image& src, OpKind op, const StructuringElement& se, const BorderPolicy& border,
                      PassAlgorithm h_algo, PassAlgorithm v_algo, VerticalStrategy v_strategy);
Image morph_separable(const Image& src, OpKind op, const StructuringElement& se, const BorderPolicy& border,
                      PassAlgorithm h_algo = PassAlgorithm::Auto, PassAlgorithm v_algo = PassAlgorithm::Auto);

// ---- dispatch + compound ops (reference dispatch.hpp:11-66) -----------------------------------
enum class ThresholdSource { Paper, Calibrated };
struct DispatchConfig {
    int threshold_h = 69;
    int threshold_v = 59;
    ThresholdSource source = ThresholdSource::Paper;
};

PassAlgorithm resolve(PassAlgorithm algo, int window, Axis axis, const DispatchConfig& cfg = {});

// Config text and files (reference dispatch.hpp:46-57): "threshold_h=<int>\nthreshold_v=<int>\n
// source=paper|calibrated\n"; parse_config is the strict inverse (Errc::BadConfig), load / save
// fail with Errc::IoError naming the path.
std::string format_config(const DispatchConfig& cfg);
DispatchConfig parse_config(const std::string& text);
DispatchConfig load_config(const std::string& path);
void save_config(const std::string& path, const DispatchConfig& cfg);

// calibrate (reference dispatch.hpp:59-66) measured on the current GPU: per swept window and
// axis, the direct sliding window against van Herk (median of `reps` CUDA-event timings); the
// thresholds are the largest windows where direct still wins. Validation as the reference
// (reps < 3 -> Errc::InsufficientReps; empty, even or non-ascending windows, extents < 1).
// The operations below honour a config whose source is Calibrated (each axis's resolved
// algorithm is passed to the GPU planner); the paper's ARM thresholds (source Paper) leave the
// choice to the planner's built-in B200 crossover. Results never depend on either.
DispatchConfig calibrate(int width, int height, const std::vector<int>& windows, int reps);

Image erode(const Image& src, const StructuringElement& se, const BorderPolicy& border, const DispatchConfig& cfg = {});
Image dilate(const Image& src, const StructuringElement& se, const BorderPolicy& border, const DispatchConfig& cfg = {});
Image opening(const Image& src, const StructuringElement& se, const BorderPolicy& border, const DispatchConfig& cfg = {});
Image closing(const Image& src, const StructuringElement& se, const BorderPolicy& border, const DispatchConfig& cfg = {});
Image gradient(const Image& src, const StructuringElement& se, const BorderPolicy& border, const DispatchConfig& cfg = {});

Image16 erode(const Image16& src, const StructuringElement& se, const BorderPolicy16& border, const DispatchConfig& cfg = {});
Image16 dilate(const Image16& src, const StructuringElement& se, const BorderPolicy16& border, const DispatchConfig& cfg = {});
Image16 opening(const Image16& src, const StructuringElement& se, const BorderPolicy16& border, const DispatchConfig& cfg = {});
Image16 closing(const Image16& src, const StructuringElement& se, const BorderPolicy16& border, const DispatchConfig& cfg = {});
Image16 gradient(const Image16& src, const StructuringElement& se, const BorderPolicy16& border, const DispatchConfig& cfg = {});

// ---- transposes (reference transpose.hpp:34-43) -----------------------------------------------
void transpose_tile(std::uint8_t* data, std::size_t stride, int n);
void transpose_tile(std::uint16_t* data, std::size_t stride, int n);
void transpose_tile(std::uint32_t* data, std::size_t stride, int n);
Image transpose_image(const Image& src);
Image16 transpose_image(const Image16& src);

// ---- PGM files (reference pgm.hpp:10-24) -------------------------------------------------------
// P5 (binary) and P2 (ASCII) with maxval 255; '#' comments anywhere in the header and, for P2,
// between pixel tokens. Errors: Errc::BadMagic, BadHeader (malformed header, extents outside
// 1..2^20, P2 token > 255 or not a number), UnsupportedMaxval, TruncatedData, IoError (files,
// message names the path), BadArgument (writing an empty image). Writes are canonical:
// "P5\n<w> <h>\n255\n" + rows, or P2 with one image row per text line; never comments.
Image read_pgm(std::istream& in);
void write_pgm(std::ostream& out, const Image& img, bool binary = true);
Image load_pgm(const std::string& path);
void store_pgm(const std::string& path, const Image& img, bool binary = true);

// ---- 1-D API (reference sliding_extrema.hpp:11-44) ----------------------------------------------
struct OpCounter {
    std::uint64_t comparisons = 0;
    void reset() noexcept { comparisons = 0; }
};
// The counter receives the comparison count of the named reference algorithm for this call
// (linear: (w-1)*n, van Herk: 2*(len-blocks)+n), the closed forms of sliding_extrema.cpp:131,139.
void linear_window_1d(const std::uint8_t* in, std::size_t n, int window, OpKind op, const BorderPolicy& border,
                      std::uint8_t* out, OpCounter* counter = nullptr);
void van_herk_1d(const std::uint8_t* in, std::size_t n, int window, OpKind op, const BorderPolicy& border,
                 std::uint8_t* out, OpCounter* counter = nullptr);
std::vector<std::uint8_t> linear_window_1d(const std::vector<std::uint8_t>& in, int window, OpKind op,
                                           const BorderPolicy& border, OpCounter* counter = nullptr);
std::vector<std::uint8_t> van_herk_1d(const std::vector<std::uint8_t>& in, int window, OpKind op,
                                      const BorderPolicy& border, OpCounter* counter = nullptr);

}  // namespace rectmorph

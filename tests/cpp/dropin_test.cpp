// Drop-in check: code written against the reference's public API (namespace rectmorph,
// core/include/rectmorph/*.hpp) compiles unchanged against rectmorph_b200.hpp and runs on the
// GPU. Cases are the reference's own known answers (test_reference.cpp:34-55,
// test_sliding_extrema.cpp:18-28, test_transpose.cpp:77-133) plus an exhaustive brute-force
// sweep written with rectmorph::sample (reference.cpp:7-27 semantics).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rectmorph_b200.hpp"

using namespace rectmorph;

static int failures = 0;
#define CHECK(c)                                                      \
    do {                                                              \
        if (!(c)) {                                                   \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);   \
            ++failures;                                               \
        }                                                             \
    } while (0)

static Image brute(const Image& src, OpKind op, const StructuringElement& se, const BorderPolicy& b) {
    Image dst(src.width(), src.height());
    for (int y = 0; y < src.height(); ++y)
        for (int x = 0; x < src.width(); ++x) {
            int acc = op == OpKind::Erode ? 255 : 0;
            for (int dy = -se.wing_y(); dy <= se.wing_y(); ++dy)
                for (int dx = -se.wing_x(); dx <= se.wing_x(); ++dx) {
                    int v = sample(src, x + dx, y + dy, b);
                    acc = op == OpKind::Erode ? std::min(acc, v) : std::max(acc, v);
                }
            dst.at(x, y) = std::uint8_t(acc);
        }
    return dst;
}

int main() {
    // ramp 3x3 erode (test_reference.cpp:34-41)
    Image ramp = Image::from_pixels(3, 3, {9, 8, 7, 6, 5, 4, 3, 2, 1});
    Image e = erode(ramp, make_se(3, 3), BorderPolicy::replicate());
    CHECK(e.to_pixels() == (std::vector<std::uint8_t>{5, 4, 4, 2, 1, 1, 2, 1, 1}));
    CHECK(e.stride() == 16);
    // constant borders (test_reference.cpp:43-55)
    Image sq = Image::from_pixels(2, 2, {128, 128, 128, 128});
    CHECK(erode(sq, make_se(3, 3), BorderPolicy::constant(5)).at(0, 0) == 5);
    CHECK(dilate(sq, make_se(3, 3), BorderPolicy::constant(200)).at(1, 1) == 200);
    // 1-D (test_sliding_extrema.cpp:18-28)
    std::vector<std::uint8_t> sig{4, 2, 6, 1, 3, 5, 0, 7};
    OpCounter c;
    CHECK(linear_window_1d(sig, 3, OpKind::Erode, BorderPolicy::replicate(), &c) ==
          (std::vector<std::uint8_t>{2, 2, 1, 1, 1, 0, 0, 0}));
    CHECK(c.comparisons == 16);
    CHECK(van_herk_1d(sig, 3, OpKind::Dilate, BorderPolicy::replicate()) ==
          (std::vector<std::uint8_t>{4, 6, 6, 6, 5, 5, 7, 7}));
    // in-place 1-D (test_sliding_extrema.cpp:126-140)
    std::vector<std::uint8_t> inplace = sig;
    linear_window_1d(inplace.data(), inplace.size(), 3, OpKind::Erode, BorderPolicy::replicate(), inplace.data());
    CHECK(inplace == (std::vector<std::uint8_t>{2, 2, 1, 1, 1, 0, 0, 0}));
    // transposes (test_transpose.cpp:77-84, 127-133)
    Image t = transpose_image(Image::from_pixels(3, 2, {1, 2, 3, 4, 5, 6}));
    CHECK(t.width() == 2 && t.height() == 3 && t.to_pixels() == (std::vector<std::uint8_t>{1, 4, 2, 5, 3, 6}));
    std::vector<std::uint16_t> tile(64);
    for (int i = 0; i < 64; ++i) tile[i] = std::uint16_t(i);
    transpose_tile(tile.data(), 8, 8);
    bool ok = true;
    for (int r = 0; r < 8; ++r)
        for (int cc = 0; cc < 8; ++cc) ok = ok && tile[r * 8 + cc] == 8 * cc + r;
    CHECK(ok);
    // errors thrown where the reference throws
    bool threw = false;
    try { make_se(4, 3); } catch (const Error& err) { threw = err.code() == Errc::EvenExtent; }
    CHECK(threw);
    threw = false;
    std::uint8_t buf[25] = {};
    try { transpose_tile(buf, 5, 5); } catch (const Error& err) { threw = err.code() == Errc::UnsupportedTile; }
    CHECK(threw);
    // exhaustive small sweep vs sample()-based brute force, all borders
    unsigned s = 12345;
    for (int w = 1; w <= 12; ++w)
        for (int h = 1; h <= 12; h += 3) {
            std::vector<std::uint8_t> px(std::size_t(w) * h);
            for (auto& p : px) p = std::uint8_t((s = s * 1103515245u + 12345u) >> 16);
            Image img = Image::from_pixels(w, h, px);
            for (int sw = 1; sw <= 9; sw += 2)
                for (int sh = 1; sh <= 9; sh += 4)
                    for (OpKind op : {OpKind::Erode, OpKind::Dilate})
                        for (BorderPolicy b : {BorderPolicy::replicate(), BorderPolicy::constant(77)}) {
                            const StructuringElement se = make_se(sw, sh);
                            const Image got = op == OpKind::Erode ? erode(img, se, b) : dilate(img, se, b);
                            CHECK(equal_pixels(got, brute(img, op, se, b)));
                        }
        }
    // opening idempotence + 16-bit extension
    Image16 im16(40, 30);
    for (int y = 0; y < 30; ++y)
        for (int x = 0; x < 40; ++x) im16.at(x, y) = std::uint16_t((x * 7919 + y * 104729) & 0xFFFF);
    Image16 o = opening(im16, make_se(5, 5), BorderPolicy16::replicate());
    CHECK(equal_pixels(opening(o, make_se(5, 5), BorderPolicy16::replicate()), o));
    Image16 t16 = transpose_image(im16);
    CHECK(t16.width() == 30 && t16.at(3, 5) == im16.at(5, 3));
    {  // morph_separable with every explicit algorithm / strategy (separable.hpp:44-55): same pixels
        Image src(97, 61);
        for (int y = 0; y < 61; ++y)
            for (int x = 0; x < 97; ++x) src.at(x, y) = std::uint8_t((x * 37 + y * 101 + x * y) & 0xFF);
        const StructuringElement se = make_se(21, 13);
        const Image want = brute(src, OpKind::Dilate, se, BorderPolicy::constant(9));
        for (auto h : {PassAlgorithm::Auto, PassAlgorithm::Linear, PassAlgorithm::VanHerk})
            for (auto v : {PassAlgorithm::Auto, PassAlgorithm::Linear, PassAlgorithm::VanHerk})
                for (auto st : {VerticalStrategy::Direct, VerticalStrategy::ViaTranspose})
                    CHECK(equal_pixels(morph_separable(src, OpKind::Dilate, se, BorderPolicy::constant(9), h, v, st),
                                       want));
        DispatchConfig cal;
        cal.threshold_h = 99;
        cal.threshold_v = 3;
        cal.source = ThresholdSource::Calibrated;
        CHECK(equal_pixels(dilate(src, se, BorderPolicy::constant(9), cal), want));
    }
    if (failures == 0) std::printf("ALL PASS\n");
    return failures == 0 ? 0 : 1;
}

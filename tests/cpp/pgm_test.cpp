// PGM check, CPU only: code written against the reference's pgm.hpp (core/include/rectmorph/
// pgm.hpp:10-24) compiles unchanged against rectmorph_b200.hpp and behaves like it. Cases follow
// the reference's tests/test_pgm.cpp:35-135 (minimal P5 / P2 reads, canonical writes, round trips,
// comments, whitespace-looking binary bytes, every typed error, path in file errors) -- written
// anew here.
#include <cstdio>
#include <sstream>
#include <string>

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

static Image from(const std::string& s) {
    std::istringstream in(s, std::ios::binary);
    return read_pgm(in);
}
static std::string to(const Image& img, bool binary) {
    std::ostringstream out(std::ios::binary);
    write_pgm(out, img, binary);
    return out.str();
}
static bool read_fails_with(const std::string& s, Errc want) {
    try {
        (void)from(s);
    } catch (const Error& e) {
        return e.code() == want;
    }
    return false;
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    {
        const Image a = from(std::string("P5\n1 1\n255\n\x2a", 12));
        CHECK(a.width() == 1 && a.height() == 1 && a.at(0, 0) == 42);
        const Image b = from("P2\n3 1\n255\n0 128 255\n");
        CHECK(b.width() == 3 && b.at(0, 0) == 0 && b.at(1, 0) == 128 && b.at(2, 0) == 255);
    }
    CHECK(to(Image::from_pixels(1, 1, {200}), true) == std::string("P5\n1 1\n255\n\xc8", 12));
    CHECK(to(Image::from_pixels(2, 2, {1, 20, 255, 0}), false) == "P2\n2 2\n255\n1 20\n255 0\n");
    for (int k = 0; k < 12; ++k) {  // round trips, deterministic, canonical
        const int w = 1 + (k * 11) % 37, h = 1 + (k * 7) % 23;
        Image img(w, h);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) img.at(x, y) = std::uint8_t((x * 31 + y * 17 + k * 5) & 0xFF);
        for (bool bin : {true, false}) {
            const std::string bytes = to(img, bin);
            CHECK(equal_pixels(from(bytes), img));
            CHECK(to(from(bytes), bin) == bytes);
        }
    }
    {  // comments anywhere in the header (and between P2 tokens), never written
        const Image c = from("P2 # m\n# line\n2 # w\n1\n# x\n255\n# d\n5 # p\n6\n");
        CHECK(c.width() == 2 && c.at(0, 0) == 5 && c.at(1, 0) == 6);
        CHECK(to(c, true).find('#') == std::string::npos && to(c, false).find('#') == std::string::npos);
    }
    {  // binary pixels that look like separators are data
        const Image ws = Image::from_pixels(2, 2, {'\n', '#', '\t', ' '});
        CHECK(equal_pixels(from(to(ws, true)), ws));
    }
    CHECK(read_fails_with("P3\n1 1\n255\n1\n", Errc::BadMagic));
    CHECK(read_fails_with("", Errc::BadMagic));
    CHECK(read_fails_with("p5\n1 1\n255\nx", Errc::BadMagic));
    CHECK(read_fails_with("P5", Errc::BadHeader));
    CHECK(read_fails_with("P5\n1 0\n255\nx", Errc::BadHeader));
    CHECK(read_fails_with("P5\n-1 1\n255\nx", Errc::BadHeader));
    CHECK(read_fails_with("P5\nw 1\n255\nx", Errc::BadHeader));
    CHECK(read_fails_with("P5\n1048577 1\n255\n", Errc::BadHeader));
    CHECK(read_fails_with("P5\n1 123456789012345678901\n255\n", Errc::BadHeader));
    CHECK(read_fails_with("P5\n1 1\n255x", Errc::BadHeader));
    CHECK(read_fails_with("P5\n1 1\n256\nx", Errc::UnsupportedMaxval));
    CHECK(read_fails_with("P5\n1 1\n15\nx", Errc::UnsupportedMaxval));
    CHECK(read_fails_with(std::string("P5\n3 1\n255\nab", 13), Errc::TruncatedData));
    CHECK(read_fails_with("P2\n2 1\n255\n7\n", Errc::TruncatedData));
    CHECK(read_fails_with("P2\n1 1\n255\n256\n", Errc::BadHeader));
    CHECK(read_fails_with("P2\n1 1\n255\nq\n", Errc::BadHeader));
    try {
        std::ostringstream out;
        write_pgm(out, Image(), true);
        CHECK(false);
    } catch (const Error& e) {
        CHECK(e.code() == Errc::BadArgument);
    }
    {  // files
        Image img(9, 4);
        for (int y = 0; y < 4; ++y)
            for (int x = 0; x < 9; ++x) img.at(x, y) = std::uint8_t(x * y + 3);
        store_pgm(dir + "/rt.pgm", img);
        CHECK(equal_pixels(load_pgm(dir + "/rt.pgm"), img));
        store_pgm(dir + "/rt2.pgm", img, false);
        CHECK(equal_pixels(load_pgm(dir + "/rt2.pgm"), img));
        try {
            (void)load_pgm(dir + "/absent.pgm");
            CHECK(false);
        } catch (const Error& e) {
            CHECK(e.code() == Errc::IoError && std::string(e.what()).find("absent.pgm") != std::string::npos);
        }
        try {
            store_pgm(dir + "/no/such/dir/x.pgm", img);
            CHECK(false);
        } catch (const Error& e) {
            CHECK(e.code() == Errc::IoError);
        }
    }
    if (failures) {
        std::printf("%d failures\n", failures);
        return 1;
    }
    std::printf("pgm_test ok\n");
    return 0;
}

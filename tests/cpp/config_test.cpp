// Dispatch-config check, CPU only: code written against the reference's config API
// (core/include/rectmorph/dispatch.hpp:46-66) compiles unchanged against rectmorph_b200.hpp and
// behaves like it. The cases follow the reference's tests/test_dispatch.cpp:134-224 (text round
// trip, comments / blank lines / stray spaces, every malformed form, file persistence and the
// missing-file error, calibrate's input validation) -- written anew here, not copied.
#include <cstdio>
#include <cstdlib>
#include <string>
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

template <class F>
static bool throws_code(F&& f, Errc want) {
    try {
        f();
    } catch (const Error& e) {
        return e.code() == want;
    } catch (...) {
        return false;
    }
    return false;
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    {  // round trip of a calibrated config
        DispatchConfig c;
        c.threshold_h = 17;
        c.threshold_v = 203;
        c.source = ThresholdSource::Calibrated;
        const std::string t = format_config(c);
        CHECK(t == "threshold_h=17\nthreshold_v=203\nsource=calibrated\n");
        const DispatchConfig p = parse_config(t);
        CHECK(p.threshold_h == 17 && p.threshold_v == 203 && p.source == ThresholdSource::Calibrated);
        CHECK(format_config(DispatchConfig{}) == "threshold_h=69\nthreshold_v=59\nsource=paper\n");
    }
    {  // comments, blank lines, spaces around keys and values, CRLF
        const DispatchConfig p = parse_config("# b200\n\n  threshold_v = 7\r\nsource =paper\nthreshold_h= 9 \n");
        CHECK(p.threshold_h == 9 && p.threshold_v == 7 && p.source == ThresholdSource::Paper);
    }
    // every malformed form is Errc::BadConfig
    const char* bad[] = {
        "threshold_h=9\nthreshold_v=7\n",                          // source missing
        "threshold_h=9\nthreshold_v=7\nsource=paper\nfoo=1\n",     // unknown key
        "threshold_h=8\nthreshold_v=7\nsource=paper\n",            // even
        "threshold_h=0\nthreshold_v=7\nsource=paper\n",            // not positive
        "threshold_h=-9\nthreshold_v=7\nsource=paper\n",           // negative
        "threshold_h=9x\nthreshold_v=7\nsource=paper\n",           // trailing garbage
        "threshold_h=\nthreshold_v=7\nsource=paper\n",             // empty value
        "threshold_v=7\nthreshold_v=7\nthreshold_h=9\nsource=paper\n",  // duplicate
        "threshold_h=9\nthreshold_v=7\nsource=measured\n",         // bad source
        "threshold_h:9\nthreshold_v=7\nsource=paper\n",            // no '='
        "",                                                        // nothing
    };
    for (const char* t : bad) CHECK(throws_code([&] { (void)parse_config(t); }, Errc::BadConfig));
    {  // files
        DispatchConfig c;
        c.threshold_h = 31;
        c.threshold_v = 5;
        c.source = ThresholdSource::Calibrated;
        const std::string path = dir + "/dispatch_cfg.txt";
        save_config(path, c);
        const DispatchConfig l = load_config(path);
        CHECK(l.threshold_h == 31 && l.threshold_v == 5 && l.source == ThresholdSource::Calibrated);
        const std::string missing = dir + "/no_such_config.txt";
        CHECK(throws_code([&] { (void)load_config(missing); }, Errc::IoError));
        try {
            (void)load_config(missing);
        } catch (const Error& e) {
            CHECK(std::string(e.what()).find("no_such_config.txt") != std::string::npos);
        }
        CHECK(throws_code([&] { save_config(dir + "/no_dir/x/cfg.txt", c); }, Errc::IoError));
    }
    // calibrate validates before touching a device
    CHECK(throws_code([] { (void)calibrate(32, 32, {3, 5}, 2); }, Errc::InsufficientReps));
    CHECK(throws_code([] { (void)calibrate(32, 32, {5, 3}, 3); }, Errc::BadArgument));
    CHECK(throws_code([] { (void)calibrate(32, 32, {3, 4}, 3); }, Errc::EvenExtent));
    CHECK(throws_code([] { (void)calibrate(32, 32, {}, 3); }, Errc::BadArgument));
    CHECK(throws_code([] { (void)calibrate(0, 32, {3}, 3); }, Errc::BadArgument));
    // resolve with a calibrated config (dispatch.cpp:14-20)
    DispatchConfig c;
    c.threshold_h = 7;
    c.threshold_v = 9;
    CHECK(resolve(PassAlgorithm::Auto, 7, Axis::Horizontal, c) == PassAlgorithm::Linear);
    CHECK(resolve(PassAlgorithm::Auto, 9, Axis::Horizontal, c) == PassAlgorithm::VanHerk);
    CHECK(resolve(PassAlgorithm::Auto, 9, Axis::Vertical, c) == PassAlgorithm::Linear);
    if (argc > 2 && std::string(argv[2]) == "--gpu") {
        // on a GPU: thresholds come from the swept set and are marked calibrated (test_dispatch.cpp:227-235)
        const DispatchConfig g = calibrate(256, 192, {3, 5, 7, 9, 15}, 3);
        CHECK(g.source == ThresholdSource::Calibrated);
        const std::vector<int> ok = {1, 3, 5, 7, 9, 15};
        bool hok = false, vok = false;
        for (int w : ok) {
            hok |= g.threshold_h == w;
            vok |= g.threshold_v == w;
        }
        CHECK(hok && vok);
        std::printf("calibrated threshold_h=%d threshold_v=%d\n", g.threshold_h, g.threshold_v);
    }
    if (failures) {
        std::printf("%d failures\n", failures);
        return 1;
    }
    std::printf("config_test ok\n");
    return 0;
}

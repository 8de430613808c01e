// rectmorph_cli_b200.cpp -- the reference's command-line front end on the GPU (reference
// tools/rectmorph_cli.cpp:105-308): `apply` filters a PGM file, `bench` times the direct and van
// Herk kernels of both passes over a window sweep into the reference's CSV schema (plus the
// device time of each call), `calibrate` writes a dispatch config measured on this GPU.
//
//   rectmorph_b200 apply --op erode|dilate|open|close|gradient --se WxH
//                        [--border replicate|constant:V] [--config FILE] INPUT.pgm OUTPUT.pgm
//   rectmorph_b200 bench --windows MIN..MAX[:STEP] --out FILE.csv [--width W] [--height H]
//                        [--reps N] [--seed S] [--transpose]
//   rectmorph_b200 calibrate --windows MIN..MAX[:STEP] --out FILE [--width W] [--height H] [--reps N]
//
// Failures print one line "rectmorph: <message>" on stderr and exit 1 (reference CLI contract,
// tests/test_cli.cpp). The pixels go through the drop-in library (librectmorph_b200) and the
// C-ABI (librmgpu); there is no CPU path.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "rectmorph_b200.hpp"
#include "rmgpu.h"

namespace rm = rectmorph;

namespace {

[[noreturn]] void usage_error(const std::string& msg) { throw rm::Error(rm::Errc::BadArgument, msg); }

int to_int(const std::string& text, const std::string& what) {
    std::size_t used = 0;
    long v = 0;
    try {
        v = std::stol(text, &used);
    } catch (...) {
        used = std::string::npos;
    }
    if (used != text.size() || text.empty() || v < -2147483647L || v > 2147483647L)
        usage_error(what + ": expected an integer, got '" + text + "'");
    return int(v);
}

rm::StructuringElement parse_se(const std::string& t) {
    const std::size_t x = t.find('x');
    if (x == std::string::npos || x == 0 || x + 1 >= t.size())
        usage_error("structuring element must be WxH, e.g. 7x5");
    return rm::make_se(to_int(t.substr(0, x), "structuring element width"),
                       to_int(t.substr(x + 1), "structuring element height"));
}

rm::BorderPolicy parse_border(const std::string& t) {
    if (t == "replicate") return rm::BorderPolicy::replicate();
    if (t.rfind("constant:", 0) == 0) {
        const int v = to_int(t.substr(9), "border value");
        if (v < 0 || v > 255) usage_error("border value must lie in 0..255");
        return rm::BorderPolicy::constant(std::uint8_t(v));
    }
    usage_error("border must be 'replicate' or 'constant:V'");
}

// MIN..MAX[:STEP]: odd endpoints >= 1, MIN <= MAX, even step >= 2 (default 2)
std::vector<int> parse_windows(const std::string& t) {
    const std::size_t dots = t.find("..");
    if (dots == std::string::npos) usage_error("window range must be MIN..MAX[:STEP]");
    std::string rest = t.substr(dots + 2);
    int step = 2;
    const std::size_t colon = rest.find(':');
    if (colon != std::string::npos) {
        step = to_int(rest.substr(colon + 1), "window step");
        rest = rest.substr(0, colon);
    }
    const int lo = to_int(t.substr(0, dots), "window minimum"), hi = to_int(rest, "window maximum");
    if (lo < 1 || lo % 2 == 0 || hi % 2 == 0) usage_error("window endpoints must be odd and >= 1");
    if (lo > hi) usage_error("window minimum exceeds maximum");
    if (step < 2 || step % 2) usage_error("window step must be even and >= 2");
    std::vector<int> w;
    for (int v = lo; v <= hi; v += step) w.push_back(v);
    return w;
}

// --key value options, --flag flags and positionals of one subcommand
struct Args {
    std::map<std::string, std::string> opt;
    std::set<std::string> flags;
    std::vector<std::string> pos;
    std::string get(const std::string& k, const std::string& dflt = "") const {
        auto it = opt.find(k);
        return it == opt.end() ? dflt : it->second;
    }
    bool has(const std::string& k) const { return opt.count(k) != 0; }
};

Args parse_args(int argc, char** argv, int first, const std::set<std::string>& keys,
                const std::set<std::string>& flag_names) {
    Args a;
    for (int i = first; i < argc; ++i) {
        const std::string s = argv[i];
        if (s.rfind("--", 0) == 0) {
            std::string k = s.substr(2), v;
            const std::size_t eq = k.find('=');
            if (eq != std::string::npos) {
                v = k.substr(eq + 1);
                k = k.substr(0, eq);
            }
            if (flag_names.count(k)) {
                a.flags.insert(k);
                continue;
            }
            if (!keys.count(k)) usage_error("unknown option --" + k);
            if (eq == std::string::npos) {
                if (i + 1 >= argc) usage_error("option --" + k + " needs a value");
                v = argv[++i];
            }
            if (a.opt.count(k)) usage_error("option --" + k + " given twice");
            a.opt[k] = v;
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

const char* kUsage =
    "usage: rectmorph_b200 <apply|bench|calibrate> [options]\n"
    "  apply     --op erode|dilate|open|close|gradient --se WxH [--border replicate|constant:V]\n"
    "            [--config FILE] INPUT.pgm OUTPUT.pgm\n"
    "  bench     --windows MIN..MAX[:STEP] --out FILE.csv [--width W] [--height H] [--reps N]\n"
    "            [--seed S] [--transpose]\n"
    "  calibrate --windows MIN..MAX[:STEP] --out FILE [--width W] [--height H] [--reps N]\n";

void run_apply(const Args& a) {
    if (a.pos.size() != 2) usage_error("apply needs INPUT and OUTPUT paths");
    if (!a.has("op")) usage_error("apply needs --op");
    if (!a.has("se")) usage_error("apply needs --se");
    const std::string op = a.get("op");
    if (op != "erode" && op != "dilate" && op != "open" && op != "close" && op != "gradient")
        usage_error("--op must be one of erode, dilate, open, close, gradient");
    const rm::StructuringElement se = parse_se(a.get("se"));
    const rm::BorderPolicy border = parse_border(a.get("border", "replicate"));
    const rm::DispatchConfig cfg = a.has("config") ? rm::load_config(a.get("config")) : rm::DispatchConfig{};
    const rm::Image src = rm::load_pgm(a.pos[0]);
    rm::Image out;
    if (op == "erode") out = rm::erode(src, se, border, cfg);
    else if (op == "dilate") out = rm::dilate(src, se, border, cfg);
    else if (op == "open") out = rm::opening(src, se, border, cfg);
    else if (op == "close") out = rm::closing(src, se, border, cfg);
    else out = rm::gradient(src, se, border, cfg);
    rm::store_pgm(a.pos[1], out);
}

int extent(const Args& a, const char* key, int dflt) {
    const int v = a.has(key) ? to_int(a.get(key), std::string("--") + key) : dflt;
    if (v < 1 || v > (1 << 20)) usage_error(std::string("--") + key + " must lie in 1..1048576");
    return v;
}

int reps_of(const Args& a) {
    const int v = a.has("reps") ? to_int(a.get("reps"), "--reps") : 21;
    if (v < 1 || v > 10000) usage_error("--reps must lie in 1..10000");
    return v;
}

std::uint64_t median(std::vector<std::uint64_t> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw rm::GpuError(RMGPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// One bench row: the host-buffer call (drop-in path, H2D + kernels + D2H) timed on the host
// clock like the reference's timing::median_ns, and the same pass on device buffers timed with
// CUDA events (device_median_ns, the GPU column added to the reference's schema).
struct Bench {
    const rm::Image& img;
    int reps;
    void* d_src = nullptr;
    void* d_dst = nullptr;
    size_t pitch = 0;
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    std::vector<std::uint8_t> host_out;

    explicit Bench(const rm::Image& i, int r) : img(i), reps(r) {
        pitch = img.stride();
        cuda_check(cudaMalloc(&d_src, pitch * img.height()), "cudaMalloc");
        cuda_check(cudaMalloc(&d_dst, pitch * img.height()), "cudaMalloc");
        cuda_check(cudaMemcpy(d_src, img.row(0), pitch * img.height(), cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaStreamCreate(&s), "stream");
        cuda_check(cudaEventCreate(&e0), "event");
        cuda_check(cudaEventCreate(&e1), "event");
        host_out.resize(pitch * img.height());
    }
    ~Bench() {
        cudaFree(d_src);
        cudaFree(d_dst);
        cudaStreamDestroy(s);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    // pass of window w along one axis with an explicit algorithm hint; returns {host ns, device ns}
    std::pair<std::uint64_t, std::uint64_t> pass(bool horizontal, int w, int algo) {
        const int wx = horizontal ? w : 1, wy = horizontal ? 1 : w;
        const int ah = horizontal ? algo : RMGPU_ALGO_AUTO, av = horizontal ? RMGPU_ALGO_AUTO : algo;
        std::vector<std::uint64_t> th, td;
        for (int k = 0; k <= reps; ++k) {  // k = 0: warm-up
            const auto t0 = std::chrono::steady_clock::now();
            int rc = rmgpu_morph_host_u8(img.row(0), pitch, host_out.data(), pitch, img.width(), img.height(), wx, wy,
                                         RMGPU_ERODE, RMGPU_BORDER_REPLICATE, 0, ah, av);
            const auto t1 = std::chrono::steady_clock::now();
            if (rc) throw rm::GpuError(rc, rmgpu_last_error());
            cuda_check(cudaEventRecord(e0, s), "record");
            rc = rmgpu_morph_u8(d_src, pitch, d_dst, pitch, img.width(), img.height(), wx, wy, RMGPU_ERODE,
                                RMGPU_BORDER_REPLICATE, 0, ah, av, s);
            if (rc) throw rm::GpuError(rc, rmgpu_last_error());
            cuda_check(cudaEventRecord(e1, s), "record");
            cuda_check(cudaEventSynchronize(e1), "sync");
            float ms = 0;
            cuda_check(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
            if (k) {
                th.push_back(std::uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count()));
                td.push_back(std::uint64_t(ms * 1e6));
            }
        }
        return {median(th), median(td)};
    }
};

void run_bench(const Args& a) {
    if (!a.has("windows")) usage_error("bench needs --windows");
    if (!a.has("out")) usage_error("bench needs --out");
    const std::vector<int> windows = parse_windows(a.get("windows"));
    const int w = extent(a, "width", 800), h = extent(a, "height", 600), reps = reps_of(a);
    const std::uint32_t seed = a.has("seed") ? std::uint32_t(to_int(a.get("seed"), "--seed")) : 1u;
    rm::Image img(w, h);
    std::mt19937 rng(seed);
    std::uniform_int_distribution<int> dist(0, 255);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) img.at(x, y) = std::uint8_t(dist(rng));
    std::ofstream csv(a.get("out"), std::ios::binary);
    if (!csv) throw rm::Error(rm::Errc::IoError, "cannot open '" + a.get("out") + "' for writing");
    // the reference's columns (rectmorph_cli.cpp:163) + the device time of the same call
    csv << "axis,algorithm,window,image_w,image_h,reps,median_ns,device_median_ns\n";
    Bench b(img, reps);
    for (int win : windows) {
        for (int axis = 0; axis < 2; ++axis)
            for (int algo : {RMGPU_ALGO_LINEAR, RMGPU_ALGO_VANHERK}) {
                const auto t = b.pass(axis == 0, win, algo);
                csv << (axis == 0 ? "horizontal" : "vertical") << ',' << (algo == RMGPU_ALGO_LINEAR ? "linear" : "vanherk")
                    << ',' << win << ',' << w << ',' << h << ',' << reps << ',' << t.first << ',' << t.second << '\n';
            }
    }
    if (a.flags.count("transpose")) {
        std::vector<std::uint64_t> th;
        for (int k = 0; k <= reps; ++k) {
            const auto t0 = std::chrono::steady_clock::now();
            rm::Image t = rm::transpose_image(img);
            const auto t1 = std::chrono::steady_clock::now();
            if (k) th.push_back(std::uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count()));
            (void)t;
        }
        csv << "transpose,tiled,0," << w << ',' << h << ',' << reps << ',' << median(th) << ",\n";
    }
    csv.flush();
    if (!csv) throw rm::Error(rm::Errc::IoError, "failed writing '" + a.get("out") + "'");
}

void run_calibrate(const Args& a) {
    if (!a.has("windows")) usage_error("calibrate needs --windows");
    if (!a.has("out")) usage_error("calibrate needs --out");
    const std::vector<int> windows = parse_windows(a.get("windows"));
    const rm::DispatchConfig cfg = rm::calibrate(extent(a, "width", 800), extent(a, "height", 600), windows, reps_of(a));
    rm::save_config(a.get("out"), cfg);
    std::cout << rm::format_config(cfg);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) usage_error("a subcommand is required: apply, bench or calibrate");
        const std::string cmd = argv[1];
        if (cmd == "--help" || cmd == "-h") {
            std::cout << kUsage;
            return 0;
        }
        for (int i = 2; i < argc; ++i)
            if (std::string(argv[i]) == "--help" || std::string(argv[i]) == "-h") {
                std::cout << kUsage;
                return 0;
            }
        if (cmd == "apply") run_apply(parse_args(argc, argv, 2, {"op", "se", "border", "config"}, {}));
        else if (cmd == "bench")
            run_bench(parse_args(argc, argv, 2, {"width", "height", "windows", "reps", "seed", "out"}, {"transpose"}));
        else if (cmd == "calibrate")
            run_calibrate(parse_args(argc, argv, 2, {"width", "height", "windows", "reps", "out"}, {}));
        else usage_error("unknown subcommand '" + cmd + "' (apply, bench or calibrate)");
        return 0;
    } catch (const std::exception& e) {
        std::string msg = e.what();
        for (char& c : msg)
            if (c == '\n') c = ' ';
        std::cerr << "rectmorph: " << msg << '\n';
        return 1;
    }
}

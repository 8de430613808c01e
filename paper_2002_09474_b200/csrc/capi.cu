// capi.cu -- the extern "C" boundary declared in include/rmgpu.h.
//
// Validation mirrors the reference before any work is done (make_se image.cpp:18-24,
// validate_window sliding_extrema.cpp:9-14, check_tile_side transpose.cpp:7-10,
// Image::Image image.cpp:26-31); then the planner picks a kernel. No CPU fallback exists: every
// pixel of every result is produced by a kernel in this library.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/rmgpu.h"
#include "common.cuh"
#include "kernels.h"

namespace rmgpu {
std::atomic<unsigned long long> g_launch_count{0};
}


namespace rmgpu {
namespace {
struct OccKey {
    const void* kern;
    int dev, threads, smem;
    bool operator==(const OccKey& o) const {
        return kern == o.kern && dev == o.dev && threads == o.threads && smem == o.smem;
    }
};
struct OccHash {
    size_t operator()(const OccKey& k) const {
        return std::hash<const void*>()(k.kern) ^ ((size_t)k.dev << 48) ^ ((size_t)k.threads << 32) ^ (size_t)k.smem;
    }
};
std::mutex g_occ_mu;
std::unordered_map<OccKey, int, OccHash> g_occ;
std::unordered_map<OccKey, int, OccHash> g_smem_set;  // (kern, dev) -> dynamic smem limit set so far
int g_sms[64];
}  // namespace

namespace {
std::mutex g_tune_mu;
std::map<std::string, int> g_tune;
}  // namespace

int tune(const char* name, int dflt) {
    {
        std::lock_guard<std::mutex> g(g_tune_mu);
        auto it = g_tune.find(name);
        if (it != g_tune.end()) return it->second;
    }
    std::string env = "RMGPU_";
    for (const char* c = name; *c; ++c) env += (char)toupper((unsigned char)*c);
    const char* v = getenv(env.c_str());
    return v ? atoi(v) : dflt;
}

int kernel_occupancy(const void* kern, int threads, int smem, cudaError_t* err) {
    int dev = 0;
    *err = cudaGetDevice(&dev);
    if (*err != cudaSuccess) return 0;
    const OccKey key{kern, dev, threads, smem};
    {
        std::lock_guard<std::mutex> g(g_occ_mu);
        auto it = g_occ.find(key);
        if (it != g_occ.end()) return it->second;
    }
    {
        // the limit only ever grows: a smaller later setting would break cached larger launches
        std::lock_guard<std::mutex> g(g_occ_mu);
        int& cur = g_smem_set[OccKey{kern, dev, 0, 0}];
        if (smem > cur) {
            *err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (*err != cudaSuccess) return 0;
            cur = smem;
        }
    }
    int occ = 0;
    *err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    if (*err != cudaSuccess) return 0;
    std::lock_guard<std::mutex> g(g_occ_mu);
    g_occ[key] = occ;
    return occ;
}

int device_sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev < 0 || dev >= 64) return 148;
    int v = __atomic_load_n(&g_sms[dev], __ATOMIC_RELAXED);
    if (v) return v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    __atomic_store_n(&g_sms[dev], v, __ATOMIC_RELAXED);
    return v;
}
}  // namespace rmgpu

using rmgpu::MorphJob;

namespace {

thread_local std::string t_last_error;
// Test / tuning hooks: RMGPU_DISABLE_STREAM=1 routes around the TMA kernels (exercises the
// fallback kernels).
const bool g_disable_stream = [] {
    const char* v = getenv("RMGPU_DISABLE_STREAM");
    return v && v[0] == '1';
}();
int fail(int status, const std::string& msg) {
    t_last_error = msg;
    return status;
}

int cuda_fail(cudaError_t e, const char* where) {
    t_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? RMGPU_ERR_OUT_OF_MEMORY : RMGPU_ERR_CUDA;
}

#define RM_CUDA(call)                                   \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// make_se (image.cpp:18-24): zero check on both extents first, then parity.
int check_se(int wx, int wy) {
    if (wx < 1 || wy < 1) return fail(RMGPU_ERR_ZERO_EXTENT, "structuring element extents must be >= 1");
    if (wx % 2 == 0 || wy % 2 == 0) return fail(RMGPU_ERR_EVEN_EXTENT, "structuring element extents must be odd");
    return RMGPU_OK;
}

int check_window(int w) {  // validate_window (sliding_extrema.cpp:9-14)
    if (w < 1) return fail(RMGPU_ERR_ZERO_EXTENT, "window extent must be >= 1");
    if (w % 2 == 0) return fail(RMGPU_ERR_EVEN_EXTENT, "window extent must be odd");
    return RMGPU_OK;
}

int check_device() {
    static std::once_flag once;
    static int status = RMGPU_OK;
    static std::string msg;
    std::call_once(once, [] {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0) {
            status = RMGPU_ERR_NO_DEVICE;
            msg = std::string("no CUDA device: ") + cudaGetErrorString(e);
            return;
        }
    });
    if (status != RMGPU_OK) return fail(status, msg);
    // the architecture of the device the caller is using (cached per device)
    static int arch_ok[64] = {};  // 0 unknown, 1 sm_100, 2 other
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(RMGPU_ERR_NO_DEVICE, "cudaGetDevice failed");
    int ok = (dev >= 0 && dev < 64) ? __atomic_load_n(&arch_ok[dev], __ATOMIC_RELAXED) : 0;
    int major = 0, minor = 0;
    if (!ok) {
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        ok = major == 10 ? 1 : 2;
        if (dev >= 0 && dev < 64) __atomic_store_n(&arch_ok[dev], ok, __ATOMIC_RELAXED);
    }
    if (ok != 1)
        return fail(RMGPU_ERR_NO_DEVICE, "librmgpu is built for sm_100a only; device " + std::to_string(dev) +
                                             " is not sm_100" + (major ? " (sm_" + std::to_string(major) +
                                                                 std::to_string(minor) + ")" : std::string()));
    return RMGPU_OK;
}

int check_image(const void* src, size_t sp, const void* dst, size_t dp, int W, int H, int elem) {
    if (W < 0 || H < 0) return fail(RMGPU_ERR_BAD_ARGUMENT, "image dimensions must be non-negative");
    if (W == 0 || H == 0) return RMGPU_OK;
    if (!src || !dst) return fail(RMGPU_ERR_BAD_ARGUMENT, "null image pointer");
    if (sp < (size_t)W * elem || dp < (size_t)W * elem || sp % elem || dp % elem)
        return fail(RMGPU_ERR_BAD_ARGUMENT, "pitch smaller than a row or not a multiple of the pixel size");
    return RMGPU_OK;
}

int check_op_border(int op, int border, unsigned bval, int elem) {
    if (op < RMGPU_ERODE || op > RMGPU_GRADIENT) return fail(RMGPU_ERR_BAD_ARGUMENT, "unknown morphology op");
    if (border != RMGPU_BORDER_REPLICATE && border != RMGPU_BORDER_CONSTANT)
        return fail(RMGPU_ERR_BAD_ARGUMENT, "unknown border mode");
    if (border == RMGPU_BORDER_CONSTANT && bval > (elem == 1 ? 0xFFu : 0xFFFFu))
        return fail(RMGPU_ERR_BAD_ARGUMENT, "constant border value out of pixel range");
    return RMGPU_OK;
}

// Scratch buffers (compound-op intermediates, two-pass fallback, host-entry staging) come from a
// private stream-ordered pool per device that keeps freed blocks cached between calls, so repeated
// calls never go back to the driver and the application's default pool is left untouched.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> g(mu);
        if (!pools[dev]) {
            cudaMemPoolProps props = {};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&pools[dev], &props);
            if (e != cudaSuccess) return e;
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

// One erode / dilate / gradient over the job's rows. Window-1 axes are a copy
// (separable.cpp:66,88); a 1x1 gradient is all zeros.
int run_single(MorphJob j) {
    static const bool force_kernel = getenv("RMGPU_FORCE_KERNEL") != nullptr;  // tuning: 1x1 through the kernel
    if (j.gx == 0 && j.gy == 0 && !force_kernel) {
        for (int b = 0; b < j.batch; ++b) {
            char* d = static_cast<char*>(j.dst) + (size_t)b * j.dimg;
            const char* s = static_cast<const char*>(j.src) + (size_t)b * j.simg;
            if (j.mode == rmgpu::MODE_GRAD) RM_CUDA(cudaMemset2DAsync(d, j.dp, 0, (size_t)j.W * j.elem, j.H, j.stream));
            else RM_CUDA(cudaMemcpy2DAsync(d, j.dp, s, j.sp, (size_t)j.W * j.elem, j.H, cudaMemcpyDeviceToDevice, j.stream));
        }
        return RMGPU_OK;
    }
    cudaError_t e = cudaSuccess;
    // Pitches / pointers that are not 16-byte aligned (the reference pads rows to 16 bytes,
    // image.cpp:9-14, so only foreign layouts hit this): stage through aligned scratch copies
    // (one 2-D copy in, one out) and run the TMA / vectorised kernels on those, instead of
    // scalar fallback kernels.
    {
        const uintptr_t s0 = reinterpret_cast<uintptr_t>(j.src) - (uintptr_t)((ptrdiff_t)j.above * (ptrdiff_t)j.sp);
        const bool al = ((s0 | reinterpret_cast<uintptr_t>(j.dst) | j.sp | j.dp | (j.batch > 1 ? (j.simg | j.dimg) : 0)) &
                         15) == 0;
        if (!al && !g_disable_stream) {
            const size_t rb = (size_t)j.W * j.elem, tp = (rb + 255) & ~size_t(255);
            const int rin = j.above + j.H + j.below;
            const size_t simg = tp * (size_t)rin, dimg = tp * (size_t)j.H;
            char* buf = nullptr;
            RM_CUDA(scratch_alloc(reinterpret_cast<void**>(&buf), (simg + dimg) * (size_t)j.batch, j.stream));
            int rc = RMGPU_OK;
            for (int b = 0; rc == RMGPU_OK && b < j.batch; ++b) {
                e = cudaMemcpy2DAsync(buf + b * simg, tp, reinterpret_cast<const char*>(s0) + (size_t)b * j.simg, j.sp, rb,
                                      rin, cudaMemcpyDeviceToDevice, j.stream);
                if (e != cudaSuccess) rc = cuda_fail(e, "staging copy in");
            }
            MorphJob k = j;
            k.src = buf + (size_t)j.above * tp;
            k.sp = tp;
            k.simg = simg;
            k.dst = buf + simg * (size_t)j.batch;
            k.dp = tp;
            k.dimg = dimg;
            if (rc == RMGPU_OK) rc = run_single(k);
            for (int b = 0; rc == RMGPU_OK && b < j.batch; ++b) {
                e = cudaMemcpy2DAsync(static_cast<char*>(j.dst) + (size_t)b * j.dimg, j.dp,
                                      static_cast<char*>(k.dst) + b * dimg, tp, rb, j.H, cudaMemcpyDeviceToDevice,
                                      j.stream);
                if (e != cudaSuccess) rc = cuda_fail(e, "staging copy out");
            }
            cudaError_t fe = cudaFreeAsync(buf, j.stream);
            if (rc == RMGPU_OK && fe != cudaSuccess) rc = cuda_fail(fe, "cudaFreeAsync");
            return rc;
        }
    }
    // Explicit algorithm hints (rmgpu.h): Linear on an axis whose wing is >= 4 runs that axis as a
    // direct sliding window (generic pass kernel), the other axis through the planner, via one
    // intermediate; everything else (Auto, VanHerk, Linear on short wings -- where the planner's
    // kernels are direct windows already) is the planner's choice. Results are identical.
    const bool direct_h = j.algo_h == RMGPU_ALGO_LINEAR && j.gx >= 4;
    const bool direct_v = j.algo_v == RMGPU_ALGO_LINEAR && j.gy >= 4;
    if ((direct_h || direct_v) && j.mode != rmgpu::MODE_GRAD) {
        const size_t tp = ((size_t)j.W * j.elem + 255) & ~size_t(255), timg = tp * (size_t)j.H;
        void* tmp = nullptr;
        if (j.gx && j.gy) RM_CUDA(scratch_alloc(&tmp, timg * j.batch, j.stream));
        MorphJob v = j, h = j;
        v.gx = 0;
        v.algo_h = v.algo_v = RMGPU_ALGO_AUTO;
        h.gy = 0;
        h.algo_h = h.algo_v = RMGPU_ALGO_AUTO;
        h.above = h.below = 0;
        if (j.gx && j.gy) {
            v.dst = tmp; v.dp = tp; v.dimg = timg;
            h.src = tmp; h.sp = tp; h.simg = timg;
        }
        int rc = RMGPU_OK;
        if (j.gy) {
            if (direct_v) {
                e = rmgpu::launch_pass_cols(v);
                if (e != cudaSuccess) rc = cuda_fail(e, "direct vertical pass");
            } else {
                rc = run_single(v);
            }
        }
        if (rc == RMGPU_OK && j.gx) {
            if (direct_h) {
                e = rmgpu::launch_pass_rows(h);
                if (e != cudaSuccess) rc = cuda_fail(e, "direct horizontal pass");
            } else {
                rc = run_single(h);
            }
        }
        if (tmp) {
            cudaError_t fe = cudaFreeAsync(tmp, j.stream);
            if (rc == RMGPU_OK && fe != cudaSuccess) rc = cuda_fail(fe, "cudaFreeAsync");
        }
        return rc;
    }
    if (!g_disable_stream && rmgpu::col::launch(j, &e)) {
        if (e != cudaSuccess) return cuda_fail(e, "register-streaming morph kernel");
        return RMGPU_OK;
    }
    // tuning knob: u16 through the phase kernel first (cfg4, 21x21 opening x512: K3 1719 us vs K2
    // 1921 us, so K3 is the default)
    if (!g_disable_stream && j.elem == 2 && rmgpu::tune("u16_phase_first", 0) && rmgpu::phase::launch(j, &e)) {
        if (e != cudaSuccess) return cuda_fail(e, "phase morph kernel");
        return RMGPU_OK;
    }
    if (!g_disable_stream && rmgpu::fuse::launch(j, &e)) {
        if (e != cudaSuccess) return cuda_fail(e, "fused separable kernel");
        return RMGPU_OK;
    }
    if (!g_disable_stream && rmgpu::sep::applicable(j)) {
        const size_t tb = rmgpu::sep::scratch_bytes(j);
        void* tmp = nullptr;
        if (tb) RM_CUDA(scratch_alloc(&tmp, tb, j.stream));
        e = rmgpu::sep::run(j, tmp);
        cudaError_t fe = tb ? cudaFreeAsync(tmp, j.stream) : cudaSuccess;
        if (e != cudaSuccess) return cuda_fail(e, "separable streaming passes");
        if (fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
        return RMGPU_OK;
    }
    if (!g_disable_stream && rmgpu::phase::launch(j, &e)) {
        if (e != cudaSuccess) return cuda_fail(e, "phase morph kernel");
        return RMGPU_OK;
    }
    if (j.mode == rmgpu::MODE_GRAD && !g_disable_stream) {
        // large-window gradient: dilation into scratch and erosion into dst (K3, else the phase
        // kernel), then dst = dilation - erosion (dispatch.cpp:58-71; never negative, no wrap)
        auto minmax = [&](const MorphJob& m, int* rc) -> bool {  // false: neither kernel takes it
            if (rmgpu::sep::applicable(m)) {
                const size_t tb = rmgpu::sep::scratch_bytes(m);
                void* tmp = nullptr;
                cudaError_t ae = tb ? scratch_alloc(&tmp, tb, m.stream) : cudaSuccess;
                if (ae != cudaSuccess) {
                    *rc = cuda_fail(ae, "scratch");
                    return true;
                }
                cudaError_t re = rmgpu::sep::run(m, tmp);
                cudaError_t fe = tb ? cudaFreeAsync(tmp, m.stream) : cudaSuccess;
                if (re != cudaSuccess) *rc = cuda_fail(re, "separable streaming passes (gradient)");
                else if (fe != cudaSuccess) *rc = cuda_fail(fe, "cudaFreeAsync");
                return true;
            }
            cudaError_t pe = cudaSuccess;
            if (!rmgpu::phase::launch(m, &pe)) return false;
            if (pe != cudaSuccess) *rc = cuda_fail(pe, "phase morph kernel (gradient)");
            return true;
        };
        const size_t rb = (size_t)j.W * j.elem, tp = (rb + 255) & ~size_t(255), timg = tp * (size_t)j.H;
        MorphJob mx = j, mn = j;
        mx.mode = rmgpu::MODE_MAX;
        mn.mode = rmgpu::MODE_MIN;
        {
            void* hi = nullptr;
            RM_CUDA(scratch_alloc(&hi, timg * j.batch, j.stream));
            mx.dst = hi; mx.dp = tp; mx.dimg = timg;
            // K3 needs 16-byte aligned pitches on both sides: the scratch has them; when dst does not,
            // sep::applicable(mn) is false and the phase kernel (or the fallbacks below) take over
            int rc = RMGPU_OK;
            if (!minmax(mx, &rc) || (rc == RMGPU_OK && !minmax(mn, &rc))) {
                cudaFreeAsync(hi, j.stream);  // neither kernel takes this shape: the fallbacks below do
                goto gradient_fallback;
            }
            for (int b = 0; rc == RMGPU_OK && b < j.batch; ++b) {
                char* d = static_cast<char*>(j.dst) + b * j.dimg;
                e = rmgpu::launch_subtract(static_cast<char*>(hi) + b * timg, tp, d, j.dp, d, j.dp, j.W, j.H, j.elem,
                                           j.stream);
                if (e != cudaSuccess) rc = cuda_fail(e, "subtract");
            }
            cudaError_t fe = cudaFreeAsync(hi, j.stream);
            if (rc == RMGPU_OK && fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
            return rc;
        }
    }
gradient_fallback:
    if (rmgpu::generic_tile_fits(j)) {
        e = rmgpu::launch_generic_tile(j);
        if (e != cudaSuccess) return cuda_fail(e, "generic morph kernel");
        return RMGPU_OK;
    }
    // Very large windows: two global 1-D passes through an intermediate buffer.
    const size_t row_bytes = (size_t)j.W * j.elem;
    const size_t tmp_pitch = (row_bytes + 255) & ~size_t(255);
    const size_t tmp_img = tmp_pitch * (size_t)j.H;
    const int nbuf = j.mode == rmgpu::MODE_GRAD ? 3 : 1;
    void* tmp = nullptr;
    RM_CUDA(scratch_alloc(&tmp, tmp_img * j.batch * nbuf, j.stream));
    auto run_pair = [&](int mode, void* out, size_t out_pitch, size_t out_img) -> int {
        MorphJob v = j;
        v.mode = mode;
        v.dst = tmp;
        v.dp = tmp_pitch;
        v.dimg = tmp_img;
        e = rmgpu::launch_pass_cols(v);
        if (e != cudaSuccess) return cuda_fail(e, "vertical pass");
        MorphJob h = j;
        h.mode = mode;
        h.src = tmp;
        h.sp = tmp_pitch;
        h.simg = tmp_img;
        h.above = h.below = 0;
        h.dst = out;
        h.dp = out_pitch;
        h.dimg = out_img;
        e = rmgpu::launch_pass_rows(h);
        if (e != cudaSuccess) return cuda_fail(e, "horizontal pass");
        return RMGPU_OK;
    };
    int rc;
    if (j.mode != rmgpu::MODE_GRAD) {
        rc = run_pair(j.mode, j.dst, j.dp, j.dimg);
    } else {
        char* hi = static_cast<char*>(tmp) + tmp_img * j.batch;
        char* lo = hi + tmp_img * j.batch;
        rc = run_pair(rmgpu::MODE_MAX, hi, tmp_pitch, tmp_img);
        if (rc == RMGPU_OK) rc = run_pair(rmgpu::MODE_MIN, lo, tmp_pitch, tmp_img);
        for (int b = 0; rc == RMGPU_OK && b < j.batch; ++b) {
            e = rmgpu::launch_subtract(hi + b * tmp_img, tmp_pitch, lo + b * tmp_img, tmp_pitch,
                                       static_cast<char*>(j.dst) + b * j.dimg, j.dp, j.W, j.H, j.elem, j.stream);
            if (e != cudaSuccess) rc = cuda_fail(e, "subtract");
        }
    }
    cudaError_t fe = cudaFreeAsync(tmp, j.stream);
    if (rc == RMGPU_OK && fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
    return rc;
}

// Full op (erode/dilate/open/close/gradient) over a whole image, batch or row band.
int run_morph(const void* src, size_t sp, size_t simg, void* dst, size_t dp, size_t dimg, int batch, int W,
              int H, int above, int below, int wx, int wy, int op, int border, unsigned bval, int elem,
              cudaStream_t stream, int algo_h = RMGPU_ALGO_AUTO, int algo_v = RMGPU_ALGO_AUTO) {
    int rc;
    if ((rc = check_se(wx, wy))) return rc;
    if ((rc = check_op_border(op, border, bval, elem))) return rc;
    if ((rc = check_image(src, sp, dst, dp, W, H, elem))) return rc;
    if (above < 0 || below < 0 || batch < 0) return fail(RMGPU_ERR_BAD_ARGUMENT, "negative halo or batch");
    if (W == 0 || H == 0 || batch == 0) return RMGPU_OK;
    {
        // context rows past the ones a window can reach are never read (every valid tap of every
        // output row is already inside [-reach, H + reach)): drop them, so a caller that passes a
        // whole image as context pays only for the halo (compound ops reach two wings)
        const int reach = (op == RMGPU_OPEN || op == RMGPU_CLOSE) ? 2 * (wy / 2) : wy / 2;
        above = std::min(above, reach);
        below = std::min(below, reach);
    }
    if ((rc = check_device())) return rc;

    MorphJob j;
    j.src = src; j.sp = sp; j.dst = dst; j.dp = dp; j.W = W; j.H = H;
    j.above = above; j.below = below;
    // Wings past the valid extent change nothing (every valid tap is already inside the window and
    // at least one tap is outside it), so clamp them to keep tiles bounded.
    j.gx = std::min(wx / 2, W);
    j.gy = std::min(wy / 2, H + above + below);
    j.cmode = border; j.bval = bval; j.elem = elem; j.batch = batch; j.simg = simg; j.dimg = dimg;
    j.stream = stream;
    if (algo_h < RMGPU_ALGO_AUTO || algo_h > RMGPU_ALGO_VANHERK || algo_v < RMGPU_ALGO_AUTO ||
        algo_v > RMGPU_ALGO_VANHERK)
        return fail(RMGPU_ERR_BAD_ARGUMENT, "unknown pass algorithm");
    j.algo_h = algo_h;
    j.algo_v = algo_v;

    if (op == RMGPU_ERODE || op == RMGPU_DILATE || op == RMGPU_GRADIENT) {
        j.mode = op == RMGPU_ERODE ? rmgpu::MODE_MIN : op == RMGPU_DILATE ? rmgpu::MODE_MAX : rmgpu::MODE_GRAD;
        return run_single(j);
    }
    if (!g_disable_stream && above == 0 && below == 0 && algo_h != RMGPU_ALGO_LINEAR && algo_v != RMGPU_ALGO_LINEAR) {
        MorphJob c = j;
        c.mode = op == RMGPU_OPEN ? rmgpu::MODE_MIN : rmgpu::MODE_MAX;
        if (rmgpu::sep::compound_applicable(c)) {
            void* tmp = nullptr;
            RM_CUDA(scratch_alloc(&tmp, rmgpu::sep::compound_scratch_bytes(c), stream));
            cudaError_t ce = rmgpu::sep::run_compound(c, tmp);
            cudaError_t fe = cudaFreeAsync(tmp, stream);
            if (ce != cudaSuccess) return cuda_fail(ce, "opening/closing (K3, fused horizontal passes)");
            if (fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
            return RMGPU_OK;
        }
    }
    // opening = dilate(erode(x)), closing = erode(dilate(x)) (dispatch.cpp:48-56): the first stage
    // runs over the band plus up to one wing of halo rows, its result is a real image whose border
    // (the true image border) is re-applied by the second stage.
    const int ia = std::min(above, j.gy), ib = std::min(below, j.gy);
    const int IH = H + ia + ib;
    const size_t row_bytes = (size_t)W * elem;
    const size_t tp = (row_bytes + 255) & ~size_t(255);
    const size_t timg = tp * (size_t)IH;
    void* tmp = nullptr;
    RM_CUDA(scratch_alloc(&tmp, timg * batch, stream));
    MorphJob a = j;
    a.mode = op == RMGPU_OPEN ? rmgpu::MODE_MIN : rmgpu::MODE_MAX;
    a.src = static_cast<const char*>(src) - (ptrdiff_t)ia * (ptrdiff_t)sp;
    a.H = IH;
    a.above = above - ia;
    a.below = below - ib;
    a.gy = std::min(wy / 2, IH + a.above + a.below);
    a.dst = tmp; a.dp = tp; a.dimg = timg;
    rc = run_single(a);
    if (rc == RMGPU_OK) {
        MorphJob b = j;
        b.mode = op == RMGPU_OPEN ? rmgpu::MODE_MAX : rmgpu::MODE_MIN;
        b.src = static_cast<const char*>(tmp) + (size_t)ia * tp;
        b.sp = tp; b.simg = timg;
        b.above = ia; b.below = ib;
        b.gy = std::min(wy / 2, H + ia + ib);
        rc = run_single(b);
    }
    cudaError_t fe = cudaFreeAsync(tmp, stream);
    if (rc == RMGPU_OK && fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
    return rc;
}

// Internal per-thread streams + cached pool for the synchronous host entry points: `stream` runs
// the kernels, `up` / `down` carry the host->device and device->host copies of a pipelined call.
struct HostCtx {
    int device = -1;
    cudaStream_t stream = nullptr, up = nullptr, down = nullptr;
    std::vector<cudaEvent_t> events;
};
thread_local HostCtx t_ctx;

int host_stream(cudaStream_t* out) {
    int rc = check_device();
    if (rc) return rc;
    int dev = 0;
    RM_CUDA(cudaGetDevice(&dev));
    if (t_ctx.stream == nullptr || t_ctx.device != dev) {
        RM_CUDA(cudaStreamCreateWithFlags(&t_ctx.stream, cudaStreamNonBlocking));
        RM_CUDA(cudaStreamCreateWithFlags(&t_ctx.up, cudaStreamNonBlocking));
        RM_CUDA(cudaStreamCreateWithFlags(&t_ctx.down, cudaStreamNonBlocking));
        t_ctx.events.clear();
        t_ctx.device = dev;
    }
    *out = t_ctx.stream;
    return RMGPU_OK;
}

int host_events(size_t n) {
    while (t_ctx.events.size() < n) {
        cudaEvent_t e;
        RM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        t_ctx.events.push_back(e);
    }
    return RMGPU_OK;
}

struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() { if (p) cudaFreeAsync(p, s); }
};

// The band pipeline of one host call, enqueued on `s` (+ the thread's `up` / `down` copy streams,
// forked from and joined back into `s`): band k uploads on `up` as two copies -- its first `halo`
// rows (what band k-1 needs below it) and the rest -- and is computed on `s` once it and the first
// rows of band k+1 have arrived; its result downloads on `down` while later bands still upload, so
// the two copy directions overlap each other and the kernels. The scratch images are allocated and
// freed on `s`.
int enqueue_host_pipeline(const void* hsrc, size_t sp, void* hdst, size_t dp, int W, int H, int wx, int wy,
                          int op, int border, unsigned bval, int elem, int algo_h, int algo_v, size_t pitch,
                          const std::vector<int>& starts, int halo, cudaStream_t s) {
    const int nb = (int)starts.size() - 1;
    int rc;
    const size_t rb = (size_t)W * elem;
    if ((rc = host_events(3 * (size_t)nb + 2))) return rc;
    cudaEvent_t* ev_head = t_ctx.events.data();   // band k's first `halo` rows uploaded
    cudaEvent_t* ev_band = ev_head + nb;          // band k uploaded
    cudaEvent_t* ev_out = ev_band + nb;           // band k computed
    cudaEvent_t ev_start = ev_out[nb], ev_end = ev_out[nb + 1];
    char *a = nullptr, *b = nullptr;
    RM_CUDA(scratch_alloc(reinterpret_cast<void**>(&a), pitch * H, s));
    RM_CUDA(scratch_alloc(reinterpret_cast<void**>(&b), pitch * H, s));
    RM_CUDA(cudaEventRecord(ev_start, s));
    RM_CUDA(cudaStreamWaitEvent(t_ctx.up, ev_start, 0));
    RM_CUDA(cudaStreamWaitEvent(t_ctx.down, ev_start, 0));
    const bool flat_in = sp == rb && pitch == rb, flat_out = dp == rb && pitch == rb;
    auto upload = [&](int r0, int n) -> cudaError_t {
        char* d = a + (size_t)r0 * pitch;
        const char* h = static_cast<const char*>(hsrc) + (size_t)r0 * sp;
        return flat_in ? cudaMemcpyAsync(d, h, rb * n, cudaMemcpyHostToDevice, t_ctx.up)
                       : cudaMemcpy2DAsync(d, pitch, h, sp, rb, n, cudaMemcpyHostToDevice, t_ctx.up);
    };
    for (int k = 0; k < nb; ++k) {
        const int r0 = starts[k], n = starts[k + 1] - r0, head = std::min(n, halo);
        if (head > 0 && head < n) RM_CUDA(upload(r0, head));
        RM_CUDA(cudaEventRecord(ev_head[k], t_ctx.up));
        RM_CUDA(upload(r0 + (head < n ? head : 0), head < n ? n - head : n));
        RM_CUDA(cudaEventRecord(ev_band[k], t_ctx.up));
    }
    for (int k = 0; rc == RMGPU_OK && k < nb; ++k) {
        const int r0 = starts[k], n = starts[k + 1] - r0;
        RM_CUDA(cudaStreamWaitEvent(s, ev_band[k], 0));
        if (k + 1 < nb) RM_CUDA(cudaStreamWaitEvent(s, ev_head[k + 1], 0));  // halo rows below
        const int above = std::min(halo, r0), below = std::min(halo, H - r0 - n);
        rc = run_morph(a + (size_t)r0 * pitch, pitch, 0, b + (size_t)r0 * pitch, pitch, 0, 1, W, n, above, below, wx,
                       wy, op, border, bval, elem, s, algo_h, algo_v);
        if (rc) break;
        RM_CUDA(cudaEventRecord(ev_out[k], s));
        RM_CUDA(cudaStreamWaitEvent(t_ctx.down, ev_out[k], 0));
        char* h = static_cast<char*>(hdst) + (size_t)r0 * dp;
        const char* d = b + (size_t)r0 * pitch;
        if (flat_out) RM_CUDA(cudaMemcpyAsync(h, d, rb * n, cudaMemcpyDeviceToHost, t_ctx.down));
        else RM_CUDA(cudaMemcpy2DAsync(h, dp, d, pitch, rb, n, cudaMemcpyDeviceToHost, t_ctx.down));
    }
    // join both copy streams back into `s` before the buffers go back to the pool
    RM_CUDA(cudaEventRecord(ev_end, t_ctx.down));
    RM_CUDA(cudaStreamWaitEvent(s, ev_end, 0));
    RM_CUDA(cudaEventRecord(ev_start, t_ctx.up));
    RM_CUDA(cudaStreamWaitEvent(s, ev_start, 0));
    cudaError_t fa = cudaFreeAsync(a, s), fb = cudaFreeAsync(b, s);
    if (rc) return rc;
    if (fa != cudaSuccess) return cuda_fail(fa, "cudaFreeAsync");
    if (fb != cudaSuccess) return cuda_fail(fb, "cudaFreeAsync");
    return RMGPU_OK;
}

// Repeated host calls with the same arguments (a loop over frames, a benchmark) replay the whole
// band pipeline as one CUDA graph: one launch instead of ~10 API calls per band, which lets the
// pipeline use finer bands (shorter fill and drain) without becoming CPU-bound.
struct HostGraphKey {
    const void* hsrc;
    void* hdst;
    size_t sp, dp;
    int W, H, wx, wy, op, border, elem, algo_h, algo_v, nb, dev;
    unsigned bval;
    bool operator==(const HostGraphKey& o) const { return memcmp(this, &o, sizeof o) == 0; }
};
struct HostGraphEntry {
    HostGraphKey key;
    cudaGraphExec_t exec;  // nullptr: capture not possible for this call, run it directly
};
thread_local std::vector<HostGraphEntry> t_graphs;
thread_local std::vector<HostGraphKey> t_seen;  // keys met once (not captured yet)
// host calls in flight (all threads): concurrent callers already keep both PCIe directions busy
std::atomic<int> g_host_inflight{0};
struct InflightGuard {
    int n;
    InflightGuard() : n(g_host_inflight.fetch_add(1, std::memory_order_relaxed) + 1) {}
    ~InflightGuard() { g_host_inflight.fetch_sub(1, std::memory_order_relaxed); }
};

int host_morph(const void* hsrc, size_t sp, void* hdst, size_t dp, int W, int H, int wx, int wy, int op,
               int border, unsigned bval, int elem, int algo_h, int algo_v) {
    int rc;
    if ((rc = check_se(wx, wy))) return rc;
    if ((rc = check_op_border(op, border, bval, elem))) return rc;
    if ((rc = check_image(hsrc, sp, hdst, dp, W, H, elem))) return rc;
    if (W == 0 || H == 0) return RMGPU_OK;
    cudaStream_t s;
    if ((rc = host_stream(&s))) return rc;
    // device rows as tight as the kernels allow (16-byte pitch): a host image whose rows are
    // already that tight then moves as one flat copy instead of a 2-D copy of H short rows
    const size_t rb = (size_t)W * elem, pitch = rb % 16 == 0 ? rb : (rb + 255) & ~size_t(255);
    const int halo = (op == RMGPU_OPEN || op == RMGPU_CLOSE) ? 2 * (wy / 2) : wy / 2;
    const bool big = rb * (size_t)H >= ((size_t)8 << 20);
    const bool graphs = rmgpu::tune("host_graph", 1) != 0;
    // bands (4096^2 u8, tools/e2e_probe.py): the fill (first band up) and drain (last band down)
    // shrink with more bands but every copy has a fixed cost on the copy engines: 2-4 bands with the
    // head rows uploaded separately measured best (0.52-0.56 ms per call; 6 bands 0.55-0.59,
    // 16 bands 0.72; round 1's 6 bands without the head split 0.58)
    // Concurrent callers (other threads inside a host call right now): whole-image calls, the
    // callers' uploads and downloads interleave on their own (2 threads, 4096^2 u8: 42.3 Gpix/s
    // unbanded = 98% of the measured duplex PCIe rate, 35.6 with 3 bands each; a single caller
    // 31.4 with 3 bands, 25.8 unbanded).
    const InflightGuard inflight;
    // Images of hundreds of MB: a band per 64 MB up to 16 (the fill and drain are one band each and
    // the per-copy cost no longer matters: 1 GiB in 16 bands ~ 1/16 of the transfer time exposed).
    const int by_size = (int)std::min<size_t>(16, std::max<size_t>(3, (rb * (size_t)H) >> 26));
    const int nb_target = rmgpu::tune("host_bands", big ? (inflight.n > 1 ? 1 : by_size) : 1);
    const int R = std::max({halo, 64, (H + nb_target - 1) / std::max(1, nb_target)});
    const int nb = (H + R - 1) / R;
    // band rows: the first and last bands half as tall as the others (weights 1, 2, ..., 2, 1), so
    // the pipeline's fill (first band up before any kernel) and drain (last band down after the
    // last kernel) shrink without adding copies
    std::vector<int> starts(1, 0);
    if (nb >= 3 && rmgpu::tune("host_taper", 1)) {
        const double unit = (double)H / (2.0 * nb - 2.0);
        for (int k = 1; k < nb; ++k) starts.push_back((int)std::lround(unit * (2.0 * k - 1.0)));
    } else {
        for (int k = 1; k < nb; ++k) starts.push_back(std::min(H, k * R));
    }
    starts.push_back(H);
    for (int k = 1; k <= nb; ++k)  // every band at least one halo (and 16 rows) tall
        if (starts[k] - starts[k - 1] < std::max(halo, 16)) {
            starts.assign(1, 0);
            for (int m = 1; m < nb; ++m) starts.push_back(std::min(H, m * R));
            starts.push_back(H);
            break;
        }
    if (nb < 2) {
        DevBuf a, b;
        a.s = b.s = s;
        RM_CUDA(scratch_alloc(&a.p, pitch * H, s));
        RM_CUDA(scratch_alloc(&b.p, pitch * H, s));
        if (sp == rb && pitch == rb) RM_CUDA(cudaMemcpyAsync(a.p, hsrc, rb * H, cudaMemcpyHostToDevice, s));
        else RM_CUDA(cudaMemcpy2DAsync(a.p, pitch, hsrc, sp, rb, H, cudaMemcpyHostToDevice, s));
        rc = run_morph(a.p, pitch, 0, b.p, pitch, 0, 1, W, H, 0, 0, wx, wy, op, border, bval, elem, s, algo_h, algo_v);
        if (rc) return rc;
        if (dp == rb && pitch == rb) RM_CUDA(cudaMemcpyAsync(hdst, b.p, rb * H, cudaMemcpyDeviceToHost, s));
        else RM_CUDA(cudaMemcpy2DAsync(hdst, dp, b.p, pitch, rb, H, cudaMemcpyDeviceToHost, s));
        RM_CUDA(cudaStreamSynchronize(s));
        return RMGPU_OK;
    }
    auto direct = [&]() -> int {
        int r = enqueue_host_pipeline(hsrc, sp, hdst, dp, W, H, wx, wy, op, border, bval, elem, algo_h, algo_v, pitch,
                                      starts, halo, s);
        // on an error, wait for everything queued (copies may still use the freed buffers' memory)
        cudaError_t e1 = cudaStreamSynchronize(t_ctx.up), e2 = cudaStreamSynchronize(t_ctx.down);
        cudaError_t e3 = cudaStreamSynchronize(s);
        if (r) return r;
        if (e1 != cudaSuccess) return cuda_fail(e1, "host pipeline (uploads)");
        if (e2 != cudaSuccess) return cuda_fail(e2, "host pipeline (downloads)");
        if (e3 != cudaSuccess) return cuda_fail(e3, "host pipeline");
        return RMGPU_OK;
    };
    if (!graphs) return direct();
    // graphs only for page-locked host buffers (memcpy nodes from pageable memory are not async)
    for (const void* hp : {hsrc, static_cast<const void*>(hdst)}) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, hp) != cudaSuccess || at.type != cudaMemoryTypeHost) {
            cudaGetLastError();
            return direct();
        }
    }
    HostGraphKey key{};
    memset(&key, 0, sizeof key);
    key.hsrc = hsrc; key.hdst = hdst; key.sp = sp; key.dp = dp; key.W = W; key.H = H; key.wx = wx; key.wy = wy;
    key.op = op; key.border = border; key.elem = elem; key.algo_h = algo_h; key.algo_v = algo_v; key.nb = nb;
    key.bval = bval;
    RM_CUDA(cudaGetDevice(&key.dev));
    for (size_t gi = 0; gi < t_graphs.size(); ++gi)
        if (t_graphs[gi].key == key) {
            const HostGraphEntry g = t_graphs[gi];
            if (gi + 1 != t_graphs.size()) {  // most recently used last
                t_graphs.erase(t_graphs.begin() + (ptrdiff_t)gi);
                t_graphs.push_back(g);
            }
            if (!g.exec) return direct();
            RM_CUDA(cudaGraphLaunch(g.exec, s));
            RM_CUDA(cudaStreamSynchronize(s));
            return RMGPU_OK;
        }
    // A key seen for the first time runs directly and is only remembered: a caller that streams new
    // buffers through (every call a new key) never pays for captures it would not replay. The second
    // call with the same key captures the pipeline; a call that cannot be captured runs directly
    // from then on.
    bool seen_once = false;
    for (size_t gi = 0; gi < t_seen.size(); ++gi)
        if (t_seen[gi] == key) {
            seen_once = true;
            t_seen.erase(t_seen.begin() + (ptrdiff_t)gi);
            break;
        }
    if (!seen_once) {
        if (t_seen.size() >= 64) t_seen.erase(t_seen.begin());
        t_seen.push_back(key);
        return direct();
    }
    cudaGraphExec_t exec = nullptr;
    cudaError_t ce = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (ce == cudaSuccess) {
        rc = enqueue_host_pipeline(hsrc, sp, hdst, dp, W, H, wx, wy, op, border, bval, elem, algo_h, algo_v, pitch,
                                   starts, halo, s);
        cudaGraph_t graph = nullptr;
        ce = cudaStreamEndCapture(s, &graph);
        if (rc == RMGPU_OK && ce == cudaSuccess && graph) ce = cudaGraphInstantiate(&exec, graph, 0);
        if (graph) cudaGraphDestroy(graph);
        if (rc != RMGPU_OK || ce != cudaSuccess) exec = nullptr;
    }
    cudaGetLastError();  // a failed capture leaves a sticky-free error behind
    // least recently used out; room for a sweep of windows and ops over one pair of buffers (a
    // cache of 8 thrashed on the 16 operations of a cfg2 step: every call captured again)
    if (t_graphs.size() >= (size_t)std::max(1, rmgpu::tune("host_graph_cache", 64))) {
        if (t_graphs.front().exec) cudaGraphExecDestroy(t_graphs.front().exec);
        t_graphs.erase(t_graphs.begin());
    }
    t_graphs.push_back({key, exec});
    if (!exec) return direct();
    RM_CUDA(cudaGraphLaunch(exec, s));
    RM_CUDA(cudaStreamSynchronize(s));
    return RMGPU_OK;
}

int pass_impl(int which, const void* src, size_t sp, void* dst, size_t dp, int W, int H, int window, int op,
              int border, unsigned bval, cudaStream_t s) {
    int rc;
    if ((rc = check_window(window))) return rc;
    if (which < RMGPU_PASS_HORIZONTAL || which > RMGPU_PASS_VERTICAL_VIA_TRANSPOSE)
        return fail(RMGPU_ERR_BAD_ARGUMENT, "unknown pass");
    if (op != RMGPU_ERODE && op != RMGPU_DILATE) return fail(RMGPU_ERR_BAD_ARGUMENT, "pass op must be erode or dilate");
    const int wx = which == RMGPU_PASS_HORIZONTAL ? window : 1;
    const int wy = which == RMGPU_PASS_HORIZONTAL ? 1 : window;
    return run_morph(src, sp, 0, dst, dp, 0, 1, W, H, 0, 0, wx, wy, op, border, bval, 1, s);
}

}  // namespace

// =================================================================================================
extern "C" {

int rmgpu_abi_version(void) { return RMGPU_ABI_VERSION; }

const char* rmgpu_last_error(void) { return t_last_error.c_str(); }

const char* rmgpu_status_string(int status) {
    switch (status) {
    case RMGPU_OK: return "ok";
    case RMGPU_ERR_ZERO_EXTENT: return "ZeroExtent";
    case RMGPU_ERR_EVEN_EXTENT: return "EvenExtent";
    case RMGPU_ERR_UNSUPPORTED_TILE: return "UnsupportedTile";
    case RMGPU_ERR_BAD_CONFIG: return "BadConfig";
    case RMGPU_ERR_BAD_ARGUMENT: return "BadArgument";
    case RMGPU_ERR_CUDA: return "CudaError";
    case RMGPU_ERR_NO_DEVICE: return "NoDevice";
    case RMGPU_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    default: return "unknown";
    }
}

unsigned long long rmgpu_launch_count(void) { return rmgpu::g_launch_count.load(); }

// Debug: record a clock64 timeline of one CTA of the streaming kernel into a device buffer of
// >= 1024 int64 (nullptr disables). Not part of the reference API.
void rmgpu_debug_trace(void* device_buf, int cta) { rmgpu::stream::set_trace((long long*)device_buf, cta); }

void rmgpu_debug_set(const char* knob, int value) {
    if (!knob) return;
    std::lock_guard<std::mutex> g(rmgpu::g_tune_mu);
    if (value < 0) rmgpu::g_tune.erase(knob);
    else rmgpu::g_tune[knob] = value;
}

int rmgpu_format_config(int threshold_h, int threshold_v, int source, char* buf, size_t cap) {
    const std::string text = "threshold_h=" + std::to_string(threshold_h) + "\nthreshold_v=" +
                             std::to_string(threshold_v) + "\nsource=" +
                             (source == RMGPU_SOURCE_CALIBRATED ? "calibrated" : "paper") + "\n";
    if (buf && cap) {
        const size_t n = std::min(cap - 1, text.size());
        memcpy(buf, text.data(), n);
        buf[n] = 0;
    }
    return (int)text.size();
}

int rmgpu_parse_config(const char* text, int* threshold_h, int* threshold_v, int* source) {
    if (!text) return fail(RMGPU_ERR_BAD_ARGUMENT, "null config text");
    auto strip = [](std::string v) {
        size_t a = 0, b = v.size();
        while (a < b && (v[a] == ' ' || v[a] == '\t')) ++a;
        while (b > a && (v[b - 1] == ' ' || v[b - 1] == '\t' || v[b - 1] == '\r')) --b;
        return v.substr(a, b - a);
    };
    auto bad = [](int line, const std::string& what) {
        return fail(RMGPU_ERR_BAD_CONFIG, "config line " + std::to_string(line) + ": " + what);
    };
    int th = 0, tv = 0, src = RMGPU_SOURCE_PAPER;
    bool have_h = false, have_v = false, have_s = false;
    const std::string all(text);
    size_t pos = 0;
    int line = 0;
    while (pos <= all.size()) {
        size_t nl = all.find('\n', pos);
        if (nl == std::string::npos) nl = all.size();
        const std::string ln = strip(all.substr(pos, nl - pos));
        ++line;
        pos = nl + 1;
        if (ln.empty() || ln[0] == '#') {
            if (nl == all.size()) break;
            continue;
        }
        const size_t eq = ln.find('=');
        if (eq == std::string::npos) return bad(line, "expected key=value");
        const std::string key = strip(ln.substr(0, eq)), val = strip(ln.substr(eq + 1));
        if (key == "threshold_h" || key == "threshold_v") {
            bool& seen = key == "threshold_h" ? have_h : have_v;
            if (seen) return bad(line, "duplicate key '" + key + "'");
            // a whole decimal integer (optional sign), positive and odd
            bool ok = !val.empty();
            long long v = 0;
            size_t i = (val[0] == '-' || val[0] == '+') ? 1 : 0;
            if (i == val.size()) ok = false;
            for (; ok && i < val.size(); ++i) {
                if (val[i] < '0' || val[i] > '9') ok = false;
                else if ((v = v * 10 + (val[i] - '0')) > 0x7fffffff) ok = false;
            }
            if (!ok) return bad(line, "expected an integer, got '" + val + "'");
            if (val[0] == '-') v = -v;
            if (v < 1 || v % 2 == 0) return bad(line, "threshold must be a positive odd integer");
            (key == "threshold_h" ? th : tv) = (int)v;
            seen = true;
        } else if (key == "source") {
            if (have_s) return bad(line, "duplicate key 'source'");
            if (val == "paper") src = RMGPU_SOURCE_PAPER;
            else if (val == "calibrated") src = RMGPU_SOURCE_CALIBRATED;
            else return bad(line, "source must be 'paper' or 'calibrated'");
            have_s = true;
        } else {
            return bad(line, "unknown key '" + key + "'");
        }
        if (nl == all.size()) break;
    }
    if (!have_h || !have_v || !have_s) return fail(RMGPU_ERR_BAD_CONFIG, "config must set threshold_h, threshold_v and source");
    if (threshold_h) *threshold_h = th;
    if (threshold_v) *threshold_v = tv;
    if (source) *source = src;
    return RMGPU_OK;
}

int rmgpu_calibrate(int width, int height, const int* windows, int n_windows, int reps, int* threshold_h,
                    int* threshold_v) {
    // validation in the reference's order (dispatch.cpp:182-194), before any device work
    if (width < 1 || height < 1) return fail(RMGPU_ERR_BAD_ARGUMENT, "calibration image extents must be >= 1");
    if (reps < 3) return fail(RMGPU_ERR_INSUFFICIENT_REPS, "calibration needs at least 3 repetitions");
    if (n_windows < 1 || !windows) return fail(RMGPU_ERR_BAD_ARGUMENT, "calibration needs at least one window");
    for (int i = 0; i < n_windows; ++i) {
        int rc = check_window(windows[i]);
        if (rc) return rc;
        if (i > 0 && windows[i] <= windows[i - 1])
            return fail(RMGPU_ERR_BAD_ARGUMENT, "calibration windows must be strictly ascending");
    }
    int rc = check_device();
    if (rc) return rc;
    cudaStream_t s = nullptr;
    RM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    } sg{s};
    const size_t pitch = ((size_t)width + 255) & ~size_t(255);
    void *src = nullptr, *dst = nullptr;
    RM_CUDA(cudaMallocAsync(&src, pitch * height, s));
    RM_CUDA(cudaMallocAsync(&dst, pitch * height, s));
    struct BufGuard {
        void *a, *b;
        cudaStream_t s;
        ~BufGuard() { cudaFreeAsync(a, s); cudaFreeAsync(b, s); }
    } bg{src, dst, s};
    // deterministic pixels: repeated calibrations time identical data (dispatch.cpp:196-201)
    RM_CUDA(rmgpu::launch_generate(src, pitch, width, height, 0x7261746Dull, 0, 1, s));
    cudaEvent_t e0, e1;
    RM_CUDA(cudaEventCreate(&e0));
    RM_CUDA(cudaEventCreate(&e1));
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); }
    } eg{e0, e1};
    // median over reps of one pass (erosion, replicate) with the given axis / algorithm
    auto median_ms = [&](int wx, int wy, int ah, int av, float* out) -> int {
        std::vector<float> t;
        for (int k = 0; k <= reps; ++k) {  // k = 0: warm-up (planner caches, first launch)
            RM_CUDA(cudaEventRecord(e0, s));
            int r = run_morph(src, pitch, 0, dst, pitch, 0, 1, width, height, 0, 0, wx, wy, RMGPU_ERODE,
                              RMGPU_BORDER_REPLICATE, 0, 1, s, ah, av);
            if (r) return r;
            RM_CUDA(cudaEventRecord(e1, s));
            RM_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            RM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (k) t.push_back(ms);
        }
        std::sort(t.begin(), t.end());
        *out = t[t.size() / 2];
        return RMGPU_OK;
    };
    int best_h = 1, best_v = 1;
    for (int i = 0; i < n_windows; ++i) {
        const int w = windows[i];
        float lin = 0, vh = 0;
        // horizontal pass: w x 1. Wings < 4 have no van Herk kernel: Linear wins by default.
        if ((rc = median_ms(w, 1, RMGPU_ALGO_LINEAR, RMGPU_ALGO_AUTO, &lin))) return rc;
        if (w / 2 >= 4) {
            if ((rc = median_ms(w, 1, RMGPU_ALGO_VANHERK, RMGPU_ALGO_AUTO, &vh))) return rc;
        } else {
            vh = lin;
        }
        if (lin <= vh) best_h = std::max(best_h, w);
        if ((rc = median_ms(1, w, RMGPU_ALGO_AUTO, RMGPU_ALGO_LINEAR, &lin))) return rc;
        if (w / 2 >= 4) {
            if ((rc = median_ms(1, w, RMGPU_ALGO_AUTO, RMGPU_ALGO_VANHERK, &vh))) return rc;
        } else {
            vh = lin;
        }
        if (lin <= vh) best_v = std::max(best_v, w);
    }
    if (threshold_h) *threshold_h = best_h;
    if (threshold_v) *threshold_v = best_v;
    return RMGPU_OK;
}

int rmgpu_resolve(int algo, int window, int axis, int threshold_h, int threshold_v) {
    if (algo != RMGPU_ALGO_AUTO) return algo;  // dispatch.cpp:14-20
    const int t = axis == RMGPU_AXIS_HORIZONTAL ? threshold_h : threshold_v;
    return window <= t ? RMGPU_ALGO_LINEAR : RMGPU_ALGO_VANHERK;
}

const char* rmgpu_plan_name(int elem_bytes, int width, int height, int wx, int wy, int op) {
    MorphJob j;
    j.W = width; j.H = height; j.elem = elem_bytes;
    j.gx = std::min(wx / 2, width);
    j.gy = std::min(wy / 2, height);
    j.mode = op == RMGPU_ERODE ? rmgpu::MODE_MIN : op == RMGPU_DILATE ? rmgpu::MODE_MAX : rmgpu::MODE_GRAD;
    if (op == RMGPU_OPEN || op == RMGPU_CLOSE) j.mode = rmgpu::MODE_MIN;
    if (j.gx == 0 && j.gy == 0) return "copy";
    if (!g_disable_stream)
        if (const char* n = rmgpu::col::plan_name(j)) return n;
    if (!g_disable_stream && j.elem == 2 && rmgpu::tune("u16_phase_first", 0))
        if (const char* n = rmgpu::phase::plan_name(j)) return n;
    if (!g_disable_stream)
        if (const char* n = rmgpu::fuse::plan_name(j)) return n;
    if (!g_disable_stream)
        if (const char* n = rmgpu::sep::plan_name(j)) return n;
    if (!g_disable_stream)
        if (const char* n = rmgpu::phase::plan_name(j)) return n;
    if (j.mode == rmgpu::MODE_GRAD && !g_disable_stream) {
        MorphJob m = j;
        m.mode = rmgpu::MODE_MAX;
        const char* n = rmgpu::sep::plan_name(m);
        if (!n) n = rmgpu::phase::plan_name(m);
        if (n) {
            static thread_local std::string g;
            g = std::string("gradient[2x ") + n + " + subtract]";
            return g.c_str();
        }
    }
    if (rmgpu::generic_tile_fits(j)) return "generic_tile";
    return "two_pass_global";
}

#define MORPH_ENTRY(SFX, ELEM)                                                                          \
    int rmgpu_morph_##SFX(const void* src, size_t sp, void* dst, size_t dp, int W, int H, int wx, int wy,   \
                          int op, int border, unsigned bval, int algo_h, int algo_v, void* stream) {     \
        return run_morph(src, sp, 0, dst, dp, 0, 1, W, H, 0, 0, wx, wy, op, border, bval, ELEM,           \
                         (cudaStream_t)stream, algo_h, algo_v);                                           \
    }                                                                                                     \
    int rmgpu_morph_batched_##SFX(const void* src, size_t sp, size_t simg, void* dst, size_t dp,          \
                                  size_t dimg, int batch, int W, int H, int wx, int wy, int op,           \
                                  int border, unsigned bval, void* stream) {                              \
        return run_morph(src, sp, simg, dst, dp, dimg, batch, W, H, 0, 0, wx, wy, op, border, bval, ELEM, \
                         (cudaStream_t)stream);                                                           \
    }                                                                                                     \
    int rmgpu_morph_band_##SFX(const void* src, size_t sp, void* dst, size_t dp, int W, int rows,         \
                               int above, int below, int wx, int wy, int op, int border, unsigned bval,   \
                               void* stream) {                                                            \
        return run_morph(src, sp, 0, dst, dp, 0, 1, W, rows, above, below, wx, wy, op, border, bval,      \
                         ELEM, (cudaStream_t)stream);                                                     \
    }                                                                                                     \
    int rmgpu_morph_host_##SFX(const void* hsrc, size_t sp, void* hdst, size_t dp, int W, int H, int wx,  \
                               int wy, int op, int border, unsigned bval, int algo_h, int algo_v) {       \
        return host_morph(hsrc, sp, hdst, dp, W, H, wx, wy, op, border, bval, ELEM, algo_h, algo_v);      \
    }

MORPH_ENTRY(u8, 1)
MORPH_ENTRY(u16, 2)

int rmgpu_pass_u8(int which, const void* src, size_t sp, void* dst, size_t dp, int W, int H, int window,
                  int op, int border, unsigned bval, int algo, void* stream) {
    (void)algo;
    return pass_impl(which, src, sp, dst, dp, W, H, window, op, border, bval, (cudaStream_t)stream);
}

int rmgpu_window_1d_u8(const void* in, size_t n, int window, int op, int border, unsigned bval, int algo,
                       void* out, void* stream) {
    (void)algo;
    int rc;
    if ((rc = check_window(window))) return rc;
    if (n == 0) return RMGPU_OK;
    if (n > 0x7fffffff) return fail(RMGPU_ERR_BAD_ARGUMENT, "1-D signal too long");
    if (in != out)
        return pass_impl(RMGPU_PASS_HORIZONTAL, in, n, out, n, (int)n, 1, window, op, border, bval,
                         (cudaStream_t)stream);
    cudaStream_t s = (cudaStream_t)stream;
    void* tmp = nullptr;
    RM_CUDA(scratch_alloc(&tmp, n, s));
    RM_CUDA(cudaMemcpyAsync(tmp, in, n, cudaMemcpyDeviceToDevice, s));
    rc = pass_impl(RMGPU_PASS_HORIZONTAL, tmp, n, out, n, (int)n, 1, window, op, border, bval, s);
    cudaFreeAsync(tmp, s);
    return rc;
}

int rmgpu_transpose_u8(const void* src, size_t sp, void* dst, size_t dp, int W, int H, void* stream) {
    int rc;
    if (W < 0 || H < 0) return fail(RMGPU_ERR_BAD_ARGUMENT, "image dimensions must be non-negative");
    if (W == 0 || H == 0) return RMGPU_OK;
    if (!src || !dst || sp < (size_t)W || dp < (size_t)H) return fail(RMGPU_ERR_BAD_ARGUMENT, "bad transpose buffers");
    if ((rc = check_device())) return rc;
    cudaError_t e = rmgpu::launch_transpose(src, sp, dst, dp, W, H, 1, (cudaStream_t)stream);
    return e == cudaSuccess ? RMGPU_OK : cuda_fail(e, "transpose");
}

int rmgpu_transpose_u16(const void* src, size_t sp, void* dst, size_t dp, int W, int H, void* stream) {
    int rc;
    if (W < 0 || H < 0) return fail(RMGPU_ERR_BAD_ARGUMENT, "image dimensions must be non-negative");
    if (W == 0 || H == 0) return RMGPU_OK;
    if (!src || !dst || sp < 2 * (size_t)W || dp < 2 * (size_t)H || (sp | dp) & 1)
        return fail(RMGPU_ERR_BAD_ARGUMENT, "bad transpose buffers");
    if ((rc = check_device())) return rc;
    cudaError_t e = rmgpu::launch_transpose(src, sp, dst, dp, W, H, 2, (cudaStream_t)stream);
    return e == cudaSuccess ? RMGPU_OK : cuda_fail(e, "transpose");
}

static int tiles_impl(void* data, size_t n_tiles, int n, size_t rs, size_t step, int elem, void* stream) {
    int rc;
    if (n != 4 && n != 8 && n != 16) return fail(RMGPU_ERR_UNSUPPORTED_TILE, "tile side must be 4, 8 or 16");
    if (n_tiles == 0) return RMGPU_OK;
    if (!data || rs < (size_t)n) return fail(RMGPU_ERR_BAD_ARGUMENT, "bad tile buffer");
    if ((rc = check_device())) return rc;
    cudaError_t e = rmgpu::launch_transpose_tiles(data, n_tiles, n, rs, step, elem, (cudaStream_t)stream);
    return e == cudaSuccess ? RMGPU_OK : cuda_fail(e, "transpose_tiles");
}

int rmgpu_transpose_tiles_u8(void* d, size_t nt, int n, size_t rs, size_t step, void* s) { return tiles_impl(d, nt, n, rs, step, 1, s); }
int rmgpu_transpose_tiles_u16(void* d, size_t nt, int n, size_t rs, size_t step, void* s) { return tiles_impl(d, nt, n, rs, step, 2, s); }
int rmgpu_transpose_tiles_u32(void* d, size_t nt, int n, size_t rs, size_t step, void* s) { return tiles_impl(d, nt, n, rs, step, 4, s); }

static int transpose_host(const void* hsrc, size_t sp, void* hdst, size_t dp, int W, int H, int elem) {
    int rc;
    if (W < 0 || H < 0) return fail(RMGPU_ERR_BAD_ARGUMENT, "image dimensions must be non-negative");
    if (W == 0 || H == 0) return RMGPU_OK;
    if (!hsrc || !hdst || sp < (size_t)W * elem || dp < (size_t)H * elem)
        return fail(RMGPU_ERR_BAD_ARGUMENT, "bad transpose buffers");
    cudaStream_t s;
    if ((rc = host_stream(&s))) return rc;
    const size_t pa = ((size_t)W * elem + 255) & ~size_t(255), pb = ((size_t)H * elem + 255) & ~size_t(255);
    DevBuf a, b;
    a.s = b.s = s;
    RM_CUDA(scratch_alloc(&a.p, pa * H, s));
    RM_CUDA(scratch_alloc(&b.p, pb * W, s));
    RM_CUDA(cudaMemcpy2DAsync(a.p, pa, hsrc, sp, (size_t)W * elem, H, cudaMemcpyHostToDevice, s));
    cudaError_t e = rmgpu::launch_transpose(a.p, pa, b.p, pb, W, H, elem, s);
    if (e != cudaSuccess) return cuda_fail(e, "transpose");
    RM_CUDA(cudaMemcpy2DAsync(hdst, dp, b.p, pb, (size_t)H * elem, W, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaStreamSynchronize(s));
    return RMGPU_OK;
}

int rmgpu_transpose_host_u8(const void* hsrc, size_t sp, void* hdst, size_t dp, int W, int H) {
    return transpose_host(hsrc, sp, hdst, dp, W, H, 1);
}

int rmgpu_transpose_host_u16(const void* hsrc, size_t sp, void* hdst, size_t dp, int W, int H) {
    return transpose_host(hsrc, sp, hdst, dp, W, H, 2);
}

int rmgpu_transpose_tiles_host(void* hdata, int elem, size_t n_tiles, int n, size_t rs, size_t step) {
    int rc;
    if (n != 4 && n != 8 && n != 16) return fail(RMGPU_ERR_UNSUPPORTED_TILE, "tile side must be 4, 8 or 16");
    if (elem != 1 && elem != 2 && elem != 4) return fail(RMGPU_ERR_BAD_ARGUMENT, "element size must be 1, 2 or 4");
    if (n_tiles == 0) return RMGPU_OK;
    if (rs < (size_t)n) return fail(RMGPU_ERR_BAD_ARGUMENT, "bad tile stride");
    cudaStream_t s;
    if ((rc = host_stream(&s))) return rc;
    // Only the tiles' own elements travel (transpose_tile touches nothing else, transpose.cpp:14-27,
    // and concurrent calls on neighbouring tiles of one image must not lose each other's updates):
    // contiguous tiles as one copy, tiles stacked at a uniform row pitch as one 2-D copy, anything
    // else tile by tile. On the device the tiles are packed (row stride n, tile step n * n).
    const size_t tb = (size_t)n * n * elem, rowb = (size_t)n * elem;
    DevBuf a;
    a.s = s;
    RM_CUDA(scratch_alloc(&a.p, tb * n_tiles, s));
    char* h = static_cast<char*>(hdata);
    char* d = static_cast<char*>(a.p);
    const bool packed = rs == (size_t)n && step == (size_t)n * n;
    const bool stacked = step == (size_t)n * rs;
    if (packed) {
        RM_CUDA(cudaMemcpyAsync(d, h, tb * n_tiles, cudaMemcpyHostToDevice, s));
    } else if (stacked) {
        RM_CUDA(cudaMemcpy2DAsync(d, rowb, h, rs * elem, rowb, (size_t)n * n_tiles, cudaMemcpyHostToDevice, s));
    } else {
        for (size_t t = 0; t < n_tiles; ++t)
            RM_CUDA(cudaMemcpy2DAsync(d + t * tb, rowb, h + t * step * elem, rs * elem, rowb, n, cudaMemcpyHostToDevice, s));
    }
    if ((rc = tiles_impl(a.p, n_tiles, n, n, (size_t)n * n, elem, s))) return rc;
    if (packed) {
        RM_CUDA(cudaMemcpyAsync(h, d, tb * n_tiles, cudaMemcpyDeviceToHost, s));
    } else if (stacked) {
        RM_CUDA(cudaMemcpy2DAsync(h, rs * elem, d, rowb, rowb, (size_t)n * n_tiles, cudaMemcpyDeviceToHost, s));
    } else {
        for (size_t t = 0; t < n_tiles; ++t)
            RM_CUDA(cudaMemcpy2DAsync(h + t * step * elem, rs * elem, d + t * tb, rowb, rowb, n, cudaMemcpyDeviceToHost, s));
    }
    RM_CUDA(cudaStreamSynchronize(s));
    return RMGPU_OK;
}

int rmgpu_pass_host_u8(int which, const void* hsrc, size_t sp, void* hdst, size_t dp, int W, int H, int window,
                       int op, int border, unsigned bval, int algo) {
    (void)algo;
    int rc;
    if ((rc = check_window(window))) return rc;
    if ((rc = check_image(hsrc, sp, hdst, dp, W, H, 1))) return rc;
    if (W == 0 || H == 0) return RMGPU_OK;
    cudaStream_t s;
    if ((rc = host_stream(&s))) return rc;
    const size_t pitch = ((size_t)W + 255) & ~size_t(255);
    DevBuf a, b;
    a.s = b.s = s;
    RM_CUDA(scratch_alloc(&a.p, pitch * H, s));
    RM_CUDA(scratch_alloc(&b.p, pitch * H, s));
    RM_CUDA(cudaMemcpy2DAsync(a.p, pitch, hsrc, sp, W, H, cudaMemcpyHostToDevice, s));
    if ((rc = pass_impl(which, a.p, pitch, b.p, pitch, W, H, window, op, border, bval, s))) return rc;
    RM_CUDA(cudaMemcpy2DAsync(hdst, dp, b.p, pitch, W, H, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaStreamSynchronize(s));
    return RMGPU_OK;
}

int rmgpu_window_1d_host_u8(const void* in, size_t n, int window, int op, int border, unsigned bval, int algo,
                            void* out) {
    (void)algo;
    int rc;
    if ((rc = check_window(window))) return rc;
    if (n == 0) return RMGPU_OK;
    if (n > 0x7fffffff) return fail(RMGPU_ERR_BAD_ARGUMENT, "1-D signal too long");
    return rmgpu_pass_host_u8(RMGPU_PASS_HORIZONTAL, in, n, out, n, (int)n, 1, window, op, border, bval, algo);
}

int rmgpu_generate_u8(void* dst, size_t pitch, int W, int H, uint64_t seed, uint64_t sid, void* stream) {
    int rc;
    if (W < 0 || H < 0 || (W && H && (!dst || pitch < (size_t)W))) return fail(RMGPU_ERR_BAD_ARGUMENT, "bad generate args");
    if ((rc = check_device())) return rc;
    cudaError_t e = rmgpu::launch_generate(dst, pitch, W, H, seed, sid, 1, (cudaStream_t)stream);
    return e == cudaSuccess ? RMGPU_OK : cuda_fail(e, "generate");
}

int rmgpu_generate_u16(void* dst, size_t pitch, int W, int H, uint64_t seed, uint64_t sid, void* stream) {
    int rc;
    if (W < 0 || H < 0 || (W && H && (!dst || pitch < 2 * (size_t)W || pitch & 1)))
        return fail(RMGPU_ERR_BAD_ARGUMENT, "bad generate args");
    if ((rc = check_device())) return rc;
    cudaError_t e = rmgpu::launch_generate(dst, pitch, W, H, seed, sid, 2, (cudaStream_t)stream);
    return e == cudaSuccess ? RMGPU_OK : cuda_fail(e, "generate");
}

}  // extern "C"

// morph_generic.cu -- generic (any window, any pitch) GPU paths.
//
// The fallbacks behind the TMA kernels (K1 / K3 / K2), reached only when those decline a job
// (RMGPU_DISABLE_STREAM, windows beyond their register budgets); unaligned pitches are staged
// into aligned scratch and go to the TMA kernels instead (capi.cu run_single):
//   * morph_generic_tile: one fused kernel, input tile + halo staged in shared memory with the
//     border rule resolved at load time (image.cpp:58-66), vertical then horizontal pass
//     (separable.cpp:141-145) as direct window loops.
//   * pass_rows / pass_cols: single 1-D direct passes straight from global memory, for windows
//     too large for a shared-memory tile, and the direct sliding window an explicit Linear
//     algorithm hint asks for on a long wing (rmgpu.h).
#include "common.cuh"
#include "kernels.h"

namespace rmgpu {

namespace {

constexpr int kGTX = 64;   // output tile width
constexpr int kGTY = 32;   // output tile height
constexpr int kGThreads = 256;
constexpr size_t kMaxSmem = 200 * 1024;

// Border-resolved fetch. Valid rows are [row_lo, row_hi) relative to output row 0 (row bands
// carry real halo rows there), valid columns [0, W).
template <typename T>
__device__ __forceinline__ uint32_t fetch(const T* __restrict__ src, size_t sp, int W, int row_lo,
                                          int row_hi, int x, int y, int cmode, uint32_t bval) {
    if (cmode && (x < 0 || x >= W || y < row_lo || y >= row_hi)) return bval;
    x = min(max(x, 0), W - 1);
    y = min(max(y, row_lo), row_hi - 1);
    return src[(ptrdiff_t)y * (ptrdiff_t)sp + x];
}

template <typename T, int MODE>
__global__ void __launch_bounds__(kGThreads)
morph_generic_tile(const T* __restrict__ src, size_t sp, T* __restrict__ dst, size_t dp, int W,
                   int H, int row_lo, int row_hi, int gx, int gy, int cmode, uint32_t bval,
                   size_t simg, size_t dimg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    src += blockIdx.z * simg;
    dst += blockIdx.z * dimg;
    const int IW = kGTX + 2 * gx, IH = kGTY + 2 * gy;
    T* tin = reinterpret_cast<T*>(smem_raw);
    T* vlo = tin + IH * IW;
    T* vhi = vlo + kGTY * IW;  // MODE_GRAD only
    const int x0 = blockIdx.x * kGTX, y0 = blockIdx.y * kGTY;
    const int tid = threadIdx.x;

    for (int i = tid; i < IH * IW; i += kGThreads) {
        const int r = i / IW, c = i - r * IW;
        tin[i] = (T)fetch<T>(src, sp, W, row_lo, row_hi, x0 - gx + c, y0 - gy + r, cmode, bval);
    }
    __syncthreads();

    // vertical pass over every tile column (halo columns included)
    for (int i = tid; i < kGTY * IW; i += kGThreads) {
        const int r = i / IW, c = i - r * IW;
        const T* col = tin + r * IW + c;
        uint32_t lo = col[0], hi = col[0];
        for (int k = 1; k <= 2 * gy; ++k) {
            const uint32_t v = col[k * IW];
            lo = min(lo, v);
            hi = max(hi, v);
        }
        if (MODE == MODE_MIN) vlo[i] = (T)lo;
        else if (MODE == MODE_MAX) vlo[i] = (T)hi;
        else { vlo[i] = (T)lo; vhi[i] = (T)hi; }
    }
    __syncthreads();

    // horizontal pass + store
    for (int i = tid; i < kGTY * kGTX; i += kGThreads) {
        const int r = i / kGTX, c = i - r * kGTX;
        const int y = y0 + r, x = x0 + c;
        if (y >= H || x >= W) continue;
        const T* rl = vlo + r * IW + c;
        uint32_t acc = rl[0];
        for (int k = 1; k <= 2 * gx; ++k) acc = red2<MODE == MODE_MAX ? MODE_MAX : MODE_MIN>(acc, rl[k]);
        if (MODE == MODE_GRAD) {
            const T* rh = vhi + r * IW + c;
            uint32_t hacc = rh[0];
            for (int k = 1; k <= 2 * gx; ++k) hacc = max(hacc, (uint32_t)rh[k]);
            acc = hacc - acc;
        }
        dst[(ptrdiff_t)y * (ptrdiff_t)dp + x] = (T)acc;
    }
}

size_t generic_smem(const MorphJob& j) {
    const size_t IW = kGTX + 2 * (size_t)j.gx, IH = kGTY + 2 * (size_t)j.gy;
    const size_t nv = j.mode == MODE_GRAD ? 2 : 1;
    return (IH * IW + nv * kGTY * IW) * (size_t)j.elem;
}

template <typename T, int MODE>
cudaError_t launch_tile_t(const MorphJob& j) {
    const size_t smem = generic_smem(j);
    auto kern = morph_generic_tile<T, MODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
    if (e != cudaSuccess) return e;
    dim3 grid(cdiv(j.W, kGTX), cdiv(j.H, kGTY), j.batch);
    kern<<<grid, kGThreads, smem, j.stream>>>(
        static_cast<const T*>(j.src), j.sp / sizeof(T), static_cast<T*>(j.dst), j.dp / sizeof(T),
        j.W, j.H, -j.above, j.H + j.below, j.gx, j.gy, j.cmode, j.bval, j.simg / sizeof(T),
        j.dimg / sizeof(T));
    count_launch();
    return cudaGetLastError();
}

// ---- single 1-D passes from global memory ---------------------------------------------------
template <typename T, int MODE, bool ROWS>
__global__ void __launch_bounds__(256)
pass_generic(const T* __restrict__ src, size_t sp, T* __restrict__ dst, size_t dp, int W, int H,
             int row_lo, int row_hi, int g, int cmode, uint32_t bval, size_t simg, size_t dimg) {
    src += blockIdx.z * simg;
    dst += blockIdx.z * dimg;
    const int x = blockIdx.x * 64 + (threadIdx.x & 63);
    const int y = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (x >= W || y >= H) return;
    uint32_t lo = identity<T, MODE_MIN>(), hi = 0;
    for (int k = -g; k <= g; ++k) {
        const uint32_t v = ROWS ? fetch<T>(src, sp, W, row_lo, row_hi, x + k, y, cmode, bval)
                                : fetch<T>(src, sp, W, row_lo, row_hi, x, y + k, cmode, bval);
        lo = min(lo, v);
        hi = max(hi, v);
    }
    dst[(ptrdiff_t)y * (ptrdiff_t)dp + x] = (T)(MODE == MODE_MIN ? lo : MODE == MODE_MAX ? hi : hi - lo);
}

template <typename T, bool ROWS>
cudaError_t launch_pass_t(const MorphJob& j) {
    dim3 grid(cdiv(j.W, 64), cdiv(j.H, 4), j.batch);
    const int g = ROWS ? j.gx : j.gy;
    const size_t si = j.simg / sizeof(T), di = j.dimg / sizeof(T);
    const T* s = static_cast<const T*>(j.src);
    T* d = static_cast<T*>(j.dst);
    const size_t sp = j.sp / sizeof(T), dp = j.dp / sizeof(T);
    const int lo = ROWS ? 0 : -j.above, hi = ROWS ? j.H : j.H + j.below;
    switch (j.mode) {
    case MODE_MIN:
        pass_generic<T, MODE_MIN, ROWS><<<grid, 256, 0, j.stream>>>(s, sp, d, dp, j.W, j.H, lo, hi, g, j.cmode, j.bval, si, di);
        break;
    case MODE_MAX:
        pass_generic<T, MODE_MAX, ROWS><<<grid, 256, 0, j.stream>>>(s, sp, d, dp, j.W, j.H, lo, hi, g, j.cmode, j.bval, si, di);
        break;
    default:
        return cudaErrorInvalidValue;
    }
    count_launch();
    return cudaGetLastError();
}

template <typename T>
__global__ void subtract_kernel(const T* __restrict__ a, size_t ap, const T* b, size_t bp, T* d, size_t dp,
                                int W, int H) {  // b may alias d (in-place gradient)
    const int x = blockIdx.x * 64 + (threadIdx.x & 63);
    const int y = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (x >= W || y >= H) return;
    d[(ptrdiff_t)y * dp + x] = (T)(a[(ptrdiff_t)y * ap + x] - b[(ptrdiff_t)y * bp + x]);
}

// a - b for 16-byte vectors of u8 or u16 pixels where every pixel of a is >= the one of b.
__global__ void subtract16_kernel(const uint8_t* __restrict__ a, size_t ap, const uint8_t* b, size_t bp, uint8_t* d,
                                  size_t dp, int vpr, int H) {
    const int v = blockIdx.x * 64 + (threadIdx.x & 63);
    const int y = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (v >= vpr || y >= H) return;
    const uint4 x = *reinterpret_cast<const uint4*>(a + (size_t)y * ap + (size_t)v * 16);
    const uint4 z = *reinterpret_cast<const uint4*>(b + (size_t)y * bp + (size_t)v * 16);
    *reinterpret_cast<uint4*>(d + (size_t)y * dp + (size_t)v * 16) = make_uint4(x.x - z.x, x.y - z.y, x.z - z.z, x.w - z.w);
}

}  // namespace

bool generic_tile_fits(const MorphJob& j) { return generic_smem(j) <= kMaxSmem; }

cudaError_t launch_generic_tile(const MorphJob& j) {
    if (!generic_tile_fits(j)) return cudaErrorInvalidValue;
    if (j.elem == 1) {
        switch (j.mode) {
        case MODE_MIN: return launch_tile_t<uint8_t, MODE_MIN>(j);
        case MODE_MAX: return launch_tile_t<uint8_t, MODE_MAX>(j);
        default: return launch_tile_t<uint8_t, MODE_GRAD>(j);
        }
    }
    switch (j.mode) {
    case MODE_MIN: return launch_tile_t<uint16_t, MODE_MIN>(j);
    case MODE_MAX: return launch_tile_t<uint16_t, MODE_MAX>(j);
    default: return launch_tile_t<uint16_t, MODE_GRAD>(j);
    }
}

cudaError_t launch_pass_rows(const MorphJob& j) {
    return j.elem == 1 ? launch_pass_t<uint8_t, true>(j) : launch_pass_t<uint16_t, true>(j);
}

cudaError_t launch_pass_cols(const MorphJob& j) {
    return j.elem == 1 ? launch_pass_t<uint8_t, false>(j) : launch_pass_t<uint16_t, false>(j);
}

cudaError_t launch_subtract(const void* a, size_t ap, const void* b, size_t bp, void* dst, size_t dp,
                            int W, int H, int elem, cudaStream_t s) {
    const size_t rb = (size_t)W * elem;
    const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(dst) |
                       ap | bp | dp | rb) & 15) == 0;
    if (vec) {  // 16 bytes per thread; bytewise max >= min, so lane-wise 32-bit subtracts never borrow
        const int vpr = (int)(rb / 16);
        dim3 grid(cdiv(vpr, 64), cdiv(H, 4));
        subtract16_kernel<<<grid, 256, 0, s>>>((const uint8_t*)a, ap, (const uint8_t*)b, bp, (uint8_t*)dst, dp, vpr, H);
    } else if (elem == 1) {
        dim3 grid(cdiv(W, 64), cdiv(H, 4));
        subtract_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)a, ap, (const uint8_t*)b, bp,
                                                       (uint8_t*)dst, dp, W, H);
    } else {
        dim3 grid(cdiv(W, 64), cdiv(H, 4));
        subtract_kernel<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)a, ap / 2, (const uint16_t*)b,
                                                        bp / 2, (uint16_t*)dst, dp / 2, W, H);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace rmgpu

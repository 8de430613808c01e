// common.cuh -- shared device helpers for the rmgpu kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace rmgpu {

// Reduction selector. Erosion = window minimum, dilation = window maximum
// (rectmorph OpKind, core/include/rectmorph/image.hpp:11-19). GRAD computes
// both and stores max - min (dispatch.cpp:58-71).
enum Mode : int { MODE_MIN = 0, MODE_MAX = 1, MODE_GRAD = 2 };

template <typename T>
struct PixelTraits;
template <>
struct PixelTraits<uint8_t> {
    static constexpr uint32_t kMax = 0xFFu;
};
template <>
struct PixelTraits<uint16_t> {
    static constexpr uint32_t kMax = 0xFFFFu;
};

template <int MODE>
__device__ __forceinline__ uint32_t red2(uint32_t a, uint32_t b) {
    return MODE == MODE_MIN ? min(a, b) : max(a, b);
}

// Identity of the reduction (identity_value, image.hpp:17-19) at width T.
template <typename T, int MODE>
__host__ __device__ constexpr uint32_t identity() {
    return MODE == MODE_MIN ? PixelTraits<T>::kMax : 0u;
}

// Packed 16-bit-lane reductions: one VIMNMX.U16x2 / VIMNMX3.U16x2 on sm_100a.
template <int MODE>
__device__ __forceinline__ uint32_t red2_u16x2(uint32_t a, uint32_t b) {
    return MODE == MODE_MIN ? __vminu2(a, b) : __vmaxu2(a, b);
}
template <int MODE>
__device__ __forceinline__ uint32_t red3_u16x2(uint32_t a, uint32_t b, uint32_t c) {
    return MODE == MODE_MIN ? __vimin3_u16x2(a, b, c) : __vimax3_u16x2(a, b, c);
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    return __byte_perm(a, b, sel);
}

__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }

// Host-side bookkeeping shared by all launch sites.
extern std::atomic<unsigned long long> g_launch_count;
inline void count_launch(unsigned long long n = 1) { g_launch_count.fetch_add(n, std::memory_order_relaxed); }

}  // namespace rmgpu

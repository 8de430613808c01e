// generate.cu -- counter-based synthetic input generator, bit-identical to
// oracle/rmoracle.c orc_generate_*, so multi-GPU ranks can create their inputs on device and
// the CPU checker still sees the same bytes.
#include "common.cuh"
#include "kernels.h"

namespace rmgpu {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void __launch_bounds__(256)
generate_kernel(T* __restrict__ dst, size_t pitch, int W, int y0, uint64_t seed, uint64_t stream_id) {
    constexpr int PER = 8 / sizeof(T);  // pixels per 64-bit word
    const int x = blockIdx.x * 256 + threadIdx.x;
    const int y = y0 + (int)blockIdx.y;
    if (x >= W) return;
    const uint64_t i = (uint64_t)y * (uint64_t)W + (uint64_t)x;
    const uint64_t word = splitmix64((seed * 0xD1B54A32D192ED03ull) ^ (stream_id << 40) ^ (i / PER));
    dst[(size_t)y * pitch + x] = (T)(word >> (8 * sizeof(T) * (i % PER)));
}

}  // namespace

cudaError_t launch_generate(void* dst, size_t pitch, int W, int H, uint64_t seed, uint64_t stream_id,
                            int elem, cudaStream_t s) {
    if (W == 0 || H == 0) return cudaSuccess;
    for (int y0 = 0; y0 < H; y0 += 65535) {
        const int rows = H - y0 < 65535 ? H - y0 : 65535;
        dim3 grid(cdiv(W, 256), rows);
        if (elem == 1)
            generate_kernel<uint8_t><<<grid, 256, 0, s>>>((uint8_t*)dst, pitch, W, y0, seed, stream_id);
        else
            generate_kernel<uint16_t><<<grid, 256, 0, s>>>((uint16_t*)dst, pitch / 2, W, y0, seed, stream_id);
        count_launch();
    }
    return cudaGetLastError();
}

}  // namespace rmgpu

// pipes.cu -- issue-rate microbenchmark of the instructions the morphology kernels are made of
// (which pipe each one occupies, and which pairs co-issue). nvcc -arch=sm_100a -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define ITER 4096
#define NACC 8

__device__ __forceinline__ uint32_t hmin2u(uint32_t a, uint32_t b) {
    __half2 r = __hmin2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hmax2u(uint32_t a, uint32_t b) {
    __half2 r = __hmax2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hfmarelu2u(uint32_t a, uint32_t b, uint32_t c) {
    __half2 r = __hfma2_relu(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b), *reinterpret_cast<__half2*>(&c));
    return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hadd2u(uint32_t a, uint32_t b) {
    __half2 r = __hadd2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
}

// every accumulator is combined with its neighbour's previous value: nothing folds, NACC
// independent chains
template <int KIND>
__device__ __forceinline__ void step(uint32_t (&a)[NACC], uint32_t b, uint32_t c) {
    uint32_t n[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
        const uint32_t x = a[i], y = a[(i + 1) % NACC], z = a[(i + 3) % NACC];
        uint32_t r = x;
        if (KIND == 0) r = __vminu2(x, y);
        if (KIND == 1) r = __vimin3_u16x2(x, y, z);
        if (KIND == 17) r = __vimax3_u16x2(x, y, z);
        if (KIND == 2) r = hmin2u(x, y);
        if (KIND == 15) r = hmax2u(x, y);
        if (KIND == 3) r = hfmarelu2u(x, c, y);
        if (KIND == 16) r = hadd2u(x, y);
        if (KIND == 4) r = __byte_perm(x, y, 0x3715);
        if (KIND == 5) r = x * b + y;
        if (KIND == 10) r = (x << 8) ^ y;   // SHF/SHL + LOP3 (2 alu instr)
        if (KIND == 11) r = x + y;
        if (KIND == 12) r = max(x, y);
        if (KIND == 13) r = __shfl_up_sync(0xffffffffu, x, 1);
        if (KIND == 18) r = __vminu4(x, y);
        if (KIND == 6) r = (i & 1) ? __vminu2(x, y) : hmin2u(x, y);
        if (KIND == 7) r = (i & 1) ? __vminu2(x, y) : x * b + y;
        if (KIND == 8) r = (i & 1) ? __vminu2(x, y) : hfmarelu2u(x, c, y);
        if (KIND == 9) r = (i & 1) ? __vminu2(x, y) : __byte_perm(x, y, 0x3715);
        if (KIND == 19) r = (i & 1) ? __vminu2(x, y) : hadd2u(x, y);
        if (KIND == 14) r = (i & 3) ? __vminu2(x, y) : __shfl_up_sync(0xffffffffu, x, 1);
        if (KIND == 20) r = (i & 1) ? __vimin3_u16x2(x, y, z) : hmin2u(x, y);
        n[i] = r;
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = n[i];
}

template <int KIND>
__global__ void bench(uint32_t* out, uint32_t b, uint32_t c, long long* cyc) {
    uint32_t a[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = threadIdx.x * 2654435761u + i;
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 8
    for (int it = 0; it < ITER; ++it) step<KIND>(a, b, c);
    const long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int KIND>
void run(const char* name, int per_step, uint32_t* out, long long* cyc) {
    const int threads = 512;  // 16 warps per SM, 4 per SMSP
    bench<KIND><<<148, threads>>>(out, 0x01020304u, 0x3c003c00u, cyc);
    cudaDeviceSynchronize();
    bench<KIND><<<148, threads>>>(out, 0x01020304u, 0x3c003c00u, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    const double winstr = (double)ITER * per_step * (threads / 32);  // warp instructions per SM
    printf("%-34s %8.3f warp-instr/clk/SM  (%.3f per SMSP)\n", name, winstr / c, winstr / c / 4);
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 8);
    run<0>("min.u16x2 (VIMNMX)", NACC, out, cyc);
    run<1>("min3 via 2x min.u16x2 (VIMNMX3?)", NACC, out, cyc);
    run<17>("max3 via 2x max.u16x2", NACC, out, cyc);
    run<2>("min.f16x2 (HMNMX2)", NACC, out, cyc);
    run<15>("max.f16x2", NACC, out, cyc);
    run<3>("fma.relu.f16x2 (HFMA2.RELU)", NACC, out, cyc);
    run<16>("add.f16x2", NACC, out, cyc);
    run<4>("prmt", NACC, out, cyc);
    run<5>("mad.lo.u32 (IMAD)", NACC, out, cyc);
    run<10>("shl+xor (2 instr)", 2 * NACC, out, cyc);
    run<11>("add.u32", NACC, out, cyc);
    run<12>("max.u32", NACC, out, cyc);
    run<13>("shfl.up", NACC, out, cyc);
    run<18>("vmin4 (emulated)", NACC, out, cyc);
    run<6>("min.u16x2 + min.f16x2 1:1", NACC, out, cyc);
    run<7>("min.u16x2 + mad 1:1", NACC, out, cyc);
    run<8>("min.u16x2 + fma.relu.f16x2 1:1", NACC, out, cyc);
    run<9>("min.u16x2 + prmt 1:1", NACC, out, cyc);
    run<19>("min.u16x2 + add.f16x2 1:1", NACC, out, cyc);
    run<20>("vimin3 + min.f16x2 1:1", NACC, out, cyc);
    run<14>("min.u16x2 x3 + shfl x1", NACC, out, cyc);
    return 0;
}

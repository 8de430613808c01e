// transpose.cu -- K4 whole-image transpose and K5 batched in-place tile transpose.
//
// K4 replaces rectmorph::transpose_image (core/src/transpose.cpp:29-53): out-of-place, dst is
// H x W. A CTA moves one 64x64-element tile through shared memory: 16-byte coalesced loads of
// input rows, column gathers out of shared memory, 16-byte coalesced stores of output rows.
//
// K5 replaces rectmorph::transpose_tile (transpose.cpp:14-27) batched over many tiles. The
// reference transposes in place by log2(n) rounds of block interleaves
// (transpose.hpp:19-30); on the GPU one thread owns a whole tile in registers and the same
// permutation becomes (a) a 4x4-byte / 2x2-half transpose inside each group of words via PRMT
// and (b) a compile-time renaming of the word groups. Tiles are contiguous (row stride n, tile
// step n*n) on the fast path; any stride/step uses a shared-memory path.
#include "common.cuh"
#include "kernels.h"

namespace rmgpu {

namespace {

// ------------------------------------------------------------------------------------------
// K4: image transpose
// ------------------------------------------------------------------------------------------
constexpr int kTT = 64;  // tile side in elements

template <typename T>
__global__ void __launch_bounds__(256)
transpose_image_kernel(const T* __restrict__ src, size_t sp, T* __restrict__ dst, size_t dp, int W,
                       int H, int vec_ok) {
    constexpr int VE = 16 / sizeof(T);          // elements per 16-byte vector
    constexpr int PITCH = kTT + VE;             // smem row pitch (elements), 16-B multiple
    __shared__ __align__(16) T tile[kTT * PITCH];
    const int x0 = blockIdx.x * kTT, y0 = blockIdx.y * kTT;
    const int tid = threadIdx.x;
    const bool full = vec_ok && (x0 + kTT <= W) && (y0 + kTT <= H);

    // load 64 rows x 64 elements
    constexpr int VPR = kTT / VE;               // vectors per tile row
    if (full) {
        for (int v = tid; v < kTT * VPR; v += 256) {
            const int r = v / VPR, c = (v % VPR) * VE;
            const uint4 val = *reinterpret_cast<const uint4*>(src + (size_t)(y0 + r) * sp + x0 + c);
            *reinterpret_cast<uint4*>(tile + r * PITCH + c) = val;
        }
    } else {
        for (int i = tid; i < kTT * kTT; i += 256) {
            const int r = i / kTT, c = i % kTT;
            if (y0 + r < H && x0 + c < W) tile[r * PITCH + c] = src[(size_t)(y0 + r) * sp + x0 + c];
        }
    }
    __syncthreads();

    // store: output row (x0 + c) holds input column c, rows y0 .. y0+63
    if (full) {
        // warp w: segment (w % VPR) of output rows; lanes = consecutive output rows (columns c)
        for (int v = tid; v < kTT * VPR; v += 256) {
            const int lane = v & 31, w = v >> 5;
            const int seg = w % VPR, c = (w / VPR) * 32 + lane;
            T vals[VE];
#pragma unroll
            for (int k = 0; k < VE; ++k) vals[k] = tile[(seg * VE + k) * PITCH + c];
            *reinterpret_cast<uint4*>(dst + (size_t)(x0 + c) * dp + y0 + seg * VE) =
                *reinterpret_cast<const uint4*>(vals);
        }
    } else {
        for (int i = tid; i < kTT * kTT; i += 256) {
            const int c = i / kTT, r = i % kTT;
            if (y0 + r < H && x0 + c < W) dst[(size_t)(x0 + c) * dp + y0 + r] = tile[r * PITCH + c];
        }
    }
}

// ------------------------------------------------------------------------------------------
// Register butterfly: a group of lanes (16 for u8, 8 for u16) each holding one 16-byte row of a
// 16x16 u8 / 8x8 u16 block ends up holding one column (= one row of the transposed block).
// Stage s (lane mask): lanes with (lane & s) == 0 keep the left half of every 2s-column block
// and receive the partner's left half into the right half; the others keep the right half.
// ------------------------------------------------------------------------------------------
template <int ELEM>  // 1 = u8 16x16 (masks 8,4,2,1), 2 = u16 8x8 (masks 4,2,1)
__device__ __forceinline__ void butterfly_rows(uint32_t (&w)[4], int lane) {
    constexpr int TOP = ELEM == 1 ? 8 : 4;
    {   // 2-word blocks
        const bool lo = !(lane & TOP);
        const uint32_t s0 = lo ? w[2] : w[0], s1 = lo ? w[3] : w[1];
        const uint32_t r0 = __shfl_xor_sync(0xffffffffu, s0, TOP), r1 = __shfl_xor_sync(0xffffffffu, s1, TOP);
        if (lo) { w[2] = r0; w[3] = r1; } else { w[0] = r0; w[1] = r1; }
    }
    {   // 1-word blocks
        const bool lo = !(lane & (TOP / 2));
        const uint32_t s0 = lo ? w[1] : w[0], s1 = lo ? w[3] : w[2];
        const uint32_t r0 = __shfl_xor_sync(0xffffffffu, s0, TOP / 2), r1 = __shfl_xor_sync(0xffffffffu, s1, TOP / 2);
        if (lo) { w[1] = r0; w[3] = r1; } else { w[0] = r0; w[2] = r1; }
    }
    {   // half-word blocks
        const uint32_t sel = (lane & (TOP / 4)) ? 0x3276u : 0x5410u;
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = prmt(w[k], __shfl_xor_sync(0xffffffffu, w[k], TOP / 4), sel);
    }
    if constexpr (ELEM == 1) {  // bytes
        const uint32_t sel = (lane & 1) ? 0x3715u : 0x6240u;
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = prmt(w[k], __shfl_xor_sync(0xffffffffu, w[k], 1), sel);
    }
}

// Contiguous 16x16 u8 tiles (cfg3) / 8x8 u16 tiles: a warp moves 512 contiguous bytes per step
// (2 u8 tiles / 4 u16 tiles, one 16-byte row per lane), transposes them with the register
// butterfly and writes them back in place: fully coalesced 128-bit loads and stores.
template <int ELEM>
__global__ void __launch_bounds__(256)
tiles_warp_kernel(uint8_t* __restrict__ data, size_t n_groups) {
    const int lane = threadIdx.x & 31;
    const size_t warps = (size_t)gridDim.x * (blockDim.x >> 5);
    for (size_t g = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < n_groups; g += warps) {
        uint4* p = reinterpret_cast<uint4*>(data + g * 512) + lane;
        const uint4 v = __ldcs(p);
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
        butterfly_rows<ELEM>(w, lane);
        __stcs(p, make_uint4(w[0], w[1], w[2], w[3]));
    }
}

// Image transpose, full 64x64 (u8) / 64x64 (u16) tiles: coalesced 128-bit loads into a padded
// shared tile, 16-byte rows of 16x16 (u8) / 8x8 (u16) blocks into registers, register butterfly,
// 128-bit stores of output rows (lane groups paired so every output row gets 32 / 64 contiguous
// bytes per warp store).
template <typename T>
__global__ void __launch_bounds__(256)
transpose_image_bfly_kernel(const T* __restrict__ src, size_t sp, T* __restrict__ dst, size_t dp, int W, int H) {
    constexpr int ELEM = sizeof(T);
    constexpr int TBY = 64;                      // tile rows
    constexpr int RB = 256;                      // tile row bytes (256 u8 / 128 u16 columns)
    constexpr int TBX = RB / ELEM;
    constexpr int PB = RB + 16;                  // padded smem row pitch (bank-conflict free)
    constexpr int BS = 16 / ELEM;                // block side (16 u8 / 8 u16)
    constexpr int NBX = TBX / BS, NBY = TBY / BS;
    __shared__ __align__(16) unsigned char tile[TBY * PB];
    const int x0 = blockIdx.x * TBX, y0 = blockIdx.y * TBY;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned char* s8 = reinterpret_cast<const unsigned char*>(src);
    unsigned char* d8 = reinterpret_cast<unsigned char*>(dst);
    constexpr int CPR = RB / 16;                 // 16-byte chunks per tile row
    constexpr int LPT = TBY * CPR / 256;         // loads per thread (4), all issued before the stores
    uint4 v[LPT];
#pragma unroll
    for (int k = 0; k < LPT; ++k) {
        const int c = tid + 256 * k, r = c / CPR, cc = c % CPR;
        v[k] = __ldcs(reinterpret_cast<const uint4*>(s8 + (size_t)(y0 + r) * sp + (size_t)x0 * ELEM + cc * 16));
    }
#pragma unroll
    for (int k = 0; k < LPT; ++k) {
        const int c = tid + 256 * k, r = c / CPR, cc = c % CPR;
        *reinterpret_cast<uint4*>(tile + r * PB + cc * 16) = v[k];
    }
    __syncthreads();
    // blocks (b, c): b = block row (input rows), c = block column (input columns). A warp job is
    // GPW consecutive b for one c; lane group g = lane / BS handles b = bq * GPW + g, so one
    // output row receives GPW * 16 contiguous bytes per warp store.
    constexpr int GPW = 32 / BS;
    constexpr int JOBS = NBX * NBY / GPW;
    const int i = lane % BS, g = lane / BS;
#pragma unroll
    for (int job = warp; job < JOBS; job += 8) {
        const int c = job % NBX, bq = job / NBX;
        const int b = bq * GPW + g;
        const uint4 t = *reinterpret_cast<const uint4*>(tile + (b * BS + i) * PB + c * 16);
        uint32_t w[4] = {t.x, t.y, t.z, t.w};
        butterfly_rows<ELEM>(w, i);
        // lane holds input column c*BS + i, rows b*BS .. b*BS+BS-1 = output row x0 + c*BS + i
        __stcs(reinterpret_cast<uint4*>(d8 + (size_t)(x0 + c * BS + i) * dp + (size_t)(y0 + b * BS) * ELEM),
               make_uint4(w[0], w[1], w[2], w[3]));
    }
}

// 4x4 byte transpose of four row words a[0..3] -> column words b[0..3].
__device__ __forceinline__ void t4x4_u8(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t& b0, uint32_t& b1, uint32_t& b2, uint32_t& b3) {
    const uint32_t t0 = prmt(a0, a1, 0x5140), t1 = prmt(a0, a1, 0x7362);
    const uint32_t t2 = prmt(a2, a3, 0x5140), t3 = prmt(a2, a3, 0x7362);
    b0 = prmt(t0, t2, 0x5410);
    b1 = prmt(t0, t2, 0x7632);
    b2 = prmt(t1, t3, 0x5410);
    b3 = prmt(t1, t3, 0x7632);
}

// Image transpose, full tiles, block version (replaces the shuffle butterfly, which ncu showed
// MIO-throttled: 16 SHFL per 16 bytes). A CTA stages TH input rows x 128 bytes in shared memory
// (coalesced 128-bit loads, 8-byte chunks XOR-swizzled by row block so the column-block reads are
// conflict-free); each thread then reads one 8x8 u8 / 4x4 u16 block with 64-bit shared loads,
// transposes it in registers with byte / half-word permutes and writes it as 8 / 4 output row
// pieces of 8 bytes -- the 16 lanes of a half warp cover 128 contiguous bytes of an output row.
template <typename T>
__global__ void __launch_bounds__(256)
transpose_image_blk_kernel(const T* __restrict__ src, size_t sp, T* __restrict__ dst, size_t dp) {
    constexpr int ELEM = sizeof(T);
    constexpr int BR = ELEM == 1 ? 8 : 4;        // block rows (8x8 u8, 4x4 u16: 8 bytes per row)
    constexpr int TH = 16 * BR;                  // tile rows (16 row blocks)
    constexpr int RB = 128;                      // tile row bytes (16 chunks of 8 bytes)
    constexpr int TX = RB / ELEM;                // tile columns
    __shared__ __align__(16) unsigned char tile[TH * RB];
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TH;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned char* s8 = reinterpret_cast<const unsigned char*>(src);
    unsigned char* d8 = reinterpret_cast<unsigned char*>(dst);
    constexpr int LPT = TH * RB / 16 / 256;      // 16-byte loads per thread (4 u8, 2 u16)
    uint4 v[LPT];
#pragma unroll
    for (int k = 0; k < LPT; ++k) {
        const int c = tid + 256 * k, r = c >> 3, q = c & 7;  // row, 16-byte chunk
        v[k] = __ldcs(reinterpret_cast<const uint4*>(s8 + (size_t)(y0 + r) * sp + (size_t)x0 * ELEM + q * 16));
    }
#pragma unroll
    for (int k = 0; k < LPT; ++k) {
        const int c = tid + 256 * k, r = c >> 3, q = c & 7;
        const int sw = (r / BR) & 15;            // 8-byte chunk 2q / 2q+1 -> (2q) ^ sw / (2q+1) ^ sw
        const int p = (2 * q) ^ sw;
        const uint4 w = (p & 1) ? make_uint4(v[k].z, v[k].w, v[k].x, v[k].y) : v[k];
        *reinterpret_cast<uint4*>(tile + r * RB + (p & ~1) * 8) = w;
    }
    __syncthreads();
    const int by = lane & 15, bx = warp * 2 + (lane >> 4);  // row block, 8-byte column block
    uint2 r[BR];
#pragma unroll
    for (int i = 0; i < BR; ++i)
        r[i] = *reinterpret_cast<const uint2*>(tile + (by * BR + i) * RB + ((bx ^ by) * 8));
    // output row o (input column x0 + bx * (8 / ELEM) + o) gets this block's BR rows
    unsigned char* drow = d8 + (size_t)(x0 + bx * (8 / ELEM)) * dp + (size_t)(y0 + by * BR) * ELEM;
    if constexpr (ELEM == 1) {
        uint32_t lo[8], hi[8];
        t4x4_u8(r[0].x, r[1].x, r[2].x, r[3].x, lo[0], lo[1], lo[2], lo[3]);
        t4x4_u8(r[0].y, r[1].y, r[2].y, r[3].y, lo[4], lo[5], lo[6], lo[7]);
        t4x4_u8(r[4].x, r[5].x, r[6].x, r[7].x, hi[0], hi[1], hi[2], hi[3]);
        t4x4_u8(r[4].y, r[5].y, r[6].y, r[7].y, hi[4], hi[5], hi[6], hi[7]);
#pragma unroll
        for (int o = 0; o < 8; ++o) __stcs(reinterpret_cast<uint2*>(drow + (size_t)o * dp), make_uint2(lo[o], hi[o]));
    } else {
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int wi = o >> 1;
            const uint32_t sel = (o & 1) ? 0x7632u : 0x5410u;
            const uint32_t a0 = wi ? r[0].y : r[0].x, a1 = wi ? r[1].y : r[1].x;
            const uint32_t a2 = wi ? r[2].y : r[2].x, a3 = wi ? r[3].y : r[3].x;
            __stcs(reinterpret_cast<uint2*>(drow + (size_t)o * dp), make_uint2(prmt(a0, a1, sel), prmt(a2, a3, sel)));
        }
    }
}

// ------------------------------------------------------------------------------------------
// K5: batched tile transposes, one tile per thread (contiguous tiles)
// ------------------------------------------------------------------------------------------

// u8 tile of side N (4, 8, 16): N rows x N/4 words.
template <int N>
__global__ void __launch_bounds__(128)
tiles_u8_kernel(uint8_t* __restrict__ data, size_t n_tiles) {
    constexpr int WPR = N / 4;             // words per row
    constexpr int NW = N * WPR;            // words per tile
    constexpr int NV = NW / 4;             // uint4 per tile
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    uint4* p = reinterpret_cast<uint4*>(data + t * (size_t)(N * N));
    uint32_t w[NW], o[NW];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const uint4 q = p[v];
        w[4 * v + 0] = q.x; w[4 * v + 1] = q.y; w[4 * v + 2] = q.z; w[4 * v + 3] = q.w;
    }
    // word (r, k) = w[r*WPR + k] holds columns 4k..4k+3 of row r. Block (m, k) = rows 4m..4m+3
    // of word column k transposes into output rows 4k..4k+3, word column m.
#pragma unroll
    for (int m = 0; m < WPR; ++m)
#pragma unroll
        for (int k = 0; k < WPR; ++k)
            t4x4_u8(w[(4 * m + 0) * WPR + k], w[(4 * m + 1) * WPR + k], w[(4 * m + 2) * WPR + k],
                    w[(4 * m + 3) * WPR + k], o[(4 * k + 0) * WPR + m], o[(4 * k + 1) * WPR + m],
                    o[(4 * k + 2) * WPR + m], o[(4 * k + 3) * WPR + m]);
#pragma unroll
    for (int v = 0; v < NV; ++v) p[v] = make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
}

// u16 tile of side N (4, 8): N rows x N/2 words; 2x2 half-word blocks.
template <int N>
__global__ void __launch_bounds__(128)
tiles_u16_kernel(uint16_t* __restrict__ data, size_t n_tiles) {
    constexpr int WPR = N / 2;
    constexpr int NW = N * WPR;
    constexpr int NV = NW / 4;
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    uint4* p = reinterpret_cast<uint4*>(data + t * (size_t)(N * N));
    uint32_t w[NW], o[NW];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const uint4 q = p[v];
        w[4 * v + 0] = q.x; w[4 * v + 1] = q.y; w[4 * v + 2] = q.z; w[4 * v + 3] = q.w;
    }
#pragma unroll
    for (int m = 0; m < WPR; ++m)
#pragma unroll
        for (int k = 0; k < WPR; ++k) {
            const uint32_t a = w[(2 * m) * WPR + k], b = w[(2 * m + 1) * WPR + k];
            o[(2 * k) * WPR + m] = prmt(a, b, 0x5410);
            o[(2 * k + 1) * WPR + m] = prmt(a, b, 0x7632);
        }
#pragma unroll
    for (int v = 0; v < NV; ++v) p[v] = make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
}

// Any element type, stride and step: one CTA per group of tiles through shared memory.
template <typename T>
__global__ void __launch_bounds__(256)
tiles_generic_kernel(T* __restrict__ data, size_t n_tiles, int n, size_t row_stride, size_t step) {
    __shared__ T buf[256];
    const int per = 256 / (n * n);   // tiles per CTA pass
    const int tid = threadIdx.x;
    const int local = tid / (n * n), e = tid % (n * n);
    const int r = e / n, c = e % n;
    for (size_t base = (size_t)blockIdx.x * per; base < n_tiles; base += (size_t)gridDim.x * per) {
        const size_t t = base + local;
        const bool live = local < per && t < n_tiles;
        if (live) buf[tid] = data[t * step + (size_t)r * row_stride + c];
        __syncthreads();
        if (live) data[t * step + (size_t)r * row_stride + c] = buf[local * n * n + c * n + r];
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_transpose(const void* src, size_t sp, void* dst, size_t dp, int W, int H, int elem,
                             cudaStream_t s) {
    const int vec_ok = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | sp | dp) & 15) == 0;
    const bool bfly = tune("transpose_bfly", 0) != 0;  // the earlier shuffle-butterfly kernel
    const int TX = bfly ? 256 / elem : 128 / elem;            // full tile: columns x rows
    const int TY = bfly ? kTT : (elem == 1 ? 128 : 64);
    const int FW = vec_ok ? W / TX * TX : 0, FH = vec_ok ? H / TY * TY : 0;  // full-tile region
    if (FW && FH) {
        dim3 grid(FW / TX, FH / TY);
        if (bfly) {
            if (elem == 1)
                transpose_image_bfly_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)src, sp, (uint8_t*)dst, dp, W, H);
            else
                transpose_image_bfly_kernel<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)src, sp, (uint16_t*)dst, dp, W,
                                                                          H);
        } else if (elem == 1) {
            transpose_image_blk_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)src, sp, (uint8_t*)dst, dp);
        } else {
            transpose_image_blk_kernel<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)src, sp, (uint16_t*)dst, dp);
        }
        count_launch();
    }
    // ragged right columns / bottom rows (and unaligned images): the shared-memory tile kernel
    auto ragged = [&](int xs, int ys, int w, int h) {
        if (w <= 0 || h <= 0) return;
        dim3 grid(cdiv(w, kTT), cdiv(h, kTT));
        const char* sb = static_cast<const char*>(src) + (size_t)ys * sp + (size_t)xs * elem;
        char* db = static_cast<char*>(dst) + (size_t)xs * dp + (size_t)ys * elem;
        const int v = ((reinterpret_cast<uintptr_t>(sb) | reinterpret_cast<uintptr_t>(db) | sp | dp) & 15) == 0;
        if (elem == 1)
            transpose_image_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)sb, sp, (uint8_t*)db, dp, w, h, v);
        else
            transpose_image_kernel<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)sb, sp / 2, (uint16_t*)db, dp / 2, w, h,
                                                                  v);
        count_launch();
    };
    ragged(FW, 0, W - FW, H);   // right strip, all rows
    ragged(0, FH, FW, H - FH);  // bottom strip under the full tiles
    return cudaGetLastError();
}

cudaError_t launch_transpose_tiles(void* data, size_t n_tiles, int n, size_t row_stride, size_t tile_step,
                                   int elem, cudaStream_t s) {
    if (n_tiles == 0) return cudaSuccess;
    const bool contiguous = row_stride == (size_t)n && tile_step == (size_t)n * n &&
                            (reinterpret_cast<uintptr_t>(data) & 15) == 0;
    const unsigned blocks = (unsigned)((n_tiles + 127) / 128);
    if (contiguous && ((elem == 1 && n == 16) || (elem == 2 && n == 8)) && n_tiles % (elem == 1 ? 2 : 4) == 0) {
        const size_t groups = n_tiles * n * n * elem / 512;
        const size_t want = (groups + 7) / 8;
        const unsigned grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
        if (elem == 1) tiles_warp_kernel<1><<<grid, 256, 0, s>>>((uint8_t*)data, groups);
        else tiles_warp_kernel<2><<<grid, 256, 0, s>>>((uint8_t*)data, groups);
        count_launch();
        return cudaGetLastError();
    }
    if (contiguous && elem == 1) {
        if (n == 4) tiles_u8_kernel<4><<<blocks, 128, 0, s>>>((uint8_t*)data, n_tiles);
        else if (n == 8) tiles_u8_kernel<8><<<blocks, 128, 0, s>>>((uint8_t*)data, n_tiles);
        else tiles_u8_kernel<16><<<blocks, 128, 0, s>>>((uint8_t*)data, n_tiles);
        count_launch();
        return cudaGetLastError();
    }
    if (contiguous && elem == 2 && n <= 8) {
        if (n == 4) tiles_u16_kernel<4><<<blocks, 128, 0, s>>>((uint16_t*)data, n_tiles);
        else tiles_u16_kernel<8><<<blocks, 128, 0, s>>>((uint16_t*)data, n_tiles);
        count_launch();
        return cudaGetLastError();
    }
    const size_t per = 256 / ((size_t)n * n);
    const size_t want = (n_tiles + per - 1) / per;
    const unsigned grid = (unsigned)(want < 148 * 64 ? want : 148 * 64);
    if (elem == 1) tiles_generic_kernel<uint8_t><<<grid, 256, 0, s>>>((uint8_t*)data, n_tiles, n, row_stride, tile_step);
    else if (elem == 2) tiles_generic_kernel<uint16_t><<<grid, 256, 0, s>>>((uint16_t*)data, n_tiles, n, row_stride, tile_step);
    else tiles_generic_kernel<uint32_t><<<grid, 256, 0, s>>>((uint32_t*)data, n_tiles, n, row_stride, tile_step);
    count_launch();
    return cudaGetLastError();
}

}  // namespace rmgpu

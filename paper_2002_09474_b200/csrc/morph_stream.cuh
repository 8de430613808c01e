// morph_stream.cuh -- shared infrastructure of the TMA-fed fused kernels (phase K2, col K1):
// strip geometry, 16-bit-lane min/max words, PTX helpers (mbarrier, bulk / tensor copies), work items
// and border-column selectors. (Originally the header of the v2 warp-specialised kernel.)
#pragma once

#include <algorithm>

#include <cuda.h>  // CUtensorMap (type only; encoded through the runtime's driver entry point)

#include "common.cuh"
#include "kernels.h"

namespace rmgpu {
namespace stream {

constexpr int QMAX = 6;                // whole blocks between suffix run and prefix block (registers)
constexpr int VCH = 16;                // rows per iteration for the direct vertical variants
constexpr int HC = 8;                  // horizontal lane chunk (block variant)


template <typename T>
struct SG;
template <>
struct SG<uint8_t> {
    static constexpr int PX = 4;     // pixels per 32-bit column word
    static constexpr int GR = 4;     // rows per transposed entry
    static constexpr int TW = 256;   // strip width (pixels)
    static constexpr int ESZ = 8;    // bytes per transposed entry (4 rows x 16-bit lanes)
    static constexpr int SWB = 16;   // entries per 128-byte swizzle row
};
template <>
struct SG<uint16_t> {
    static constexpr int PX = 2;
    static constexpr int GR = 2;
    static constexpr int TW = 128;
    static constexpr int ESZ = 4;
    static constexpr int SWB = 32;
};

// ---- lane words (16-bit lanes; one VIMNMX(3).U16x2 per min/max) ------------------------------
template <typename T>
struct LW;
template <>
struct LW<uint8_t> {
    uint32_t a, b;  // 4 pixels (row-major: a = {p0,p2}, b = {p1,p3}) or 4 rows of a column
};
template <>
struct LW<uint16_t> {
    uint32_t a;     // 2 pixels or 2 rows
};

template <int MODE>
__device__ __forceinline__ LW<uint8_t> lop(LW<uint8_t> x, LW<uint8_t> y) {
    return {red2_u16x2<MODE>(x.a, y.a), red2_u16x2<MODE>(x.b, y.b)};
}
template <int MODE>
__device__ __forceinline__ LW<uint16_t> lop(LW<uint16_t> x, LW<uint16_t> y) {
    return {red2_u16x2<MODE>(x.a, y.a)};
}
template <int MODE>
__device__ __forceinline__ LW<uint8_t> lop3(LW<uint8_t> x, LW<uint8_t> y, LW<uint8_t> z) {
    return {red3_u16x2<MODE>(x.a, y.a, z.a), red3_u16x2<MODE>(x.b, y.b, z.b)};
}
template <int MODE>
__device__ __forceinline__ LW<uint16_t> lop3(LW<uint16_t> x, LW<uint16_t> y, LW<uint16_t> z) {
    return {red3_u16x2<MODE>(x.a, y.a, z.a)};
}
template <typename T, int MODE>
__device__ __forceinline__ LW<T> lid() {
    LW<T> r;
    r.a = MODE == MODE_MIN ? 0xFFFFFFFFu : 0u;
    if constexpr (sizeof(T) == 1) r.b = r.a;
    return r;
}
__device__ __forceinline__ LW<uint8_t> unpack_w(uint32_t w, uint8_t*) { return {prmt(w, 0u, 0x4240), prmt(w, 0u, 0x4341)}; }
__device__ __forceinline__ LW<uint16_t> unpack_w(uint32_t w, uint16_t*) { return {w}; }

// ---- PTX helpers -------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "RM_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra RM_DONE;\n"
        "bra RM_WAIT;\n"
        "RM_DONE:\n"
        "}\n" ::"r"(saddr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(bar))
                 : "memory");
}
// One TMA tensor copy of a box {RP/4 words, B rows} (3-D map: words, rows, images).
__device__ __forceinline__ void tma_box(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            saddr(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(saddr(bar))
        : "memory");
}
// TMA tensor store of a box {TW*sz bytes, B rows} from shared memory (3-D map: bytes, rows, images).
__device__ __forceinline__ void tma_store_box(const CUtensorMap* map, int x, int y, int z, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map),
                 "r"(x), "r"(y), "r"(z), "r"(saddr(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// ---- layout ---------------------------------------------------------------------------------
struct StreamParams {
    const uint8_t* src;
    size_t sp;
    uint8_t* dst;
    size_t dp;
    int W, H;
    int row_lo, row_hi;   // valid input rows (relative to output row 0 of the image)
    int gx, gy;
    int cmode;
    uint32_t bval;
    size_t simg, dimg;
    int rh;               // output rows per CTA
    int pf;               // input blocks prefetched ahead of the leading block (TMA bytes in flight)
    long long* trace;     // debug timeline (nullptr normally): CTA (trace_cta) records clock64 stamps
    int trace_cta;
    int use_tma;          // interior blocks through one 2-D tensor copy (map rows start at row_lo)
    int use_tma_out;      // full output chunks through one TMA tensor store
    int batch;            // images
};

#ifdef RMGPU_TRACE
#define RM_TRACE(slot)                                                                                   \
    do {                                                                                                 \
        if (p.trace && blockIdx.x == (unsigned)p.trace_cta && (threadIdx.x & 31) == 0) p.trace[(slot)] = clock64(); \
    } while (0)
#else
#define RM_TRACE(slot) \
    do {               \
    } while (0)
#endif

// Compile-time geometry of one horizontal class HB: 1/3/5/7 = direct window (gx = (HB-1)/2),
// 8 / 9 = lane-chunk block algorithm for gx up to GXMAX (small / large halo).
template <typename T, int HB>
struct HG {
    static constexpr int sz = sizeof(T);
    static constexpr int TW = SG<T>::TW;
    static constexpr int GXMAX = HB <= 7 ? (HB - 1) / 2 : (HB == 8 ? (sz == 1 ? 48 : 24) : (sz == 1 ? 64 : 32));
    static constexpr int RP = ((TW * sz + 2 * GXMAX * sz + 31) / 16) * 16;  // ring row pitch (bytes)
    static constexpr int NCH = (TW + 2 * GXMAX + 7) / 8 + 2;                // 8-column chunks (+ slack)
    static constexpr int NCHP = NCH | 1;                                     // odd: conflict-free lanes
    static constexpr int VTG = 8 * NCHP;                                     // entries per row group
    static constexpr int LPG = TW / 8;                                       // lanes per row group
    static constexpr int NVW = (RP / (2 * sz) + 31) / 32;                    // vertical warps (2 px/thread)
};

// Shared-memory plan, identical on host and device (B and q runtime -> NSB; rest compile-time).


// Column fix-up for a 2-pixel word at image column c: byte source nibbles over (raw, Z), where Z
// bytes 0 (and 1 for u16) hold the constant border value. Returns the ring byte offset to load.
template <typename T>
__device__ __forceinline__ void col_fix(int c, int W, int cmode, int xs_col, int& load_off, uint32_t& nib,
                                        bool& fix) {
    constexpr int sz = sizeof(T);
    fix = !(c >= 0 && c + 1 < W);
    const int cc0 = min(max(c, 0), W - 1);
    const int cl = fix ? (cc0 / 2) * 2 : c;
    load_off = (cl - xs_col) * sz;
    nib = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int col = c + j;
#pragma unroll
        for (int b = 0; b < sz; ++b) {
            int n;
            if (!fix) n = j * sz + b;
            else if (cmode && (col < 0 || col >= W)) n = 4 + b;
            else n = (min(max(col, 0), W - 1) - cl) * sz + b;
            nib |= (uint32_t)n << (4 * (j * sz + b));
        }
    }
}

__device__ __forceinline__ uint32_t nib_at(uint32_t nib, int k) { return (nib >> (4 * k)) & 0xF; }

struct Item {
    int x0, y0, rh, b;
    int xs_b, xs_col, copy_len, cb0, nwv, off, y_first, Lend, Lf;
};

template <typename T>
__device__ __forceinline__ Item make_item(const StreamParams& p, int idx, int nstrips, int nrowb, int B, int w1,
                                          int s) {
    constexpr int TW = SG<T>::TW, sz = sizeof(T);
    Item it;
    const int per_img = nstrips * nrowb;
    it.b = idx / per_img;
    const int rem = idx - it.b * per_img;
    const int ry = rem / nstrips;
    it.x0 = (rem - ry * nstrips) * TW;
    it.y0 = ry * p.rh;
    it.rh = min(p.rh, p.H - it.y0);
    const int xb = (it.x0 - p.gx) * sz;
    it.xs_b = xb >= 0 ? (xb / 16) * 16 : -(((-xb) + 15) / 16) * 16;
    it.xs_col = it.xs_b / sz;
    const int xe_b = ((it.x0 + TW + p.gx) * sz + 15) / 16 * 16;
    const int w_b16 = (p.W * sz + 15) / 16 * 16;
    it.cb0 = max(it.xs_b, 0);
    it.copy_len = min(xe_b, w_b16) - it.cb0;
    it.nwv = (xe_b - it.xs_b) / (2 * sz);
    it.off = (it.x0 - p.gx) - it.xs_col;
    it.y_first = it.y0 - p.gy;
    it.Lend = (it.rh - 1 + w1 - s) / B;
    int Lf = 0;
    while (s + Lf * B - w1 + B - 1 < 0) ++Lf;
    it.Lf = Lf;
    return it;
}

extern long long* g_trace;   // debug timeline buffer (device), set by rmgpu_debug_trace
extern int g_trace_cta;
// Encodes the 3-D tensor map {words, rows, images} of the job's valid input rows (host).
bool encode_input_map(const MorphJob& j, int box_words, int box_rows, CUtensorMap* map);
// 3-D byte-granular map {bytes, rows, images} of the output (box = one full chunk of the strip).
bool encode_output_map(const MorphJob& j, int box_bytes, int box_rows, CUtensorMap* map);

inline int stream_gxmax(int elem, int hb) {
    return elem == 1 ? (hb <= 7 ? (hb - 1) / 2 : hb == 8 ? HG<uint8_t, 8>::GXMAX : HG<uint8_t, 9>::GXMAX)
                     : (hb <= 7 ? (hb - 1) / 2 : hb == 8 ? HG<uint16_t, 8>::GXMAX : HG<uint16_t, 9>::GXMAX);
}

template <typename T>
inline int stream_ring_row(int hb) {
    switch (hb) {
    case 1: return HG<T, 1>::RP;
    case 3: return HG<T, 3>::RP;
    case 5: return HG<T, 5>::RP;
    case 7: return HG<T, 7>::RP;
    case 8: return HG<T, 8>::RP;
    default: return HG<T, 9>::RP;
    }
}

}  // namespace stream
}  // namespace rmgpu

// morph_stream.cuh -- K1/K2 v2: warp-specialised, TMA-fed, strip-streaming fused separable
// erosion / dilation (u8, u16). Design notes in morph_stream.cu.
#pragma once

#include <algorithm>

#include <cuda.h>  // CUtensorMap (type only; encoded through the runtime's driver entry point)

#include "common.cuh"
#include "kernels.h"

namespace rmgpu {
namespace stream {

// horizontal warps: one per 4-row group of a chunk of B rows (2..8)
__host__ __device__ constexpr int nhw_of(int B) { return B / 4 < 2 ? 2 : (B / 4 > 8 ? 8 : B / 4); }
constexpr int QMAX = 6;                // whole blocks between suffix run and prefix block (registers)
constexpr int VCH = 16;                // rows per iteration for the direct vertical variants
constexpr int HC = 8;                  // horizontal lane chunk (block variant)

// named barrier ids (0 is __syncthreads)
constexpr int BAR_VW = 1, BAR_FULL0 = 2, BAR_EMPTY0 = 4, BAR_HW = 6;

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
    int sleep_ns;         // phase kernel: producer back-off when it has nothing to issue
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
struct Plan {
    int NSB, off_ring, off_vt, off_hs, off_out, total;
};

template <typename T, int HB>
__host__ __device__ inline Plan make_plan(int B, int q, int PF) {
    using H = HG<T, HB>;
    using G = SG<T>;
    Plan p;
    p.NSB = q + 2 + PF;
    int o = 64 * 8;  // mbarriers
    p.off_ring = o;
    o += p.NSB * B * H::RP;
    p.off_vt = o;
    o += 2 * (B / G::GR) * H::VTG * G::ESZ;
    p.off_hs = o;
    if (HB > 7) o += nhw_of(B) * (32 / H::LPG) * (H::VTG + H::NCHP) * G::ESZ;
    o = (o + 127) / 128 * 128;
    p.off_out = o;
    o += 2 * B * G::TW * (int)sizeof(T);
    p.total = o;
    return p;
}

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

// ---- the kernel ------------------------------------------------------------------------------
// VB: vertical variant: 1/3/5/7 = direct window (VCH rows per iteration), 8/16/24 = block size B.
// HB: horizontal class (HG).
template <typename T, int VB, int HB>
struct KG {  // per-kernel thread layout
    static constexpr int B = VB <= 7 ? VCH : VB;
    static constexpr int NHW = nhw_of(B);
    static constexpr int NVW = HG<T, HB>::NVW;
    static constexpr int NTH = 32 * (NVW + NHW);
};

// Work item = (strip, row range, image); items are processed persistently by the CTAs of a 1-D
// grid (CTA c takes items c, c + G, ...), and the TMA block stream runs on across items so the
// next item's first rows arrive while the current one finishes.
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

template <int MODE>
__device__ __forceinline__ uint32_t tree_min(uint32_t a, uint32_t b, uint32_t c) {
    return red3_u16x2<MODE>(a, b, c);
}

template <typename T, int MODE, int VB, int HB>
__global__ void __launch_bounds__(KG<T, VB, HB>::NTH)
morph_stream_kernel(const StreamParams p, const __grid_constant__ CUtensorMap tmap,
                    const __grid_constant__ CUtensorMap omap) {
    using G = SG<T>;
    using H = HG<T, HB>;
    constexpr int GR = G::GR, TW = G::TW, ESZ = G::ESZ;
    constexpr int sz = sizeof(T);
    constexpr bool VDIRECT = VB <= 7;
    constexpr int B = VDIRECT ? VCH : VB;
    constexpr int NGC = B / GR;          // row groups per chunk
    constexpr int OUTP = TW * sz;        // output tile row pitch (packed: TMA store box)
    constexpr int RP = H::RP, NCHP = H::NCHP, VTG = H::VTG, LPG = H::LPG;
    constexpr int NVW = KG<T, VB, HB>::NVW, NTH = KG<T, VB, HB>::NTH, NHW = KG<T, VB, HB>::NHW;
    constexpr int SUBG = 32 / LPG;       // row groups per warp pass
    extern __shared__ __align__(128) unsigned char smem[];

    const int gy = p.gy;
    const int w1 = 2 * gy, w1x = 2 * p.gx;
    const int q = VDIRECT ? 0 : w1 / B;
    const int r = VDIRECT ? w1 : w1 - q * B;
    const int s = r & 3;
    const int PF = p.pf;
    const Plan pl = make_plan<T, HB>(B, q, PF);
    const int NSB = pl.NSB;
    const int nstrips = (p.W + TW - 1) / TW;
    const int nrowb = (p.H + p.rh - 1) / p.rh;
    const int nitems = nstrips * nrowb * p.batch;
    const int G0 = (int)gridDim.x;

    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    unsigned char* ring = smem + pl.off_ring;
    unsigned char* vt = smem + pl.off_vt;
    unsigned char* hs = smem + pl.off_hs;
    unsigned char* outbase = smem + pl.off_out;

    const uint32_t bv = sz == 1 ? (p.bval & 0xFF) : (p.bval & 0xFFFF);

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int k = 0; k < NSB; ++k) mbar_init(&full[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int warp = tid >> 5, lane = tid & 31;
    auto item_at = [&](int n) { return (int)blockIdx.x + n * G0; };  // n-th item of this CTA

    if (warp < NVW) {
        // ================= vertical role: producer (warp 0) + streaming column sweeps =========
        // ---- producer cursor (warp 0): block pk of this CTA's item pn ------------------------
        int pn = 0, pk = -1;
        Item pit;
        bool pvalid = item_at(0) < nitems;
        if (pvalid) pit = make_item<T>(p, item_at(0), nstrips, nrowb, B, w1, s);
        int pslot = 0;  // ring slot of the next block to issue
        auto issue_next = [&]() {
            if (!pvalid) return;
            const int slot = pslot;
            unsigned char* base = ring + (size_t)slot * B * RP;
            const int yb = pit.y_first + s + pk * B;
            if (p.use_tma && yb >= p.row_lo && yb + B <= p.row_hi) {
                if (lane == 0) {
                    mbar_arrive_tx(&full[slot], (uint32_t)(B * RP));
                    tma_box(base, &tmap, pit.xs_b / 4, yb - p.row_lo, pit.b, &full[slot]);
                }
            } else {
                const uint8_t* src = p.src + (size_t)pit.b * p.simg;
                const int y = yb + lane;
                const bool inrow = lane < B;
                const bool outside = p.cmode && (y < p.row_lo || y >= p.row_hi);
                const unsigned cp = __ballot_sync(0xffffffffu, inrow && !outside);
                unsigned fillm = __ballot_sync(0xffffffffu, inrow && outside);
                while (fillm) {  // constant rows outside the image: the warp writes the border value
                    const int m = __ffs(fillm) - 1;
                    fillm &= fillm - 1;
                    const uint32_t bw = sz == 1 ? bv * 0x01010101u : bv * 0x00010001u;
                    uint4* row = reinterpret_cast<uint4*>(base + (size_t)m * RP);
                    for (int c = lane; c < RP / 16; c += 32) row[c] = make_uint4(bw, bw, bw, bw);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_tx(&full[slot], (uint32_t)(__popc(cp) * pit.copy_len));
                __syncwarp();
                if (inrow && !outside) {
                    const int yc = min(max(y, p.row_lo), p.row_hi - 1);
                    bulk_g2s(base + (size_t)lane * RP + (pit.cb0 - pit.xs_b),
                             src + (ptrdiff_t)yc * (ptrdiff_t)p.sp + pit.cb0, (uint32_t)pit.copy_len, &full[slot]);
                }
            }
            pslot = pslot + 1 == NSB ? 0 : pslot + 1;
            if (++pk > pit.Lend) {
                ++pn;
                pk = -1;
                pvalid = item_at(pn) < nitems;
                if (pvalid) pit = make_item<T>(p, item_at(pn), nstrips, nrowb, B, w1, s);
            }
        };
        if (warp == 0) {
            if (lane == 0 && p.use_tma) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap) : "memory");
            for (int k = 0; k <= PF; ++k) issue_next();  // blocks seq 0 .. PF
        }

        auto op2 = [](uint32_t x, uint32_t y) { return red2_u16x2<MODE>(x, y); };
        auto op3 = [](uint32_t x, uint32_t y, uint32_t z) { return red3_u16x2<MODE>(x, y, z); };
        constexpr uint32_t IDV = MODE == MODE_MIN ? 0xFFFFFFFFu : 0u;

        // consumed block stream: slot/parity of the current block and of blocks -1, -q, -q-1
        int seq = 0, sL = 0, ph = 0;
        int sL1 = NSB - 1, sQ = ((-q) % NSB + NSB) % NSB, sQ1 = ((-q - 1) % NSB + NSB) % NSB;
        auto advance = [&]() {
            ++seq;
            sL1 = sL;
            sL = sL + 1 == NSB ? 0 : sL + 1;
            ph ^= sL == 0;
            sQ1 = sQ;
            sQ = sQ + 1 == NSB ? 0 : sQ + 1;
        };
        int chunk = 0;
        for (int n = 0; item_at(n) < nitems; ++n) {
            const Item it = make_item<T>(p, item_at(n), nstrips, nrowb, B, w1, s);
            // thread t owns image columns xs_col + 2t, +1 as one u16x2 word (u8 unpacked on load)
            const int t = tid;
            const bool active = t < it.nwv;
            int load_off = 0;
            uint32_t nib = 0;
            bool fix = false;
            col_fix<T>(it.xs_col + 2 * (active ? t : 0), p.W, p.cmode, it.xs_col, load_off, nib, fix);
            const uint32_t selU =
                sz == 1 ? ((nib & 0xF) | (5u << 4) | (((nib >> 4) & 0xF) << 8) | (5u << 12)) : nib;
            const uint32_t Z = bv;
            int voff0, voff1;
            {
                const int pos0 = 2 * t - it.off, pos1 = pos0 + 1;
                voff0 = (active && pos0 >= 0 && pos0 < 8 * H::NCH) ? ((pos0 & 7) * NCHP + (pos0 >> 3)) * ESZ : -1;
                voff1 = (active && pos1 >= 0 && pos1 < 8 * H::NCH) ? ((pos1 & 7) * NCHP + (pos1 >> 3)) * ESZ : -1;
            }
            auto ldw = [&](const unsigned char* a) -> uint32_t {
                if constexpr (sz == 1) {
                    const uint32_t raw = *reinterpret_cast<const uint16_t*>(a);
                    return prmt(raw, Z, selU);
                } else {
                    const uint32_t raw = *reinterpret_cast<const uint32_t*>(a);
                    return fix ? prmt(raw, Z, selU) : raw;
                }
            };
            const unsigned char* rbase = ring + load_off;
            auto sbase = [&](int slot) { return rbase + (size_t)slot * (B * RP); };

            // block -1 of this item: never a leading block, wait for it before its trailing use
            // producer stays exactly PF blocks ahead: consuming seq g issues seq g + PF (the
            // prologue covered 0..PF), whose slot held seq g + PF - NSB = g - q - 2: dead.
            bar_sync(BAR_VW, NVW * 32);
            if (warp == 0 && seq > 0) issue_next();
            mbar_wait(&full[sL], (uint32_t)ph);
            advance();

            uint32_t M[QMAX];
#pragma unroll
            for (int k = 0; k < QMAX; ++k) M[k] = IDV;
            for (int L = 0; L <= it.Lend; ++L, advance()) {
                if (warp == 0 && L < 60 && n == 0) RM_TRACE(L * 8 + 0);
                bar_sync(BAR_VW, NVW * 32);  // iteration L-1 done by every vertical thread
                if (warp == 0) issue_next();
                if (warp == 0 && L < 60 && n == 0) RM_TRACE(L * 8 + 1);
                mbar_wait(&full[sL], (uint32_t)ph);
                if (warp == 0 && L < 60 && n == 0) RM_TRACE(L * 8 + 2);
                const bool emit = L >= it.Lf;
                const int buf = chunk & 1;
                if (emit) bar_sync(BAR_EMPTY0 + buf, NTH);
                if (warp == 0 && L < 60 && n == 0) RM_TRACE(L * 8 + 3);
                if (active) {
                    const unsigned char* lead = sbase(sL);
                    unsigned char* vb = vt + (size_t)buf * NGC * VTG * ESZ;
                    uint32_t grp[GR];
                    auto flush = [&](int m0) {
                        unsigned char* rowg = vb + (m0 / GR) * VTG * ESZ;
                        if constexpr (sz == 1) {
                            if (voff0 >= 0)
                                *reinterpret_cast<uint2*>(rowg + voff0) =
                                    make_uint2(prmt(grp[0], grp[2], 0x5410), prmt(grp[1], grp[3], 0x5410));
                            if (voff1 >= 0)
                                *reinterpret_cast<uint2*>(rowg + voff1) =
                                    make_uint2(prmt(grp[0], grp[2], 0x7632), prmt(grp[1], grp[3], 0x7632));
                        } else {
                            if (voff0 >= 0) *reinterpret_cast<uint32_t*>(rowg + voff0) = prmt(grp[0], grp[1], 0x5410);
                            if (voff1 >= 0) *reinterpret_cast<uint32_t*>(rowg + voff1) = prmt(grp[0], grp[1], 0x7632);
                        }
                    };
                    if constexpr (VDIRECT) {
                        constexpr int WD = VB;
                        uint32_t X[B + WD - 1];
                        const unsigned char* prev = sbase(sL1);
#pragma unroll
                        for (int k = 0; k < WD - 1; ++k) X[k] = ldw(prev + (B - (WD - 1) + k) * RP);
#pragma unroll
                        for (int m = 0; m < B; ++m) X[WD - 1 + m] = ldw(lead + m * RP);
                        if (emit) {
#pragma unroll
                            for (int m = 0; m < B; ++m) {
                                uint32_t o;
                                if constexpr (WD == 1) o = X[m];
                                else if constexpr (WD == 3) o = op3(X[m], X[m + 1], X[m + 2]);
                                else if constexpr (WD == 5) o = op3(op3(X[m], X[m + 1], X[m + 2]), X[m + 3], X[m + 4]);
                                else o = op3(op3(X[m], X[m + 1], X[m + 2]), op3(X[m + 3], X[m + 4], X[m + 5]), X[m + 6]);
                                grp[m % GR] = o;
                                if (m % GR == GR - 1) flush(m - (GR - 1));
                            }
                        }
                    } else {
                        uint32_t P[B];
                        P[0] = ldw(lead);
#pragma unroll
                        for (int m = 1; m < B; ++m) P[m] = op2(P[m - 1], ldw(lead + m * RP));
                        if (emit) {
                            // gap = tail r rows of block L-q + whole blocks L-q+1 .. L-1 (tree-reduced)
                            const unsigned char* tb = sbase(sQ);  // block L-q
                            const unsigned char* tt = tb + (B - r) * RP;
                            uint32_t v[B + QMAX];
#pragma unroll
                            for (int i = 0; i < B - 1; ++i) v[i] = i < r ? ldw(tt + i * RP) : IDV;
#pragma unroll
                            for (int k = 0; k < QMAX - 1; ++k) v[B - 1 + k] = k < q - 1 ? M[k] : IDV;
                            constexpr int NV = B - 1 + QMAX - 1;
                            uint32_t gap = IDV;
#pragma unroll
                            for (int i = 0; i < NV; i += 3) {
                                const uint32_t x = v[i], y = i + 1 < NV ? v[i + 1] : IDV, z = i + 2 < NV ? v[i + 2] : IDV;
                                v[i / 3] = op3(x, y, z);
                            }
#pragma unroll
                            for (int i = 0; i < (NV + 2) / 3; i += 3) {
                                const int nv2 = (NV + 2) / 3;
                                const uint32_t x = v[i], y = i + 1 < nv2 ? v[i + 1] : IDV, z = i + 2 < nv2 ? v[i + 2] : IDV;
                                gap = op3(gap, op3(x, y, z), IDV);
                            }
                            // trailing run rows oL + m: block L-q-1 row B-r+m (m < r), block L-q row m-r
                            const unsigned char* ta = sbase(sQ1) + (B - r) * RP;
                            const unsigned char* tbb = tb - r * RP;
                            uint32_t acc = gap;
#pragma unroll
                            for (int m = B - 1; m >= 0; --m) {
                                acc = op2(acc, ldw((m < r ? ta : tbb) + m * RP));
                                grp[m % GR] = op2(acc, P[m]);
                                if (m % GR == 0) flush(m);
                            }
                        }
#pragma unroll
                        for (int k = QMAX - 1; k > 0; --k) M[k] = M[k - 1];
                        M[0] = P[B - 1];
                    }
                }
                if (warp == 0 && L < 60 && n == 0) RM_TRACE(L * 8 + 4);
                if (emit) {
                    bar_arrive(BAR_FULL0 + buf, NTH);
                    ++chunk;
                }
            }
        }
        // balance the horizontal side's extra releases so every barrier generation completes
        bar_sync(BAR_EMPTY0 + (chunk & 1), NTH);
        bar_sync(BAR_EMPTY0 + ((chunk + 1) & 1), NTH);
    } else {
        // ================= horizontal role ========================================================
        const int hw = warp - NVW;
        bar_arrive(BAR_EMPTY0 + 0, NTH);
        bar_arrive(BAR_EMPTY0 + 1, NTH);
        const int sub = lane / LPG;       // row group within the warp pass
        const int lam = lane % LPG;       // 8-column chunk owned by this lane
        unsigned char* scr = hs + (size_t)(hw * SUBG + sub) * (VTG + NCHP) * ESZ;  // P scratch, then M
        unsigned char* msc = scr + (size_t)VTG * ESZ;
        const int q8 = w1x >> 3, r8 = w1x & 7;
        auto ld8 = [&](const unsigned char* a) -> LW<T> {
            LW<T> v;
            if constexpr (sz == 1) {
                const uint2 u = *reinterpret_cast<const uint2*>(a);
                v.a = u.x;
                v.b = u.y;
            } else {
                v.a = *reinterpret_cast<const uint32_t*>(a);
            }
            return v;
        };
        auto st8 = [&](unsigned char* a, LW<T> v) {
            if constexpr (sz == 1) *reinterpret_cast<uint2*>(a) = make_uint2(v.a, v.b);
            else *reinterpret_cast<uint32_t*>(a) = v.a;
        };
        int chunk = 0;
        for (int n = 0; item_at(n) < nitems; ++n) {
            const Item it = make_item<T>(p, item_at(n), nstrips, nrowb, B, w1, s);
            uint8_t* dst = p.dst + (size_t)it.b * p.dimg;
            for (int L = it.Lf; L <= it.Lend; ++L, ++chunk) {
                const int buf = chunk & 1;
                if (hw == 0 && L < 60 && n == 0) RM_TRACE(480 + L * 8 + 0);
                // the previous chunk's TMA store must have finished reading its output buffer
                if (p.use_tma_out && tid == NVW * 32) bulk_wait_read0();
                bar_sync(BAR_FULL0 + buf, NTH);
                unsigned char* outt = outbase + (size_t)buf * B * OUTP;
                if (hw == 0 && L < 60 && n == 0) RM_TRACE(480 + L * 8 + 1);
                const int oL = s + L * B - w1;
                const unsigned char* vb = vt + (size_t)buf * NGC * VTG * ESZ;
                for (int g0 = hw * SUBG; g0 < NGC; g0 += NHW * SUBG) {
                    const int g = g0 + sub;
                    const int o_g = oL + g * GR;
                    const bool live = g < NGC && o_g + GR - 1 >= 0 && o_g < it.rh;
                    const unsigned char* rowg = vb + (size_t)(g < NGC ? g : 0) * VTG * ESZ;
                    auto emit4 = [&](int a, LW<T> c0, LW<T> c1, LW<T> c2, LW<T> c3) {
                        unsigned char* po = outt + (size_t)(g * GR) * OUTP + (size_t)a * sz;
                        if constexpr (sz == 1) {
                            const uint32_t a01 = prmt(c0.a, c1.a, 0x6240), a23 = prmt(c2.a, c3.a, 0x6240);
                            const uint32_t b01 = prmt(c0.b, c1.b, 0x6240), b23 = prmt(c2.b, c3.b, 0x6240);
                            *reinterpret_cast<uint32_t*>(po) = prmt(a01, a23, 0x5410);
                            *reinterpret_cast<uint32_t*>(po + OUTP) = prmt(b01, b23, 0x5410);
                            *reinterpret_cast<uint32_t*>(po + 2 * OUTP) = prmt(a01, a23, 0x7632);
                            *reinterpret_cast<uint32_t*>(po + 3 * OUTP) = prmt(b01, b23, 0x7632);
                        } else {  // u16: two columns per call (c2, c3 unused)
                            *reinterpret_cast<uint32_t*>(po) = prmt(c0.a, c1.a, 0x5410);
                            *reinterpret_cast<uint32_t*>(po + OUTP) = prmt(c0.a, c1.a, 0x7632);
                        }
                    };
                    auto emit8 = [&](const LW<T> (&o)[8]) {
#pragma unroll
                        for (int j = 0; j < 8; j += GR) {
                            if constexpr (GR == 4) emit4(8 * lam + j, o[j], o[j + 1], o[j + 2], o[j + 3]);
                            else emit4(8 * lam + j, o[j], o[j + 1], o[j], o[j]);
                        }
                    };
                    if constexpr (HB <= 7) {
                        constexpr int WD = HB;
                        LW<T> X[8 + WD - 1];
                        const unsigned char* b0 = rowg + lam * ESZ;
#pragma unroll
                        for (int i = 0; i < 8 + WD - 1; ++i) X[i] = ld8(b0 + ((i & 7) * NCHP + (i >> 3)) * ESZ);
                        LW<T> o[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if constexpr (WD == 1) o[j] = X[j];
                            else if constexpr (WD == 3) o[j] = lop3<MODE>(X[j], X[j + 1], X[j + 2]);
                            else if constexpr (WD == 5) o[j] = lop3<MODE>(lop3<MODE>(X[j], X[j + 1], X[j + 2]), X[j + 3], X[j + 4]);
                            else o[j] = lop3<MODE>(lop3<MODE>(X[j], X[j + 1], X[j + 2]), lop3<MODE>(X[j + 3], X[j + 4], X[j + 5]), X[j + 6]);
                        }
                        if (live) emit8(o);
                    } else {
                        const int nch = (TW + w1x + 7) >> 3;
                        LW<T> S[8];
                        for (int k = lam; k < nch; k += LPG) {
                            LW<T> x[8];
                            const unsigned char* b0 = rowg + k * ESZ;
#pragma unroll
                            for (int j = 0; j < 8; ++j) x[j] = ld8(b0 + j * NCHP * ESZ);
                            LW<T> pre = x[0];
                            unsigned char* pb = scr + k * ESZ;
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                if (j) pre = lop<MODE>(pre, x[j]);
                                st8(pb + j * NCHP * ESZ, pre);
                            }
                            st8(msc + k * ESZ, pre);
                            if (k == lam) {
                                S[7] = x[7];
#pragma unroll
                                for (int j = 6; j >= 0; --j) S[j] = lop<MODE>(S[j + 1], x[j]);
                            }
                        }
                        __syncwarp();
                        {
                            const int k = lam;
                            // chunk minima strictly between (k, k+q8[+1]): tree of predicated loads
                            constexpr int QM8 = H::GXMAX / 4 + 1;
                            LW<T> mv[QM8 + 2];
#pragma unroll
                            for (int i = 0; i < QM8 + 2; ++i) mv[i] = lid<T, MODE>();
#pragma unroll
                            for (int i = 1; i < QM8; ++i)
                                if (i < q8) mv[i - 1] = ld8(msc + (k + i) * ESZ);
                            LW<T> Fa = lid<T, MODE>();
#pragma unroll
                            for (int i = 0; i < QM8; i += 3) Fa = lop<MODE>(Fa, lop3<MODE>(mv[i], mv[i + 1], mv[i + 2]));
                            const LW<T> Fb = lop<MODE>(Fa, ld8(msc + (k + q8) * ESZ));
                            const unsigned char* pa = scr + (r8 * NCHP + k + q8) * ESZ;
                            const unsigned char* pbb = scr + ((r8 - 8) * NCHP + k + q8 + 1) * ESZ;
                            LW<T> o[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const bool lo = j < 8 - r8;
                                o[j] = lop3<MODE>(S[j], lo ? Fa : Fb, ld8((lo ? pa : pbb) + j * NCHP * ESZ));
                            }
                            if (live) emit8(o);
                        }
                        __syncwarp();
                    }
                }
                if (hw == 0 && L < 60 && n == 0) RM_TRACE(480 + L * 8 + 2);
                bar_arrive(BAR_EMPTY0 + buf, NTH);
                const int rlo = max(0, -oL), rhi = min(B, it.rh - oL);
                // TMA stores only full chunks of full-width strips: the hardware rounds the right
                // clip edge to 16 bytes, which would touch the caller's row padding
                const bool full_chunk = p.use_tma_out && rlo == 0 && rhi == B && it.x0 + TW <= p.W;
                if (full_chunk) fence_async_smem();  // emits visible to the TMA (async proxy)
                bar_sync(BAR_HW, NHW * 32);
                if (hw == 0 && L < 60 && n == 0) RM_TRACE(480 + L * 8 + 3);
                if (full_chunk) {
                    if (tid == NVW * 32) {
                        tma_store_box(&omap, it.x0 * sz, it.y0 + oL, it.b, outt);
                        bulk_commit();
                    }
                } else {
                    const int htid = tid - NVW * 32;  // horizontal thread index
                    const int cols = min(TW, p.W - it.x0);
                    const int row_bytes = cols * sz;
                    const bool vec = (((uintptr_t)dst | p.dp) & 15) == 0 && cols == TW;
                    if (vec) {
                        constexpr int CPR = TW * sz / 16;
                        for (int i = rlo * CPR + htid; i < rhi * CPR; i += NHW * 32) {
                            const int rr = i / CPR, ch = i % CPR;
                            const uint4 v = *reinterpret_cast<const uint4*>(outt + (size_t)rr * OUTP + ch * 16);
                            *reinterpret_cast<uint4*>(dst + (size_t)(it.y0 + oL + rr) * p.dp + (size_t)it.x0 * sz + ch * 16) = v;
                        }
                    } else {
                        for (int i = rlo * row_bytes + htid; i < rhi * row_bytes; i += NHW * 32) {
                            const int rr = i / row_bytes, b = i % row_bytes;
                            dst[(size_t)(it.y0 + oL + rr) * p.dp + (size_t)it.x0 * sz + b] = outt[(size_t)rr * OUTP + b];
                        }
                    }
                }
                if (hw == 0 && L < 60 && n == 0) RM_TRACE(480 + L * 8 + 4);
            }
        }
        if (p.use_tma_out && tid == NVW * 32) bulk_wait_all();
    }
}

// ---- host launch ------------------------------------------------------------------------------
extern long long* g_trace;   // debug timeline buffer (device), set by rmgpu_debug_trace
extern int g_trace_cta;
// Encodes the 3-D tensor map {words, rows, images} of the job's valid input rows (host).
bool encode_input_map(const MorphJob& j, int box_words, int box_rows, CUtensorMap* map);
// 3-D byte-granular map {bytes, rows, images} of the output (box = one full chunk of the strip).
bool encode_output_map(const MorphJob& j, int box_bytes, int box_rows, CUtensorMap* map);

template <typename T, int MODE, int VB, int HB>
cudaError_t launch_stream_variant(const MorphJob& j, int rh, int B, int q, int pf) {
    using G = SG<T>;
    StreamParams p;
    p.src = static_cast<const uint8_t*>(j.src);
    p.sp = j.sp;
    p.dst = static_cast<uint8_t*>(j.dst);
    p.dp = j.dp;
    p.W = j.W;
    p.H = j.H;
    p.row_lo = -j.above;
    p.row_hi = j.H + j.below;
    p.gx = j.gx;
    p.gy = j.gy;
    p.cmode = j.cmode;
    p.bval = j.bval;
    p.simg = j.simg;
    p.dimg = j.dimg;
    p.rh = rh;
    p.pf = pf;
    p.trace = g_trace;
    p.trace_cta = g_trace_cta;
    CUtensorMap map;
    p.use_tma = encode_input_map(j, HG<T, HB>::RP / 4, B, &map) ? 1 : 0;
    CUtensorMap omap;
    p.use_tma_out = encode_output_map(j, G::TW * (int)sizeof(T), B, &omap) ? 1 : 0;
    const Plan pl = make_plan<T, HB>(B, q, pf);
    auto kern = morph_stream_kernel<T, MODE, VB, HB>;
    cudaError_t e = cudaSuccess;
    const int occ = kernel_occupancy((const void*)kern, KG<T, VB, HB>::NTH, pl.total, &e);
    if (e != cudaSuccess) return e;
    const int sms = device_sm_count();
    const long items = (long)cdiv(j.W, G::TW) * cdiv(j.H, rh) * j.batch;
    const long ctas = std::max(1L, std::min(items, (long)sms * std::max(1, occ)));
    dim3 grid((unsigned)ctas, 1, 1);
    p.batch = j.batch;
    kern<<<grid, KG<T, VB, HB>::NTH, pl.total, j.stream>>>(p, map, omap);
    count_launch();
    return cudaGetLastError();
}

#define RM_STREAM_V(X) X(1) X(3) X(5) X(7) X(8) X(16) X(24)
#define RM_STREAM_H(X) X(1) X(3) X(5) X(7) X(8) X(9)

template <typename T, int MODE, int VB>
cudaError_t stream_dispatch_h(const MorphJob& j, int hb, int rh, int B, int q, int pf) {
    switch (hb) {
#define RM_CASE(H) \
    case H: return launch_stream_variant<T, MODE, VB, H>(j, rh, B, q, pf);
        RM_STREAM_H(RM_CASE)
#undef RM_CASE
    }
    return cudaErrorInvalidValue;
}

template <typename T, int MODE>
cudaError_t stream_dispatch(const MorphJob& j, int vb, int hb, int rh, int B, int q, int pf) {
    switch (vb) {
#define RM_CASE(V) \
    case V: return stream_dispatch_h<T, MODE, V>(j, hb, rh, B, q, pf);
        RM_STREAM_V(RM_CASE)
#undef RM_CASE
    }
    return cudaErrorInvalidValue;
}

// Host-side planning helpers shared with morph_stream.cu
inline int stream_gxmax(int elem, int hb) {
    return elem == 1 ? (hb <= 7 ? (hb - 1) / 2 : hb == 8 ? HG<uint8_t, 8>::GXMAX : HG<uint8_t, 9>::GXMAX)
                     : (hb <= 7 ? (hb - 1) / 2 : hb == 8 ? HG<uint16_t, 8>::GXMAX : HG<uint16_t, 9>::GXMAX);
}

template <typename T>
inline int stream_smem(int hb, int B, int q, int pf) {
    switch (hb) {
    case 1: return make_plan<T, 1>(B, q, pf).total;
    case 3: return make_plan<T, 3>(B, q, pf).total;
    case 5: return make_plan<T, 5>(B, q, pf).total;
    case 7: return make_plan<T, 7>(B, q, pf).total;
    case 8: return make_plan<T, 8>(B, q, pf).total;
    default: return make_plan<T, 9>(B, q, pf).total;
    }
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

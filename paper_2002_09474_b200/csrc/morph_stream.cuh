// morph_stream.cuh -- K1/K2 v2: warp-specialised, TMA-fed, strip-streaming fused separable
// erosion / dilation (u8, u16). Design notes in morph_stream.cu.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace rmgpu {
namespace stream {

constexpr int NVW = 4;                 // vertical warps
constexpr int NHW = 4;                 // horizontal warps
constexpr int NTH = 32 * (NVW + NHW);  // threads per CTA
constexpr int PF = 2;                  // input blocks prefetched ahead of the leading block
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
};

// Shared-memory plan, identical on host and device.
struct Plan {
    int B;        // rows per iteration (block size)
    int NSB;      // ring slots (blocks)
    int RP;       // ring row pitch (bytes)
    int VTWE;     // transposed-tile row length (entries)
    int NGC;      // row groups per chunk
    int off_ring, off_vt, off_hs, off_out, total;
    int HSE;      // per-warp horizontal scratch entries
};

template <typename T>
__host__ __device__ inline Plan make_plan(int B, int q, int gx, bool hblock) {
    using G = SG<T>;
    Plan p;
    p.B = B;
    p.NSB = q + 2 + PF;
    const int sz = (int)sizeof(T);
    p.RP = ((G::TW * sz + 2 * gx * sz + 31) / 16) * 16;
    const int cols = p.RP / sz;
    p.VTWE = ((cols + HC + 16 + G::SWB - 1) / G::SWB) * G::SWB;  // slack: last lane chunk may overrun
    p.NGC = B / G::GR;
    p.HSE = hblock ? ((G::TW + 2 * gx + HC + G::SWB - 1) / G::SWB) * G::SWB : 0;
    int o = 64 * 8;  // mbarriers
    p.off_ring = o;
    o += p.NSB * B * p.RP;
    p.off_vt = o;
    o += 2 * p.NGC * p.VTWE * G::ESZ;
    p.off_hs = o;
    o += hblock ? NHW * (p.HSE + 64) * G::ESZ : 0;
    p.off_out = o;
    o += B * (G::TW * sz + 16);
    p.total = o;
    return p;
}

template <typename T>
__device__ __forceinline__ int swz(int e) {
    constexpr int S = SG<T>::SWB;
    return (e & ~(S - 1)) | ((e & (S - 1)) ^ ((e / S) & (S - 1)));
}

// Column fix-up for a word at image column c: returns ring byte offset to load (relative to
// the strip's first byte xs_b) and a PRMT selector over (raw, bword).
template <typename T>
__device__ __forceinline__ void col_fix(int c, int W, int cmode, int xs_col, int& load_off, uint32_t& sel, bool& fix) {
    constexpr int PX = SG<T>::PX;
    constexpr int sz = sizeof(T);
    if (c >= 0 && c + PX - 1 < W) {
        load_off = (c - xs_col) * sz;
        sel = 0x3210;
        fix = false;
        return;
    }
    fix = true;
    const int cc0 = min(max(c, 0), W - 1);
    const int cl = (cc0 / PX) * PX;
    load_off = (cl - xs_col) * sz;
    sel = 0;
#pragma unroll
    for (int j = 0; j < PX; ++j) {
        const int col = c + j;
#pragma unroll
        for (int b = 0; b < sz; ++b) {
            int nib;
            if (cmode && (col < 0 || col >= W)) nib = 4 + b;
            else nib = (min(max(col, 0), W - 1) - cl) * sz + b;
            sel |= (uint32_t)nib << (4 * (j * sz + b));
        }
    }
}

// ---- the kernel ------------------------------------------------------------------------------
// VB: vertical variant: 1/3/5/7 = direct window (VCH rows per iteration), 8/16/24 = block size.
// HB: horizontal variant: 1/3/5/7 = direct window, 8 = lane-chunk block algorithm (HC = 8).
template <typename T, int MODE, int VB, int HB>
__global__ void __launch_bounds__(NTH)
morph_stream_kernel(StreamParams p) {
    using G = SG<T>;
    constexpr int PX = G::PX, GR = G::GR, TW = G::TW, ESZ = G::ESZ;
    constexpr int sz = sizeof(T);
    constexpr bool VDIRECT = VB <= 7;
    constexpr int B = VDIRECT ? VCH : VB;
    constexpr int OUTP = TW * sz + 16;
    extern __shared__ __align__(128) unsigned char smem[];

    const int gx = p.gx, gy = p.gy;
    const int w1 = 2 * gy, w1x = 2 * gx;
    const int q = VDIRECT ? 0 : w1 / B;
    const int r = VDIRECT ? w1 : w1 - q * B;
    const int s = r & 3;
    const Plan pl = make_plan<T>(B, q, gx, HB > 7);

    const uint8_t* src = p.src + blockIdx.z * p.simg;
    uint8_t* dst = p.dst + blockIdx.z * p.dimg;
    const int x0 = blockIdx.x * TW;
    const int y0 = blockIdx.y * p.rh;
    const int rh = min(p.rh, p.H - y0);
    // strip bytes [xs_b, xe_b) of every input row, 16-byte aligned
    const int xb = (x0 - gx) * sz;
    const int xs_b = xb >= 0 ? (xb / 16) * 16 : -(((-xb) + 15) / 16) * 16;
    const int xs_col = xs_b / sz;
    const int xe_b = ((x0 + TW + gx) * sz + 15) / 16 * 16;
    const int w_b16 = (p.W * sz + 15) / 16 * 16;
    const int cb0 = max(xs_b, 0);
    const int cb1 = min(xe_b, w_b16);
    const int copy_len = cb1 - cb0;  // bytes copied per row (multiple of 16, > 0)
    const int nwv = (xe_b - xs_b) / 4;
    const int y_first = y0 - gy;     // image row of input index 0
    const int Lend = (rh - 1 + w1 - s) / B;
    int Lf = 0;
    while (s + Lf * B - w1 + B - 1 < 0) ++Lf;

    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    unsigned char* ring = smem + pl.off_ring;
    unsigned char* vt = smem + pl.off_vt;
    unsigned char* hs = smem + pl.off_hs;
    unsigned char* outt = smem + pl.off_out;

    uint32_t bword = p.bval & 0xFF;
    if constexpr (sz == 1) bword *= 0x01010101u;
    else bword = (p.bval & 0xFFFF) * 0x00010001u;

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int k = 0; k < pl.NSB; ++k) mbar_init(&full[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int warp = tid >> 5, lane = tid & 31;

    if (warp < NVW) {
        // ================= vertical role: producer (warp 0) + streaming column sweeps =========
        const int t = tid;  // column word
        const bool active = t < nwv;
        int load_off = 0;
        uint32_t sel = 0x3210;
        bool fix = false;
        if (active) col_fix<T>(xs_col + PX * t, p.W, p.cmode, xs_col, load_off, sel, fix);

        // issue block k (rows [s + kB, s + kB + B) of the input index space) into its slot
        auto issue = [&](int k) {
            const int slot = (k + 1) % pl.NSB;
            unsigned char* base = ring + (size_t)slot * B * pl.RP;
            uint32_t bytes = 0;
            if (lane == 0) {
                for (int m = 0; m < B; ++m) {
                    const int y = y_first + s + k * B + m;
                    if (!(p.cmode && (y < p.row_lo || y >= p.row_hi))) bytes += copy_len;
                }
            }
            // constant rows outside the image: the warp fills them with the border value
            for (int m = 0; m < B; ++m) {
                const int y = y_first + s + k * B + m;
                if (p.cmode && (y < p.row_lo || y >= p.row_hi)) {
                    uint4* row = reinterpret_cast<uint4*>(base + (size_t)m * pl.RP);
                    for (int c = lane; c < pl.RP / 16; c += 32) row[c] = make_uint4(bword, bword, bword, bword);
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_tx(&full[slot], bytes);
                for (int m = 0; m < B; ++m) {
                    const int y = y_first + s + k * B + m;
                    if (p.cmode && (y < p.row_lo || y >= p.row_hi)) continue;
                    const int yc = min(max(y, p.row_lo), p.row_hi - 1);
                    bulk_g2s(base + (size_t)m * pl.RP + (cb0 - xs_b), src + (ptrdiff_t)yc * (ptrdiff_t)p.sp + cb0,
                             (uint32_t)copy_len, &full[slot]);
                }
            }
        };
        if (warp == 0) {
            for (int k = -1; k < PF && k <= Lend; ++k) issue(k);
        }

        auto slot_base = [&](int k) -> const unsigned char* {
            return ring + (size_t)((k + 1) % pl.NSB) * B * pl.RP + load_off;
        };
        auto ldw = [&](const unsigned char* a) -> LW<T> {
            uint32_t raw = *reinterpret_cast<const uint32_t*>(a);
            if (fix) raw = prmt(raw, bword, sel);
            return unpack_w(raw, (T*)nullptr);
        };

        LW<T> M[QMAX];
#pragma unroll
        for (int k = 0; k < QMAX; ++k) M[k] = lid<T, MODE>();
        int chunk = 0;
        for (int L = 0; L <= Lend; ++L) {
            bar_sync(BAR_VW, NVW * 32);  // iteration L-1 done by every vertical thread
            if (warp == 0 && L + PF <= Lend) issue(L + PF);
            const int slot = (L + 1) % pl.NSB;
            mbar_wait(&full[slot], ((L + 1) / pl.NSB) & 1);
            const bool emit = L >= Lf;
            const int buf = chunk & 1;
            if (emit) bar_sync(BAR_EMPTY0 + buf, NTH);
            if (active) {
                const unsigned char* lead = slot_base(L);
                const int oL = s + L * B - w1;
                LW<T> out[B];
                if constexpr (VDIRECT) {
                    constexpr int WD = VB;
                    LW<T> X[B + WD - 1];
                    const unsigned char* prev = slot_base(L - 1);
#pragma unroll
                    for (int k = 0; k < WD - 1; ++k) X[k] = ldw(prev + (size_t)(B - (WD - 1) + k) * pl.RP);
#pragma unroll
                    for (int m = 0; m < B; ++m) X[WD - 1 + m] = ldw(lead + (size_t)m * pl.RP);
                    if (emit) {
#pragma unroll
                        for (int m = 0; m < B; ++m) {
                            if constexpr (WD == 1) out[m] = X[m];
                            else if constexpr (WD == 3) out[m] = lop3<MODE>(X[m], X[m + 1], X[m + 2]);
                            else if constexpr (WD == 5) out[m] = lop3<MODE>(lop3<MODE>(X[m], X[m + 1], X[m + 2]), X[m + 3], X[m + 4]);
                            else out[m] = lop3<MODE>(lop3<MODE>(X[m], X[m + 1], X[m + 2]), lop3<MODE>(X[m + 3], X[m + 4], X[m + 5]), X[m + 6]);
                        }
                    }
                } else {
                    LW<T> P[B];
                    P[0] = ldw(lead);
#pragma unroll
                    for (int m = 1; m < B; ++m) P[m] = lop<MODE>(P[m - 1], ldw(lead + (size_t)m * pl.RP));
                    if (emit) {
                        // gap = tail r rows of block L-q + whole blocks L-q+1 .. L-1
                        LW<T> gap = lid<T, MODE>();
                        const unsigned char* tb = slot_base(L - q);
                        for (int i = 0; i < r; ++i) gap = lop<MODE>(gap, ldw(tb + (size_t)(B - r + i) * pl.RP));
#pragma unroll
                        for (int k = 0; k < QMAX - 1; ++k)
                            if (k < q - 1) gap = lop<MODE>(gap, M[k]);
                        // trailing run rows oL + m: block L-q-1 row B-r+m (m < r), block L-q row m-r
                        const unsigned char* ta = slot_base(L - q - 1) + (size_t)(B - r) * pl.RP;
                        const unsigned char* tbb = tb - (size_t)r * pl.RP;
                        LW<T> acc = gap;
#pragma unroll
                        for (int m = B - 1; m >= 0; --m) {
                            const unsigned char* a = (m < r ? ta : tbb) + (size_t)m * pl.RP;
                            acc = lop<MODE>(acc, ldw(a));
                            out[m] = lop<MODE>(acc, P[m]);
                        }
                    }
#pragma unroll
                    for (int k = QMAX - 1; k > 0; --k) M[k] = M[k - 1];
                    M[0] = P[B - 1];
                }
                if (emit) {
                    // transpose GR x PX blocks and store into VT[buf] (rows oL.. of this chunk)
                    unsigned char* vb = vt + (size_t)buf * pl.NGC * pl.VTWE * ESZ;
#pragma unroll
                    for (int g = 0; g < B / GR; ++g) {
                        unsigned char* rowg = vb + (size_t)g * pl.VTWE * ESZ;
                        const int e0 = PX * t;
                        if constexpr (sz == 1) {
                            const LW<uint8_t> r0 = out[4 * g], r1 = out[4 * g + 1], r2 = out[4 * g + 2], r3 = out[4 * g + 3];
                            *reinterpret_cast<uint2*>(rowg + swz<T>(e0 + 0) * ESZ) =
                                make_uint2(prmt(r0.a, r2.a, 0x5410), prmt(r1.a, r3.a, 0x5410));
                            *reinterpret_cast<uint2*>(rowg + swz<T>(e0 + 1) * ESZ) =
                                make_uint2(prmt(r0.b, r2.b, 0x5410), prmt(r1.b, r3.b, 0x5410));
                            *reinterpret_cast<uint2*>(rowg + swz<T>(e0 + 2) * ESZ) =
                                make_uint2(prmt(r0.a, r2.a, 0x7632), prmt(r1.a, r3.a, 0x7632));
                            *reinterpret_cast<uint2*>(rowg + swz<T>(e0 + 3) * ESZ) =
                                make_uint2(prmt(r0.b, r2.b, 0x7632), prmt(r1.b, r3.b, 0x7632));
                        } else {
                            const LW<uint16_t> r0 = out[2 * g], r1 = out[2 * g + 1];
                            *reinterpret_cast<uint32_t*>(rowg + swz<T>(e0 + 0) * ESZ) = prmt(r0.a, r1.a, 0x5410);
                            *reinterpret_cast<uint32_t*>(rowg + swz<T>(e0 + 1) * ESZ) = prmt(r0.a, r1.a, 0x7632);
                        }
                    }
                }
            }
            if (emit) {
                bar_arrive(BAR_FULL0 + buf, NTH);
                ++chunk;
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
        unsigned char* scr = hs + (size_t)hw * (pl.HSE + 64) * ESZ;  // P scratch, then M scratch
        unsigned char* msc = scr + (size_t)pl.HSE * ESZ;
        const int off = (x0 - gx) - xs_col;
        int chunk = 0;
        for (int L = Lf; L <= Lend; ++L, ++chunk) {
            const int buf = chunk & 1;
            bar_sync(BAR_FULL0 + buf, NTH);
            const int oL = s + L * B - w1;
            const unsigned char* vb = vt + (size_t)buf * pl.NGC * pl.VTWE * ESZ;
            for (int g = hw; g < pl.NGC; g += NHW) {
                const int o_g = oL + g * GR;
                if (o_g + GR - 1 < 0 || o_g >= rh) continue;
                const unsigned char* rowg = vb + (size_t)g * pl.VTWE * ESZ;
                auto ldv = [&](int xv) -> LW<T> {
                    LW<T> v;
                    if constexpr (sz == 1) {
                        const uint2 u = *reinterpret_cast<const uint2*>(rowg + swz<T>(xv) * ESZ);
                        v.a = u.x;
                        v.b = u.y;
                    } else {
                        v.a = *reinterpret_cast<const uint32_t*>(rowg + swz<T>(xv) * ESZ);
                    }
                    return v;
                };
                // emit GR output columns (a..a+GR-1) of rows g*GR.. into the output tile
                // emit GR output columns (a..a+GR-1) of rows g*GR.. into the output tile
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
                if constexpr (HB <= 7) {
                    // direct window: each lane owns TW/32 consecutive output columns
                    constexpr int WD = HB;
                    constexpr int NO = TW / 32;
                    LW<T> X[NO + WD - 1];
                    const int a0 = lane * NO;
#pragma unroll
                    for (int i = 0; i < NO + WD - 1; ++i) X[i] = ldv(off + a0 + i);
                    LW<T> o[NO];
#pragma unroll
                    for (int j = 0; j < NO; ++j) {
                        if constexpr (WD == 1) o[j] = X[j];
                        else if constexpr (WD == 3) o[j] = lop3<MODE>(X[j], X[j + 1], X[j + 2]);
                        else if constexpr (WD == 5) o[j] = lop3<MODE>(lop3<MODE>(X[j], X[j + 1], X[j + 2]), X[j + 3], X[j + 4]);
                        else o[j] = lop3<MODE>(lop3<MODE>(X[j], X[j + 1], X[j + 2]), lop3<MODE>(X[j + 3], X[j + 4], X[j + 5]), X[j + 6]);
                    }
#pragma unroll
                    for (int j = 0; j < NO; j += GR) {
                        if constexpr (GR == 4) emit4(a0 + j, o[j], o[j + 1], o[j + 2], o[j + 3]);
                        else emit4(a0 + j, o[j], o[j + 1], o[j], o[j]);
                    }
                } else {
                    // lane-chunk van Herk: chunk k = inputs [kC, kC+C); prefix -> scratch, suffix kept
                    constexpr int C = HC;
                    const int nch = (TW + w1x + C - 1) / C;
                    LW<T> S[C];
                    for (int k = lane; k < nch; k += 32) {
                        LW<T> x[C];
#pragma unroll
                        for (int j = 0; j < C; ++j) x[j] = ldv(off + k * C + j);
                        LW<T> pre = x[0];
#pragma unroll
                        for (int j = 0; j < C; ++j) {
                            if (j) pre = lop<MODE>(pre, x[j]);
                            if constexpr (sz == 1)
                                *reinterpret_cast<uint2*>(scr + swz<T>(k * C + j) * ESZ) = make_uint2(pre.a, pre.b);
                            else
                                *reinterpret_cast<uint32_t*>(scr + swz<T>(k * C + j) * ESZ) = pre.a;
                        }
                        if constexpr (sz == 1)
                            *reinterpret_cast<uint2*>(msc + k * ESZ) = make_uint2(pre.a, pre.b);
                        else
                            *reinterpret_cast<uint32_t*>(msc + k * ESZ) = pre.a;
                        if (k == lane) {
                            S[C - 1] = x[C - 1];
#pragma unroll
                            for (int j = C - 2; j >= 0; --j) S[j] = lop<MODE>(S[j + 1], x[j]);
                        }
                    }
                    __syncwarp();
                    const int k = lane;
                    if (k * C < TW) {
                        const int qc = w1x / C, rc = w1x - qc * C;
                        auto ldm = [&](int kk) -> LW<T> {
                            LW<T> v;
                            if constexpr (sz == 1) {
                                const uint2 u = *reinterpret_cast<const uint2*>(msc + kk * ESZ);
                                v.a = u.x;
                                v.b = u.y;
                            } else {
                                v.a = *reinterpret_cast<const uint32_t*>(msc + kk * ESZ);
                            }
                            return v;
                        };
                        auto ldp = [&](int e) -> LW<T> {
                            LW<T> v;
                            if constexpr (sz == 1) {
                                const uint2 u = *reinterpret_cast<const uint2*>(scr + swz<T>(e) * ESZ);
                                v.a = u.x;
                                v.b = u.y;
                            } else {
                                v.a = *reinterpret_cast<const uint32_t*>(scr + swz<T>(e) * ESZ);
                            }
                            return v;
                        };
                        LW<T> Fa = lid<T, MODE>();
                        for (int i = 1; i < qc; ++i) Fa = lop<MODE>(Fa, ldm(k + i));
                        const LW<T> Fb = lop<MODE>(Fa, ldm(k + qc));
                        LW<T> o[C];
#pragma unroll
                        for (int j = 0; j < C; ++j) {
                            const int a = k * C + j;
                            o[j] = lop3<MODE>(S[j], j < C - rc ? Fa : Fb, ldp(a + w1x));
                        }
#pragma unroll
                        for (int j = 0; j < C; j += GR) {
                            if constexpr (GR == 4) emit4(k * C + j, o[j], o[j + 1], o[j + 2], o[j + 3]);
                            else emit4(k * C + j, o[j], o[j + 1], o[j], o[j]);
                        }
                    }
                    __syncwarp();
                }
            }
            bar_arrive(BAR_EMPTY0 + buf, NTH);
            bar_sync(BAR_HW, NHW * 32);
            // store the valid rows of the chunk
            {
                const int htid = tid - NVW * 32;
                const int cols = min(TW, p.W - x0);
                const int row_bytes = cols * sz;
                const bool vec = (((uintptr_t)dst | p.dp) & 15) == 0 && cols == TW;
                const int rlo = max(0, -oL), rhi = min(B, rh - oL);
                if (vec) {
                    constexpr int CPR = TW * sz / 16;
                    for (int i = rlo * CPR + htid; i < rhi * CPR; i += NHW * 32) {
                        const int rr = i / CPR, ch = i % CPR;
                        const uint4 v = *reinterpret_cast<const uint4*>(outt + (size_t)rr * OUTP + ch * 16);
                        *reinterpret_cast<uint4*>(dst + (size_t)(y0 + oL + rr) * p.dp + (size_t)x0 * sz + ch * 16) = v;
                    }
                } else {
                    for (int i = rlo * row_bytes + htid; i < rhi * row_bytes; i += NHW * 32) {
                        const int rr = i / row_bytes, b = i % row_bytes;
                        dst[(size_t)(y0 + oL + rr) * p.dp + (size_t)x0 * sz + b] = outt[(size_t)rr * OUTP + b];
                    }
                }
            }
            bar_sync(BAR_HW, NHW * 32);
        }
    }
}

// ---- host launch ------------------------------------------------------------------------------
template <typename T, int MODE, int VB, int HB>
cudaError_t launch_stream_variant(const MorphJob& j, int rh, int B, int q) {
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
    const Plan pl = make_plan<T>(B, q, j.gx, HB > 7);
    auto kern = morph_stream_kernel<T, MODE, VB, HB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.total);
    if (e != cudaSuccess) return e;
    dim3 grid(cdiv(j.W, G::TW), cdiv(j.H, rh), j.batch);
    kern<<<grid, NTH, pl.total, j.stream>>>(p);
    count_launch();
    return cudaGetLastError();
}

#define RM_STREAM_V(X) X(1) X(3) X(5) X(7) X(8) X(16) X(24)
#define RM_STREAM_H(X) X(1) X(3) X(5) X(7) X(8)

template <typename T, int MODE, int VB>
cudaError_t stream_dispatch_h(const MorphJob& j, int hb, int rh, int B, int q) {
    switch (hb) {
#define RM_CASE(H) \
    case H: return launch_stream_variant<T, MODE, VB, H>(j, rh, B, q);
        RM_STREAM_H(RM_CASE)
#undef RM_CASE
    }
    return cudaErrorInvalidValue;
}

template <typename T, int MODE>
cudaError_t stream_dispatch(const MorphJob& j, int vb, int hb, int rh, int B, int q) {
    switch (vb) {
#define RM_CASE(V) \
    case V: return stream_dispatch_h<T, MODE, V>(j, hb, rh, B, q);
        RM_STREAM_V(RM_CASE)
#undef RM_CASE
    }
    return cudaErrorInvalidValue;
}

}  // namespace stream
}  // namespace rmgpu

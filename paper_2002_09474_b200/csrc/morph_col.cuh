// morph_col.cuh -- K1 v4: register-streaming fused separable erosion / dilation for small
// windows (both wings <= 3, i.e. w <= 7), u8 and u16. Design notes in morph_col.cu.
#pragma once

#include <algorithm>
#include <type_traits>

#include "morph_stream.cuh"  // PTX helpers (mbarrier, TMA), tensor-map encoders, red*_u16x2

namespace rmgpu {
namespace col {

using stream::bulk_g2s;
using stream::fence_async_smem;
using stream::mbar_arrive_tx;
using stream::mbar_init;
using stream::mbar_wait;
using stream::tma_box;

#ifndef RM_COL_BR
#define RM_COL_BR 8
#endif
#ifndef RM_COL_NS
#define RM_COL_NS 3
#endif
#ifndef RM_COL_WPB
#define RM_COL_WPB 4
#endif
constexpr int WPB = RM_COL_WPB;      // warps per CTA (independent pipelines sharing one smem block)
constexpr int BR = RM_COL_BR;        // rows per TMA block
constexpr int NS = RM_COL_NS;        // ring slots per warp
constexpr int SB = 512;              // strip bytes per row (32 lanes x 16 B)
constexpr int HDR = 128;             // mbarriers
// Slot layout: the 8 staged rows' 512 strip bytes (dense, one 512-byte-aligned TMA box) and, when
// the horizontal window needs neighbours, the 16 bytes left / right of the strip for each row in
// two small regions (two 16-byte-wide TMA boxes), so the big box stays aligned to whole 128-byte
// lines. Slot = 4096 (+ 2 x 128) bytes, a multiple of 128.
template <int GX>
struct ColGeo {
    static constexpr int HALO = GX == 0 ? 0 : 16;
    static constexpr int MAINB = BR * SB;
    static constexpr int LEFT = MAINB, RIGHT = MAINB + BR * 16;
    static constexpr int SLOTB = MAINB + (HALO ? 2 * BR * 16 : 0);
    static constexpr int WARPB = NS * SLOTB;
    static constexpr int SMEM = HDR + WPB * WARPB;
};
constexpr int GMAX = 3;  // largest wing handled here (windows up to 7 x 7)

struct ColParams {
    const uint8_t* src;  // output row 0 of image 0
    size_t sp;
    uint8_t* dst;
    size_t dp;
    int W, H;
    int row_lo, row_hi;  // valid input rows relative to output row 0
    int cmode;
    uint32_t bval;
    size_t simg, dimg;
    int batch;
    int R;               // output rows per item
    int nstrips, nbands;
    int use_tma;
    // item walk (host-computed): a warp visits items gw, gw + nwarps, ...; divisions by the strip
    // count and the items per image use multiply-high magic numbers
    int ds, dband, db;
    uint32_t strip_m, img_m;
    int strip_s, img_s;
};

// q = n / d for 0 <= n < 2^31 with host-computed (m, s): q = (umulhi(n, m) + n) >> s
struct FastDivHost {
    uint32_t m;
    int s;
    static FastDivHost make(uint32_t d) {
        FastDivHost f;
        int s = 0;
        while ((1ull << s) < d) ++s;
        f.s = s;
        f.m = (uint32_t)((((1ull << s) - d) << 32) / d + 1);
        return f;
    }
};
__device__ __forceinline__ int fdiv(int n, uint32_t m, int s) {
    return (int)((__umulhi((uint32_t)n, m) + (uint64_t)(uint32_t)n) >> s);
}

// Work item cursor: item n -> (image, band, strip), strips fastest so neighbouring warps share
// halo rows in L2. A warp walks items gw, gw + nwarps, ... with mixed-radix increments (the
// divisions happen once per warp).
struct Cursor {
    int b, band, strip;
    __device__ __forceinline__ void init(const ColParams& p, int n) {
        b = fdiv(n, p.img_m, p.img_s);
        const int rem = n - b * p.nstrips * p.nbands;
        band = fdiv(rem, p.strip_m, p.strip_s);
        strip = rem - band * p.nstrips;
    }
    __device__ __forceinline__ void step(const ColParams& p) {
        strip += p.ds;
        int carry = 0;
        if (strip >= p.nstrips) {
            strip -= p.nstrips;
            carry = 1;
        }
        band += p.dband + carry;
        carry = 0;
        if (band >= p.nbands) {
            band -= p.nbands;
            carry = 1;
        }
        b += p.db + carry;
    }
    __device__ __forceinline__ bool valid(const ColParams& p) const { return b < p.batch; }
};

struct CItem {
    int b, y0, x0, rows_out, nblk;
};
template <typename T, int GY>
__device__ __forceinline__ CItem col_item(const ColParams& p, const Cursor& c) {
    CItem it;
    it.b = c.b;
    it.y0 = c.band * p.R;
    it.x0 = c.strip * (SB / (int)sizeof(T));
    it.rows_out = min(p.R, p.H - it.y0);
    it.nblk = (it.rows_out + 2 * GY + BR - 1) / BR;
    return it;
}

template <int MODE>
__device__ __forceinline__ uint32_t op2(uint32_t a, uint32_t b) {
    return red2_u16x2<MODE>(a, b);
}
template <int MODE>
__device__ __forceinline__ uint32_t op3(uint32_t a, uint32_t b, uint32_t c) {
    return red3_u16x2<MODE>(a, b, c);
}
// reduction over N consecutive words of a list (N odd, <= 7)
template <int MODE, int N>
__device__ __forceinline__ uint32_t opn(const uint32_t* v) {
    if constexpr (N == 1) return v[0];
    else if constexpr (N == 3) return op3<MODE>(v[0], v[1], v[2]);
    else if constexpr (N == 5) return op3<MODE>(op3<MODE>(v[0], v[1], v[2]), v[3], v[4]);
    else return op3<MODE>(op3<MODE>(op3<MODE>(v[0], v[1], v[2]), v[3], v[4]), v[5], v[6]);
}

// Two windows of N (5 or 7) consecutive words whose starts are D (1 or 2) apart, a = v[0..N) and
// b = v[D..N+D): the words both contain are reduced once and each window adds its own with one
// three-input instruction -- N == 7: 4 instructions for both instead of 6, N == 5: 3 instead of 4.
template <int MODE, int N, int D>
__device__ __forceinline__ void opn_pair(const uint32_t* v, uint32_t& a, uint32_t& b) {
    static_assert((N == 5 || N == 7) && (D == 1 || D == 2), "paired windows");
    uint32_t c = op3<MODE>(v[2], v[3], v[4]);
    if constexpr (N == 7) c = op3<MODE>(c, v[5], v[6]);
    a = op3<MODE>(c, v[0], v[1]);
    if constexpr (D == 1) b = op3<MODE>(c, v[1], v[N]);
    else b = op3<MODE>(c, v[N], v[N + 1]);
}

// ---------------------------------------------------------------------------------------------
// Per-row word sets. u8: a lane owns 16 pixels = 4 raw words; min/max run on 16-bit lanes of
// the raw word (odd pixels, in the high bytes: the high byte of a 16-bit min/max is the min/max
// of the high bytes) and of its byte-swapped copy (even pixels) -- one PRMT per 4 pixels, no
// unpacking. u16: a lane owns 8 pixels = 4 u16x2 words. Both carry 2 extra words: the column
// word(s) just left of the strip (lane 0) / right of it (lane 31).
// ---------------------------------------------------------------------------------------------
// x << 8 as a multiply: IMAD on the FMA pipe instead of a permute / shift on the ALU pipe
__device__ __forceinline__ uint32_t shl8_fma(uint32_t x) {
    uint32_t y;
    asm("mul.lo.u32 %0, %1, 256;" : "=r"(y) : "r"(x));
    return y;
}

template <typename T>
struct RowW;
template <>
struct RowW<uint8_t> {
    static constexpr int N = 10;  // S0..S3 (even pixels), R0..R3 (odd pixels), XS, XR
};
template <>
struct RowW<uint16_t> {
    static constexpr int N = 6;   // w0..w3, X0, X1
};

template <typename T, int MODE, int GX, int GY>
struct ColCore {
    static constexpr int NW = RowW<T>::N;
    static constexpr int WV = 2 * GY + 1;
    static constexpr int sz = sizeof(T);
    static constexpr int PXL = 16 / sz;  // pixels per lane

    // load one staged row into expanded words
    using CG = ColGeo<GX>;
    static __device__ __forceinline__ void load_row(const unsigned char* slot, int r, int lane, uint32_t* e) {
        const uint4 m = *reinterpret_cast<const uint4*>(slot + r * SB + lane * 16);
        const uint32_t w[4] = {m.x, m.y, m.z, m.w};
        uint2 xx = make_uint2(0, 0);  // halo words (lane 0: left of the strip, lane 31: right)
        if constexpr (GX > 0)
            xx = *reinterpret_cast<const uint2*>(slot + (lane == 0 ? CG::LEFT + 8 : CG::RIGHT) + r * 16);
        if constexpr (sz == 1) {
            const uint32_t x = lane == 0 ? xx.y : xx.x;  // left: bytes x0-4..x0-1; right: x0+512..
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                e[k] = shl8_fma(w[k]);            // even pixels into the high bytes: x * 256 on the FMA
                                                  // pipe (the min / max and permutes saturate the ALU pipe)
                e[4 + k] = w[k];                  // odd pixels already there
            }
            e[8] = shl8_fma(x);
            e[9] = x;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) e[k] = w[k];
            e[4] = xx.x;
            e[5] = xx.y;
        }
    }

    // horizontal window over one vertically reduced row; returns the 4 packed output words
    static __device__ __forceinline__ uint4 horizontal(const uint32_t* v, int lane) {
        uint32_t o[4];
        if constexpr (sz == 1) {
            // S(k) / R(k) for k = -1..4 (k = -1 / 4 from the neighbouring lanes or the extra word)
            uint32_t S[6], Rr[6];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                S[k + 1] = v[k];
                Rr[k + 1] = v[4 + k];
            }
            S[0] = S[5] = Rr[0] = Rr[5] = 0;
            if constexpr (GX >= 1) {  // R(-1), S(4)
                const uint32_t rl = __shfl_up_sync(0xffffffffu, v[7], 1);
                const uint32_t sr = __shfl_down_sync(0xffffffffu, v[0], 1);
                Rr[0] = lane == 0 ? v[9] : rl;
                S[5] = lane == 31 ? v[8] : sr;
            }
            if constexpr (GX >= 2) {  // S(-1), R(4)
                const uint32_t sl = __shfl_up_sync(0xffffffffu, v[3], 1);
                const uint32_t rr = __shfl_down_sync(0xffffffffu, v[4], 1);
                S[0] = lane == 0 ? v[8] : sl;
                Rr[5] = lane == 31 ? v[9] : rr;
            }
            // U(i) = {p_i, p_{i+2}} for i = -GX .. 13+GX; U(4k)=S(k), U(4k+1)=R(k),
            // U(4k+2)=PRMT(S(k),S(k+1)), U(4k+3)=PRMT(R(k),R(k+1))
            constexpr int UB = GX;  // U index offset
            uint32_t U[14 + 2 * GX];
#pragma unroll
            for (int i = -GX; i < 14 + GX; ++i) {
                const int k = (i + 4) / 4 - 1, m = (i + 4) % 4;
                uint32_t u;
                if (m == 0) u = S[k + 1];
                else if (m == 1) u = Rr[k + 1];
                else if (m == 2) u = prmt(S[k + 1], S[k + 2], 0x5432);
                else u = prmt(Rr[k + 1], Rr[k + 2], 0x5432);
                U[i + UB] = u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t oe, oo;  // windows of the even / odd pixel pairs: one U index apart
                if constexpr (GX >= 2) {
                    opn_pair<MODE, 2 * GX + 1, 1>(&U[4 * k - GX + UB], oe, oo);
                } else {
                    oe = opn<MODE, 2 * GX + 1>(&U[4 * k - GX + UB]);
                    oo = opn<MODE, 2 * GX + 1>(&U[4 * k + 1 - GX + UB]);
                }
                o[k] = prmt(oe, oo, 0x7351);
            }
        } else {
            // Wf(k) for k = -2..5
            uint32_t Wf[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) Wf[k + 2] = v[k];
            if constexpr (GX >= 1) {
                const uint32_t l1 = __shfl_up_sync(0xffffffffu, v[3], 1);
                const uint32_t r0 = __shfl_down_sync(0xffffffffu, v[0], 1);
                Wf[1] = lane == 0 ? v[5] : l1;
                Wf[6] = lane == 31 ? v[4] : r0;
                if constexpr (GX >= 3) {
                    const uint32_t l2 = __shfl_up_sync(0xffffffffu, v[2], 1);
                    const uint32_t r1 = __shfl_down_sync(0xffffffffu, v[1], 1);
                    Wf[0] = lane == 0 ? v[4] : l2;
                    Wf[7] = lane == 31 ? v[5] : r1;
                } else {
                    Wf[0] = Wf[7] = 0;
                }
            } else {
                Wf[0] = Wf[1] = Wf[6] = Wf[7] = 0;
            }
            // U(i) = {p_i, p_{i+1}} for i = -GX .. 6+GX
            constexpr int UB = GX;
            uint32_t U[7 + 2 * GX];
#pragma unroll
            for (int i = -GX; i < 7 + GX; ++i) {
                const int k = (i + 4) / 2 - 2, m = (i + 4) % 2;
                U[i + UB] = m == 0 ? Wf[k + 2] : prmt(Wf[k + 2], Wf[k + 3], 0x5432);
            }
            if constexpr (GX >= 2) {  // neighbouring output words: windows two U indices apart
#pragma unroll
                for (int k = 0; k < 4; k += 2) opn_pair<MODE, 2 * GX + 1, 2>(&U[2 * k - GX + UB], o[k], o[k + 1]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] = opn<MODE, 2 * GX + 1>(&U[2 * k - GX + UB]);
            }
        }
        return make_uint4(o[0], o[1], o[2], o[3]);
    }
};

// Ragged right edge: only the lane's first nbytes output bytes are inside the image.
static __device__ __noinline__ void store_partial(uint8_t* d, uint4 out, int nbytes) {
    if (nbytes <= 0) return;
    const uint32_t ow[4] = {out.x, out.y, out.z, out.w};
    for (int b = 0; b < nbytes; ++b) d[b] = (uint8_t)(ow[b >> 2] >> (8 * (b & 3)));
}

// Border strips: overwrite the staged out-of-image columns of one block in shared memory
// (replicate: the row's first / last pixel; constant: the border value), so the row loop itself
// has no border logic. Lane-parallel, border strips only.
template <typename T, int GX>
__device__ __forceinline__ unsigned char* staged_byte(unsigned char* slot, int r, int m) {
    using CG = ColGeo<GX>;
    return m < 0 ? slot + CG::LEFT + r * 16 + (m + 16)
                 : (m < SB ? slot + r * SB + m : slot + CG::RIGHT + r * 16 + (m - SB));
}
template <typename T, int GX>
__device__ __forceinline__ void fix_block_columns(unsigned char* slot, int lane, int x0, int W, int cmode, uint32_t bv) {
    constexpr int sz = sizeof(T);
    constexpr int HALO = ColGeo<GX>::HALO;
    if (HALO > 0 && x0 == 0) {  // 16 halo bytes left of column 0: 8 rows x 4 words = one word per lane
        const int r = lane >> 2, wI = lane & 3;
        uint32_t f = bv;
        if (cmode == 0)
            f = sz == 1 ? slot[r * SB] * 0x01010101u : *reinterpret_cast<const uint16_t*>(slot + r * SB) * 0x00010001u;
        __syncwarp();
        reinterpret_cast<uint32_t*>(slot + ColGeo<GX>::LEFT + r * 16)[wI] = f;
    }
    const int start = (W - x0) * sz;  // first staged byte (from the strip start) at column >= W
    if (start < SB + HALO) {
        for (int r = 0; r < BR; ++r) {
            uint32_t f = bv;
            if (cmode == 0)
                f = sz == 1 ? *staged_byte<T, GX>(slot, r, start - 1) * 0x01010101u
                            : *reinterpret_cast<const uint16_t*>(staged_byte<T, GX>(slot, r, start - 2)) * 0x00010001u;
            __syncwarp();
            for (int m = start + lane; m < SB + HALO; m += 32) *staged_byte<T, GX>(slot, r, m) = (uint8_t)(f >> (8 * (m & 3)));
        }
    }
    __syncwarp();
}

template <typename T, int MODE, int GX, int GY>
__global__ void __launch_bounds__(WPB * 32)
morph_col_kernel(const ColParams p, const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap hmap) {
    constexpr int sz = sizeof(T);
    constexpr int PXL = 16 / sz;
    constexpr int SWPX = SB / sz;
    constexpr int WV = 2 * GY + 1;
    constexpr int RING = WV == 1 ? 1 : (WV <= 4 ? 4 : 8);  // power of two dividing BR: compile-time slots
    constexpr int NW = RowW<T>::N;
    using C = ColCore<T, MODE, GX, GY>;
    using CG = ColGeo<GX>;
    constexpr int HALO = CG::HALO, SLOTB = CG::SLOTB, WARPB = CG::WARPB;
    extern __shared__ __align__(128) unsigned char smem[];

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + wib * NS;
    unsigned char* ring = smem + HDR + wib * WARPB;
    const int nwarps = gridDim.x * WPB;
    const int gw = blockIdx.x * WPB + wib;
    const int nitems = p.nstrips * p.nbands * p.batch;
    if (gw >= nitems) return;
    if (lane == 0) {
        for (int k = 0; k < NS; ++k) mbar_init(&bars[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    const uint32_t bv = sz == 1 ? (p.bval & 0xFF) * 0x01010101u : (p.bval & 0xFFFF) * 0x00010001u;

    // ---- producer side (warp-collective; lane 0 / lanes < BR issue) -----------------------------
    Cursor ic;
    ic.init(p, gw);
    const Cursor c0 = ic;
    CItem iit = col_item<T, GY>(p, ic);
    bool ivalid = true;
    int ib = 0, islot = 0;
    auto issue = [&]() {
        if (!ivalid) return;
        unsigned char* dstb = ring + islot * SLOTB;
        uint64_t* bar = &bars[islot];
        const int yb = iit.y0 - GY + ib * BR;
        const int xb = iit.x0 * sz;  // byte column of the strip start
        if (p.use_tma && yb >= p.row_lo && yb + BR <= p.row_hi) {
            if (lane == 0) {
                mbar_arrive_tx(bar, (uint32_t)SLOTB);
                tma_box(dstb, &tmap, xb / 4, yb - p.row_lo, iit.b, bar);
                if constexpr (HALO > 0) {
                    tma_box(dstb + CG::LEFT, &hmap, (xb - 16) / 4, yb - p.row_lo, iit.b, bar);
                    tma_box(dstb + CG::RIGHT, &hmap, (xb + SB) / 4, yb - p.row_lo, iit.b, bar);
                }
            }
        } else {
            // border block: bulk copies per row (clamped row / constant fill), clipped columns
            const int y = yb + lane;
            const bool inrow = lane < BR;
            const bool outside = p.cmode && (y < p.row_lo || y >= p.row_hi);
            const int len = min(SB, (int)p.sp - xb);
            const bool lft = HALO > 0 && xb >= 16, rgt = HALO > 0 && xb + SB + 16 <= (int)p.sp;
            const bool cp = inrow && !outside;
            const int bytes = __reduce_add_sync(0xffffffffu, cp ? len + (lft ? 16 : 0) + (rgt ? 16 : 0) : 0);
            unsigned fillm = __ballot_sync(0xffffffffu, inrow && outside);
            while (fillm) {
                const int r = __ffs(fillm) - 1;
                fillm &= fillm - 1;
                reinterpret_cast<uint4*>(dstb + r * SB)[lane] = make_uint4(bv, bv, bv, bv);
                if (HALO > 0 && lane < 2)
                    *reinterpret_cast<uint4*>(dstb + (lane ? CG::RIGHT : CG::LEFT) + r * 16) = make_uint4(bv, bv, bv, bv);
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_tx(bar, (uint32_t)bytes);
            __syncwarp();
            if (cp) {
                const int yc = min(max(y, p.row_lo), p.row_hi - 1);
                const uint8_t* srow = p.src + (size_t)iit.b * p.simg + (ptrdiff_t)yc * (ptrdiff_t)p.sp;
                bulk_g2s(dstb + lane * SB, srow + xb, (uint32_t)len, bar);
                if (lft) bulk_g2s(dstb + CG::LEFT + lane * 16, srow + xb - 16, 16u, bar);
                if (rgt) bulk_g2s(dstb + CG::RIGHT + lane * 16, srow + xb + SB, 16u, bar);
            }
        }
        islot = islot + 1 == NS ? 0 : islot + 1;
        if (++ib == iit.nblk) {
            ib = 0;
            ic.step(p);
            ivalid = ic.valid(p);
            if (ivalid) iit = col_item<T, GY>(p, ic);
        }
    };
    for (int k = 0; k < NS; ++k) issue();

    // ---- consumer --------------------------------------------------------------------------------
    int cslot = 0;
    uint32_t cpar = 0;
    uint32_t E[RING][NW];
    Cursor cc = c0;
    for (; cc.valid(p); cc.step(p)) {
        const CItem it = col_item<T, GY>(p, cc);
        const bool edge = it.x0 == 0 || it.x0 + SWPX + 4 > p.W;
        const int store_bytes = max(0, min(16, (p.W - it.x0 - lane * PXL) * sz));
        // destination of input row t: output row t - 2*GY
        const ptrdiff_t dp = (ptrdiff_t)p.dp;
        uint8_t* drow = p.dst + (size_t)it.b * p.dimg + (size_t)it.x0 * sz + (size_t)lane * 16 +
                        (ptrdiff_t)(it.y0 - 2 * GY) * (ptrdiff_t)p.dp;
        int o = -2 * GY;
        for (int blk = 0; blk < it.nblk; ++blk) {
            mbar_wait(&bars[cslot], cpar);
            const unsigned char* rows = ring + cslot * SLOTB;
            if (edge) fix_block_columns<T, GX>(ring + cslot * SLOTB, lane, it.x0, p.W, p.cmode, bv);
            // 8 rows; the row-validity test only in blocks with warm-up rows or rows past the band
            // vertically reduced words of row r -> horizontal window -> one 16-byte store
            auto emit = [&](uint8_t* d, const uint32_t* vmin, const uint32_t* vmax, const uint32_t* v) {
                uint4 out;
                if constexpr (MODE == MODE_GRAD) {
                    // morphological gradient from one read: dilation - erosion. Bytes (u8) /
                    // halves (u16) of max are >= those of min, so one 32-bit subtract per
                    // word never borrows across pixels.
                    const uint4 lo = ColCore<T, MODE_MIN, GX, GY>::horizontal(vmin, lane);
                    const uint4 hi = ColCore<T, MODE_MAX, GX, GY>::horizontal(vmax, lane);
                    out = make_uint4(hi.x - lo.x, hi.y - lo.y, hi.z - lo.z, hi.w - lo.w);
                } else {
                    out = C::horizontal(v, lane);
                }
                if (store_bytes == 16) *reinterpret_cast<uint4*>(d) = out;
                else store_partial(d, out, store_bytes);
            };
            auto block = [&](auto check_tag) {
                constexpr bool CHECK = decltype(check_tag)::value;
                if constexpr (WV >= 5) {
                    // rows in pairs: the two vertical windows share WV - 1 rows (opn_pair)
#pragma unroll
                    for (int r = 0; r < BR; r += 2) {
                        C::load_row(rows, r, lane, E[r % RING]);
                        C::load_row(rows, r + 1, lane, E[(r + 1) % RING]);
                        const bool ok0 = !CHECK || (unsigned)(o + r) < (unsigned)it.rows_out;
                        const bool ok1 = !CHECK || (unsigned)(o + r + 1) < (unsigned)it.rows_out;
                        if (ok0 || ok1) {
                            uint32_t a0[NW], a1[NW], b0[NW], b1[NW];  // rows r / r + 1 (b*: max for the gradient)
#pragma unroll
                            for (int w = 0; w < NW; ++w) {
                                uint32_t col[WV + 1];  // rows r + 1, r, ..., r + 1 - WV
#pragma unroll
                                for (int k = 0; k <= WV; ++k) col[k] = E[(r + 1 - k + 8 * RING) % RING][w];
                                if constexpr (MODE == MODE_GRAD) {
                                    opn_pair<MODE_MIN, WV, 1>(col, a1[w], a0[w]);
                                    opn_pair<MODE_MAX, WV, 1>(col, b1[w], b0[w]);
                                } else {
                                    opn_pair<MODE, WV, 1>(col, a1[w], a0[w]);
                                }
                            }
                            if (ok0) emit(drow, a0, b0, a0);
                            if (ok1) emit(drow + dp, a1, b1, a1);
                        }
                        drow += 2 * dp;
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        C::load_row(rows, r, lane, E[r % RING]);
                        if (!CHECK || (unsigned)(o + r) < (unsigned)it.rows_out) {
                            uint32_t a0[NW], b0[NW];
#pragma unroll
                            for (int w = 0; w < NW; ++w) {
                                uint32_t col[WV];
#pragma unroll
                                for (int k = 0; k < WV; ++k) col[k] = E[(r - k + 8 * RING) % RING][w];
                                if constexpr (MODE == MODE_GRAD) {
                                    a0[w] = opn<MODE_MIN, WV>(col);
                                    b0[w] = opn<MODE_MAX, WV>(col);
                                } else {
                                    a0[w] = opn<MODE, WV>(col);
                                }
                            }
                            emit(drow, a0, b0, a0);
                        }
                        drow += dp;
                    }
                }
            };
            if (o >= 0 && o + BR <= it.rows_out) block(std::false_type{});
            else block(std::true_type{});
            o += BR;
            // block fully read by every lane: hand the slot back (the TMA refill is ordered after
            // these generic-proxy reads by program order + the warp barrier)
            __syncwarp();
            cslot = cslot + 1 == NS ? 0 : cslot + 1;
            cpar ^= cslot == 0;
            issue();
        }
    }
}

// ---------------------------------------------------------------------------------------------
template <typename T, int MODE, int GX, int GY>
cudaError_t launch_col_variant(const MorphJob& j, int R) {
    ColParams p{};
    p.src = static_cast<const uint8_t*>(j.src);
    p.sp = j.sp;
    p.dst = static_cast<uint8_t*>(j.dst);
    p.dp = j.dp;
    p.W = j.W;
    p.H = j.H;
    p.row_lo = -j.above;
    p.row_hi = j.H + j.below;
    p.cmode = j.cmode;
    p.bval = j.bval;
    p.simg = j.simg;
    p.dimg = j.dimg;
    p.batch = j.batch;
    p.nstrips = cdiv(j.W * (int)sizeof(T), SB);
    CUtensorMap map;
    using CG = ColGeo<GX>;
    constexpr int SMEM = CG::SMEM;
    CUtensorMap hmap;
    p.use_tma = stream::encode_input_map(j, SB / 4, BR, &map) ? 1 : 0;
    if (p.use_tma && CG::HALO > 0) p.use_tma = stream::encode_input_map(j, 4, BR, &hmap) ? 1 : 0;
    else memset(&hmap, 0, sizeof(hmap));
    auto kern = morph_col_kernel<T, MODE, GX, GY>;
    cudaError_t e = cudaSuccess;
    const int occ = kernel_occupancy((const void*)kern, WPB * 32, SMEM, &e);
    if (e != cudaSuccess) return e;
    const int sms = device_sm_count();
    if (R <= 0) {
        // rows per item (R + 2*GY a multiple of BR): the warps run in waves of (SMs x resident
        // warps) items; minimise waves x staged rows per item (ties go to the shorter item). A fixed
        // per-item switch cost of 8 rows was in this model until round 2; measured without it:
        // 4096^2 7x7 13.6 -> 12.7 us, 8192^2 3x3 31.1 -> 29.6, nothing more than 1% slower
        // (knob col_switch)
        const long slots = (long)sms * std::max(1, occ) * WPB;
        const long strips = (long)p.nstrips * j.batch;
        double best = 1e30;
        for (int m = 1; m <= 64; ++m) {
            const int r = m * BR - 2 * GY;
            if (r < 1) continue;
            const long items = strips * cdiv(j.H, r);
            const long waves = (items + slots - 1) / slots;
            const double t = (double)waves * (m * BR + tune("col_switch", 0));
            if (t < best - 1e-9) {
                best = t;
                R = r;
            }
            if (r >= j.H) break;
        }
        R = std::min(R, std::max(1, j.H));
    }
    p.R = R;
    p.nbands = cdiv(j.H, R);
    const long items = (long)p.nstrips * p.nbands * j.batch;
    const long ctas = std::max(1L, std::min((items + WPB - 1) / WPB, (long)sms * std::max(1, occ)));
    const long nwarps = ctas * WPB;
    const long per_img = (long)p.nstrips * p.nbands;
    p.db = (int)(nwarps / per_img);
    const long r2 = nwarps - (long)p.db * per_img;
    p.dband = (int)(r2 / p.nstrips);
    p.ds = (int)(r2 - (long)p.dband * p.nstrips);
    const FastDivHost fs = FastDivHost::make((uint32_t)p.nstrips), fi = FastDivHost::make((uint32_t)per_img);
    p.strip_m = fs.m;
    p.strip_s = fs.s;
    p.img_m = fi.m;
    p.img_s = fi.s;
    kern<<<dim3((unsigned)ctas), WPB * 32, SMEM, j.stream>>>(p, map, hmap);
    count_launch();
    return cudaGetLastError();
}

template <typename T, int MODE, int GY>
cudaError_t col_dispatch_x(const MorphJob& j, int R) {
    switch (j.gx) {
    case 0: return launch_col_variant<T, MODE, 0, GY>(j, R);
    case 1: return launch_col_variant<T, MODE, 1, GY>(j, R);
    case 2: return launch_col_variant<T, MODE, 2, GY>(j, R);
    case 3: return launch_col_variant<T, MODE, 3, GY>(j, R);
    }
    return cudaErrorInvalidValue;
}

template <typename T, int MODE>
cudaError_t col_dispatch(const MorphJob& j, int R) {
    switch (j.gy) {
    case 0: return col_dispatch_x<T, MODE, 0>(j, R);
    case 1: return col_dispatch_x<T, MODE, 1>(j, R);
    case 2: return col_dispatch_x<T, MODE, 2>(j, R);
    case 3: return col_dispatch_x<T, MODE, 3>(j, R);
    }
    return cudaErrorInvalidValue;
}

}  // namespace col
}  // namespace rmgpu

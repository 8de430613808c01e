// morph_fast.cuh -- shared implementation of the fused kernel (see morph_fast.cu for the design notes).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace rmgpu {
namespace fast {

constexpr int NT = 256;     // threads per CTA
constexpr int TH = 64;      // tile rows
constexpr int QMAX = 6;     // whole blocks between suffix run and prefix block kept in registers

// ---- per-thread lane words ------------------------------------------------------------------
template <typename T>
struct LW;
template <>
struct LW<uint8_t> {   // 4 pixels (or 4 rows of one column), 16-bit lanes: a = {0, 2}, b = {1, 3}
    uint32_t a, b;
};
template <>
struct LW<uint16_t> {  // 2 pixels (or 2 rows of one column): a = {0, 1}
    uint32_t a;
};

template <typename T>
struct Geo;
template <>
struct Geo<uint8_t> {
    static constexpr int PX = 4;    // pixels per global word
    static constexpr int GR = 4;    // rows per transposed entry
    static constexpr int TW = 256;  // tile width (pixels)
    static constexpr int NG = TH / 4;
    static constexpr int SHIFT = 2;
};
template <>
struct Geo<uint16_t> {
    static constexpr int PX = 2;
    static constexpr int GR = 2;
    static constexpr int TW = 128;
    static constexpr int NG = TH / 2;
    static constexpr int SHIFT = 1;
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

// u8 word -> 16-bit lanes and back
__device__ __forceinline__ LW<uint8_t> unpack(uint32_t w, uint8_t*) {
    return {prmt(w, 0u, 0x4240), prmt(w, 0u, 0x4341)};
}
__device__ __forceinline__ LW<uint16_t> unpack(uint32_t w, uint16_t*) { return {w}; }

// ---- kernel parameters ---------------------------------------------------------------------
struct FastParams {
    const uint8_t* src;
    size_t sp;            // bytes
    uint8_t* dst;
    size_t dp;            // bytes
    int W, H;
    int row_lo, row_hi;   // valid input rows (relative to output row 0)
    int gx, gy;
    int cmode;
    uint32_t bval;
    size_t simg, dimg;    // bytes between batch images
    int vs;               // vertical units per column word (row split)
    int hsegs;            // horizontal streaming segments (direct variants)
};

// ---- the 1-D sweeps ------------------------------------------------------------------------
// Emitter interface: em.group(o0, LW<T> g[GR]) receives GR consecutive outputs o0..o0+GR-1
// (o0 multiple of GR, possibly outside [0, n_out): the emitter filters).

// Direct window W3 in {3, 5}: forward stream, groups of GR outputs.
template <typename T, int MODE, int WD, class Load, class Emit>
__device__ __forceinline__ void sweep_direct(int n_out, const Load& ld, Emit& em) {
    constexpr int GR = Geo<T>::GR;
    LW<T> win[GR + WD - 1];
#pragma unroll
    for (int k = 0; k < WD - 1; ++k) win[k] = ld(k);
    for (int o0 = 0; o0 < n_out; o0 += GR) {
#pragma unroll
        for (int k = 0; k < GR; ++k) win[WD - 1 + k] = ld(o0 + WD - 1 + k);
        LW<T> out[GR];
#pragma unroll
        for (int k = 0; k < GR; ++k) {
            if constexpr (WD == 1) out[k] = win[k];
            else if constexpr (WD == 3) out[k] = lop3<MODE>(win[k], win[k + 1], win[k + 2]);
            else out[k] = lop<MODE>(lop3<MODE>(win[k], win[k + 1], win[k + 2]), lop<MODE>(win[k + 3], win[k + 4]));
        }
        em.group(o0, out);
#pragma unroll
        for (int k = 0; k < WD - 1; ++k) win[k] = win[k + GR];
    }
}

// Block (van Herk / Gil-Werman) emission for leading block L. P[] holds the prefix of block L.
template <typename T, int MODE, int B, class Load, class Emit>
__device__ __forceinline__ void vh_emit(int oL, LW<T> gap, const LW<T> (&P)[B], const Load& ld, Emit& em) {
    constexpr int GR = Geo<T>::GR;
    LW<T> acc = gap;
    LW<T> grp[GR];
#pragma unroll
    for (int m = B - 1; m >= 0; --m) {
        acc = lop<MODE>(acc, ld(oL + m));
        grp[m % GR] = lop<MODE>(acc, P[m]);
        if (m % GR == 0) em.group(oL + m, grp);
    }
}

// Streaming block sweep: n_out outputs; window w = 2g+1 >= B+1; inputs x[i], i >= 0, where output
// o covers x[o .. o+w-1].
template <typename T, int MODE, int B, class Load, class Emit>
__device__ __forceinline__ void sweep_block(int n_out, int w1, const Load& ld, Emit& em) {
    const int q = w1 / B, r = w1 - q * B;
    const int s = r & 3;                               // emission starts stay multiples of 4
    const int Lend = q + (n_out - 1 + r - s) / B;      // last leading block with an emission
    LW<T> M[QMAX];                                     // M[k] = min of block L-1-k
#pragma unroll
    for (int k = 0; k < QMAX; ++k) M[k] = lid<T, MODE>();
    for (int L = 0; L <= Lend; ++L) {
        const int base = s + L * B;
        LW<T> P[B];
        P[0] = ld(base);
#pragma unroll
        for (int m = 1; m < B; ++m) P[m] = lop<MODE>(P[m - 1], ld(base + m));
        const int oL = base - w1;
        if (oL + B - 1 >= 0) {
            LW<T> gap = lid<T, MODE>();
            const int t0 = oL + B;
            for (int i = 0; i < r; ++i) gap = lop<MODE>(gap, ld(t0 + i));
#pragma unroll
            for (int k = 0; k < QMAX - 1; ++k)
                if (k < q - 1) gap = lop<MODE>(gap, M[k]);
            vh_emit<T, MODE, B>(oL, gap, P, ld, em);
        }
#pragma unroll
        for (int k = QMAX - 1; k > 0; --k) M[k] = M[k - 1];
        M[0] = P[B - 1];
    }
}

// ---- vertical pass: loader from global + emitter into the transposed tile --------------------
template <typename T>
struct VLoad {
    const uint8_t* col;   // byte address of (image row 0, this thread's load column)
    size_t sp;
    int ybase;            // image row of input index 0
    int row_lo, row_hi;
    int cmode;
    uint32_t bword;       // constant border value replicated over the word
    uint32_t sel;         // byte permutation of (raw, bword) for border columns
    bool fix;
    __device__ __forceinline__ LW<T> operator()(int i) const {
        const int y = ybase + i;
        uint32_t raw;
        if (cmode && (y < row_lo || y >= row_hi)) {
            raw = bword;
        } else {
            const int yc = min(max(y, row_lo), row_hi - 1);
            raw = __ldg(reinterpret_cast<const uint32_t*>(col + (ptrdiff_t)yc * (ptrdiff_t)sp));
            if (fix) raw = prmt(raw, bword, sel);
        }
        return unpack(raw, (T*)nullptr);
    }
};

template <typename T>
struct VEmit;

template <>
struct VEmit<uint8_t> {
    uint2* vt;      // transposed tile, entry (xv, g) at vt[xv * NG + (g ^ swz)]
    int t;          // column word index (xv = 4t + c)
    int row0;       // tile row of output 0 of this unit
    int n_out;
    __device__ __forceinline__ void group(int o0, const LW<uint8_t> (&r)[4]) {
        if (o0 < 0 || o0 >= n_out) return;
        constexpr int NG = Geo<uint8_t>::NG;
        const int g = ((row0 + o0) >> 2) ^ (t & (NG - 1));
        uint2* base = vt + (size_t)(4 * t) * NG + g;
        // rows r0..r3 of columns 4t..4t+3 -> per column {rows 0,2 | rows 1,3}
        base[0 * NG] = make_uint2(prmt(r[0].a, r[2].a, 0x5410), prmt(r[1].a, r[3].a, 0x5410));
        base[1 * NG] = make_uint2(prmt(r[0].b, r[2].b, 0x5410), prmt(r[1].b, r[3].b, 0x5410));
        base[2 * NG] = make_uint2(prmt(r[0].a, r[2].a, 0x7632), prmt(r[1].a, r[3].a, 0x7632));
        base[3 * NG] = make_uint2(prmt(r[0].b, r[2].b, 0x7632), prmt(r[1].b, r[3].b, 0x7632));
    }
};

template <>
struct VEmit<uint16_t> {
    uint32_t* vt;
    int t;          // xv = 2t + c
    int row0;
    int n_out;
    __device__ __forceinline__ void group(int o0, const LW<uint16_t> (&r)[2]) {
        if (o0 < 0 || o0 >= n_out) return;
        constexpr int NG = Geo<uint16_t>::NG;
        const int g = ((row0 + o0) >> 1) ^ (t & (NG - 1));
        uint32_t* base = vt + (size_t)(2 * t) * NG + g;
        base[0] = prmt(r[0].a, r[1].a, 0x5410);
        base[NG] = prmt(r[0].a, r[1].a, 0x7632);
    }
};

// ---- horizontal pass: loader from the transposed tile + emitter into the output tile ---------
template <typename T>
struct HLoad;
template <>
struct HLoad<uint8_t> {
    const uint2* vt;
    int g, off, xmax;
    __device__ __forceinline__ LW<uint8_t> operator()(int i) const {
        constexpr int NG = Geo<uint8_t>::NG;
        const int xv = max(0, min(off + i, xmax));
        const uint2 v = vt[(size_t)xv * NG + (g ^ ((xv >> 2) & (NG - 1)))];
        return {v.x, v.y};
    }
};
template <>
struct HLoad<uint16_t> {
    const uint32_t* vt;
    int g, off, xmax;
    __device__ __forceinline__ LW<uint16_t> operator()(int i) const {
        constexpr int NG = Geo<uint16_t>::NG;
        const int xv = max(0, min(off + i, xmax));
        return {vt[(size_t)xv * NG + (g ^ ((xv >> 1) & (NG - 1)))]};
    }
};

template <typename T>
struct HEmit;
template <>
struct HEmit<uint8_t> {
    uint8_t* out;   // output tile, row pitch OUTP bytes
    int outp;
    int g;          // row group (rows 4g..4g+3)
    int col0;       // tile column of output 0
    int n_out;
    __device__ __forceinline__ void group(int o0, const LW<uint8_t> (&c)[4]) {
        if (o0 < 0 || o0 >= n_out) return;
        // c[k] = column o0+k: a = {row0,row2}, b = {row1,row3}
        const uint32_t a01 = prmt(c[0].a, c[1].a, 0x6240), a23 = prmt(c[2].a, c[3].a, 0x6240);
        const uint32_t b01 = prmt(c[0].b, c[1].b, 0x6240), b23 = prmt(c[2].b, c[3].b, 0x6240);
        uint8_t* p = out + (size_t)(4 * g) * outp + col0 + o0;
        *reinterpret_cast<uint32_t*>(p) = prmt(a01, a23, 0x5410);
        *reinterpret_cast<uint32_t*>(p + outp) = prmt(b01, b23, 0x5410);
        *reinterpret_cast<uint32_t*>(p + 2 * outp) = prmt(a01, a23, 0x7632);
        *reinterpret_cast<uint32_t*>(p + 3 * outp) = prmt(b01, b23, 0x7632);
    }
};
template <>
struct HEmit<uint16_t> {
    uint8_t* out;
    int outp;
    int g;          // rows 2g, 2g+1
    int col0;
    int n_out;
    __device__ __forceinline__ void group(int o0, const LW<uint16_t> (&c)[2]) {
        if (o0 < 0 || o0 >= n_out) return;
        uint8_t* p = out + (size_t)(2 * g) * outp + 2 * (col0 + o0);
        *reinterpret_cast<uint32_t*>(p) = prmt(c[0].a, c[1].a, 0x5410);
        *reinterpret_cast<uint32_t*>(p + outp) = prmt(c[0].a, c[1].a, 0x7632);
    }
};

// ---- per-axis variant selection ------------------------------------------------------------
// V: 1 = copy (window 1), 3 / 5 = direct, 4..32 (multiple of 4) = block size B.
template <typename T, int MODE, int V, class Load, class Emit>
__device__ __forceinline__ void sweep(int n_out, int w1, const Load& ld, Emit& em) {
    if constexpr (V == 1) sweep_direct<T, MODE, 1>(n_out, ld, em);
    else if constexpr (V == 3) sweep_direct<T, MODE, 3>(n_out, ld, em);
    else if constexpr (V == 5) sweep_direct<T, MODE, 5>(n_out, ld, em);
    else sweep_block<T, MODE, V>(n_out, w1, ld, em);
}

__host__ __device__ constexpr int outp_bytes(int tw_bytes) { return tw_bytes + 16; }

template <typename T>
__host__ __device__ constexpr int entry_bytes() { return sizeof(T) == 1 ? 8 : 4; }

// Column fix-up for a word starting at image column c (u8: 4 px, u16: 2 px).
template <typename T>
__device__ __forceinline__ void column_fixup(int c, int W, int cmode, int& c_load, uint32_t& sel, bool& fix) {
    constexpr int PX = Geo<T>::PX;
    if (c >= 0 && c + PX - 1 < W) {
        c_load = c;
        sel = 0x3210;
        fix = false;
        return;
    }
    fix = true;
    const int cc0 = min(max(c, 0), W - 1);
    c_load = (cc0 / PX) * PX;
    sel = 0;
#pragma unroll
    for (int j = 0; j < PX; ++j) {
        const int col = c + j;
        int nib[sizeof(T)];
        if (cmode && (col < 0 || col >= W)) {
#pragma unroll
            for (int b = 0; b < (int)sizeof(T); ++b) nib[b] = 4 + b;   // bytes of bword
        } else {
            const int cc = min(max(col, 0), W - 1) - c_load;
#pragma unroll
            for (int b = 0; b < (int)sizeof(T); ++b) nib[b] = cc * (int)sizeof(T) + b;
        }
#pragma unroll
        for (int b = 0; b < (int)sizeof(T); ++b) sel |= (uint32_t)nib[b] << (4 * (j * sizeof(T) + b));
    }
}

template <typename T, int MODE, int VV, int HV>
__global__ void __launch_bounds__(NT)
morph_fast_kernel(FastParams p) {
    using G = Geo<T>;
    constexpr int PX = G::PX, GR = G::GR, TW = G::TW, NG = G::NG;
    constexpr int OUTP = outp_bytes(TW * sizeof(T));
    extern __shared__ __align__(16) unsigned char smem[];

    const uint8_t* src = p.src + blockIdx.z * p.simg;
    uint8_t* dst = p.dst + blockIdx.z * p.dimg;
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
    const int gx = p.gx, gy = p.gy;
    const int xs = ((x0 - gx) >= 0) ? ((x0 - gx) / PX) * PX : -(((gx - x0) + PX - 1) / PX) * PX;
    const int nwv = (x0 + TW + gx - xs + PX - 1) / PX;   // column words incl. halo
    const int vtw = nwv * PX;

    unsigned char* vt = smem;                                      // vtw * NG entries
    uint8_t* outt = smem + (size_t)vtw * NG * entry_bytes<T>();    // TH x OUTP
    outt = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(outt) + 15) & ~uintptr_t(15));

    uint32_t bword = p.bval & 0xFF;
    if constexpr (sizeof(T) == 1) bword = bword * 0x01010101u;
    else bword = (p.bval & 0xFFFF) * 0x00010001u;

    // 1. vertical pass -------------------------------------------------------------------------
    {
        const int rows_per = TH / p.vs;
        for (int u = threadIdx.x; u < nwv * p.vs; u += NT) {
            const int t = u % nwv, v = u / nwv;
            int c_load;
            uint32_t sel;
            bool fix;
            column_fixup<T>(xs + PX * t, p.W, p.cmode, c_load, sel, fix);
            VLoad<T> ld{src + (size_t)c_load * sizeof(T), p.sp, y0 + v * rows_per - gy, p.row_lo, p.row_hi,
                        p.cmode, bword, sel, fix};
            if constexpr (sizeof(T) == 1) {
                VEmit<uint8_t> em{reinterpret_cast<uint2*>(vt), t, v * rows_per, rows_per};
                sweep<T, MODE, VV>(rows_per, 2 * gy, ld, em);
            } else {
                VEmit<uint16_t> em{reinterpret_cast<uint32_t*>(vt), t, v * rows_per, rows_per};
                sweep<T, MODE, VV>(rows_per, 2 * gy, ld, em);
            }
        }
    }
    __syncthreads();

    // 2. horizontal pass -----------------------------------------------------------------------
    {
        const int off = (x0 - gx) - xs;
        const int seg = TW / p.hsegs;
        for (int u = threadIdx.x; u < NG * p.hsegs; u += NT) {
            const int g = u % NG, sgi = u / NG;
            if constexpr (sizeof(T) == 1) {
                HLoad<uint8_t> ld{reinterpret_cast<const uint2*>(vt), g, off + sgi * seg, vtw - 1};
                HEmit<uint8_t> em{outt, OUTP, g, sgi * seg, seg};
                sweep<T, MODE, HV>(seg, 2 * gx, ld, em);
            } else {
                HLoad<uint16_t> ld{reinterpret_cast<const uint32_t*>(vt), g, off + sgi * seg, vtw - 1};
                HEmit<uint16_t> em{outt, OUTP, g, sgi * seg, seg};
                sweep<T, MODE, HV>(seg, 2 * gx, ld, em);
            }
        }
    }
    __syncthreads();

    // 3. store the tile -----------------------------------------------------------------------
    {
        const int rows = min(TH, p.H - y0);
        const int cols = min(TW, p.W - x0);
        const int row_bytes = cols * (int)sizeof(T);
        const bool vec = (((uintptr_t)(dst) | p.dp) & 15) == 0 && row_bytes == TW * (int)sizeof(T);
        if (vec) {
            constexpr int CPR = TW * sizeof(T) / 16;    // 16-byte chunks per row
            for (int i = threadIdx.x; i < rows * CPR; i += NT) {
                const int rr = i / CPR, ch = i % CPR;
                const uint4 v = *reinterpret_cast<const uint4*>(outt + (size_t)rr * OUTP + ch * 16);
                *reinterpret_cast<uint4*>(dst + (size_t)(y0 + rr) * p.dp + (size_t)x0 * sizeof(T) + ch * 16) = v;
            }
        } else {
            for (int i = threadIdx.x; i < rows * row_bytes; i += NT) {
                const int rr = i / row_bytes, b = i % row_bytes;
                dst[(size_t)(y0 + rr) * p.dp + (size_t)x0 * sizeof(T) + b] = outt[(size_t)rr * OUTP + b];
            }
        }
    }
}

// ---- host side -------------------------------------------------------------------------------
template <typename T>
size_t fast_smem(int gx) {
    using G = Geo<T>;
    const int xs_slack = 2 * G::PX;
    const int vtw = G::TW + 2 * gx + xs_slack;
    return (size_t)vtw * G::NG * entry_bytes<T>() + 16 + (size_t)TH * outp_bytes(G::TW * sizeof(T));
}

// Variant for one axis given the wing g (window 2g+1).
inline int pick_variant(int g) {
    const int w1 = 2 * g;
    if (g == 0) return 1;
    if (g == 1) return 3;
    if (g == 2) return 5;
    // block size: largest of the compiled sizes with 1 <= q <= QMAX, preferring small (r+q)/B
    static const int sizes[] = {4, 8, 16, 24, 32};
    int best = 0;
    double best_cost = 1e30;
    for (int B : sizes) {
        if (B > w1) continue;
        const int q = w1 / B, r = w1 - q * B;
        if (q > QMAX) continue;
        const double cost = 3.0 + (double)(r + q) / B + 0.02 * B;   // small bias against huge blocks
        if (cost < best_cost) {
            best_cost = cost;
            best = B;
        }
    }
    return best;  // 0 = not covered
}

template <typename T, int MODE, int VV, int HV>
cudaError_t launch_variant(const MorphJob& j) {
    using G = Geo<T>;
    FastParams p;
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
    // vertical units per column word: enough to fill the CTA, keeping >= 16 rows per unit
    const int nwv = (G::TW + 2 * j.gx + 2 * G::PX) / G::PX;
    int vs = 1;
    while (vs < 4 && nwv * vs * 2 <= NT + NT / 2 && (TH / (vs * 2)) >= 16 && (VV <= 5 || 2 * j.gy <= TH / (vs * 2)))
        vs *= 2;
    p.vs = vs;
    p.hsegs = 1;
    if (HV <= 5) {
        int hs = 1;
        while (hs < 16 && G::NG * hs * 2 <= NT && G::TW / (hs * 2) >= 16) hs *= 2;
        p.hsegs = hs;
    } else {
        int hs = 1;
        while (hs < 8 && G::NG * hs * 2 <= NT && G::TW / (hs * 2) >= 32) hs *= 2;
        p.hsegs = hs;
    }
    const size_t smem = fast_smem<T>(j.gx);
    auto kern = morph_fast_kernel<T, MODE, VV, HV>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(cdiv(j.W, G::TW), cdiv(j.H, TH), j.batch);
    kern<<<grid, NT, smem, j.stream>>>(p);
    count_launch();
    return cudaGetLastError();
}

#define RM_FAST_VARIANTS(X) X(1) X(3) X(5) X(4) X(8) X(16) X(24) X(32)

template <typename T, int MODE, int VV>
cudaError_t dispatch_h(const MorphJob& j, int hv) {
    switch (hv) {
#define RM_CASE(H) case H: return launch_variant<T, MODE, VV, H>(j);
        RM_FAST_VARIANTS(RM_CASE)
#undef RM_CASE
    }
    return cudaErrorInvalidValue;
}

template <typename T, int MODE>
cudaError_t dispatch_v(const MorphJob& j, int vv, int hv) {
    switch (vv) {
#define RM_CASE(V) case V: return dispatch_h<T, MODE, V>(j, hv);
        RM_FAST_VARIANTS(RM_CASE)
#undef RM_CASE
    }
    return cudaErrorInvalidValue;
}


}  // namespace fast
}  // namespace rmgpu

// morph_sep.cuh -- K3: the separable rectangle as two streaming passes that hand over through L2.
//
// The reference computes a w_x x w_y erosion/dilation as a vertical pass into a full intermediate
// image followed by a horizontal pass (separable.cpp:130-157; van Herk / Gil-Werman for long
// windows, sliding_extrema.cpp:58-132). The passes commute (the border clamp is per axis), and on
// B200 the intermediate of a 4096^2 u8 image (16 MB) fits the 126 MB L2 many times over, so K3
// runs the two passes as barrier-free, shared-memory-free streaming kernels (planner and pass
// order in morph_sep.cu: horizontal first on whole images and row bands):
//
//  * V (vertical pass): one thread per 4-pixel column word streams down a band of rows with
//    plain coalesced loads. Block van Herk with blocks of B rows: out = T[m] u G u P[m] where
//    P is the prefix of the leading block, T the suffix of the trailing rows (re-read: they
//    were loaded w_y rows earlier and are still in L2) and G the r tail rows plus the minimum of
//    the q-1 whole blocks in between (block minima kept in registers). The rows are folded in
//    pairs with three-input min / max (vblock_reduce): 2 VIMNMX3 per row and 16-bit-lane word --
//    all min / max, byte permutes, selects and shifts share the ALU pipe (one warp instruction
//    every second cycle per scheduler, tools/ubench/pipes.cu), so shifts and row addresses go to
//    the FMA pipe (IMAD.SHL / IMAD.WIDE). Reading the strip-major
//    intermediate (128-pixel strips) the row pitch is a compile-time constant, so every row of a
//    block is an immediate offset from one register. Large images: the same algorithm fed by a
//    per-warp TMA pipeline (tensor boxes or 1-D bulk copies, output by TMA store).
//  * H (horizontal pass): one warp per (group of 4 rows, column part) sweeps segments of 32 lane
//    chunks of C columns. Each lane transposes its 4 x C pixels in registers (PRMT) so that the two
//    16-bit lanes of a word hold different ROWS of one column, scans prefix and suffix along its C
//    columns, and fetches the far suffix / prefix / chunk minima from the lanes a = g / C away with
//    SHFL (g mod C is a template parameter, so every register index is compile-time). STAGES = 2
//    runs an opening's / closing's two horizontal passes in one sweep.
//  * Pixels use 16-bit SIMD lanes (VIMNMX(3).U16x2). u8 words keep their raw bytes: the 16-bit
//    min/max of raw words is exact in the high byte of each lane, so a word A = raw carries pixels
//    1 and 3 and A << 8 carries pixels 0 and 2 (no unpacking; one PRMT repacks).
//
// The intermediate is a private scratch buffer that is consumed while it is still in L2 (measured
// DRAM traffic of a 4096^2 op: 33.9 MB for 33.5 MB algorithmic; profiles/traffic_cfg2.json).
#pragma once

#include "morph_stream.cuh"  // TMA / mbarrier helpers, tensor-map encoders

namespace rmgpu {
namespace sep {

struct SepParams {
    const uint8_t* src;
    size_t sp;
    uint8_t* dst;
    size_t dp;
    int W, H;            // output extent of one image
    int row_lo, row_hi;  // V: valid input rows relative to output row 0 ([-above, H + below))
    int g;               // wing along the pass axis
    int q, r;            // V: 2g = q*B + r
    int rb;              // V: output rows per band (multiple of B)
    int cmode;
    uint32_t bval;
    size_t simg, dimg;
    int nwords;          // V: 4-pixel column words per row
    int groups;          // H: 4-row groups per image
    int parts, pw;       // H: column parts per row group (one warp each), output columns per part
    int batch;
    int discard;         // H: discard the source lines after use (source = private scratch)
    int pdl;             // launched as a programmatic dependent of the previous pass (same op)
    size_t sstride;      // V: source strip stride (strip-major intermediate) or 0 (row-major)
    size_t dsstride;     // H: destination strip stride (strip-major intermediate) or 0 (row-major)
    int nstrips, nbands; // V (TMA): 128-pixel strips per row, bands per image
    int nsl, nst;        // V (TMA): leading / trailing ring slots per warp
    int wsmem;           // V (TMA): shared-memory bytes per warp
};

// 4 pixels of one row (V) in two 16-bit-lane words.
template <typename T>
struct W4;
template <>
struct W4<uint8_t> {
    static __device__ __forceinline__ uint2 load(const uint8_t* p) {
        const uint32_t raw = __ldg(reinterpret_cast<const unsigned int*>(p));
        return make_uint2(raw, raw << 8);
    }
    static __device__ __forceinline__ void store(uint8_t* p, uint2 v) {
        *reinterpret_cast<uint32_t*>(p) = prmt(v.x, v.y, 0x3715);
    }
    static __device__ __forceinline__ uint2 splat(uint32_t b) {
        const uint32_t w = b * 0x01010101u;
        return make_uint2(w, w);
    }
    static __device__ __forceinline__ uint32_t pixel(uint2 v, int k) {  // pixel k of a word pair
        return k & 1 ? (v.x >> (8 * k)) & 0xFF : (v.y >> (8 * k + 8)) & 0xFF;
    }
};
template <>
struct W4<uint16_t> {
    static __device__ __forceinline__ uint2 load(const uint8_t* p) {
        return __ldg(reinterpret_cast<const uint2*>(p));
    }
    static __device__ __forceinline__ void store(uint8_t* p, uint2 v) { *reinterpret_cast<uint2*>(p) = v; }
    static __device__ __forceinline__ uint2 splat(uint32_t b) {
        const uint32_t w = b * 0x00010001u;
        return make_uint2(w, w);
    }
    static __device__ __forceinline__ uint32_t pixel(uint2 v, int k) {
        const uint32_t w = k < 2 ? v.x : v.y;
        return (w >> (16 * (k & 1))) & 0xFFFF;
    }
};

template <int MODE>
__device__ __forceinline__ uint2 op2(uint2 a, uint2 b) {
    return make_uint2(red2_u16x2<MODE>(a.x, b.x), red2_u16x2<MODE>(a.y, b.y));
}
template <int MODE>
__device__ __forceinline__ uint2 op3(uint2 a, uint2 b, uint2 c) {
    return make_uint2(red3_u16x2<MODE>(a.x, b.x, c.x), red3_u16x2<MODE>(a.y, b.y, c.y));
}
template <int MODE>
__device__ __forceinline__ uint2 ident2() {
    const uint32_t v = MODE == MODE_MIN ? 0xFFFFFFFFu : 0u;
    return make_uint2(v, v);
}

constexpr int VT = 128;  // threads per V block
constexpr int HT = 128;  // threads per H block (4 warps, one 4-row group each)

// ================================ V: vertical pass ==============================================
// Raw row words: u8 = one 32-bit word (4 pixels), u16 = two (4 pixels).
template <typename T>
struct VW;
template <>
struct VW<uint8_t> {
    using Raw = uint32_t;
    static __device__ __forceinline__ Raw load(const uint8_t* p) { return __ldg(reinterpret_cast<const unsigned int*>(p)); }
    static __device__ __forceinline__ uint2 unpack(Raw r) { return make_uint2(r, r << 8); }
    static __device__ __forceinline__ Raw splat(uint32_t b) { return b * 0x01010101u; }
    static __device__ __forceinline__ Raw sel(bool c, Raw a, Raw b) { return c ? a : b; }
};
template <>
struct VW<uint16_t> {
    using Raw = uint2;
    static __device__ __forceinline__ Raw load(const uint8_t* p) { return __ldg(reinterpret_cast<const uint2*>(p)); }
    static __device__ __forceinline__ uint2 unpack(Raw r) { return r; }
    static __device__ __forceinline__ Raw splat(uint32_t b) { return make_uint2(b * 0x00010001u, b * 0x00010001u); }
    static __device__ __forceinline__ Raw sel(bool c, Raw a, Raw b) { return make_uint2(c ? a.x : b.x, c ? a.y : b.y); }
};

// Ragged last column word (W % 4 != 0): the pixels past W are computed from in-pitch garbage and
// dropped here, one pixel store each.
template <typename T>
__device__ __forceinline__ void store_partial(uint8_t* p, uint2 v, int n) {
    for (int k = 0; k < n; ++k) reinterpret_cast<T*>(p)[k] = (T)W4<T>::pixel(v, k);
}

constexpr int VRMAX = 4;  // tail rows r = 2g mod B folded from re-read rows (planner keeps r <= 4)

// G op= the n most recent whole-block minima M[0..n) (n warp-uniform, <= 4): one branch instead of
// a select per register.
template <int MODE, int QM>
__device__ __forceinline__ uint2 fold_minima(uint2 G, const uint2 (&M)[QM], int n) {
    static_assert(QM >= 4, "block minima");
    switch (n) {
    case 4: return op3<MODE>(op3<MODE>(G, M[0], M[1]), M[2], M[3]);
    case 3: return op3<MODE>(op2<MODE>(G, M[0]), M[1], M[2]);
    case 2: return op3<MODE>(G, M[0], M[1]);
    case 1: return op2<MODE>(G, M[0]);
    default: return G;
    }
}

// The reductions of one block of B (even) output rows in 2 three-input min / max per row and
// 16-bit-lane word (VIMNMX3 issues at the rate of the two-input form): rows are folded in pairs,
//   T2[j] = G u trailing rows 2j .. B-1       = op3(T2[j+1], xt[2j], xt[2j+1]),   T2[B/2] = G
//   P2[j] = leading rows 0 .. 2j+1            = op3(P2[j-1], xl[2j], xl[2j+1])
//   out[2j]   = op3(T2[j], P2[j-1], xl[2j]),   out[2j+1] = op3(xt[2j+1], T2[j+1], P2[j])
// with G = the r tail rows and the q-1 whole-block minima. XT / XR / XL return unpacked rows.
template <typename T, int MODE, int B, int QM, typename XT, typename XR, typename XL, typename ST>
__device__ __forceinline__ void vblock_reduce(int q, int r, uint2 (&M)[QM], XT xt, XR xr, XL xl, ST st) {
    static_assert(B % 2 == 0, "rows are folded in pairs");
    constexpr int HB = B / 2;
    uint2 G = ident2<MODE>();
    switch (r) {  // warp-uniform
    case 4: G = op3<MODE>(op3<MODE>(G, xr(0), xr(1)), xr(2), xr(3)); break;
    case 3: G = op3<MODE>(xr(0), xr(1), xr(2)); break;
    case 2: G = op2<MODE>(xr(0), xr(1)); break;
    case 1: G = xr(0); break;
    default: break;
    }
    G = fold_minima<MODE, QM>(G, M, q - 1);
    uint2 T2[HB + 1];
    T2[HB] = G;
#pragma unroll
    for (int j = HB - 1; j >= 0; --j) T2[j] = op3<MODE>(T2[j + 1], xt(2 * j), xt(2 * j + 1));
    uint2 P2 = xl(0);
    st(0, op2<MODE>(T2[0], P2));
    P2 = op2<MODE>(P2, xl(1));
    st(1, op3<MODE>(xt(1), T2[1], P2));
#pragma unroll
    for (int j = 1; j < HB; ++j) {
        const uint2 xe = xl(2 * j), xo = xl(2 * j + 1);
        st(2 * j, op3<MODE>(T2[j], P2, xe));
        P2 = op3<MODE>(P2, xe, xo);
        st(2 * j + 1, op3<MODE>(xt(2 * j + 1), T2[j + 1], P2));
    }
#pragma unroll
    for (int k = QM - 1; k > 0; --k) M[k] = M[k - 1];
    M[0] = P2;
}

// B rows of one column word starting at row0 (border-aware on edge bands).
template <typename T, int B, bool EDGE, int SPC>
__device__ __forceinline__ void vload_rows(const SepParams& p, const uint8_t* s, int row0,
                                           typename VW<T>::Raw (&x)[B]) {
    using V = VW<T>;
    using Raw = typename V::Raw;
    const ptrdiff_t sp = SPC ? (ptrdiff_t)SPC : (ptrdiff_t)p.sp;
    if constexpr (EDGE) {  // border-aware (edge bands): clamp, then substitute the constant
        const Raw CW = V::splat(p.bval);
#pragma unroll
        for (int m = 0; m < B; ++m) {
            const int i = row0 + m;
            const int ic = min(max(i, p.row_lo), p.row_hi - 1);
            const Raw v = V::load(s + (ptrdiff_t)ic * sp);
            x[m] = V::sel(p.cmode && ic != i, CW, v);
        }
    } else if constexpr (SPC != 0) {
        const uint8_t* pl = s + (ptrdiff_t)row0 * sp;
#pragma unroll
        for (int m = 0; m < B; ++m) x[m] = V::load(pl + m * SPC);  // immediate offsets
    } else {
        const uint8_t* pl = s + (ptrdiff_t)row0 * sp;
#pragma unroll
        for (int m = 0; m < B; ++m)  // base + m * pitch: one 64-bit multiply-add (FMA pipe) per row
            x[m] = V::load(pl + (size_t)(uint32_t)m * (size_t)(uint32_t)sp);
    }
}

// One block of B output rows. Window of output m (leading input row base+m):
//   rows [base+m-2g, base+m] = T[m] u G u P[m] with
//   T[m] = suffix of the trailing batch [base-2g, base-2g+B) from m,
//   G    = the r rows [base-2g+B, base-(q-1)B) u whole blocks L-q+1 .. L-1 (minima M[0..q-2]),
//   P[m] = prefix of the leading block [base, base+m].
// SPC: compile-time source row pitch (0 = runtime p.sp). With SPC every row of a block is a
// compile-time offset from one base register (the strip-major intermediate of the H-first order).
// All 2B (+r) loads of a block are issued before its first reduction. (Measured: loading the next
// block's leading rows one block ahead -- B more live registers -- is slower: 4096^2 1x31 11.8 vs
// 10.1 us, 63x63 19.8 vs 18.8 us.)
template <typename T, int MODE, int B, int QM, bool EDGE, bool FULL, int SPC>
__device__ __forceinline__ void vblock(const SepParams& p, const uint8_t* s, uint8_t* drow, int base, int nst,
                                       int nvalid, uint2 (&M)[QM]) {
    using V = VW<T>;
    using Raw = typename V::Raw;
    const int w1 = 2 * p.g, q = p.q, r = p.r;
    const ptrdiff_t sp = SPC ? (ptrdiff_t)SPC : (ptrdiff_t)p.sp;
    Raw xt[B], xr[VRMAX], xl[B];
    const int tb = base - w1;  // first trailing row; the r tail rows follow the batch directly
    vload_rows<T, B, EDGE, SPC>(p, s, tb, xt);
    if constexpr (EDGE) {
        const Raw CW = V::splat(p.bval);
#pragma unroll
        for (int t = 0; t < VRMAX; ++t)
            if (t < r) {
                const int i = tb + B + t;
                const int ic = min(max(i, p.row_lo), p.row_hi - 1);
                xr[t] = V::sel(p.cmode && ic != i, CW, V::load(s + (ptrdiff_t)ic * sp));
            }
    } else {
        const uint8_t* pt = s + (ptrdiff_t)(tb + B) * sp;
#pragma unroll
        for (int t = 0; t < VRMAX; ++t)
            if (t < r) xr[t] = V::load(pt + (size_t)(uint32_t)t * (size_t)(uint32_t)sp);
    }
    vload_rows<T, B, EDGE, SPC>(p, s, base, xl);
    vblock_reduce<T, MODE, B, QM>(
        q, r, M, [&](int m) { return V::unpack(xt[m]); }, [&](int t) { return V::unpack(xr[t]); },
        [&](int m) { return V::unpack(xl[m]); },
        [&](int m, uint2 o) {
            // row m of the block: base + m * pitch as one 64-bit multiply-add (FMA pipe), not a
            // chain of 64-bit adds on the ALU pipe the min / max instructions saturate
            uint8_t* d = drow + (size_t)(uint32_t)m * (size_t)(uint32_t)p.dp;
            if constexpr (FULL) {
                W4<T>::store(d, o);
            } else if (m < nst) {
                if (nvalid == 4) W4<T>::store(d, o);
                else store_partial<T>(d, o, nvalid);
            }
        });
}

template <typename T, int MODE, int B, int QM, bool EDGE, int SPC = 0>
__device__ __forceinline__ void vpass_body(const SepParams& p, const uint8_t* s, uint8_t* d, int y0, int y1,
                                           int nvalid) {
    using V = VW<T>;
    const ptrdiff_t sp = SPC ? (ptrdiff_t)SPC : (ptrdiff_t)p.sp;
    const int i0 = y0 + p.g;  // leading input row of output row y0
    const uint2 ID = ident2<MODE>();
    uint2 M[QM];
#pragma unroll
    for (int k = 0; k < QM; ++k) M[k] = ID;
    // warm-up: minima of the q-1 whole blocks before block 0
    for (int L = -(p.q - 1); L < 0; ++L) {
        typename V::Raw xl[B];
        vload_rows<T, B, EDGE, SPC>(p, s, i0 + L * B, xl);
        uint2 P = op2<MODE>(V::unpack(xl[0]), V::unpack(xl[1]));
#pragma unroll
        for (int m = 2; m + 1 < B; m += 2) P = op3<MODE>(P, V::unpack(xl[m]), V::unpack(xl[m + 1]));
#pragma unroll
        for (int k = QM - 1; k > 0; --k) M[k] = M[k - 1];
        M[0] = P;
    }
    (void)sp;
    for (int yb = y0; yb < y1; yb += B) {
        const int base = i0 + (yb - y0);
        uint8_t* drow = d + (ptrdiff_t)yb * (ptrdiff_t)p.dp;
        const int nst = y1 - yb;
        if (nst >= B && nvalid == 4) vblock<T, MODE, B, QM, EDGE, true, SPC>(p, s, drow, base, nst, nvalid, M);
        else vblock<T, MODE, B, QM, EDGE, false, SPC>(p, s, drow, base, nst, nvalid, M);
    }
}

// Measured (4096^2 / 16384^2 u8 1x63): 4 resident CTAs (<= 128 registers, small spills on the
// border path) with the leading loads issued after the trailing suffix beat 3 CTAs with every load
// hoisted: 12.4 vs 13-16 us, 65.5% vs 52-62% of HBM. u8 blocks of <= 14 rows fit 6 CTAs (85
// registers; one wave of the ~24-warps-per-SM band plan): 4096^2 1x31 12.1 -> 10.7 us, 31x31 17.7 ->
// 16.6, 15x15 16.9 -> 16.5; taller blocks lose at 5-6 CTAs (101x101 B20 21.0 -> 23.1 us), and so
// does u16 (cfg4 424 -> 417 Gpix/s).
#ifndef SEP_VMINB
#ifndef SEP_VMINB16
#define SEP_VMINB16 4
#endif
#define SEP_VMINB(T, B) (sizeof(T) == 1 ? ((B) <= 14 ? 6 : 4) : SEP_VMINB16)
#endif
#ifndef SEP_VHOIST
#define SEP_VSPLIT 1
#endif
template <typename T, int MODE, int B, int QM, int SPC = 0>
__global__ void __launch_bounds__(VT, SEP_VMINB(T, B)) vpass_kernel(const SepParams p) {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // a dependent may start scheduling
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // no-op unless launched as a PDL dependent
    const int c = blockIdx.x * VT + threadIdx.x;
    if (c >= p.nwords) return;
    const int y0 = blockIdx.y * p.rb;
    const int y1 = min(y0 + p.rb, p.H);
    const int nblk = (y1 - y0 + B - 1) / B;
    constexpr int sz = sizeof(T);
    // source column word c: row-major (strip stride 0) or strip-major (128-pixel strips of
    // p.sstride bytes, rows SPC bytes apart)
    const uint8_t* s = p.src + (size_t)blockIdx.z * p.simg +
                       (p.sstride ? (size_t)(c >> 5) * p.sstride + (size_t)(c & 31) * 4 * sz : (size_t)c * 4 * sz);
    uint8_t* d = p.dst + (size_t)blockIdx.z * p.dimg + (size_t)c * 4 * sz;
    // rows touched: [y0 - g, y0 + nblk*B - 1 + g]
    const bool edge = (y0 - p.g < p.row_lo) || (y0 + nblk * B + p.g > p.row_hi);
    const int nvalid = min(4, p.W - 4 * c);
    if (edge) vpass_body<T, MODE, B, QM, true, SPC>(p, s, d, y0, y1, nvalid);
    else vpass_body<T, MODE, B, QM, false, SPC>(p, s, d, y0, y1, nvalid);
}

// ---------------- V fed by TMA: one warp = one strip of 128 pixels x one band ------------------
// Every warp is an independent pipeline (no CTA barriers): lane 0 streams the leading blocks (B
// rows) and the trailing batches (B + VRMAX rows, L2 hits) into two private shared-memory rings with
// 2-D TMA boxes, PF blocks ahead; all lanes read rows with one LDS each (compile-time offsets, no
// address arithmetic) and write results into a double-buffered output tile that leaves through
// one TMA tensor store per block. Bands touching the image border take the LDG path above.
constexpr int VTW = VT / 32;  // warps per CTA

template <typename T, int MODE, int B, int QM>
__global__ void __launch_bounds__(VT) vtma_kernel(const SepParams p, const __grid_constant__ CUtensorMap lmap,
                                                  const __grid_constant__ CUtensorMap tmap,
                                                  const __grid_constant__ CUtensorMap omap) {
    using V = VW<T>;
    using Raw = typename V::Raw;
    using namespace stream;
    constexpr int sz = sizeof(T);
    constexpr int SB = 128 * sz;  // bytes per strip row
    constexpr int TB = B + VRMAX;  // rows per trailing box
    extern __shared__ __align__(128) unsigned char smem[];
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // a dependent may start scheduling
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // no-op unless launched as a PDL dependent
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wid = blockIdx.x * VTW + warp;
    const int per_img = p.nstrips * p.nbands;
    const int img = wid / per_img;
    if (img >= p.batch) return;
    const int rem = wid - img * per_img;
    const int band = rem / p.nstrips;
    const int strip = rem - band * p.nstrips;
    const int y0 = band * p.rb;
    const int y1 = min(y0 + p.rb, p.H);
    const int nblk = (y1 - y0 + B - 1) / B;
    const int g = p.g, w1 = 2 * g, q = p.q, r = p.r;
    // bands whose rows reach past the valid input rows fill the rings themselves (clamped rows /
    // the constant), synchronously; everything downstream is shared with the TMA path
    const bool edge = (y0 - g < p.row_lo) || (y0 + nblk * B + g > p.row_hi);
    const int ecw = min(strip * 32 + lane, p.nwords - 1);
    const uint8_t* ecol = p.src + (size_t)img * p.simg +
                          (p.sstride ? (size_t)(ecw >> 5) * p.sstride + (size_t)(ecw & 31) * 4 * sz : (size_t)ecw * 4 * sz);
    auto fill = [&](unsigned char* slot, int row0, int nrows) {
        const Raw CW = V::splat(p.bval);
        for (int m = 0; m < nrows; ++m) {
            const int i = row0 + m;
            const int ic = min(max(i, p.row_lo), p.row_hi - 1);
            const Raw v = V::load(ecol + (ptrdiff_t)ic * (ptrdiff_t)p.sp);
            *reinterpret_cast<Raw*>(slot + m * SB + lane * 4 * sz) = V::sel(p.cmode && ic != i, CW, v);
        }
        __syncwarp();
    };
    const int NSL = p.nsl, NST = p.nst;
    unsigned char* wbase = smem + (size_t)warp * p.wsmem;
    unsigned char* lring = wbase;
    unsigned char* tring = lring + (size_t)NSL * B * SB;
    unsigned char* outb = tring + (size_t)NST * TB * SB;
    uint64_t* fl = reinterpret_cast<uint64_t*>(outb + 2 * B * SB);
    uint64_t* ft = fl + NSL;
    if (lane == 0) {
        for (int k = 0; k < NSL; ++k) mbar_init(&fl[k], 1);
        for (int k = 0; k < NST; ++k) mbar_init(&ft[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    const int i0 = y0 + g;  // leading input row of output row y0
    const int nL = q - 1 + nblk;
    const int xw = strip * (SB / 4);  // map x coordinate (32-bit words)
    // strip-major source (p.sstride): a block of a strip is one contiguous run of rows -> one 1-D
    // bulk copy, no tensor map
    const uint8_t* sstrip = p.src + (size_t)img * p.simg + (size_t)strip * p.sstride;
    auto issue_lead = [&](int jl, int slot) {
        mbar_arrive_tx(&fl[slot], (uint32_t)(B * SB));
        const int row = i0 + (jl - (q - 1)) * B;
        if (p.sstride) bulk_g2s(lring + (size_t)slot * B * SB, sstrip + (ptrdiff_t)row * SB, (uint32_t)(B * SB), &fl[slot]);
        else tma_box(lring + (size_t)slot * B * SB, &lmap, xw, row - p.row_lo, img, &fl[slot]);
    };
    auto issue_trail = [&](int L, int slot) {
        mbar_arrive_tx(&ft[slot], (uint32_t)(TB * SB));
        const int row = i0 + L * B - w1;
        if (p.sstride) bulk_g2s(tring + (size_t)slot * TB * SB, sstrip + (ptrdiff_t)row * SB, (uint32_t)(TB * SB), &ft[slot]);
        else tma_box(tring + (size_t)slot * TB * SB, &tmap, xw, row - p.row_lo, img, &ft[slot]);
    };
    if (lane == 0 && !edge) {
        if (!p.sstride) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&lmap) : "memory");
        for (int k = 0; k < NSL && k < nL; ++k) issue_lead(k, k);
        for (int k = 0; k < NST && k < nblk; ++k) issue_trail(k, k);
    }
    const uint2 ID = ident2<MODE>();
    uint2 M[QM];
#pragma unroll
    for (int k = 0; k < QM; ++k) M[k] = ID;
    const int lo = lane * 4 * sz;
    int lslot = 0, lpar = 0, tslot = 0, tpar = 0;  // ring positions of block jl / L
    for (int jl = 0; jl < nL; ++jl) {
        const int L = jl - (q - 1);
        unsigned char* lsb = lring + (size_t)lslot * B * SB;
        const unsigned char* ls = lsb + lo;
        if (edge) fill(lsb, i0 + L * B, B);
        else mbar_wait(&fl[lslot], (uint32_t)lpar);
        if (L < 0) {  // warm-up block: its minimum only
            uint2 P = V::unpack(*reinterpret_cast<const Raw*>(ls));
#pragma unroll
            for (int m = 1; m < B; ++m) P = op2<MODE>(P, V::unpack(*reinterpret_cast<const Raw*>(ls + m * SB)));
#pragma unroll
            for (int k = QM - 1; k > 0; --k) M[k] = M[k - 1];
            M[0] = P;
            __syncwarp();
            if (lane == 0 && !edge && jl + NSL < nL) issue_lead(jl + NSL, lslot);
            if (++lslot == NSL) { lslot = 0; lpar ^= 1; }
            continue;
        }
        unsigned char* tsb = tring + (size_t)tslot * TB * SB;
        const unsigned char* ts = tsb + lo;
        if (edge) fill(tsb, i0 + L * B - w1, TB);
        else mbar_wait(&ft[tslot], (uint32_t)tpar);
        // output tile L & 1: its previous TMA store (block L-2) must have finished reading it
        unsigned char* obb = outb + (size_t)(L & 1) * B * SB;
        unsigned char* ob = obb + lo;
        if (L >= 2) {
            if (lane == 0) bulk_wait_read1();
            __syncwarp();
        }
        vblock_reduce<T, MODE, B, QM>(
            q, r, M, [&](int m) { return V::unpack(*reinterpret_cast<const Raw*>(ts + m * SB)); },
            [&](int t) { return V::unpack(*reinterpret_cast<const Raw*>(ts + (B + t) * SB)); },
            [&](int m) { return V::unpack(*reinterpret_cast<const Raw*>(ls + m * SB)); },
            [&](int m, uint2 o) { W4<T>::store(ob + m * SB, o); });
        fence_async_smem();  // the tile's generic writes before the async-proxy store reads it
        __syncwarp();
        if (lane == 0) {
            tma_store_box(&omap, strip * SB, y0 + L * B, img, obb);
            bulk_commit();
            if (!edge && jl + NSL < nL) issue_lead(jl + NSL, lslot);
            if (!edge && L + NST < nblk) issue_trail(L + NST, tslot);
        }
        if (++lslot == NSL) { lslot = 0; lpar ^= 1; }
        if (++tslot == NST) { tslot = 0; tpar ^= 1; }
    }
    if (lane == 0) bulk_wait_all();
}

// ================================ H: horizontal pass ============================================
// Lane chunk geometry: C columns x 4 rows per lane. u8: C = 16 (16-byte row loads) or 8; u16: 8.
template <typename T, int C>
struct HChunk {
    static constexpr int sz = sizeof(T);
    static constexpr int RB = C * sz;        // bytes per row per lane
    static constexpr int NW = RB / 4;        // 32-bit words per row per lane
};

template <typename T, int C>
__device__ __forceinline__ void h_load_row(const uint8_t* p, uint32_t (&w)[HChunk<T, C>::NW]) {
    constexpr int NW = HChunk<T, C>::NW;
    if constexpr (NW >= 4) {  // 16 or 32 bytes
#pragma unroll
        for (int k = 0; k < NW; k += 4) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + k / 4);
            w[k] = v.x; w[k + 1] = v.y; w[k + 2] = v.z; w[k + 3] = v.w;
        }
    } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
        w[0] = v.x; w[1] = v.y;
    }
}
template <typename T, int C>
__device__ __forceinline__ void h_store_row(uint8_t* p, const uint32_t (&w)[HChunk<T, C>::NW]) {
    constexpr int NW = HChunk<T, C>::NW;
    if constexpr (NW >= 4) {
#pragma unroll
        for (int k = 0; k < NW; k += 4) reinterpret_cast<uint4*>(p)[k / 4] = make_uint4(w[k], w[k + 1], w[k + 2], w[k + 3]);
    } else {
        *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
    }
}

// Border-aware load of one lane chunk row (chunks that reach past column 0 or W-1). Chunks start
// at multiples of C, so a chunk is either wholly left of the image, wholly right of it, or holds
// the last n < C real pixels followed by border pixels.
template <typename T, int C>
__device__ __forceinline__ void h_load_row_edge(const uint8_t* row, int cx, int W, int cmode, uint32_t bval,
                                                uint32_t (&w)[HChunk<T, C>::NW]) {
    constexpr int sz = sizeof(T);
    constexpr int NW = HChunk<T, C>::NW;
    const T* rp = reinterpret_cast<const T*>(row);
    const uint32_t splat = sz == 1 ? 0x01010101u : 0x00010001u;
    if (cx + C <= 0 || cx >= W) {
        const uint32_t v = cmode ? bval : (uint32_t)rp[cx < 0 ? 0 : W - 1];
#pragma unroll
        for (int k = 0; k < NW; ++k) w[k] = v * splat;
        return;
    }
    h_load_row<T, C>(row + (ptrdiff_t)cx * sz, w);
    const uint32_t rep = (cmode ? bval : (uint32_t)rp[W - 1]) * splat;
    const int nb = (W - cx) * sz;  // real bytes in the chunk (< C * sz)
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const int kb = nb - 4 * k;
        const uint32_t keep = kb >= 4 ? 0xFFFFFFFFu : (kb <= 0 ? 0u : (1u << (8 * kb)) - 1u);
        w[k] = (w[k] & keep) | (rep & ~keep);
    }
}

// rows r0..r3 (NW words each) -> per column c: {A, B} 16-bit-lane words holding 4 rows
template <typename T, int C>
__device__ __forceinline__ void h_transpose_in(const uint32_t (&r0)[HChunk<T, C>::NW],
                                               const uint32_t (&r1)[HChunk<T, C>::NW],
                                               const uint32_t (&r2)[HChunk<T, C>::NW],
                                               const uint32_t (&r3)[HChunk<T, C>::NW], uint2 (&x)[C]) {
    if constexpr (sizeof(T) == 1) {
        // A = {row1 -> byte1, row3 -> byte3}, B = {row0 -> byte1, row2 -> byte3}
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int k = c >> 2, e = c & 3;
            const uint32_t sel = (uint32_t)(e << 4) | (uint32_t)((4 + e) << 12);
            x[c].x = prmt(r1[k], r3[k], sel);
            x[c].y = prmt(r0[k], r2[k], sel);
        }
    } else {
        // A = {row0, row1}, B = {row2, row3}
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int k = c >> 1;
            const uint32_t sel = (c & 1) ? 0x7632u : 0x5410u;
            x[c].x = prmt(r0[k], r1[k], sel);
            x[c].y = prmt(r2[k], r3[k], sel);
        }
    }
}

template <typename T, int C>
__device__ __forceinline__ void h_transpose_out(const uint2 (&o)[C], uint32_t (&r0)[HChunk<T, C>::NW],
                                                uint32_t (&r1)[HChunk<T, C>::NW], uint32_t (&r2)[HChunk<T, C>::NW],
                                                uint32_t (&r3)[HChunk<T, C>::NW]) {
    if constexpr (sizeof(T) == 1) {
#pragma unroll
        for (int k = 0; k < C / 4; ++k) {
            const uint2 a = o[4 * k], b = o[4 * k + 1], c = o[4 * k + 2], e = o[4 * k + 3];
            // B words: byte1 = row0, byte3 = row2; A words: byte1 = row1, byte3 = row3
            const uint32_t b01 = prmt(a.y, b.y, 0x7351), b23 = prmt(c.y, e.y, 0x7351);
            const uint32_t a01 = prmt(a.x, b.x, 0x7351), a23 = prmt(c.x, e.x, 0x7351);
            r0[k] = prmt(b01, b23, 0x5410);
            r2[k] = prmt(b01, b23, 0x7632);
            r1[k] = prmt(a01, a23, 0x5410);
            r3[k] = prmt(a01, a23, 0x7632);
        }
    } else {
#pragma unroll
        for (int k = 0; k < C / 2; ++k) {
            const uint2 a = o[2 * k], b = o[2 * k + 1];
            r0[k] = prmt(a.x, b.x, 0x5410);
            r1[k] = prmt(a.x, b.x, 0x7632);
            r2[k] = prmt(a.y, b.y, 0x5410);
            r3[k] = prmt(a.y, b.y, 0x7632);
        }
    }
}

__device__ __forceinline__ uint2 shup(uint2 v, int d) {
    return make_uint2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}
__device__ __forceinline__ uint2 shdn(uint2 v, int d) {
    return make_uint2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}

// One warp item = 4 rows x one column part: segments of 32 lane chunks; BX = g mod C
// (compile-time). The next segment's rows are loaded before the current one is reduced.
// One lane-chunk van Herk pass over the columns of a segment: x = this lane's C columns (4 rows
// each), o = the window result for those columns (valid where the window's chunks are loaded).
// BXS = g mod C, plus 32 for the short-wing variant (a = 0 and 2 (g mod C) < C: some windows
// lie inside this lane's chunk; the planner picks it only when the wing is that short).
template <int MODE, int C, int BXS>
__device__ __forceinline__ void h_lane_pass(const uint2 (&x)[C], int a, uint2 (&o)[C]) {
    const uint2 ID = ident2<MODE>();
    constexpr int BX = BXS & 31;
    constexpr bool SHORT = BXS >= 32;
    constexpr int HC = C / 2;
    uint2 P[C], S[C];
    if constexpr (SHORT) {
        // half-chunk scans: prefix / suffix within each half, then the chunk-wide ones from them;
        // a window inside the chunk (2*BX+1 > C/2 columns) straddles the halves, so it is the left
        // half's suffix joined with the right half's prefix (stored in o now, merged below)
        P[0] = x[0];
        P[HC] = x[HC];
        S[HC - 1] = x[HC - 1];
        S[C - 1] = x[C - 1];
#pragma unroll
        for (int c = 1; c < HC; ++c) {
            P[c] = op2<MODE>(P[c - 1], x[c]);
            P[HC + c] = op2<MODE>(P[HC + c - 1], x[HC + c]);
        }
#pragma unroll
        for (int c = HC - 2; c >= 0; --c) {
            S[c] = op2<MODE>(S[c + 1], x[c]);
            S[HC + c] = op2<MODE>(S[HC + c + 1], x[HC + c]);
        }
#pragma unroll
        for (int j = BX; j < C - BX; ++j) o[j] = op2<MODE>(S[j - BX], P[j + BX]);  // in-chunk windows
#pragma unroll
        for (int c = HC; c < C; ++c) P[c] = op2<MODE>(P[HC - 1], P[c]);
#pragma unroll
        for (int c = 0; c < HC; ++c) S[c] = op2<MODE>(S[c], S[HC]);
    } else {
        P[0] = x[0];
#pragma unroll
        for (int c = 1; c < C; ++c) P[c] = op2<MODE>(P[c - 1], x[c]);
        S[C - 1] = x[C - 1];
#pragma unroll
        for (int c = C - 2; c >= 0; --c) S[c] = op2<MODE>(S[c + 1], x[c]);
    }
    const uint2 cm = P[C - 1];
    // chunk minima strictly inside the window: lanes L-a+1 .. L+a-1, plus lane L-a when the
    // left end lies one chunk further out (dl) and lane L+a when the right end does (dr)
    uint2 base = a > 0 ? cm : ID;
    for (int dd = 1; dd < a; ++dd) base = op3<MODE>(base, shup(cm, dd), shdn(cm, dd));
    const uint2 ml = shup(cm, a), mr = shdn(cm, a);
    uint2 m00 = base, m10, m01, m11;
    if (a > 0) {
        m10 = op2<MODE>(base, ml);
        m01 = op2<MODE>(base, mr);
        m11 = op3<MODE>(base, ml, mr);
    } else {  // a = 0: only both ends one chunk out leave a whole chunk (this lane's) inside
        m10 = ID;
        m01 = ID;
        m11 = cm;
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const bool dl = j < BX;       // left end in chunk L-a-1
        const bool dr = j + BX >= C;  // right end in chunk L+a+1
        const uint2 sl = shup(S[(j - BX + C) % C], a + (dl ? 1 : 0));
        const uint2 pr = shdn(P[(j + BX) % C], a + (dr ? 1 : 0));
        const uint2 mid = dl ? (dr ? m11 : m10) : (dr ? m01 : m00);
        if (!(SHORT && !dl && !dr)) o[j] = op3<MODE>(sl, mid, pr);  // (else: in-chunk, kept)
    }
}

// The border of the intermediate image between the two horizontal passes of an opening/closing:
// columns outside [0, W) take the constant, or (replicate) the intermediate's column 0 / W-1.
template <typename T, int C>
__device__ __forceinline__ void h_border_fix(uint2 (&o)[C], int X, int cx, int HA, int W, int cmode, uint32_t bval) {
    const int lane = threadIdx.x & 31;
    const bool left = X < HA * C, right = X + (32 - HA) * C > W;  // warp-uniform
    if (!left && !right) return;
    uint2 lv, rv;
    if (cmode) {
        const uint32_t w = sizeof(T) == 1 ? bval * 0x01010101u : bval * 0x00010001u;
        lv = rv = make_uint2(w, w);
    } else {
        lv = make_uint2(__shfl_sync(0xffffffffu, o[0].x, min(31, max(0, HA - X / C))),
                        __shfl_sync(0xffffffffu, o[0].y, min(31, max(0, HA - X / C))));
        const int lw = min(31, max(0, HA + (W - 1 - X) / C)), pw = (W - 1 - X) % C;
        uint2 mine = o[0];
#pragma unroll
        for (int j = 1; j < C; ++j)
            if (j == pw) mine = o[j];
        rv = make_uint2(__shfl_sync(0xffffffffu, mine.x, lw), __shfl_sync(0xffffffffu, mine.y, lw));
    }
    (void)lane;
#pragma unroll
    for (int j = 0; j < C; ++j) {
        if (cx + j < 0) o[j] = lv;
        else if (cx + j >= W) o[j] = rv;
    }
}

// One warp item = 4 rows x one column part: segments of 32 lane chunks; BX = g mod C
// (compile-time). The next segment's rows are loaded before the current one is reduced.
// STAGES = 2: the two horizontal passes of an opening (MODE = min, then max) or closing in one
// sweep -- the first pass's result never leaves registers; halo lanes double.
template <typename T, int MODE, int C, int BXS, int STAGES = 1>
__device__ __forceinline__ void h_item(const SepParams& p, const uint8_t* srow0, size_t sp, uint8_t* drow0,
                                       int nrows, int part) {
    using HC = HChunk<T, C>;
    constexpr int NW = HC::NW, sz = sizeof(T);
    constexpr int MODE2 = MODE == MODE_MIN ? MODE_MAX : MODE_MIN;
    const int lane = threadIdx.x & 31;
    const int a = p.g / C;                   // whole chunks in the wing
    constexpr int BX = BXS & 31;
    const int A = a + (BX > 0 ? 1 : 0);      // halo lanes on each side, per pass
    const int HA = STAGES * A;
    const int OS = (32 - 2 * HA) * C;        // output columns per segment
    const int W = p.W;
    // rows past the last one re-read it; their results are never stored
    const size_t rs1 = nrows > 1 ? sp : 0, rs2 = nrows > 2 ? 2 * sp : rs1, rs3 = nrows > 3 ? 3 * sp : rs2;

    using RowW = uint32_t[NW];
    auto load_seg = [&](int X, RowW& q0, RowW& q1, RowW& q2, RowW& q3) {
        const int cx = X + (lane - HA) * C;
        if (cx >= 0 && cx + C <= W) {
            const uint8_t* b = srow0 + (ptrdiff_t)cx * sz;
            h_load_row<T, C>(b, q0);
            h_load_row<T, C>(b + rs1, q1);
            h_load_row<T, C>(b + rs2, q2);
            h_load_row<T, C>(b + rs3, q3);
        } else {
            h_load_row_edge<T, C>(srow0, cx, W, p.cmode, p.bval, q0);
            h_load_row_edge<T, C>(srow0 + rs1, cx, W, p.cmode, p.bval, q1);
            h_load_row_edge<T, C>(srow0 + rs2, cx, W, p.cmode, p.bval, q2);
            h_load_row_edge<T, C>(srow0 + rs3, cx, W, p.cmode, p.bval, q3);
        }
    };
    const int xlo = part * p.pw, xhi = min(W, xlo + p.pw);
    // reduce the segment at X held in q*, refilling q* with the segment at Xn (if any) first
    auto process = [&](int X, RowW& q0, RowW& q1, RowW& q2, RowW& q3, int Xn) {
        const int cx = X + (lane - HA) * C;  // first column of this lane's chunk
        uint2 x[C];
        h_transpose_in<T, C>(q0, q1, q2, q3, x);
        if (Xn < xhi) load_seg(Xn, q0, q1, q2, q3);
        uint2 o[C];
        h_lane_pass<MODE, C, BXS>(x, a, o);
        if constexpr (STAGES == 2) {
            h_border_fix<T, C>(o, X, cx, HA, W, p.cmode, p.bval);
            h_lane_pass<MODE2, C, BXS>(o, a, x);
#pragma unroll
            for (int k = 0; k < C; ++k) o[k] = x[k];
        }
        uint32_t o0[NW], o1[NW], o2[NW], o3[NW];
        h_transpose_out<T, C>(o, o0, o1, o2, o3);
        if (lane >= HA && lane < 32 - HA && cx < W) {
            // a chunk never straddles a 128-pixel strip (C divides 128)
            uint8_t* drow = drow0 + (p.dsstride ? (ptrdiff_t)(cx >> 7) * (ptrdiff_t)p.dsstride + (ptrdiff_t)(cx & 127) * sz
                                                : (ptrdiff_t)cx * sz);
            if (cx + C <= W) {
                h_store_row<T, C>(drow, o0);
                if (nrows > 1) h_store_row<T, C>(drow + p.dp, o1);
                if (nrows > 2) h_store_row<T, C>(drow + 2 * p.dp, o2);
                if (nrows > 3) h_store_row<T, C>(drow + 3 * p.dp, o3);
            } else {
                const int n = W - cx;
                auto part_store = [&](int k, const uint32_t (&rw)[NW]) {  // compile-time indices only
                    if (k < nrows) {
#pragma unroll
                        for (int wi = 0; wi < NW; ++wi)
#pragma unroll
                            for (int b = 0; b < 4 / sz; ++b) {
                                const int e = wi * (4 / sz) + b;
                                if (e < n) reinterpret_cast<T*>(drow + (size_t)k * p.dp)[e] = (T)(rw[wi] >> (8 * sz * b));
                            }
                    }
                };
                part_store(0, o0);
                part_store(1, o1);
                part_store(2, o2);
                part_store(3, o3);
            }
        }
    };
    // one segment in flight (measured: a second register set for two is slower -- 4096^2 63x1
    // 10.3 -> 14.4 us -- code size and registers)
    uint32_t r0[NW], r1[NW], r2[NW], r3[NW];
    load_seg(xlo, r0, r1, r2, r3);
    for (int X = xlo; X < xhi; X += OS) process(X, r0, r1, r2, r3, X + OS);
    if (p.discard) {
        // drop the source lines only this warp reads (its part minus the halos the neighbouring
        // parts read) from L2 unwritten: the source is a private scratch band
        __syncwarp();
        const int elo = part == 0 ? 0 : xlo + HA * C;
        const int ehi = part == p.parts - 1 ? W : xhi - HA * C;
        const int l0 = part == 0 ? 0 : (elo * sz + 127) / 128;
        const int l1 = part == p.parts - 1 ? (W * sz + 127) / 128 : (ehi * sz) / 128;
        for (int k = 0; k < nrows; ++k)
            for (int l = l0 + lane; l < l1; l += 32)
                asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(srow0 + (size_t)k * sp + (size_t)l * 128) : "memory");
    }
}

// One warp per (4-row group, column part).
// Resident CTAs per SM (4 warps each): one sweep, u8 16-column chunks need ~128 registers (5-6 CTAs
// spill: 4096^2 63x63 19.1 -> 20.4 / 22.6 us); u16 8-column chunks fit 6 (4096^2 21x21 27.3 -> 24.8 us).
#ifndef SEP_HMINB2C8
#define SEP_HMINB2C8 5
#endif
#ifndef SEP_HMINB_SHORT
#define SEP_HMINB_SHORT 4
#endif
#define SEP_HMINB(T, C, BX, STAGES) \
    ((STAGES) == 1 ? (sizeof(T) == 2 ? 6 : ((BX) >= 32 ? SEP_HMINB_SHORT : 4)) : ((C) == 8 ? SEP_HMINB2C8 : 2))
template <typename T, int MODE, int C, int BX, int STAGES = 1>
__global__ void __launch_bounds__(HT, SEP_HMINB(T, C, BX, STAGES)) hpass_kernel(const SepParams p) {
    const int widx = blockIdx.x * (HT / 32) + (threadIdx.x >> 5);
    const int gidx = widx / p.parts;
    const int part = widx - gidx * p.parts;
    const int img = gidx / p.groups;
    const int grp = gidx - img * p.groups;
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // a dependent V may start scheduling
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // no-op unless launched as a PDL dependent
    if (img >= p.batch) return;  // whole warp: no shuffle partner is left behind
    const int y = grp * 4;
    h_item<T, MODE, C, BX, STAGES>(p, p.src + (size_t)img * p.simg + (size_t)y * p.sp, p.sp,
                           p.dst + (size_t)img * p.dimg + (size_t)y * p.dp, min(4, p.H - y), part);
}

// Launch with programmatic stream serialization when p.pdl: the CTAs may be scheduled while the
// previous pass drains; the kernel's griddepcontrol.wait holds them until its results are visible.
template <typename... Args>
inline cudaError_t launch_pdl(void (*kern)(SepParams, Args...), dim3 grid, dim3 block, int smem, cudaStream_t s,
                              const SepParams& p, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.pdl && tune("sep_pdl", 0) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, p, args...);
}

// H launch: after a V pass into the scratch band (p.discard) H is a programmatic dependent launch
// -- its CTAs are scheduled while V's last wave drains and wait (griddepcontrol.wait) for V's
// results before reading them.
inline cudaError_t launch_hk(void (*kern)(SepParams), const SepParams& p, dim3 grid, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(HT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (p.discard || p.pdl) && tune("sep_pdl", 0) ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace sep
}  // namespace rmgpu

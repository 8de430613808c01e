// morph_fuse.cuh -- K4: the separable rectangle in ONE kernel (vertical pass, then horizontal pass,
// the intermediate never leaves shared memory).
//
// Reference: morph_separable (separable.cpp:130-157) runs vertical_pass_direct /
// vertical_pass_via_transpose into a full intermediate image `tall`, then horizontal_pass; both
// passes are van Herk / Gil-Werman windows for long windows (sliding_extrema.cpp:58-132). K3
// (morph_sep.cuh) keeps that structure as two launches handing over through L2. K4 fuses them:
//
//  * One CTA = one item = a strip of SW output columns x a band of rows of one image. A strip
//    row with its horizontal halo is exactly 512 bytes (SW = C * (32 - 2A) pixels, A halo lanes of
//    C = 16 bytes each side), so every shared-memory row below is 512 bytes.
//  * Input rows arrive by TMA (2-D boxes of 128 x 32-bit words x B rows, one per V block) into a
//    ring of NS block slots, PF blocks ahead of the block being reduced. Rows outside the image
//    (TMA zero fill) are patched by the thread that owns the column word (the identity for
//    replicate -- the clamped row is always inside the window -- or the constant).
//  * Warps 0-3 (V): one thread per 4-byte column word of the 512-byte row streams down the band,
//    block van Herk with blocks of B rows exactly as K3's V (out = T[m] u G u P[m]); the trailing
//    rows are re-read from the ring (L - q, and the last r rows of L - q - 1 through a guard copy
//    in front of slot 0, so every row of a block is a compile-time offset from one base). Results
//    go to a ring of NT tile slots (B rows x 512 bytes).
//  * Warps 4-7 (H): one warp per 4-row group of the tile: K3's lane-chunk van Herk (each lane
//    transposes its 4 rows x 16 bytes in registers, prefix / suffix along its chunk, SHFL for the
//    far ends), the column border re-applied to the vertical result first (replicate = its column
//    0 / W-1, constant = the value), results stored with 128-bit stores straight to global.
//  * V -> H: per tile slot a full mbarrier (128 V arrivals) and an empty mbarrier (128 H
//    arrivals); groups are dealt round-robin to the H warps across blocks. V -> producer: one named
//    barrier among the V warps per block frees the ring slot of the oldest trailing block.
// Every input pixel is read from HBM once (halo re-reads hit L2) and every output pixel written
// once: 2 * sizeof(T) bytes per pixel, no intermediate in global memory.
#pragma once

#include "morph_sep.cuh"

namespace rmgpu {
namespace fuse {

// One CTA per SM: 4 vertical warps, 11 horizontal warps (the horizontal pass is the heavier one:
// measured alone, 8 horizontal warps per SM ran 1.9x longer than 8 vertical warps) and the TMA
// producer warp.
#ifndef FUSE_HWARPS
#define FUSE_HWARPS 11
#endif
constexpr int NVT = 128;                 // vertical threads (one 4-byte column word each)
constexpr int NHT = 32 * FUSE_HWARPS;    // horizontal threads
constexpr int FT = NVT + NHT + 32;       // warps 0-3 vertical, then horizontal, the last one TMA
constexpr int RP = 512;   // shared-memory row pitch: one strip row with its halo (bytes)
constexpr int QM = 8;     // whole-block minima kept in registers (q - 1 <= QM)
constexpr int RMAXG = 8;  // tail rows r = 2g mod B (guard rows in front of slot 0)
constexpr int NTMAX = 8;  // tile slots (p.nt = 2, 4 or 8, as the shared memory allows)

struct FuseParams {
    uint8_t* dst;
    size_t dp, dimg;
    int W, H;
    int row_lo, row_hi;   // valid input rows relative to output row 0 ([-above, H + below))
    int gx, gy;
    int q, r, QQ;         // 2 gy = q B + r; QQ = q + (r > 0): oldest trailing block L - QQ
    int a, A, SW;         // H: whole chunks in the wing, halo lanes, output columns per strip
    // items per image: the first `extra` strips in nb + 1 bands of rba rows, the others in nb bands
    // of rbb rows (rows multiples of B), so that the grid fills whole waves of resident CTAs
    int nstrips, nb, extra, rba, rbb, per_img, batch;
    int cmode;
    uint32_t bval;
    int NS;               // ring block slots (a multiple of pair)
    int pair;             // blocks per TMA box / full barrier (1 or 2): fewer, larger TMA issues
    int nt, ntlog;        // tile slots (a power of two) and its log2
    int dbg;              // tuning only: skip the math -- 1 horizontal, 2 vertical, 3 both
    long long* trace;     // debug timeline of CTA trace_cta (tools/trace_fuse.py), normally null
    int trace_cta;
    int ring_off, tile_off, bar_off;  // shared-memory layout (bytes)
};

// x * 256 on the FMA pipe (IMAD) instead of a shift on the ALU pipe, which the min/max and byte
// permutes saturate
__device__ __forceinline__ uint32_t shl8_fma(uint32_t x) {
    uint32_t y;
    asm("mul.lo.u32 %0, %1, 256;" : "=r"(y) : "r"(x));
    return y;
}

// A 4-byte column word as 16-bit-lane reduction values.
template <typename T>
struct FV;
template <>
struct FV<uint8_t> {
    using V = uint2;  // x = raw (pixels 1, 3 in the high bytes), y = raw << 8 (pixels 0, 2)
    static __device__ __forceinline__ V ld(const unsigned char* p) {
        const uint32_t r = *reinterpret_cast<const uint32_t*>(p);
        return make_uint2(r, shl8_fma(r));
    }
    static __device__ __forceinline__ void st(unsigned char* p, V v) {
        *reinterpret_cast<uint32_t*>(p) = prmt(v.x, v.y, 0x3715);
    }
    template <int MODE>
    static __device__ __forceinline__ V op(V a, V b) { return sep::op2<MODE>(a, b); }
    template <int MODE>
    static __device__ __forceinline__ V op3(V a, V b, V c) { return sep::op3<MODE>(a, b, c); }
    template <int MODE>
    static __device__ __forceinline__ V id() { return sep::ident2<MODE>(); }
    static __device__ __forceinline__ uint32_t splat(uint32_t b) { return b * 0x01010101u; }
};
template <>
struct FV<uint16_t> {
    using V = uint32_t;  // two pixels, one per 16-bit lane
    static __device__ __forceinline__ V ld(const unsigned char* p) { return *reinterpret_cast<const uint32_t*>(p); }
    static __device__ __forceinline__ void st(unsigned char* p, V v) { *reinterpret_cast<uint32_t*>(p) = v; }
    template <int MODE>
    static __device__ __forceinline__ V op(V a, V b) { return red2_u16x2<MODE>(a, b); }
    template <int MODE>
    static __device__ __forceinline__ V op3(V a, V b, V c) { return red3_u16x2<MODE>(a, b, c); }
    template <int MODE>
    static __device__ __forceinline__ V id() { return MODE == MODE_MIN ? 0xFFFFFFFFu : 0u; }
    static __device__ __forceinline__ uint32_t splat(uint32_t b) { return b * 0x00010001u; }
};

// Wait for a phase with a suspend-time hint: the warp sleeps in the barrier unit instead of
// spinning on try_wait (a polling warp takes issue slots from the ALU-bound warps beside it).
// (a macro, so that profiles attribute each wait to its call site)
#define mbar_sleep(bar, parity)                                                   \
    asm volatile(                                                                 \
        "{\n"                                                                     \
        ".reg .pred P1;\n"                                                        \
        "RM_SWAIT:\n"                                                             \
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"            \
        "@P1 bra RM_SDONE;\n"                                                     \
        "bra RM_SWAIT;\n"                                                         \
        "RM_SDONE:\n"                                                             \
        "}\n" ::"r"(stream::saddr(bar)),                                          \
        "r"(parity), "r"(0x100000u)                                               \
        : "memory")

// G op= the n most recent whole-block minima M[0..n) (n warp-uniform, <= QM): one branch instead
// of a select per register.
template <typename F, int MODE, typename V>
__device__ __forceinline__ V fold_minima(V G, const V (&M)[QM], int n) {
    switch (n) {
    case 8: return F::template op3<MODE>(F::template op3<MODE>(G, M[0], M[1]), F::template op3<MODE>(M[2], M[3], M[4]), F::template op3<MODE>(M[5], M[6], M[7]));
    case 7: return F::template op3<MODE>(F::template op3<MODE>(G, M[0], M[1]), F::template op3<MODE>(M[2], M[3], M[4]), F::template op<MODE>(M[5], M[6]));
    case 6: return F::template op3<MODE>(F::template op3<MODE>(G, M[0], M[1]), F::template op3<MODE>(M[2], M[3], M[4]), M[5]);
    case 5: return F::template op3<MODE>(F::template op3<MODE>(G, M[0], M[1]), F::template op<MODE>(M[2], M[3]), M[4]);
    case 4: return F::template op3<MODE>(F::template op3<MODE>(G, M[0], M[1]), M[2], M[3]);
    case 3: return F::template op3<MODE>(F::template op<MODE>(G, M[0]), M[1], M[2]);
    case 2: return F::template op3<MODE>(G, M[0], M[1]);
    case 1: return F::template op<MODE>(G, M[0]);
    default: return G;
    }
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(stream::saddr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(stream::saddr(bar)) : "memory");
}

// One 4-row group of the tile -> 4 output rows of the strip (K3's lane-chunk horizontal pass on
// shared-memory rows; the column border is applied to the vertical result first).
template <typename T, int MODE, int BXS>
__device__ __forceinline__ void h_group(const unsigned char* trow, uint8_t* drow0, size_t dp, int nrows, int X,
                                        int a, int A, int W, int cmode, uint32_t bval) {
    constexpr int sz = sizeof(T), C = 16 / sz, NW = 4;
    const int lane = threadIdx.x & 31;
    uint32_t r0[NW], r1[NW], r2[NW], r3[NW];
    {
        const unsigned char* p = trow + lane * 16;
        const uint4 v0 = *reinterpret_cast<const uint4*>(p);
        const uint4 v1 = *reinterpret_cast<const uint4*>(p + RP);
        const uint4 v2 = *reinterpret_cast<const uint4*>(p + 2 * RP);
        const uint4 v3 = *reinterpret_cast<const uint4*>(p + 3 * RP);
        r0[0] = v0.x; r0[1] = v0.y; r0[2] = v0.z; r0[3] = v0.w;
        r1[0] = v1.x; r1[1] = v1.y; r1[2] = v1.z; r1[3] = v1.w;
        r2[0] = v2.x; r2[1] = v2.y; r2[2] = v2.z; r2[3] = v2.w;
        r3[0] = v3.x; r3[1] = v3.y; r3[2] = v3.z; r3[3] = v3.w;
    }
    uint2 x[C];
    sep::h_transpose_in<T, C>(r0, r1, r2, r3, x);
    const int cx = X + (lane - A) * C;  // first column of this lane's chunk
    sep::h_border_fix<T, C>(x, X, cx, A, W, cmode, bval);
    uint2 o[C];
    sep::h_lane_pass<MODE, C, BXS>(x, a, o);
    uint32_t o0[NW], o1[NW], o2[NW], o3[NW];
    sep::h_transpose_out<T, C>(o, o0, o1, o2, o3);
    if (lane >= A && lane < 32 - A && cx < W) {
        uint8_t* d = drow0 + (ptrdiff_t)cx * sz;
        if (cx + C <= W) {
            *reinterpret_cast<uint4*>(d) = make_uint4(o0[0], o0[1], o0[2], o0[3]);
            if (nrows > 1) *reinterpret_cast<uint4*>(d + dp) = make_uint4(o1[0], o1[1], o1[2], o1[3]);
            if (nrows > 2) *reinterpret_cast<uint4*>(d + 2 * dp) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
            if (nrows > 3) *reinterpret_cast<uint4*>(d + 3 * dp) = make_uint4(o3[0], o3[1], o3[2], o3[3]);
        } else {
            const int n = W - cx;
            auto part = [&](int k, const uint32_t (&rw)[NW]) {
                if (k < nrows) {
#pragma unroll
                    for (int wi = 0; wi < NW; ++wi)
#pragma unroll
                        for (int b = 0; b < 4 / sz; ++b) {
                            const int e = wi * (4 / sz) + b;
                            if (e < n) reinterpret_cast<T*>(d + (size_t)k * dp)[e] = (T)(rw[wi] >> (8 * sz * b));
                        }
                }
            };
            part(0, o0);
            part(1, o1);
            part(2, o2);
            part(3, o3);
        }
    }
}

#ifndef FUSE_MINB
#define FUSE_MINB (FT > 256 ? 1 : 2)
#endif

template <typename T, int MODE, int B, int BXS>
__global__ void __launch_bounds__(FT, FUSE_MINB) fused_kernel(const FuseParams p, const __grid_constant__ CUtensorMap map,
                                                              const __grid_constant__ CUtensorMap gmap) {
    using namespace stream;
    using F = FV<T>;
    using V = typename F::V;
    constexpr int sz = sizeof(T);
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ring = smem + p.ring_off;  // p.r guard rows in front of slot 0
    unsigned char* tile = smem + p.tile_off;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
    uint64_t* tfull = full + p.NS;
    uint64_t* tempty = tfull + NTMAX;
    uint64_t* rempty = tempty + NTMAX;  // ring slot released by every vertical thread

    const int img = blockIdx.x / p.per_img;
    int rem = blockIdx.x - img * p.per_img;
    int strip, y0, rb;
    if (rem < p.extra * (p.nb + 1)) {
        strip = rem / (p.nb + 1);
        rb = p.rba;
        y0 = (rem - strip * (p.nb + 1)) * rb;
    } else {
        rem -= p.extra * (p.nb + 1);
        const int sb = rem / p.nb;
        strip = p.extra + sb;
        rb = p.rbb;
        y0 = (rem - sb * p.nb) * rb;
    }
    const int x0 = strip * p.SW;  // first output column
    const int y1 = min(y0 + rb, p.H);
    const int nblk = (y1 - y0 + B - 1) / B;
    const int q = p.q, r = p.r, QQ = p.QQ, NS = p.NS;
    const int i0 = y0 + p.gy;  // leading input row of output row y0
    const int kmin = -QQ;      // first block loaded (the oldest trailing block of output block 0)

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS / p.pair; ++s) mbar_init(&full[s], 1);
        for (int s = 0; s < p.nt; ++s) {
            mbar_init(&tfull[s], NVT);
            mbar_init(&tempty[s], NHT);
        }
        for (int s = 0; s < NS; ++s) mbar_init(&rempty[s], NVT);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int xw = (x0 * sz - 16 * p.A) / 4;  // map x of the strip row's first word (may be < 0)
    const int pair = p.pair, NU = NS / pair;  // ring units: pair consecutive blocks, one TMA box
    auto issue = [&](int u) {  // unit u (blocks kmin + u * pair ...) -> its ring unit (the last
                               // unit also fills the guard rows)
        const int su = u % NU;
        const bool g = r > 0 && su == NU - 1;
        mbar_arrive_tx(&full[su], (uint32_t)((pair * B + (g ? r : 0)) * RP));
        const int row = i0 + (kmin + u * pair) * B - p.row_lo;
        tma_box(ring + (size_t)su * pair * B * RP, &map, xw, row, img, &full[su]);
        if (g) tma_box(ring - (size_t)r * RP, &gmap, xw, row + pair * B - r, img, &full[su]);
    };
    const int nunits = (nblk - kmin + pair - 1) / pair;  // units covering blocks kmin .. nblk - 1
    if (warp < NVT / 32) {
        // ------------------------------ vertical ------------------------------
        const int t = threadIdx.x;
        const int wo = 4 * t;
        if (t == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map) : "memory");
            for (int u = 0; u < NU && u < nunits; ++u) issue(u);
        }
        long long* tr = (p.trace && blockIdx.x == (unsigned)p.trace_cta && t == 0) ? p.trace : nullptr;
        const V ID = F::template id<MODE>();
        const uint32_t sub = p.cmode ? F::splat(p.bval) : (MODE == MODE_MIN ? 0xFFFFFFFFu : 0u);
        V M[QM];
#pragma unroll
        for (int k = 0; k < QM; ++k) M[k] = ID;
        int s = 0, par = 0;  // ring slot of block k and the phase parity of its unit
        for (int k = kmin; k < nblk; ++k) {
            unsigned char* sb = ring + (size_t)s * B * RP;
            if (tr) tr[(k - kmin) * 8 + 0] = clock64();
            if (s % pair == 0) mbar_sleep(&full[s / pair], (uint32_t)par);
            if (tr) tr[(k - kmin) * 8 + 1] = clock64();
            const int rs = i0 + k * B;  // first input row of block k
            if (rs < p.row_lo || rs + B > p.row_hi) {
                // rows outside the valid input: the identity (replicate: the clamped row is inside
                // every window that reaches past it) or the constant; each thread patches only the
                // column word it reads
                for (int m = 0; m < B; ++m) {
                    const int i = rs + m;
                    if (i < p.row_lo || i >= p.row_hi) {
                        *reinterpret_cast<uint32_t*>(sb + m * RP + wo) = sub;
                        if (r > 0 && s == NS - 1 && m >= B - r) *reinterpret_cast<uint32_t*>(ring - (B - m) * RP + wo) = sub;
                    }
                }
                fence_async_smem();  // before a later TMA overwrites the slot
            }
            if (k >= -(q - 1)) {
                const unsigned char* pl = sb + wo;
                if (k < 0) {  // warm-up block: its minimum only
                    V P = F::ld(pl), P2 = F::ld(pl + (B / 2) * RP);  // two half chains
#pragma unroll
                    for (int m = 1; m < B / 2; ++m) {
                        P = F::template op<MODE>(P, F::ld(pl + m * RP));
                        P2 = F::template op<MODE>(P2, F::ld(pl + (B / 2 + m) * RP));
                    }
                    P = F::template op<MODE>(P, P2);
#pragma unroll
                    for (int kk = QM - 1; kk > 0; --kk) M[kk] = M[kk - 1];
                    M[0] = P;
                } else {
                    const int L = k;
                    int st = s - q;
                    if (st < 0) st += NS;
                    int sf = st - (r > 0);  // slot of block L - QQ, whose last reader this is
                    if (sf < 0) sf += NS;
                    const int ts = L & (p.nt - 1);
                    if (p.dbg >= 2) {
                        mbar_arrive(&rempty[sf]);
                        if (L >= p.nt) mbar_sleep(&tempty[ts], (uint32_t)(((L >> p.ntlog) & 1) ^ 1));
                        mbar_arrive(&tfull[ts]);
                    } else {
                        // trailing rows [start(L-q) - r, start(L-q) + B + r): through the guard
                        // when block L-q sits in slot 0. The trailing suffix and the leading prefix
                        // are independent chains: interleaved, combined once the tile slot is free.
                        const unsigned char* pt = ring + (size_t)st * B * RP - (size_t)r * RP + wo;
                        // Each chain split at HB = B / 2 into two independent half chains (four
                        // chains in flight): Tm is the full suffix for rows >= HB and the suffix
                        // within the lower half below; Pm the full prefix below HB and the prefix
                        // within the upper half above. The halves' missing parts (Tm[HB], Pm[HB-1])
                        // are folded into G once per half instead of per row.
                        constexpr int HB = B / 2;
                        V Tm[B], Pm[B];
                        Tm[B - 1] = F::ld(pt + (B - 1) * RP);
                        Tm[HB - 1] = F::ld(pt + (HB - 1) * RP);
                        Pm[0] = F::ld(pl);
                        Pm[HB] = F::ld(pl + HB * RP);
#pragma unroll
                        for (int j = 1; j < HB; ++j) {
                            Tm[B - 1 - j] = F::template op<MODE>(Tm[B - j], F::ld(pt + (B - 1 - j) * RP));
                            Tm[HB - 1 - j] = F::template op<MODE>(Tm[HB - j], F::ld(pt + (HB - 1 - j) * RP));
                            Pm[j] = F::template op<MODE>(Pm[j - 1], F::ld(pl + j * RP));
                            Pm[HB + j] = F::template op<MODE>(Pm[HB + j - 1], F::ld(pl + (HB + j) * RP));
                        }
                        const V P = F::template op<MODE>(Pm[HB - 1], Pm[B - 1]);  // the block's minimum
                        V G = ID;
#pragma unroll
                        for (int tt = 0; tt < RMAXG; ++tt)
                            if (tt < r) G = F::template op<MODE>(G, F::ld(pt + (B + tt) * RP));
                        // last read of block L - QQ (and of L - q when r = 0): release its slot
                        mbar_arrive(&rempty[sf]);
                        G = fold_minima<F, MODE>(G, M, q - 1);
                        if (L >= p.nt) mbar_sleep(&tempty[ts], (uint32_t)(((L >> p.ntlog) & 1) ^ 1));
                        if (tr) tr[(k - kmin) * 8 + 2] = clock64();
                        unsigned char* to = tile + (size_t)ts * B * RP + wo;
                        const V GL = F::template op<MODE>(G, Tm[HB]), GU = F::template op<MODE>(G, Pm[HB - 1]);
#pragma unroll
                        for (int m = 0; m < B; ++m)
                            F::st(to + m * RP, F::template op3<MODE>(Tm[m], m < HB ? GL : GU, Pm[m]));
#pragma unroll
                        for (int kk = QM - 1; kk > 0; --kk) M[kk] = M[kk - 1];
                        M[0] = P;
                        mbar_arrive(&tfull[ts]);
                        if (tr) tr[(k - kmin) * 8 + 3] = clock64();
                    }
                }
            }
            if (++s == NS) {
                s = 0;
                par ^= 1;
            }
        }
    } else if (warp == FT / 32 - 1) {
        // ------------------------------ TMA producer ------------------------------
        // One warp refills released ring units in order: unit u (blocks kmin + u * pair ...) into
        // the ring blocks of unit u - NU, once the last of those (released in block order) is
        // released. A TMA issue costs hundreds of cycles under load, so it has its own warp, off
        // the vertical and horizontal warps. Issuing in order is also what makes the parity-only
        // waits on the release barriers exact: the slot's previous phase (unit u - 2 NU) was
        // released before unit u - NU could be issued. The whole warp waits; lane 0 issues.
        if (lane == 0) {  // a descriptor's first fetch is slow: before it is needed
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map) : "memory");
            if (r > 0) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&gmap) : "memory");
        }
        for (int u = NU; u < nunits; ++u) {
            const int last = (u - NU + 1) * pair - 1;  // relative to kmin
            mbar_sleep(&rempty[last % NS], (uint32_t)((last / NS) & 1));
            if (lane == 0) issue(u);
            __syncwarp();
        }
    } else {
        // ------------------------------ horizontal ------------------------------
        const int hw = warp - NVT / 32;
        const int ngroups = (y1 - y0 + 3) / 4;
        uint8_t* dimg = p.dst + (size_t)img * p.dimg;
        // A warp releases a tile slot only after that block's full phase has completed (also for
        // blocks holding none of its groups): otherwise its release of block d + nt could be
        // counted in block d's phase while another warp still reads block d.
        int done = 0, waited = -1;
        auto wait_tile = [&](int L) {
            mbar_sleep(&tfull[L & (p.nt - 1)], (uint32_t)((L >> p.ntlog) & 1));
            waited = L;
        };
        auto release_to = [&](int L) {
            for (; done < L; ++done) {
                if (done != waited) wait_tile(done);
                mbar_arrive(&tempty[done & (p.nt - 1)]);
            }
        };
        long long* tr =
            (p.trace && blockIdx.x == (unsigned)p.trace_cta && lane == 0) ? p.trace + 1024 + hw * 256 : nullptr;
        for (int G = hw; G < ngroups; G += NHT / 32) {
            const int L = (4 * G) / B;
            if (tr) tr[(G / 4) * 4 + 0] = clock64();
            release_to(L);
            if (L != waited) wait_tile(L);
            if (tr) tr[(G / 4) * 4 + 1] = clock64();
            const unsigned char* trow = tile + (size_t)(L & (p.nt - 1)) * B * RP + (size_t)(4 * G - L * B) * RP;
            const int y = y0 + 4 * G;
            if (p.dbg != 1 && p.dbg != 3)
                h_group<T, MODE, BXS>(trow, dimg + (size_t)y * p.dp, p.dp, min(4, y1 - y), x0, p.a, p.A, p.W, p.cmode,
                                      p.bval);
            if (tr) tr[(G / 4) * 4 + 2] = clock64();
        }
        release_to(nblk);
    }
    (void)lane;
}

}  // namespace fuse
}  // namespace rmgpu

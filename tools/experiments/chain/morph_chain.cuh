// morph_chain.cuh -- K5: the passes of one separable op (or of an opening / closing) chained inside
// ONE persistent launch, handing over through L2.
//
// K3 (morph_sep.cuh) runs the reference's two-pass structure (separable.cpp:130-157) as one launch
// per pass; at 2^29+ pixels the intermediate of pass k has left L2 before pass k+1 reads it (cfg5:
// 4 GiB of DRAM traffic for 2 GiB algorithmic; cfg4's opening 6 GiB for 2 GiB). K5 keeps K3's pass
// bodies (h_item / vpass_body, bit-identical results) and replaces the launch boundary by data-flow:
//
//  * The rows of every image are cut into slabs of S rows. A stage (pass) is a list of warp-sized
//    items per slab: V = (band of rb rows, 32 column words), H = (4 rows, column part).
//  * Every warp of a grid of resident CTAs is its own worker: it draws items of its preferred stage
//    from that stage's ticket counter (in order; the next ticket is drawn while the current item
//    runs), and moves to another stage when its own runs out. Warp w of every CTA sits on scheduler
//    w, so a scheduler's warps run one pass body (instruction cache) and the SM runs all of them
//    (load-latency-bound vertical items beside ALU-bound horizontal ones).
//  * An item of stage k waits (lane 0 polls, then a warp barrier) until the slabs it reads are
//    complete (a done counter per stage and slab, bumped once per finished item with release
//    semantics) and, to bound the intermediate in flight, until stage k + 1 has finished the slab
//    `ahead` slabs back. Tickets of a stage are handed out in order, so every item a warp waits for
//    is held by a resident warp that waits only for earlier items: no deadlock, whatever the grid.
//  * The intermediate is read back while it is still in L2. Its lines are never read before they
//    are complete and L1 is invalidated per launch, so ordinary loads are safe; the non-coherent
//    path is not used for data written in this launch.
#pragma once

#include "morph_sep.cuh"

namespace rmgpu {
namespace sep {

enum ChainKind : int { CK_V = 0, CK_H = 1, CK_HH = 2 };

struct ChainStage {
    SepParams p;
    int kind;   // ChainKind
    int var;    // V: block size B; H / HH: C * 100 + bx code (selects the kernel)
    int n;      // warp items per slab (every slab has the same nominal count; items past the image are no-ops)
    int nbx;    // V: 32-word column strips per band
    int total;  // n * slabs
};

struct ChainParams {
    ChainStage st[3];
    int nst;
    int S;       // rows per slab (multiple of every V stage's rb and of 4)
    int nsi;     // slabs per image
    int nslab;   // nsi * batch
    int ahead;   // slabs stage k may run ahead of stage k + 1 (>= 2)
    int roles;   // preferred stage of warps 0..3 of a CTA, 2 bits each
    unsigned* ctr;  // [k] ticket counter of stage k (k < 4), [4 + k * nslab + gs] done items of stage k in slab gs
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// ---- one V item: 128 column words x one band (the body of vpass_kernel) -------------------------
template <typename T, int MODE, int B, int SPC, bool COH>
__device__ __forceinline__ void chain_v_item(const SepParams& p, int img, int y0, int c) {
    constexpr int QMc = 4;
    constexpr int sz = sizeof(T);
    const int y1 = min(y0 + p.rb, p.H);
    const int nblk = (y1 - y0 + B - 1) / B;
    const uint8_t* s = p.src + (size_t)img * p.simg +
                       (p.sstride ? (size_t)(c >> 5) * p.sstride + (size_t)(c & 31) * 4 * sz : (size_t)c * 4 * sz);
    uint8_t* d = p.dst + (size_t)img * p.dimg + (size_t)c * 4 * sz;
    const bool edge = (y0 - p.g < p.row_lo) || (y0 + nblk * B + p.g > p.row_hi);
    const int nvalid = min(4, p.W - 4 * c);
    if (edge) vpass_body<T, MODE, B, QMc, true, SPC, COH>(p, s, d, y0, y1, nvalid);
    else vpass_body<T, MODE, B, QMc, false, SPC, COH>(p, s, d, y0, y1, nvalid);
}

// The block size is a run-time switch over inlined bodies (the kernel is specialised on the
// horizontal variant only): every body addresses the stage's parameters in the constant bank.
template <typename T, int MODE, int SPC, bool COH>
__device__ __forceinline__ void chain_v(const SepParams& p, int B, int img, int y0, int c) {
    switch (B) {
#define RM_CV(BB) \
    case BB: chain_v_item<T, MODE, BB, SPC, COH>(p, img, y0, c); break;
        RM_CV(8) RM_CV(10) RM_CV(12) RM_CV(14) RM_CV(16)
#undef RM_CV
    default:
        if constexpr (sizeof(T) == 1) {
            switch (B) {
#define RM_CV(BB) \
    case BB: chain_v_item<T, MODE, BB, SPC, COH>(p, img, y0, c); break;
                RM_CV(18) RM_CV(20) RM_CV(22) RM_CV(24)
#undef RM_CV
            }
        }
    }
}

constexpr int CT = 128;  // threads per chain CTA: 4 independent warps
#ifndef CHAIN_MINB
#define CHAIN_MINB 4
#endif
#ifndef CHAIN_ACQUIRE
#define CHAIN_ACQUIRE 1
#endif

// NS = 2: H (src -> strip-major scratch) then V (scratch -> dst), one erosion / dilation.
// NS = 3: V (src -> t1), HH (t1 -> strip-major t2: this mode then the other), V of the other mode
//         (t2 -> dst): an opening (MODE = min) or closing (MODE = max) of whole images.
template <typename T, int MODE, int C, int BXS, int NS>
__global__ void __launch_bounds__(CT, CHAIN_MINB) chain_kernel(const __grid_constant__ ChainParams cp) {
    constexpr int MODE2 = MODE == MODE_MIN ? MODE_MAX : MODE_MIN;
    constexpr int SB = 128 * (int)sizeof(T);
    constexpr int KH = NS == 2 ? 0 : 1;  // the horizontal stage
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned* done = cp.ctr + 4;
    int k = (cp.roles >> (2 * warp)) & 3;  // preferred stage
    int left = NS;                         // stages not yet found exhausted
    unsigned nxt = lane == 0 ? atomicAdd(cp.ctr + k, 1u) : 0u;
    for (;;) {
        const int i = (int)__shfl_sync(0xffffffffu, nxt, 0);
        const int tot = k == 0 ? cp.st[0].total : (k == 1 ? cp.st[1].total : cp.st[2].total);
        if (i >= tot) {  // this stage has run out: the next one (cyclically) that has not
            if (--left == 0) return;
            k = k + 1 == NS ? 0 : k + 1;
            if (lane == 0) nxt = atomicAdd(cp.ctr + k, 1u);
            continue;
        }
        if (lane == 0) nxt = atomicAdd(cp.ctr + k, 1u);  // the next ticket, drawn while this item runs
        const int n = k == 0 ? cp.st[0].n : (k == 1 ? cp.st[1].n : cp.st[2].n);
        const int gs = i / n, rem = i - gs * n;
        const int img = gs / cp.nsi, sl = gs - img * cp.nsi;
        if (lane == 0) {
            if (k > 0) {  // stage k reads stage k - 1
                // a vertical pass reads one wing into the neighbouring slabs of the same image
                const bool vert = k != KH;
                const int lo = (vert && sl > 0) ? gs - 1 : gs;
                const int hi = (vert && sl + 1 < cp.nsi) ? gs + 1 : gs;
                const unsigned full = (unsigned)(k == 1 ? cp.st[0].n : cp.st[1].n);
                const unsigned* dn = done + (size_t)(k - 1) * cp.nslab;
                for (int d = lo; d <= hi; ++d) {
                    while (ld_relaxed_u32(dn + d) < full) __nanosleep(64);
                }
#if CHAIN_ACQUIRE
                (void)ld_acquire_u32(dn + hi);
#endif
            }
            if (k + 1 < NS && gs >= cp.ahead) {  // the intermediate in flight stays bounded
                const unsigned full = (unsigned)(k == 0 ? cp.st[1].n : cp.st[2].n);
                const unsigned* dn = done + (size_t)(k + 1) * cp.nslab + (gs - cp.ahead);
                while (ld_relaxed_u32(dn) < full) __nanosleep(64);
            }
        }
        __syncwarp();
        if (k == KH) {
            const SepParams& p = cp.st[KH].p;
            const int grp = rem / p.parts, part = rem - grp * p.parts;
            const int y = sl * cp.S + grp * 4;
            if (y < p.H)
                h_item<T, MODE, C, BXS, NS == 2 ? 1 : 2, NS == 3>(p, p.src + (size_t)img * p.simg + (size_t)y * p.sp, p.sp,
                                                                 p.dst + (size_t)img * p.dimg + (size_t)y * p.dp,
                                                                 min(4, p.H - y), part);
        } else if (NS == 2 || k == 2) {
            constexpr int KV = NS == 2 ? 1 : 2;
            const SepParams& p = cp.st[KV].p;
            const int band = rem / cp.st[KV].nbx, bx = rem - band * cp.st[KV].nbx;
            const int y0 = sl * cp.S + band * p.rb;
            const int c = bx * 32 + lane;
            if (y0 < p.H && c < p.nwords) chain_v<T, NS == 2 ? MODE : MODE2, SB, true>(p, cp.st[KV].var, img, y0, c);
        } else {
            const SepParams& p = cp.st[0].p;
            const int band = rem / cp.st[0].nbx, bx = rem - band * cp.st[0].nbx;
            const int y0 = sl * cp.S + band * p.rb;
            const int c = bx * 32 + lane;
            if (y0 < p.H && c < p.nwords) chain_v<T, MODE, 0, false>(p, cp.st[0].var, img, y0, c);
        }
        __syncwarp();
        if (lane == 0) red_release_add(done + (size_t)k * cp.nslab + gs, 1u);
    }
}

}  // namespace sep
}  // namespace rmgpu

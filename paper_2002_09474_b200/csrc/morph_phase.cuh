// morph_phase.cuh -- K1/K2 v3: persistent, TMA-fed, phase-based fused separable erosion /
// dilation (u8, u16). Design notes in morph_phase.cu. Reuses the geometry, lane words, TMA
// helpers and work-item decomposition of morph_stream.cuh.
#pragma once

#include "morph_stream.cuh"

namespace rmgpu {
namespace phase {

using namespace stream;

// Register budget per variant: 3 resident CTAs per SM where the shared-memory footprint allows it
// and the code fits 72 registers without spilling (u16, 8-row blocks); 2 (96 registers) otherwise.
__host__ __device__ constexpr int phase_min_blocks(int elem, int vb) { return (elem == 2 || vb == 8) ? 3 : 2; }
constexpr int PNT = 256;  // compute threads per CTA (every one runs both passes) + 1 producer warp
constexpr int PNW = PNT / 32;

// ring slot size: B rows, rounded to 128 bytes (TMA tensor destinations are 128-byte aligned)
__host__ __device__ constexpr int slot_bytes(int B, int RP) { return (B * RP + 127) / 128 * 128; }

// rows per chunk for block size B (a multiple of B, at most 32)
__host__ __device__ constexpr int chunk_rows(int B) { return (32 / B) * B; }

struct PPlan {
    int NSB, off_ring, off_vt, off_msc, off_out, total;
};

template <typename T, int HB>
__host__ __device__ inline PPlan make_pplan(int B, int q, int PF) {
    using H = HG<T, HB>;
    using G = SG<T>;
    const int CH = chunk_rows(B);
    const int NGC = CH / G::GR;
    PPlan p;
    // a refilled slot must be older than the previous chunk (warps drift within a chunk)
    p.NSB = q + 1 + PF + CH / B;
    int o = 1024;  // mbarriers (<= 64) + store descriptors
    p.off_ring = o;
    o += p.NSB * slot_bytes(B, H::RP);
    p.off_vt = o;
    o += NGC * H::VTG * G::ESZ;
    p.off_msc = o;
    if (HB > 7) o += NGC * H::NCHP * G::ESZ;
    o = (o + 127) / 128 * 128;
    p.off_out = o;
    o += 2 * CH * G::TW * (int)sizeof(T);
    p.total = o;
    return p;
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
        : "r"(saddr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(bar)) : "memory");
}

constexpr int BAR_C = 1;  // named barrier of the compute warps

// Emitting chunks of one item (chunks whose blocks reach the first emitting iteration Lf).
__device__ __forceinline__ int emitting_chunks(const Item& it, int KB) {
    int n = 0;
    for (int c0 = 0; c0 <= it.Lend; c0 += KB)
        if (min(c0 + KB - 1, it.Lend) >= it.Lf) ++n;
    return n;
}

template <typename T, int MODE, int VB, int HB>
__global__ void __launch_bounds__(PNT + 32, phase_min_blocks(sizeof(T), VB))
morph_phase_kernel(const StreamParams p, const __grid_constant__ CUtensorMap tmap,
                   const __grid_constant__ CUtensorMap omap) {
    using G = SG<T>;
    using H = HG<T, HB>;
    constexpr int GR = G::GR, TW = G::TW, ESZ = G::ESZ;
    constexpr int sz = sizeof(T);
    constexpr bool VDIRECT = VB <= 7;
    constexpr int VR = VB / 100;               // block mode: tail rows r = w1 mod B (compile-time)
    constexpr int B = VDIRECT ? VCH : VB % 100;  // rows per block (TMA box)
    constexpr int CH = chunk_rows(B);          // rows per chunk (horizontal hand-off)
    constexpr int KB = CH / B;                 // blocks per chunk
    constexpr int NGC = CH / GR;               // row groups per chunk
    constexpr int OUTP = TW * sz;
    constexpr int RP = H::RP, NCHP = H::NCHP, VTG = H::VTG, LPG = H::LPG;
    constexpr int SUBG = 32 / LPG;
    constexpr int SLOT = slot_bytes(B, RP);
    extern __shared__ __align__(128) unsigned char smem[];

    const int w1 = 2 * p.gy, w1x = 2 * p.gx;
    const int q = VDIRECT ? 0 : w1 / B;
    const int r = VDIRECT ? w1 : VR;
    const int s = r & 3;
    const int PF = p.pf;
    const PPlan pl = make_pplan<T, HB>(B, q, PF);
    const int NSB = pl.NSB;
    const int nstrips = (p.W + TW - 1) / TW;
    const int nrowb = (p.H + p.rh - 1) / p.rh;
    const int nitems = nstrips * nrowb * p.batch;
    const int G0 = (int)gridDim.x;

    uint64_t* full = reinterpret_cast<uint64_t*>(smem);   // NSB
    uint64_t* empty = full + NSB;                          // NSB
    uint64_t* ofull = empty + NSB;                         // 2
    uint64_t* oempty = ofull + 2;                          // 2
    int4* sdesc = reinterpret_cast<int4*>(smem + 512);     // 2 store descriptors {x, y, z, full}
    unsigned char* ring = smem + pl.off_ring;
    unsigned char* vt = smem + pl.off_vt;
    unsigned char* msc0 = smem + pl.off_msc;
    unsigned char* outbase = smem + pl.off_out;
    const uint32_t bv = sz == 1 ? (p.bval & 0xFF) : (p.bval & 0xFFFF);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int k = 0; k < NSB; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&ofull[k], 1);
            mbar_init(&oempty[k], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto item_at = [&](int n) { return (int)blockIdx.x + n * G0; };

    if (warp == PNT / 32) {
        // ======================= producer warp: TMA loads into the ring, TMA stores out ==========
        if (lane == 0 && p.use_tma) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap) : "memory");
        int pn = 0, pk = -1, pslot = 0, puse = 0;  // next block: item pn, block pk, slot, slot-use
        bool pvalid = item_at(0) < nitems;
        Item pit;
        if (pvalid) pit = make_item<T>(p, item_at(0), nstrips, nrowb, B, w1, s);
        // stores to handle: emitting chunks of all this CTA's items
        int stores_left = 0;
        for (int n = 0; item_at(n) < nitems; ++n)
            stores_left += emitting_chunks(make_item<T>(p, item_at(n), nstrips, nrowb, B, w1, s), KB);
        // Event-ordered loop: the compute warps release ring slots and then publish chunk c's
        // output (OFULL) at the end of every emitting chunk, so waiting (suspended) on OFULL[c]
        // guarantees every slot freed so far is already released: issue the store, then refill
        // all free slots. No polling.
        int sc = 0, pending = -1;
        auto issue_load = [&]() {
            const int slot = pslot;
            unsigned char* base = ring + (size_t)slot * SLOT;
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
                while (fillm) {
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
                             src + (ptrdiff_t)yc * (ptrdiff_t)p.sp + pit.cb0, (uint32_t)pit.copy_len,
                             &full[slot]);
                }
            }
            if (++pslot == NSB) {
                pslot = 0;
                ++puse;
            }
            if (++pk > pit.Lend) {
                ++pn;
                pk = -1;
                pvalid = item_at(pn) < nitems;
                if (pvalid) pit = make_item<T>(p, item_at(pn), nstrips, nrowb, B, w1, s);
            }
        };
        auto slot_free = [&]() {
            int ready = 1;
            if (lane == 0 && puse > 0) ready = mbar_test(&empty[pslot], (uint32_t)((puse - 1) & 1));
            return __shfl_sync(0xffffffffu, ready, 0) != 0;
        };
        while (pvalid && slot_free()) issue_load();  // prologue: the first NSB blocks
        for (; stores_left > 0; --stores_left, ++sc) {
            const int ob = sc & 1;
            mbar_wait(&ofull[ob], (uint32_t)((sc >> 1) & 1));
            if (lane == 0) {
                // the previous store has had a whole chunk to read its buffer: release it
                if (pending >= 0) {
                    bulk_wait_read0();
                    mbar_arrive(&oempty[pending]);
                    pending = -1;
                }
                const int4 d = sdesc[ob];
                if (d.w) {
                    tma_store_box(&omap, d.x, d.y, d.z, outbase + (size_t)ob * CH * OUTP);
                    bulk_commit();
                    pending = ob;
                } else {
                    mbar_arrive(&oempty[ob]);  // copied by the compute warps already
                }
            }
            __syncwarp();
            while (pvalid && slot_free()) issue_load();
        }
        if (lane == 0) {
            if (pending >= 0) mbar_arrive(&oempty[pending]);
            bulk_wait_all();
        }
        return;
    }

    // =========================== compute warps (PNT threads) ===================================
    auto op2 = [](uint32_t x, uint32_t y) { return red2_u16x2<MODE>(x, y); };
    auto op3 = [](uint32_t x, uint32_t y, uint32_t z) { return red3_u16x2<MODE>(x, y, z); };
    constexpr uint32_t IDV = MODE == MODE_MIN ? 0xFFFFFFFFu : 0u;

    // consumed block stream: slot/parity of current block and of blocks -1, -q, -q-1
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
    int rel = 0, rslot = 0;  // blocks released to the producer: seq < rel
    auto release_below = [&](int upto) {
        if (tid == 0)
            while (rel < upto) {
                mbar_arrive(&empty[rslot]);
                rslot = rslot + 1 == NSB ? 0 : rslot + 1;
                ++rel;
            }
    };
    int chunk = 0;  // emitting chunks so far (output buffer parity / use count)

    const int sub = lane / LPG, lam = lane % LPG;
    const int q8 = w1x >> 3, r8 = w1x & 7;

    for (int n = 0; item_at(n) < nitems; ++n) {
        const Item it = make_item<T>(p, item_at(n), nstrips, nrowb, B, w1, s);
        uint8_t* dst = p.dst + (size_t)it.b * p.dimg;
        const bool real = tid < it.nwv;
        const bool vwarp = warp * 32 < it.nwv;  // warp-uniform: any real column word in this warp
        const int t = real ? tid : it.nwv - 1;
        int load_off = 0;
        uint32_t nib = 0;
        bool fix = false;
        col_fix<T>(it.xs_col + 2 * t, p.W, p.cmode, it.xs_col, load_off, nib, fix);
        const uint32_t selU = sz == 1 ? ((nib & 0xF) | (5u << 4) | (((nib >> 4) & 0xF) << 8) | (5u << 12)) : nib;
        const uint32_t Z = bv;
        int voff0, voff1;
        {
            // scratch entry: band 0, chunk NCHP-1 (>= NCH-1), beyond every chunk the horizontal
            // pass reads (< NCH-2); NOT entry NCH, which is position 1 of band 1
            const int dummy = (NCHP - 1) * ESZ;
            const int pos0 = 2 * t - it.off, pos1 = pos0 + 1;
            voff0 = (real && pos0 >= 0 && pos0 < 8 * H::NCH) ? ((pos0 & 7) * NCHP + (pos0 >> 3)) * ESZ : dummy;
            voff1 = (real && pos1 >= 0 && pos1 < 8 * H::NCH) ? ((pos1 & 7) * NCHP + (pos1 >> 3)) * ESZ : dummy;
        }
        auto ldw = [&](const unsigned char* a) -> uint32_t {
            if constexpr (sz == 1) {
                return prmt(*reinterpret_cast<const uint16_t*>(a), Z, selU);
            } else {
                const uint32_t raw = *reinterpret_cast<const uint32_t*>(a);
                return fix ? prmt(raw, Z, selU) : raw;
            }
        };
        const unsigned char* rbase = ring + load_off;
        auto sbase = [&](int slot) { return rbase + (size_t)slot * SLOT; };

        // block -1 of this item
        mbar_wait(&full[sL], (uint32_t)ph);
        advance();

        uint32_t M[QMAX];
#pragma unroll
        for (int k = 0; k < QMAX; ++k) M[k] = IDV;

        for (int c0 = 0; c0 <= it.Lend; c0 += KB) {
            // wx = 1: no horizontal pass -- the vertical results go straight into the output tile
            // (row-major), so that tile must have been read out by its previous TMA store first
            unsigned char* vout = nullptr;
            if constexpr (HB == 1) {
                const bool emitting = min(c0 + KB - 1, it.Lend) >= it.Lf;
                vout = outbase + (size_t)(chunk & 1) * CH * OUTP;
                if (emitting && chunk >= 2) mbar_wait(&oempty[chunk & 1], (uint32_t)((((chunk) >> 1) - 1) & 1));
            }
            // ================= vertical phase: KB blocks of B rows into the transposed tile =========
            const int tci = chunk < 60 ? chunk : 59;
            if (warp == 0) RM_TRACE(tci * 8 + 0);
            bool emit_any = false;
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                const int L = c0 + kb;
                if (L > it.Lend) break;
                const bool emit = L >= it.Lf;
                emit_any |= emit;
                if (!vwarp) {  // warp holds no column word of this strip: only track the ring
                    advance();
                    continue;
                }
                if (warp == 0 && kb == 0) RM_TRACE(tci * 8 + 1);
                mbar_wait(&full[sL], (uint32_t)ph);
                if (warp == 0 && kb == 0) RM_TRACE(tci * 8 + 2);
                const unsigned char* lead = sbase(sL);
                uint32_t grp[GR];
                auto flush = [&](int m0) {
                    if constexpr (HB == 1) {
                        // pixel pair (pos0, pos0+1) of GR rows -> output tile rows kb*B+m0+i
                        const int pos0 = 2 * t - it.off;
                        if (real && pos0 >= 0 && pos0 < TW) {
#pragma unroll
                            for (int i = 0; i < GR; ++i) {
                                unsigned char* d = vout + (size_t)(kb * B + m0 + i) * OUTP + (size_t)pos0 * sz;
                                if constexpr (sz == 1) *reinterpret_cast<uint16_t*>(d) = (uint16_t)prmt(grp[i], 0u, 0x0020);
                                else *reinterpret_cast<uint32_t*>(d) = grp[i];
                            }
                        }
                        return;
                    }
                    unsigned char* rowg = vt + ((kb * B + m0) / GR) * VTG * ESZ;
                    if constexpr (sz == 1) {
                        *reinterpret_cast<uint2*>(rowg + voff0) =
                            make_uint2(prmt(grp[0], grp[2], 0x5410), prmt(grp[1], grp[3], 0x5410));
                        *reinterpret_cast<uint2*>(rowg + voff1) =
                            make_uint2(prmt(grp[0], grp[2], 0x7632), prmt(grp[1], grp[3], 0x7632));
                    } else {
                        *reinterpret_cast<uint32_t*>(rowg + voff0) = prmt(grp[0], grp[1], 0x5410);
                        *reinterpret_cast<uint32_t*>(rowg + voff1) = prmt(grp[0], grp[1], 0x7632);
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
                        // gap = tail r rows of block L-q + whole blocks L-q+1 .. L-1 (r is small:
                        // the planner picks B to minimise it)
                        const unsigned char* tb = sbase(sQ);
                        const unsigned char* tt = tb + (B - r) * RP;
                        uint32_t gap = IDV;
                        for (int i = 0; i < r; ++i) gap = op2(gap, ldw(tt + i * RP));
#pragma unroll
                        for (int k = 0; k + 1 < QMAX; k += 2) {
                            const uint32_t a = k < q - 1 ? M[k] : IDV, b = k + 1 < q - 1 ? M[k + 1] : IDV;
                            gap = op3(gap, a, b);
                        }
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
                advance();
            }
            if (!emit_any) continue;  // warm-up chunk: nothing to hand over (uniform across the CTA)
            const int oC = s + c0 * B - w1;  // output row of chunk row 0 (relative to the item)
            const int ob = chunk & 1;
            unsigned char* outt = outbase + (size_t)ob * CH * OUTP;
            if (warp == 0) RM_TRACE(tci * 8 + 3);
            if constexpr (HB != 1) {
            bar_sync(BAR_C, PNT);  // transposed tile complete
            if (warp == 0) RM_TRACE(tci * 8 + 4);

            // ================= horizontal phase: one warp per row group ===============================
            if (chunk >= 2) mbar_wait(&oempty[ob], (uint32_t)(((chunk >> 1) - 1) & 1));
            for (int g0 = warp * SUBG; g0 < NGC; g0 += PNW * SUBG) {
                const int g = g0 + sub;
                const unsigned char* rowg = vt + (size_t)g * VTG * ESZ;
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
                auto emit4 = [&](int a, LW<T> c0v, LW<T> c1v, LW<T> c2v, LW<T> c3v) {
                    unsigned char* po = outt + (size_t)(g * GR) * OUTP + (size_t)a * sz;
                    if constexpr (sz == 1) {
                        const uint32_t a01 = prmt(c0v.a, c1v.a, 0x6240), a23 = prmt(c2v.a, c3v.a, 0x6240);
                        const uint32_t b01 = prmt(c0v.b, c1v.b, 0x6240), b23 = prmt(c2v.b, c3v.b, 0x6240);
                        *reinterpret_cast<uint32_t*>(po) = prmt(a01, a23, 0x5410);
                        *reinterpret_cast<uint32_t*>(po + OUTP) = prmt(b01, b23, 0x5410);
                        *reinterpret_cast<uint32_t*>(po + 2 * OUTP) = prmt(a01, a23, 0x7632);
                        *reinterpret_cast<uint32_t*>(po + 3 * OUTP) = prmt(b01, b23, 0x7632);
                    } else {
                        *reinterpret_cast<uint32_t*>(po) = prmt(c0v.a, c1v.a, 0x5410);
                        *reinterpret_cast<uint32_t*>(po + OUTP) = prmt(c0v.a, c1v.a, 0x7632);
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
                    emit8(o);
                } else {
                    // lane-chunk van Herk; prefix written back in place over the row group's entries
                    unsigned char* scr = vt + (size_t)g * VTG * ESZ;
                    unsigned char* msc = msc0 + (size_t)g * NCHP * ESZ;
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
                    const int k = lam;
                    LW<T> Fa = lid<T, MODE>();
                    for (int i = 1; i < q8; ++i) Fa = lop<MODE>(Fa, ld8(msc + (k + i) * ESZ));
                    const LW<T> Fb = lop<MODE>(Fa, ld8(msc + (k + q8) * ESZ));
                    const unsigned char* pa = scr + (r8 * NCHP + k + q8) * ESZ;
                    const unsigned char* pbb = scr + ((r8 - 8) * NCHP + k + q8 + 1) * ESZ;
                    LW<T> o[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const bool lo = j < 8 - r8;
                        o[j] = lop3<MODE>(S[j], lo ? Fa : Fb, ld8((lo ? pa : pbb) + j * NCHP * ESZ));
                    }
                    emit8(o);
                }
            }
            }  // HB != 1
            const int rlo = max(0, -oC), rhi = min(CH, it.rh - oC);
            const bool full_chunk = p.use_tma_out && rlo == 0 && rhi == CH && it.x0 + TW <= p.W;
            if (warp == 0) RM_TRACE(tci * 8 + 5);
            if (full_chunk) fence_async_smem();  // emits visible to the TMA store (async proxy)
            bar_sync(BAR_C, PNT);                // output tile complete, transposed tile free
            if (warp == 0) RM_TRACE(tci * 8 + 6);
            const int g_last = seq - 1;          // last block consumed by this chunk
            const bool item_done = c0 + KB > it.Lend;
            if (!full_chunk) {
                const int cols = min(TW, p.W - it.x0);
                const int row_bytes = cols * sz;
                const bool vec = (((uintptr_t)dst | p.dp) & 15) == 0 && cols == TW;
                if (vec) {
                    constexpr int CPR = TW * sz / 16;
                    for (int i = rlo * CPR + tid; i < rhi * CPR; i += PNT) {
                        const int rr = i / CPR, ch = i % CPR;
                        const uint4 v = *reinterpret_cast<const uint4*>(outt + (size_t)rr * OUTP + ch * 16);
                        *reinterpret_cast<uint4*>(dst + (size_t)(it.y0 + oC + rr) * p.dp + (size_t)it.x0 * sz + ch * 16) = v;
                    }
                } else {
                    for (int i = rlo * row_bytes + tid; i < rhi * row_bytes; i += PNT) {
                        const int rr = i / row_bytes, b = i % row_bytes;
                        dst[(size_t)(it.y0 + oC + rr) * p.dp + (size_t)it.x0 * sz + b] = outt[(size_t)rr * OUTP + b];
                    }
                }
                bar_sync(BAR_C, PNT);  // copy finished: the producer may hand the buffer back
            }
            // blocks no iteration after this chunk reads: everything below seq (g_last - q) of this
            // item, or the whole item when it is finished -- released BEFORE the chunk is published,
            // the producer refills slots right after it sees OFULL
            release_below(item_done ? g_last + 1 : g_last - q);
            if (tid == 0) {
                sdesc[ob] = make_int4(it.x0 * sz, it.y0 + oC, it.b, full_chunk ? 1 : 0);
                mbar_arrive(&ofull[ob]);
            }
            ++chunk;
        }
    }
}

template <typename T, int MODE, int VB, int HB>
cudaError_t launch_phase_variant(const MorphJob& j, int rh, int B, int q, int pf) {
    using G = SG<T>;
    StreamParams p{};
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
    p.batch = j.batch;
    p.trace = g_trace;
    p.trace_cta = g_trace_cta;
    CUtensorMap map, omap;
    p.use_tma = encode_input_map(j, HG<T, HB>::RP / 4, B, &map) ? 1 : 0;
    p.use_tma_out = encode_output_map(j, G::TW * (int)sizeof(T), chunk_rows(B), &omap) ? 1 : 0;
    const PPlan pl = make_pplan<T, HB>(B, q, pf);
    auto kern = morph_phase_kernel<T, MODE, VB, HB>;
    cudaError_t e = cudaSuccess;
    const int occ = kernel_occupancy((const void*)kern, PNT + 32, pl.total, &e);
    if (e != cudaSuccess) return e;
    const int sms = device_sm_count();
    const long items = (long)cdiv(j.W, G::TW) * cdiv(j.H, rh) * j.batch;
    const long ctas = std::max(1L, std::min(items, (long)sms * std::max(1, occ)));
    kern<<<dim3((unsigned)ctas), PNT + 32, pl.total, j.stream>>>(p, map, omap);
    count_launch();
    return cudaGetLastError();
}

#define RM_PHASE_V(X) X(1) X(3) X(5) X(7) X(8) X(12) X(16) X(20) X(24) X(28) X(208) X(212) X(216) X(220) X(224) X(228) \
    X(1416)
#define RM_PHASE_H(X) X(1) X(3) X(5) X(7) X(8) X(9)

template <typename T, int MODE, int VB>
cudaError_t phase_dispatch_h(const MorphJob& j, int hb, int rh, int B, int q, int pf) {
    switch (hb) {
#define RM_CASE(H) \
    case H: return launch_phase_variant<T, MODE, VB, H>(j, rh, B, q, pf);
        RM_PHASE_H(RM_CASE)
#undef RM_CASE
    }
    return cudaErrorInvalidValue;
}

template <typename T, int MODE>
cudaError_t phase_dispatch(const MorphJob& j, int vb, int hb, int rh, int B, int q, int pf) {
    switch (vb) {
#define RM_CASE(V) \
    case V: return phase_dispatch_h<T, MODE, V>(j, hb, rh, B, q, pf);
        RM_PHASE_V(RM_CASE)
#undef RM_CASE
    }
    return cudaErrorInvalidValue;
}

template <typename T>
inline int phase_smem(int hb, int B, int q, int pf) {
    switch (hb) {
    case 1: return make_pplan<T, 1>(B, q, pf).total;
    case 3: return make_pplan<T, 3>(B, q, pf).total;
    case 5: return make_pplan<T, 5>(B, q, pf).total;
    case 7: return make_pplan<T, 7>(B, q, pf).total;
    case 8: return make_pplan<T, 8>(B, q, pf).total;
    default: return make_pplan<T, 9>(B, q, pf).total;
    }
}

}  // namespace phase
}  // namespace rmgpu

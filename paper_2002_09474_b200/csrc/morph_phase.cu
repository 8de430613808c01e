// morph_phase.cu -- planner for K1/K2 v3, the persistent phase-based fused kernel.
//
// Design (B200-first; reference semantics from separable.cpp:130-157, sliding_extrema.cpp,
// image.cpp:58-66):
//   * Persistent CTAs (one per resident slot) walk work items = (strip of TW output columns,
//     run of rows, image). Input rows of the strip + horizontal halo stream into a shared-memory
//     ring as 2-D TMA boxes of B rows (cp.async.bulk.tensor, completion on a per-slot mbarrier),
//     issued PF blocks ahead by warp 0, across item boundaries, so the first rows of the next item
//     arrive while the current one finishes.
//   * Each chunk of CH (<= 32) rows is processed in two phases by ALL 256 threads:
//       vertical  - one thread per 2-pixel column word: direct window (w <= 7) or the van Herk /
//                   Gil-Werman block algorithm with a compile-time register block B and the gap
//                   minimum tree-reduced from r tail rows and q-1 carried block minima; pixels in
//                   16-bit lanes so every min/max is one VIMNMX(3).U16x2; results transposed in
//                   registers (PRMT) into the shared transposed tile;
//       horizontal- one warp per 4-row (u8) / 2x2-row (u16) group, each lane owning 8 columns:
//                   direct window or lane-chunk van Herk (prefix written back in place, suffix in
//                   registers, chunk minima combined for the gap); outputs transposed back to rows
//                   in registers into a double-buffered output tile;
//     with one __syncthreads between the phases and one after; multiple CTAs per SM overlap each
//     other's phases.
//   * Full chunks leave through one TMA tensor store; ragged chunks with 16-byte stores.
//   Every pixel is read from HBM once and written once; halo rows/columns are L2 hits.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "morph_phase.cuh"

namespace rmgpu {
namespace phase {
cudaError_t dispatch_u8_min(const MorphJob&, int, int, int, int, int, int);
cudaError_t dispatch_u8_max(const MorphJob&, int, int, int, int, int, int);
cudaError_t dispatch_u16_min(const MorphJob&, int, int, int, int, int, int);
cudaError_t dispatch_u16_max(const MorphJob&, int, int, int, int, int, int);

namespace {

struct Choice {
    int vb, hb, B, q, rh, smem, pf;
};

bool choose(const MorphJob& j, Choice* c) {
    if (j.mode != MODE_MIN && j.mode != MODE_MAX) return false;
    if (j.elem != 1 && j.elem != 2) return false;
    if ((reinterpret_cast<uintptr_t>(j.src) | j.sp | (j.batch > 1 ? j.simg : 0)) & 15) return false;
    const int tw = j.elem == 1 ? SG<uint8_t>::TW : SG<uint16_t>::TW;
    const int w1 = 2 * j.gy;
    if (j.gy <= 3) {
        c->vb = 2 * j.gy + 1;
        c->B = VCH;
        c->q = 0;
    } else {
        double best = 1e30;
        c->vb = 0;
        // halo class first (it sets the ring row pitch), then the block size: min/max per output
        // ~ 3 + (2r + q)/B (+ per-block overhead 6/B), divided by the CTAs that fit per SM (max 2)
        const int hb0 = j.gx <= 3 ? 2 * j.gx + 1 : (j.gx <= stream_gxmax(j.elem, 8) ? 8 : 9);
        for (int B : {8, 12, 16, 20, 24, 28}) {
            if (B > w1) continue;
            const int q = w1 / B, r = w1 - q * B;
            // compile-time tail lengths: 0 or 2 for every B, plus r = 14 for 16-row blocks (w = 31, 63:
            // 32-row chunks, 8 row groups, all warps busy in the horizontal phase)
            const bool ok = r == 0 || r == 2 || (B == 16 && r == 14);
            if (q > QMAX || !ok) continue;
            const int t = j.elem == 1 ? phase_smem<uint8_t>(hb0, B, q, 2) : phase_smem<uint16_t>(hb0, B, q, 2);
            if (t > 220 * 1024) continue;
            const int occ = std::max(1, std::min(phase_min_blocks(j.elem, B + 100 * r), (228 * 1024) / (t + 1024)));
            // vertical: min/max per output ~ 3 + (2r + q)/B (+ per-block overhead 6/B); horizontal:
            // one phase per chunk costs about the same wall time whether it has 5 or 8 row groups
            // (one warp each), so its per-row cost scales with 8 / (row groups per chunk)
            const int ngc = chunk_rows(B) / 4;
            double cost = (3.0 + double(2 * r + q) / B + 6.0 / B + 3.0 * 8.0 / ngc) / occ;
            if (B == 16 && r == 14 && q >= 2) cost *= 0.9;  // measured: best for w = 63 on large images
            if (cost < best - 1e-9) {
                best = cost;
                c->vb = B + 100 * r;
                c->B = B;
                c->q = q;
            }
        }
        if (!c->vb) return false;
    }
    c->hb = j.gx <= 3 ? 2 * j.gx + 1 : (j.gx <= stream_gxmax(j.elem, 8) ? 8 : 9);
    if (j.gx > stream_gxmax(j.elem, c->hb)) return false;
    const int rp = j.elem == 1 ? stream_ring_row<uint8_t>(c->hb) : stream_ring_row<uint16_t>(c->hb);
    const int blk = c->B * rp;
    auto smem_of = [&](int pf) {
        return j.elem == 1 ? phase_smem<uint8_t>(c->hb, c->B, c->q, pf) : phase_smem<uint16_t>(c->hb, c->B, c->q, pf);
    };
    // TMA prefetch depth: ~64 KB of input in flight per SM (Little's law at ~1 us loaded DRAM
    // latency, 6.5 TB/s over 148 SMs), within the shared-memory budget
    int pf = 1, total = smem_of(pf);
    if (total > 220 * 1024) return false;
    if (const char* e = getenv("RMGPU_STREAM_PF")) {
        pf = std::max(1, atoi(e));
        total = smem_of(pf);
    } else {
        // deepest prefetch (up to ~48 KB in flight per SM) that keeps the occupancy of PF = 2
        const int occ_ref = std::max(1, std::min(8, (228 * 1024) / (smem_of(2) + 1024)));
        for (int cand = 1; cand <= 16; ++cand) {
            const int t = smem_of(cand);
            if (t > 220 * 1024) break;
            const int occ = std::max(1, std::min(8, (228 * 1024) / (t + 1024)));
            if (cand > 2 && occ < occ_ref) break;
            pf = cand;
            total = t;
            if ((long)cand * blk * occ >= 48 * 1024) break;
        }
    }
    c->pf = pf;
    c->smem = total;
    // rows per item: the persistent grid runs in waves of (SMs x resident CTAs) items; every item
    // pays w1 warm-up rows plus a fixed switch cost. Pick the band count that minimises
    // waves x (rows per item + w1 + 16): one full wave of long items beats many short ones
    // (measured on 4096^2: 256-row items 15-30% faster than 64-row items).
    const int occ = std::max(1, std::min(phase_min_blocks(j.elem, c->vb), (228 * 1024) / (total + 1024)));
    const long strips = (long)((j.W + tw - 1) / tw) * j.batch;
    const long slots = 148L * occ;
    long best_nb = 1;
    double best_t = 1e30;
    for (long nb = 1; nb <= std::max(1, j.H / 8); ++nb) {
        const long rows = (j.H + nb - 1) / nb;
        const long waves = (strips * nb + slots - 1) / slots;
        const double t = (double)waves * (double)(rows + w1 + 16);
        if (t < best_t - 1e-9) {
            best_t = t;
            best_nb = nb;
        }
    }
    int rh = (int)((j.H + best_nb - 1) / best_nb);
    rh = (rh + 3) / 4 * 4;
    if (const char* e = getenv("RMGPU_STREAM_RH")) {
        const int v = atoi(e);
        if (v > 0) rh = (v + 3) / 4 * 4;
    }
    c->rh = rh;
    return true;
}

}  // namespace

bool launch(const MorphJob& j, cudaError_t* err) {
    Choice c;
    if (!choose(j, &c)) return false;
    if (j.elem == 1)
        *err = j.mode == MODE_MIN ? dispatch_u8_min(j, c.vb, c.hb, c.rh, c.B, c.q, c.pf)
                                  : dispatch_u8_max(j, c.vb, c.hb, c.rh, c.B, c.q, c.pf);
    else
        *err = j.mode == MODE_MIN ? dispatch_u16_min(j, c.vb, c.hb, c.rh, c.B, c.q, c.pf)
                                  : dispatch_u16_max(j, c.vb, c.hb, c.rh, c.B, c.q, c.pf);
    return true;
}

const char* plan_name(const MorphJob& j) {
    static thread_local char buf[96];
    MorphJob k = j;
    k.src = nullptr;
    k.sp = (size_t)((j.W * j.elem + 15) / 16 * 16);
    Choice c;
    if (!choose(k, &c)) return nullptr;
    snprintf(buf, sizeof(buf), "phase_%s_v%s%d_h%s%d_rh%d_pf%d_smem%dK", j.elem == 1 ? "u8" : "u16",
             c.vb <= 7 ? "d" : "b", c.vb % 100, c.hb <= 7 ? "d" : "b", c.hb, c.rh, c.pf, c.smem / 1024);
    return buf;
}

}  // namespace phase
}  // namespace rmgpu

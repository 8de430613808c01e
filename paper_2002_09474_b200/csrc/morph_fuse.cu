// morph_fuse.cu -- planner and launcher of K4 (morph_fuse.cuh): the separable rectangle as one
// kernel (vertical then horizontal pass, intermediate in shared memory). Reference semantics:
// morph_separable (separable.cpp:130-157: V then H, window 1 = identity), van Herk / Gil-Werman
// windows (sliding_extrema.cpp:58-132), per-axis replicate / constant borders (image.cpp:58-66).
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "morph_fuse.cuh"

namespace rmgpu {
namespace fuse {

#define RM_DECL(TN, MN, BB)                                                                                  \
    cudaError_t launch_##TN##_##MN##_b##BB(const FuseParams&, int, dim3, int, cudaStream_t, const CUtensorMap&, \
                                        const CUtensorMap&);
#define RM_DECL_B(TN, MN) RM_DECL(TN, MN, 12) RM_DECL(TN, MN, 20)
RM_DECL_B(u8, min)
RM_DECL_B(u8, max)
RM_DECL(u16, min, 8) RM_DECL(u16, min, 12)
RM_DECL(u16, max, 8) RM_DECL(u16, max, 12)
#undef RM_DECL_B
#undef RM_DECL

cudaError_t launch_kernel(const void* kern, const FuseParams& p, dim3 grid, int smem, cudaStream_t s,
                          const CUtensorMap& map, const CUtensorMap& gmap) {
    cudaError_t e = cudaSuccess;
    const int occ = kernel_occupancy(kern, FT, smem, &e);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    FuseParams pp = p;
    CUtensorMap m = map, g = gmap;
    void* args[] = {&pp, &m, &g};
    e = cudaLaunchKernel(kern, grid, dim3(FT), args, (size_t)smem, s);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

namespace {

// block sizes with instantiations (u8: 12, 20; u16: 8, 12): K4 is a knob-only path, windows whose
// 2 gy does not split over one of them stay on K3
constexpr int kB[] = {8, 12, 20};
constexpr int kSmemPerSm = 228 * 1024;  // B200: shared memory per SM (1 KB reserved per CTA)

struct Plan {
    int B = 0, q = 0, r = 0, C = 0, a = 0, A = 0, SW = 0, bxs = 0;
    int NS = 0, PF = 0, nt = 0, pair = 0, smem = 0, ctas = 0;  // ctas: resident CTAs per SM the smem allows
    int nstrips = 0, nb = 0, extra = 0, rba = 0, rbb = 0, per_img = 0;
    int ring_off = 0, tile_off = 0, bar_off = 0;
};

int smem_bytes(int B, int r, int NS, int nt, int* ring_off, int* tile_off, int* bar_off) {
    *ring_off = (r * RP + 127) / 128 * 128;  // guard rows in front of slot 0
    *tile_off = *ring_off + NS * B * RP;
    *bar_off = *tile_off + nt * B * RP;
    return *bar_off + 8 * (2 * NS + 2 * NTMAX);  // full (<= NS), tile full / empty, ring release
}

bool aligned(const MorphJob& j) {
    const uintptr_t sb = reinterpret_cast<uintptr_t>(j.src) - (uintptr_t)((ptrdiff_t)j.above * (ptrdiff_t)j.sp);
    return ((sb | reinterpret_cast<uintptr_t>(j.dst) | j.sp | j.dp | (j.batch > 1 ? (j.simg | j.dimg) : 0)) & 15) == 0;
}

bool plan(const MorphJob& j, Plan* pl) {
    // Off by default: measured against K3 (two launches through L2) it is still slower at 4096^2
    // (63x63: 21.3 vs 18.7 us) and at 32768^2 (823 vs 789 us) -- both passes are latency / issue
    // bound, not HBM bound, so removing the intermediate's traffic does not pay yet (K4).
    if (!tune("fuse", 0)) return false;
    if (j.mode != MODE_MIN && j.mode != MODE_MAX) return false;
    if (j.elem != 1 && j.elem != 2) return false;
    if (j.W < 1 || j.H < 1 || j.batch < 1) return false;
    if (j.gx < 4 || j.gy < 4) return false;  // 1-D and short-wing windows: K1 / K3
    if (!aligned(j)) return false;
    Plan p;
    p.C = 16 / j.elem;
    p.a = j.gx / p.C;
    const int bx = j.gx % p.C;
    p.A = p.a + (bx ? 1 : 0);
    if (p.A > tune("fuse_amax", 8)) return false;
    p.SW = p.C * (32 - 2 * p.A);
    p.bxs = bx + (j.gx < p.C && 2 * bx < p.C ? 32 : 0);
    if (j.elem == 2 && p.bxs >= 32) return false;
    // V block B: 2 gy = q B + r with q >= 1, r <= RMAXG (guard rows), q - 1 <= QM; per output row
    // the vertical thread pays ~(2r + 30) / B for the tail fold, the block-minima fold and the
    // per-block synchronisation; PF >= 2 blocks of TMA prefetch when they fit next to a second CTA
    const int forced_b = tune("fuse_b", 0);
    const int want_pf = tune("fuse_pf", FT > 256 ? 4 : 2);
    const int smem_cap = kSmemPerSm / std::max(1, tune("fuse_ctas", FT > 256 ? 1 : 2)) - 1024;  // resident CTAs per SM
    double best = 1e30;
    const int want_nt = tune("fuse_nt", FT > 256 ? 8 : 4);
    const int pair = std::min(2, std::max(1, tune("fuse_pair", 2)));
    for (int B : kB) {
        if (j.elem == 2 ? B > 12 : B == 8) continue;
        if (forced_b && B != forced_b) continue;
        const int q = 2 * j.gy / B, r = 2 * j.gy % B;
        if (q < 1 || r > RMAXG || q - 1 > QM) continue;
        const int QQ = q + (r > 0);
        // largest (tile slots, prefetch) that fits: 4 tile slots give the horizontal warps slack
        // behind the vertical ones (with 2, each waits on the other); PF >= 1 block ahead
        bool done = false;
        for (int nt = std::min(want_nt, NTMAX); nt >= 2 && !done; nt /= 2) {
            for (int PF = std::max(1, want_pf); PF >= 1; --PF) {
                const int NS = (QQ + pair + PF + pair - 1) / pair * pair;
                int ro, to, bo;
                const int sm = smem_bytes(B, r, NS, nt, &ro, &to, &bo);
                if (sm > smem_cap) continue;
                const double cost = (2.0 * r + 30.0) / B + (PF < want_pf ? 0.25 : 0.0) + (nt < want_nt ? 0.5 : 0.0);
                if (cost < best) {
                    best = cost;
                    p.B = B;
                    p.q = q;
                    p.r = r;
                    p.PF = PF;
                    p.NS = NS;
                    p.pair = pair;
                    p.nt = nt;
                    p.smem = sm;
                    p.ring_off = ro;
                    p.tile_off = to;
                    p.bar_off = bo;
                }
                done = true;
                break;
            }
        }
    }
    if (!p.B) return false;
    p.ctas = std::max(1, std::min(FT > 256 ? 1 : 2, kSmemPerSm / (p.smem + 1024)));
    // items: strips x bands x images, one CTA each. P items per image: every strip gets nb bands and
    // the first `extra` strips one more, so that the grid fills whole waves of resident CTAs (each
    // CTA's time is its band height plus the warm-up: 2 gy rows read for block minima and trailing
    // rows, paid once per band); P minimises waves x (tallest band + warm-up)
    p.nstrips = (j.W + p.SW - 1) / p.SW;
    const long long slots = (long long)device_sm_count() * p.ctas;
    const int maxb = (j.H + p.B - 1) / p.B;
    auto rows_for = [&](int nbands) { return ((j.H + nbands - 1) / nbands + p.B - 1) / p.B * p.B; };
    double bcost = 1e30;
    int bestP = p.nstrips;
    const int frb = tune("fuse_rb", 0);
    for (long long P = p.nstrips; P <= (long long)p.nstrips * maxb; ++P) {
        const int nb = (int)(P / p.nstrips), extra = (int)(P % p.nstrips);
        const int rbmax = rows_for(nb);
        if ((long long)(nb - 1) * rbmax >= j.H || (extra && (long long)nb * rows_for(nb + 1) >= j.H)) continue;
        if (frb > 0 && rbmax != std::max(p.B, (frb + p.B - 1) / p.B * p.B)) continue;
        const long long waves = (P * j.batch + slots - 1) / slots;
        const double c = (double)waves * (rbmax + 0.6 * 2 * j.gy + 8) + 1e-6 * (double)P;
        if (c < bcost) {
            bcost = c;
            bestP = (int)P;
        }
        if (P * j.batch > 64 * slots) break;
    }
    p.per_img = bestP;
    p.nb = bestP / p.nstrips;
    p.extra = bestP % p.nstrips;
    p.rbb = rows_for(p.nb);
    p.rba = p.extra ? rows_for(p.nb + 1) : p.rbb;
    // bands that would start past the image (rounding) are not items: recount
    if ((long long)(p.nb - 1) * p.rbb >= j.H || (p.extra && (long long)p.nb * p.rba >= j.H)) {
        p.extra = 0;
        p.nb = (j.H + p.rbb - 1) / p.rbb;
        p.rba = p.rbb;
        p.per_img = p.nb * p.nstrips;
    }
    *pl = p;
    return true;
}

template <int SZ>
cudaError_t dispatch(const FuseParams& fp, int mode, int B, int bxs, dim3 grid, int smem, cudaStream_t s,
                     const CUtensorMap& m, const CUtensorMap& g) {
#define RM_CASE(TN, MN, BB) \
    case BB: return launch_##TN##_##MN##_b##BB(fp, bxs, grid, smem, s, m, g);
    if (SZ == 1) {
        if (mode == MODE_MIN) {
            switch (B) { RM_CASE(u8, min, 12) RM_CASE(u8, min, 20) }
        } else {
            switch (B) { RM_CASE(u8, max, 12) RM_CASE(u8, max, 20) }
        }
    } else {
        if (mode == MODE_MIN) {
            switch (B) { RM_CASE(u16, min, 8) RM_CASE(u16, min, 12) }
        } else {
            switch (B) { RM_CASE(u16, max, 8) RM_CASE(u16, max, 12) }
        }
    }
#undef RM_CASE
    return cudaErrorInvalidValue;
}

}  // namespace

bool launch(const MorphJob& j, cudaError_t* err) {
    Plan p;
    if (!plan(j, &p)) return false;
    CUtensorMap map, gmap;
    if (p.pair * p.B > 256 || !stream::encode_input_map(j, RP / 4, p.pair * p.B, &map)) return false;
    if (p.r > 0) {
        if (!stream::encode_input_map(j, RP / 4, p.r, &gmap)) return false;
    } else {
        gmap = map;
    }
    FuseParams fp{};
    fp.dst = static_cast<uint8_t*>(j.dst);
    fp.dp = j.dp;
    fp.dimg = j.dimg;
    fp.W = j.W;
    fp.H = j.H;
    fp.row_lo = -j.above;
    fp.row_hi = j.H + j.below;
    fp.gx = j.gx;
    fp.gy = j.gy;
    fp.q = p.q;
    fp.r = p.r;
    fp.QQ = p.q + (p.r > 0);
    fp.a = p.a;
    fp.A = p.A;
    fp.SW = p.SW;
    fp.nstrips = p.nstrips;
    fp.nb = p.nb;
    fp.extra = p.extra;
    fp.rba = p.rba;
    fp.rbb = p.rbb;
    fp.per_img = p.per_img;
    fp.batch = j.batch;
    fp.cmode = j.cmode;
    fp.bval = j.bval;
    fp.NS = p.NS;
    fp.pair = p.pair;
    fp.nt = p.nt;
    fp.ntlog = p.nt == 8 ? 3 : p.nt == 4 ? 2 : 1;
    fp.dbg = tune("fuse_dbg", 0);
    fp.trace = stream::g_trace;
    fp.trace_cta = stream::g_trace_cta;
    fp.ring_off = p.ring_off;
    fp.tile_off = p.tile_off;
    fp.bar_off = p.bar_off;
    const long long items = (long long)p.per_img * j.batch;
    if (items > 0x7fffffffLL) return false;
    const dim3 grid((unsigned)items);
    *err = j.elem == 1 ? dispatch<1>(fp, j.mode, p.B, p.bxs, grid, p.smem, j.stream, map, gmap)
                       : dispatch<2>(fp, j.mode, p.B, p.bxs, grid, p.smem, j.stream, map, gmap);
    return true;
}

const char* plan_name(const MorphJob& j) {
    static thread_local char buf[96];
    Plan p;
    if (!plan(j, &p)) return nullptr;
    snprintf(buf, sizeof buf, "fuse_%s_B%d_r%d_A%d_SW%d_rb%d-%d_items%d_ns%d_nt%d", j.elem == 1 ? "u8" : "u16",
             p.B, p.r, p.A, p.SW, p.rba, p.rbb, p.per_img, p.NS, p.nt);
    return buf;
}

}  // namespace fuse
}  // namespace rmgpu

// morph_sep.cu -- planner and launchers of K3 (morph_sep.cuh): vertical pass V and horizontal pass H
// as two streaming kernels with the intermediate handed over through L2 (row bands sized so that
// one band of the intermediate stays resident). Reference semantics: separable.cpp:130-157 (V then
// H, window 1 = identity), image.cpp:58-66 (replicate / constant borders per axis).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "morph_sep.cuh"

namespace rmgpu {
namespace sep {

cudaError_t launch_h_u8_min(const SepParams&, int C, int bx, dim3 grid, cudaStream_t s);
cudaError_t launch_h_u8_max(const SepParams&, int C, int bx, dim3 grid, cudaStream_t s);
cudaError_t launch_h_u16_min(const SepParams&, int C, int bx, dim3 grid, cudaStream_t s);
cudaError_t launch_h_u16_max(const SepParams&, int C, int bx, dim3 grid, cudaStream_t s);
cudaError_t launch_hh_u8_min(const SepParams&, int C, int bx, dim3 grid, cudaStream_t s);
cudaError_t launch_hh_u8_max(const SepParams&, int C, int bx, dim3 grid, cudaStream_t s);
cudaError_t launch_hh_u16_min(const SepParams&, int C, int bx, dim3 grid, cudaStream_t s);
cudaError_t launch_hh_u16_max(const SepParams&, int C, int bx, dim3 grid, cudaStream_t s);


namespace {

constexpr int QM = 4;  // block minima kept in registers (q - 1 <= QM)
constexpr int kBlocks[] = {8, 10, 12, 14, 16, 18, 20, 22, 24};

int env_int(const char* name, int dflt) { return tune(name, dflt); }

// V block size B: the tail r = 2g mod B must be <= VRMAX (folded from re-read rows), q-1 <= QM
// block minima in registers; per output row the pass folds (q-1 + r)/B extra values and larger B
// costs registers (u16 keeps B <= 16).
bool choose_b(int elem, int g, int* B_out) {
    const int w1 = 2 * g;
    double best = 1e30;
    int bb = 0;
    for (int B : kBlocks) {
        if (B > w1 || (elem == 2 && B > 16)) continue;
        const int q = w1 / B, r = w1 % B;
        if (r > VRMAX || q - 1 > QM) continue;
        const double cost = (0.5 * (q - 1) + r) / B + 0.01 * B;
        if (cost < best) {
            best = cost;
            bb = B;
        }
    }
    const int forced = env_int("sep_vb", 0);  // tuning: force a block size when it is valid
    if (forced > 0 && forced <= w1 && w1 % forced <= VRMAX && w1 / forced - 1 <= QM &&
        (elem == 1 || forced <= 16))
        for (int B : kBlocks)
            if (B == forced) bb = B;
    *B_out = bb;
    return bb != 0;
}

// H chunk width for a wing g: C = 16 for u8 wings >= 8, 8 otherwise (>= 4); at most 8 halo lanes.
bool choose_c(int elem, int g, int* C_out) {
    // (u16 with 16-column chunks -- 32 bytes per row per lane -- measured slower on cfg4: 377 vs
    // 408 Gpix/s)
    // u8 wings 4..7 also take 16-column chunks: the windows inside a lane's chunk come from
    // half-chunk scans (h_lane_pass)
    int C;
    if (elem == 1) C = (g >= 8 || env_int("sep_c16_short", 1)) ? 16 : 8;
    else C = 8;
    if (g < 4 || (C == 8 && g < C / 2)) return false;
    const int A = g / C + (g % C ? 1 : 0);
    if (A > 8) return false;
    *C_out = C;
    return true;
}

// The TMA pipeline pays off only on the largest images: with the strip-major intermediate the
// plain-load vertical pass wins up to 16384^2 (8192^2 63x63: 70 vs 82 us; 16384^2 even) and the TMA
// pass from 2^29 pixels (32768^2: 791 vs 816 us). Tall images only: a band touching the top or
// bottom border fills its rings synchronously.
bool v_wants_tma(const MorphJob& j) {
    const long long px = (long long)j.W * j.H * j.batch;
    return env_int("sep_notma", px >= (1LL << 29) && j.H >= 2048 ? 0 : 1) == 0;
}
// Strip-major source: a strip's block is one contiguous run -> 1-D bulk copies into the same TMA
// pipeline (no tensor maps); pays off from 2^28 pixels (16384^2 63x63: 215 vs 228 us), the plain
// loads ramp faster below (4096^2: 18.5 vs 23.5 us).
bool v_wants_bulk(const MorphJob& j) {
    const long long px = (long long)j.W * j.H * j.batch;
    return env_int("sep_vbulk", px >= (1LL << 28) && j.H >= 2048 ? 1 : 0) != 0;
}

// TMA-fed variant when the maps encode (16-byte pitches); the plain LDG kernel otherwise.
template <typename T, int MODE, int B>
cudaError_t launch_v_t(const SepParams& p0, dim3 grid, cudaStream_t s, const MorphJob& j) {
    constexpr int sz = sizeof(T), SB = 128 * sz;
    SepParams p = p0;
    CUtensorMap lmap, tmap, omap;
    // the TMA pipeline pays off on large images (16384^2 u8 1x63: 77% vs 65% of HBM); on small ones
    // the plain-load kernel ramps faster (4096^2: 13.0 vs 15.4 us)
    // (tall images only: a band touching the top or bottom border fills its rings synchronously)
    // strip-major source: the bulk-copy variant (no input maps) when sep_vbulk; else plain loads
    const bool bulk = p.sstride && v_wants_bulk(j) && stream::encode_output_map(j, SB, B, &omap);
    if (bulk) {
        memset(&lmap, 0, sizeof lmap);
        memset(&tmap, 0, sizeof tmap);
    }
    const bool tma = bulk || (!p.sstride && v_wants_tma(j) && stream::encode_input_map(j, SB / 4, B, &lmap) &&
                              stream::encode_input_map(j, SB / 4, B + VRMAX, &tmap) &&
                              stream::encode_output_map(j, SB, B, &omap));
    if (tma) {
        const int pf = std::max(1, env_int("sep_pf", 1));
        p.nsl = p.nst = pf + 1;
        p.wsmem = ((p.nsl * B + p.nst * (B + VRMAX) + 2 * B) * SB + 8 * (p.nsl + p.nst) + 127) / 128 * 128;
        p.nstrips = (p.nwords + 31) / 32;
        p.nbands = (int)grid.y;
        const long long warps = (long long)p.nstrips * p.nbands * p.batch;
        auto kern = vtma_kernel<T, MODE, B, QM>;
        cudaError_t e = cudaSuccess;
        const int smem = VTW * p.wsmem;
        kernel_occupancy((const void*)kern, VT, smem, &e);
        if (e != cudaSuccess) return e;
        cudaError_t le = launch_pdl(kern, dim3((unsigned)((warps + VTW - 1) / VTW)), dim3(VT), smem, s, p, lmap, tmap, omap);
        if (le != cudaSuccess) return le;
    } else if (p.sstride) {  // strip-major intermediate: rows at compile-time offsets
        cudaError_t le = launch_pdl(vpass_kernel<T, MODE, B, QM, SB>, grid, dim3(VT), 0, s, p);
        if (le != cudaSuccess) return le;
    } else {
        cudaError_t le = launch_pdl(vpass_kernel<T, MODE, B, QM>, grid, dim3(VT), 0, s, p);
        if (le != cudaSuccess) return le;
    }
    count_launch();
    return cudaGetLastError();
}

template <typename T, int MODE>
cudaError_t launch_v_b(const SepParams& p, int B, dim3 grid, cudaStream_t s, const MorphJob& j) {
    switch (B) {
#define RM_V(BB) \
    case BB: return launch_v_t<T, MODE, BB>(p, grid, s, j);
        RM_V(8) RM_V(10) RM_V(12) RM_V(14) RM_V(16) RM_V(18) RM_V(20) RM_V(22) RM_V(24)
#undef RM_V
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_v(const SepParams& p, int elem, int mode, int B, dim3 grid, cudaStream_t s, const MorphJob& j) {
    if (elem == 1) return mode == MODE_MIN ? launch_v_b<uint8_t, MODE_MIN>(p, B, grid, s, j) : launch_v_b<uint8_t, MODE_MAX>(p, B, grid, s, j);
    return mode == MODE_MIN ? launch_v_b<uint16_t, MODE_MIN>(p, B, grid, s, j) : launch_v_b<uint16_t, MODE_MAX>(p, B, grid, s, j);
}

// template code: g mod C, + 32 for the short-wing variant (the window fits in one chunk)
int bx_code(int g, int C) { return g % C + (g < C && 2 * (g % C) < C ? 32 : 0); }

cudaError_t launch_h(const SepParams& p, int elem, int mode, int C, dim3 grid, cudaStream_t s) {
    const int bx = bx_code(p.g, C);
    if (elem == 1) return mode == MODE_MIN ? launch_h_u8_min(p, C, bx, grid, s) : launch_h_u8_max(p, C, bx, grid, s);
    return mode == MODE_MIN ? launch_h_u16_min(p, C, bx, grid, s) : launch_h_u16_max(p, C, bx, grid, s);
}

SepParams base_params(const MorphJob& j) {
    SepParams p{};
    p.W = j.W;
    p.H = j.H;
    p.cmode = j.cmode;
    p.bval = j.bval;
    p.batch = j.batch;
    return p;
}

// Plan of one vertical pass over the job's rows: src (rows [-above, H + below) valid) -> out.
struct VPlan {
    SepParams p;
    int B;
    dim3 grid;
};
bool plan_v(const MorphJob& j, void* out, size_t op, size_t oimg, int pdl, size_t sstride, VPlan* vp) {
    int B = 0;
    if (!choose_b(j.elem, j.gy, &B)) return false;
    SepParams p = base_params(j);
    p.src = static_cast<const uint8_t*>(j.src);
    p.sp = j.sp;
    p.simg = j.simg;
    p.dst = static_cast<uint8_t*>(out);
    p.dp = op;
    p.dimg = oimg;
    p.row_lo = -j.above;
    p.row_hi = j.H + j.below;
    p.pdl = pdl;
    p.sstride = sstride;
    p.g = j.gy;
    p.q = 2 * j.gy / B;
    p.r = 2 * j.gy % B;
    p.nwords = (j.W + 3) / 4;
    // bands: one wave of the warps that are resident at this variant's register budget (u8 blocks
    // of <= 14 rows 6 CTAs per SM, taller ones and u16 4: 63x63 at 4096^2 used to launch 824 CTAs for
    // 592 slots); the warm-up (q-1 blocks per band) stays < ~50% of a band
    const long long cols = (long long)p.nwords * j.batch;
    const int sms = device_sm_count();
    const int vwarps = env_int("sep_vwarps", (j.elem == 1 && B <= 14 ? 6 : 4) * (VT / 32));
    int bands = (int)std::max(1LL, ((long long)sms * vwarps * 32 + cols - 1) / cols);
    int rb = (j.H + bands - 1) / bands;
    // the band is at least as tall as its warm-up (q-1 blocks): 4096^2 101x101 20.5 vs 21.6 us at
    // 40 rows, 63x63 flat; a 2(q-1)B floor was slower (fewer warps)
    const bool piped = sstride ? v_wants_bulk(j) : v_wants_tma(j);  // TMA pipeline vs plain loads
    // plain loads: short bands (8192^2 63x63: rb 80 60.7 us, 160 64.2; cfg4's 1024-row images too:
    // 423 vs 406 Gpix/s with whole-image bands)
    if (!piped) rb = std::min(rb, 80);
    rb = std::max(rb, (p.q - 1) * B);
    // TMA path: bands of 320-640 rows (32768^2 63x63: rb 640 865 us, 160 895 us, one band per warp
    // per 2341 rows 1081 us)
    if (piped) rb = std::min(std::max(rb, 320), sstride ? 320 : 640);
    rb = env_int("sep_rb", rb);
    rb = std::max(B, (rb + B - 1) / B * B);
    p.rb = rb;
    vp->p = p;
    vp->B = B;
    vp->grid = dim3((unsigned)((p.nwords + VT - 1) / VT), (unsigned)((j.H + rb - 1) / rb), (unsigned)j.batch);
    return true;
}

cudaError_t run_v(const MorphJob& j, void* out, size_t op, size_t oimg, int pdl = 0, size_t sstride = 0) {
    VPlan vp;
    if (!plan_v(j, out, op, oimg, pdl, sstride, &vp)) return cudaErrorInvalidValue;
    MorphJob jo = j;  // the output side of the tensor maps
    jo.dst = out;
    jo.dp = op;
    jo.dimg = oimg;
    return launch_v(vp.p, j.elem, j.mode, vp.B, vp.grid, j.stream, jo);
}

// Plan of one horizontal pass over H rows: in -> job dst (stages = 2: this mode then the other, the
// two horizontal passes of an opening / closing).
struct HPlan {
    SepParams p;
    int C, bx;
    dim3 grid;
};
bool plan_h(const MorphJob& j, const void* in, size_t ip, size_t iimg, int discard, int stages, size_t dsstride,
            HPlan* hp) {
    int C = 0;
    if (!choose_c(j.elem, j.gx, &C)) return false;
    SepParams p = base_params(j);
    p.src = static_cast<const uint8_t*>(in);
    p.sp = ip;
    p.simg = iimg;
    p.dst = static_cast<uint8_t*>(j.dst);
    p.dp = j.dp;
    p.dimg = j.dimg;
    p.g = j.gx;
    p.groups = (j.H + 3) / 4;
    p.discard = discard;
    p.dsstride = dsstride;
    // parts: ~24 resident warps per SM, each part a whole number of segments
    const int A = stages * (j.gx / C + (j.gx % C ? 1 : 0));
    const int OS = (32 - 2 * A) * C;
    if (OS <= 0) return false;
    const int nseg = (j.W + OS - 1) / OS;
    const long long rowsw = (long long)p.groups * j.batch;
    // each warp keeps one segment in flight: parts of <= 8 segments (measured: 4096^2 u8 63x1 best
    // at 2 parts, 16384^2 at 4-5)
    int parts = (nseg + 7) / 8;
    parts = std::min(std::max(1, env_int("sep_parts", parts)), nseg);
    const int segs_per = (nseg + parts - 1) / parts;
    p.pw = segs_per * OS;
    p.parts = (nseg + segs_per - 1) / segs_per;
    const long long warps = rowsw * p.parts;
    hp->p = p;
    hp->C = C;
    hp->bx = bx_code(p.g, C);
    hp->grid = dim3((unsigned)((warps + HT / 32 - 1) / (HT / 32)));
    return true;
}

cudaError_t run_h(const MorphJob& j, const void* in, size_t ip, size_t iimg, int discard, int stages = 1,
                  size_t dsstride = 0) {
    HPlan hp;
    if (!plan_h(j, in, ip, iimg, discard, stages, dsstride, &hp)) return cudaErrorInvalidValue;
    const SepParams& p = hp.p;
    const int C = hp.C, bx = hp.bx;
    if (stages == 2) {
        if (j.elem == 1) return j.mode == MODE_MIN ? launch_hh_u8_min(p, C, bx, hp.grid, j.stream) : launch_hh_u8_max(p, C, bx, hp.grid, j.stream);
        return j.mode == MODE_MIN ? launch_hh_u16_min(p, C, bx, hp.grid, j.stream) : launch_hh_u16_max(p, C, bx, hp.grid, j.stream);
    }
    return launch_h(p, j.elem, j.mode, C, hp.grid, j.stream);
}

}  // namespace

bool applicable(const MorphJob& j) {
    const int enabled = env_int("sep", 1);
    if (!enabled) return false;
    if (j.mode != MODE_MIN && j.mode != MODE_MAX) return false;
    if (j.elem != 1 && j.elem != 2) return false;
    if (j.W < 1 || j.H < 1) return false;
    if ((reinterpret_cast<uintptr_t>(j.src) | reinterpret_cast<uintptr_t>(j.dst) | j.sp | j.dp |
         (j.batch > 1 ? (j.simg | j.dimg) : 0)) & 15)
        return false;
    if (j.gx == 0 && j.gy == 0) return false;
    int t;
    if (j.gy != 0 && !choose_b(j.elem, j.gy, &t)) return false;
    if (j.gx != 0 && !choose_c(j.elem, j.gx, &t)) return false;
    return true;
}

// Opening (j.mode = MODE_MIN first) / closing (MODE_MAX first) of whole images (no halo rows) in
// three launches instead of four: opening = Dv o (Dh o Eh) o Ev -- each separable op may run its
// passes in either order, so the two horizontal passes meet in the middle and run as one sweep
// (the intermediate between them never leaves registers; its column border is re-applied there).
bool compound_applicable(const MorphJob& j) {
    if (!applicable(j) || j.above || j.below || j.gx == 0 || j.gy == 0) return false;
    const int hh = env_int("sep_hh", 1);  // 0 off, 1 planner, 2 always (tests)
    if (!hh) return false;
    int C = 0;
    choose_c(j.elem, j.gx, &C);
    const int A = j.gx / C + (j.gx % C ? 1 : 0);
    if (2 * A > 10) return false;  // the left border fix needs the second segment clear of negative columns
    // the two-pass sweep with 16-column chunks needs 168-254 registers: on small images the four
    // passes of two H-first separable ops win (4096^2 u8 63x63 closing 35.9 vs 41.8 us; 16384^2
    // opening 429 vs 404 us)
    const long long px = (long long)j.W * j.H * j.batch;
    return hh == 2 || C == 8 || px >= (1LL << 26);
}

size_t compound_scratch_bytes(const MorphJob& j) {
    return 2 * (((size_t)j.W * j.elem + 255) & ~size_t(255)) * (size_t)j.H * (size_t)j.batch;
}

cudaError_t run_compound(const MorphJob& j, void* tmp) {
    const size_t tp = ((size_t)j.W * j.elem + 255) & ~size_t(255), timg = tp * (size_t)j.H;
    uint8_t* t1 = static_cast<uint8_t*>(tmp);
    uint8_t* t2 = t1 + timg * (size_t)j.batch;
    const int second = j.mode == MODE_MIN ? MODE_MAX : MODE_MIN;
    cudaError_t e = run_v(j, t1, tp, timg);  // first op, vertical
    if (e != cudaSuccess) return e;
    MorphJob h = j;  // first op horizontal, then second op horizontal: t1 -> t2
    h.dst = t2;
    h.dp = tp;
    h.dimg = timg;
    // the first intermediate's lines are dropped from L2 after their last read only while they can
    // still be there unwritten (on cfg4's 1 GiB they are long written back: the discards were 3% of
    // the sweep's instructions)
    const int discard = env_int("sep_discard", timg * (size_t)j.batch <= ((size_t)64 << 20) ? 1 : 0);
    if ((e = run_h(h, t1, tp, timg, discard, 2)) != cudaSuccess) return e;
    MorphJob v = j;  // second op, vertical: t2 -> dst (rows outside the image: the image border)
    v.mode = second;
    v.src = t2;
    v.sp = tp;
    v.simg = timg;
    return run_v(v, j.dst, j.dp, j.dimg, 1);
}

size_t scratch_pitch(const MorphJob& j) { return ((size_t)j.W * j.elem + 255) & ~size_t(255); }

// Rows per L2 band of the intermediate (the whole image when it fits).
int band_rows(const MorphJob& j) {
    const size_t budget = (size_t)env_int("sep_l2mb", 1 << 12) << 20;  // measured: banded launches fill the GPU worse than one pass over the image
    const size_t per_row = scratch_pitch(j) * (size_t)j.batch;
    const long long rows = std::max<long long>(64, (long long)(budget / std::max<size_t>(per_row, 1)));
    return (int)std::min<long long>(rows, j.H);
}

// H-first order (with its whole intermediate in one scratch) unless the image is too large for it
bool hfirst(const MorphJob& j) { return env_int("sep_hfirst", 1) && band_rows(j) == j.H; }

cudaError_t run(const MorphJob& j, void* tmp) {
    if (j.gy == 0) return run_h(j, j.src, j.sp, j.simg, 0);
    if (j.gx == 0) return run_v(j, j.dst, j.dp, j.dimg);
    const size_t tp = scratch_pitch(j);
    if (hfirst(j)) {
        // Horizontal pass first (src -> scratch, halo rows of a row band included), vertical second
        // (scratch -> dst). The latency-bound vertical pass then reads its 2-3 copies of every row
        // from L2 instead of HBM (4096^2: 63x63 20.9 vs 23.5 us, 101x101 23.6 vs 26.0); the scratch
        // is not discarded (several vertical bands read each row).
        // The vertical pass on loads (small / short images) reads a strip-major intermediate
        // (128-pixel strips, rows 128*sz bytes apart): every row of a block is then an immediate
        // offset from one base register.
        // (from 2^29 pixels the row-major intermediate + tensor-map TMA pass measured faster:
        // 32768^2 63x63 796 vs 809 us)
        const int IH = j.H + j.above + j.below;
        const bool smaj = !v_wants_tma(j) && env_int("sep_strip", 1) != 0;
        const size_t SB = (size_t)128 * j.elem;
        const size_t sstride = SB * (size_t)IH;
        const size_t rowp = smaj ? SB : tp;
        const size_t timg = smaj ? sstride * (size_t)((j.W + 127) / 128) : tp * (size_t)IH;
        MorphJob h = j;
        h.src = static_cast<const uint8_t*>(j.src) - (ptrdiff_t)j.above * (ptrdiff_t)j.sp;
        h.H = IH;
        h.above = h.below = 0;
        h.dst = tmp;
        h.dp = rowp;
        h.dimg = timg;
        cudaError_t e = run_h(h, h.src, j.sp, j.simg, 0, 1, smaj ? sstride : 0);
        if (e != cudaSuccess) return e;
        MorphJob v = j;  // rows [-above, H + below) of the scratch are valid
        v.src = static_cast<uint8_t*>(tmp) + (size_t)j.above * rowp;
        v.sp = rowp;
        v.simg = timg;
        return run_v(v, j.dst, j.dp, j.dimg, 1, smaj ? sstride : 0);
    }
    const int R = band_rows(j);
    const size_t timg = tp * (size_t)R;
    for (int y0 = 0; y0 < j.H; y0 += R) {
        MorphJob b = j;
        const int rows = std::min(R, j.H - y0);
        b.src = static_cast<const uint8_t*>(j.src) + (size_t)y0 * j.sp;
        b.dst = static_cast<uint8_t*>(j.dst) + (size_t)y0 * j.dp;
        b.H = rows;
        b.above = j.above + y0;
        b.below = j.below + (j.H - y0 - rows);
        cudaError_t e = run_v(b, tmp, tp, timg);
        if (e != cudaSuccess) return e;
        // discard the intermediate's lines only when the band can still be in L2 (measured: on a
        // 1 GiB intermediate the discards cost 7%)
        e = run_h(b, tmp, tp, timg, env_int("sep_discard", timg * b.batch <= (size_t)64 << 20 ? 1 : 0));
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

size_t scratch_bytes(const MorphJob& j) {
    if (j.gx == 0 || j.gy == 0) return 0;
    if (hfirst(j)) return scratch_pitch(j) * (size_t)(j.H + j.above + j.below) * (size_t)j.batch;
    return scratch_pitch(j) * (size_t)band_rows(j) * (size_t)j.batch;
}

const char* plan_name(const MorphJob& j) {
    static thread_local char buf[96];
    if (!applicable(j)) return nullptr;
    int B = 0, C = 0;
    if (j.gy) choose_b(j.elem, j.gy, &B);
    if (j.gx) choose_c(j.elem, j.gx, &C);
    snprintf(buf, sizeof buf, "sep_%s_vB%d_hC%d_band%d", j.elem == 1 ? "u8" : "u16", B, C,
             (j.gx && j.gy) ? band_rows(j) : 0);
    return buf;
}

}  // namespace sep
}  // namespace rmgpu

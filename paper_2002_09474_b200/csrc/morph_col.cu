// morph_col.cu -- planner for K1 v4, the register-streaming fused kernel for small windows.
//
// Design (B200-first; reference semantics from separable.cpp:35-83,130-146 and image.cpp:58-66):
//   * Every warp is an independent pipeline. A warp owns a strip of 512 bytes of columns
//     (512 u8 / 256 u16 pixels; 16 bytes per lane) and walks work items = (strip, band of R output
//     rows, image) persistently. Its input rows (+/- wy/2 halo rows, +/- 16 halo bytes) arrive
//     in 8-row 2-D TMA boxes in a private 3-slot shared-memory ring (one mbarrier per slot),
//     issued by the warp itself 2 blocks ahead, across item boundaries. No CTA barriers at all.
//   * Each staged row is read once with one 128-bit LDS per lane. u8 pixels stay packed: the
//     16-bit min/max of a raw word is exact in its high bytes (the odd pixels), and of its
//     byte-swapped copy (one PRMT) for the even pixels, so 2 pixels / VIMNMX(3).U16x2 with no
//     unpacking. The vertical window keeps the last wy rows in registers (ring indexed by the
//     unrolled row); the horizontal window shifts 16-bit lanes with PRMT and crosses lanes with
//     SHFL (lanes 0 / 31 use the staged halo word), then one PRMT per 4 pixels repacks bytes.
//   * Results leave with one 128-bit store per lane per row (512 contiguous bytes per warp).
//   Border strips (first / last) fix out-of-image columns with per-lane PRMT selectors (replicate:
//   the row's first / last pixel; constant: the border value); border row blocks are staged row by
//   row from clamped rows (or filled with the constant). Every pixel is read from HBM once and
//   written once; halo rows are L2 hits.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "morph_col.cuh"

namespace rmgpu {
namespace col {
cudaError_t dispatch_u8_min(const MorphJob&, int);
cudaError_t dispatch_u8_max(const MorphJob&, int);
cudaError_t dispatch_u16_min(const MorphJob&, int);
cudaError_t dispatch_u16_max(const MorphJob&, int);
cudaError_t dispatch_u8_grad(const MorphJob&, int);
cudaError_t dispatch_u16_grad(const MorphJob&, int);

namespace {

bool choose(const MorphJob& j, int* R) {
    if (j.mode != MODE_MIN && j.mode != MODE_MAX && j.mode != MODE_GRAD) return false;
    if (j.elem != 1 && j.elem != 2) return false;
    if (j.gx > GMAX || j.gy > GMAX) return false;
    if (getenv("RMGPU_NO_COL")) return false;
    const uintptr_t src0 = reinterpret_cast<uintptr_t>(j.src) - (uintptr_t)((size_t)j.above * j.sp);
    if ((src0 | j.sp | reinterpret_cast<uintptr_t>(j.dst) | j.dp) & 15) return false;
    if (j.batch > 1 && ((j.simg | j.dimg) & 15)) return false;
    // rows per item: chosen at launch from the kernel's occupancy (wave model, morph_col.cuh);
    // RMGPU_COL_BLOCKS=m forces R = m * BR - 2 * gy (tuning)
    *R = 0;
    if (const char* e = getenv("RMGPU_COL_BLOCKS")) *R = std::max(1, atoi(e) * BR - 2 * j.gy);
    return true;
}

}  // namespace

bool launch(const MorphJob& j, cudaError_t* err) {
    int R = 0;
    if (!choose(j, &R)) return false;
    if (j.elem == 1)
        *err = j.mode == MODE_MIN ? dispatch_u8_min(j, R) : j.mode == MODE_MAX ? dispatch_u8_max(j, R) : dispatch_u8_grad(j, R);
    else
        *err = j.mode == MODE_MIN ? dispatch_u16_min(j, R)
                                  : j.mode == MODE_MAX ? dispatch_u16_max(j, R) : dispatch_u16_grad(j, R);
    return true;
}

const char* plan_name(const MorphJob& j) {
    static thread_local char buf[96];
    MorphJob k = j;
    k.src = nullptr;
    k.dst = nullptr;
    k.sp = k.dp = (size_t)((j.W * j.elem + 15) / 16 * 16);
    k.simg = k.dimg = k.sp * j.H;
    int R = 0;
    if (!choose(k, &R)) return nullptr;
    snprintf(buf, sizeof(buf), "col_%s_w%dx%d_R%s_smem%dK", j.elem == 1 ? "u8" : "u16", 2 * j.gx + 1, 2 * j.gy + 1,
             R > 0 ? std::to_string(R).c_str() : "auto",
             (j.gx == 0 ? ColGeo<0>::SMEM : ColGeo<1>::SMEM) / 1024);
    return buf;
}

}  // namespace col
}  // namespace rmgpu

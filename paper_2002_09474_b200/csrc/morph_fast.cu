// morph_fast.cu -- K1/K2: the fused separable erosion / dilation kernel (u8 and u16).
//
// One CTA owns an output tile of TH rows x TW columns and does, entirely on chip:
//   1. vertical pass (separable.cpp:141-143, vertical_pass_direct / vertical_pass_via_transpose)
//      straight from global memory: one thread per (4-pixel u8 | 2-pixel u16) column word of the
//      tile plus its horizontal halo, sweeping down the rows. Border rows are resolved by clamping
//      the row index (replicate) or substituting the constant (image.cpp:58-66); border columns by a
//      per-thread byte permutation fixed at kernel start. Pixels live in 16-bit lanes so every
//      min/max is one VIMNMX(3).U16x2 (SURVEY.md finding 4).
//   2. the vertical results are written to shared memory TRANSPOSED (4x4 u8 / 2x2 u16 blocks
//      through PRMT): the paper's transpose trick done in registers, so the
//      horizontal pass is again a sweep over "columns" of words -- no global transpose.
//   3. horizontal pass (separable.cpp:62-83) over the transposed tile, one thread per row group.
//   4. the tile is transposed back in registers, staged in shared memory and written with 16-byte
//      coalesced stores. Each pixel is read from HBM once and written once.
//
// Each 1-D pass uses either a direct window (w = 3, 5: one or two 3-input min/max per output,
// the "linear" algorithm of sliding_extrema.cpp:28-37) or the van Herk / Gil-Werman block
// decomposition (sliding_extrema.cpp:58-132) re-designed for a fixed register block of B
// samples: a window [o, o+w-1] is split at the start of the block holding its right end, so
// out = op(suffix_min(x[o .. blockstart-1]), prefix_min(block[0 .. m])). The suffix runs backward
// over the B left ends of one emission, seeded with the min of the gap between them and the block
// (r tail samples plus q-1 whole-block minima). Cost per output ~3 min/max + (r+q)/B for any w,
// with B a compile-time constant (registers) and w, q, r runtime values.
#include <cstdio>

#include "morph_fast.cuh"

namespace rmgpu {
namespace fast {
cudaError_t dispatch_u8_min(const MorphJob& j, int vv, int hv);
cudaError_t dispatch_u8_max(const MorphJob& j, int vv, int hv);
cudaError_t dispatch_u16_min(const MorphJob& j, int vv, int hv);
cudaError_t dispatch_u16_max(const MorphJob& j, int vv, int hv);
}  // namespace fast

namespace {
using namespace fast;

bool covered(const MorphJob& j, int* vv, int* hv) {
    if (j.mode != MODE_MIN && j.mode != MODE_MAX) return false;
    if (j.elem != 1 && j.elem != 2) return false;
    // 4-byte aligned column words for every row: base and pitch multiples of 4 (the reference's
    // stride is a multiple of 16, image.cpp:9-14)
    if ((reinterpret_cast<uintptr_t>(j.src) | j.sp | j.simg) & 3) return false;
    // a row must hold whole words (pitch >= width rounded up to the word) so edge loads stay in-row
    const size_t px = j.elem == 1 ? 4 : 2;
    if (j.sp < ((size_t)j.W + px - 1) / px * px * j.elem) return false;
    *vv = pick_variant(j.gy);
    *hv = pick_variant(j.gx);
    if (*vv == 0 || *hv == 0) return false;
    const size_t smem = j.elem == 1 ? fast_smem<uint8_t>(j.gx) : fast_smem<uint16_t>(j.gx);
    return smem <= 200 * 1024;
}

}  // namespace

bool launch_fast(const MorphJob& j, cudaError_t* err) {
    int vv, hv;
    if (!covered(j, &vv, &hv)) return false;
    if (j.elem == 1)
        *err = j.mode == MODE_MIN ? fast::dispatch_u8_min(j, vv, hv) : fast::dispatch_u8_max(j, vv, hv);
    else
        *err = j.mode == MODE_MIN ? fast::dispatch_u16_min(j, vv, hv) : fast::dispatch_u16_max(j, vv, hv);
    return true;
}

const char* fast_plan_name(const MorphJob& j) {
    static thread_local char buf[96];
    MorphJob k = j;
    if (k.mode == MODE_GRAD) return nullptr;
    k.src = nullptr;
    k.sp = (size_t)((j.W + 3) / 4 * 4) * j.elem;
    int vv, hv;
    if (!covered(k, &vv, &hv)) return nullptr;
    snprintf(buf, sizeof(buf), "fused_%s_v%s%d_h%s%d", j.elem == 1 ? "u8" : "u16", vv <= 5 ? "d" : "b", vv,
             hv <= 5 ? "d" : "b", hv);
    return buf;
}

}  // namespace rmgpu

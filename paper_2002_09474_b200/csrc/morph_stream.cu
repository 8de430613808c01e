// morph_stream.cu -- planner for K1/K2 v2, the warp-specialised strip-streaming fused kernel.
//
// Design (B200-first; reference semantics from separable.cpp:130-157, sliding_extrema.cpp,
// image.cpp:58-66):
//   * A CTA owns a vertical strip of TW output columns (256 px u8 / 128 px u16) and a long run
//     of rows. Its input rows (strip + horizontal halo, 16-byte aligned) stream into a
//     shared-memory ring through cp.async.bulk (TMA bulk copies, one per row, completion on an
//     mbarrier per ring slot). Replicate borders clamp the source row; constant rows are filled
//     with the border value; border columns are fixed per thread with one PRMT.
//   * 4 "vertical" warps: one thread per 4-pixel (u8) / 2-pixel (u16) column word, sweeping down
//     the ring. Small windows use a direct window (3-input VIMNMX3.U16x2); larger ones the van
//     Herk / Gil-Werman decomposition with a compile-time register block of B rows: prefix of
//     the leading block, suffix of the trailing run seeded with the gap minimum (r tail rows +
//     q-1 whole-block minima carried in registers). ~3 min/max per output for any window.
//     Results are transposed in registers (PRMT) into a double-buffered shared tile.
//   * 4 "horizontal" warps: one warp per 4-row (u8) / 2-row (u16) group of a chunk. Each lane
//     owns an 8-column chunk of the strip: prefix to a per-warp scratch, suffix in registers,
//     chunk minima combined for the gap; outputs are transposed back to rows in registers,
//     staged, and written with 16-byte coalesced stores.
//   * Vertical and horizontal warps hand chunks over with named barriers, so loading, the
//     vertical sweep and the horizontal sweep of different chunks overlap. Every pixel is read
//     from HBM once and written once (halo rows/columns are re-read from L2 by neighbours).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "morph_stream.cuh"

namespace rmgpu {
namespace stream {
long long* g_trace = nullptr;
int g_trace_cta = 0;
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
        for (int B : {8, 16, 24}) {
            if (B > w1) continue;
            const int q = w1 / B, r = w1 - q * B;
            if (q > QMAX) continue;
            const double cost = 3.0 + double(r + q) / B;
            if (cost < best - 1e-9) {
                best = cost;
                c->vb = B;
                c->B = B;
                c->q = q;
            }
        }
        if (!c->vb) return false;
    }
    c->hb = j.gx <= 3 ? 2 * j.gx + 1 : (j.gx <= stream_gxmax(j.elem, 8) ? 8 : 9);
    if (j.gx > stream_gxmax(j.elem, c->hb)) return false;
    // TMA prefetch depth: keep ~56 KB of input in flight per SM (Little's law at ~1 us DRAM
    // latency under load and 6.5 TB/s over 148 SMs), within the shared-memory budget.
    const int blk = c->B * (j.elem == 1 ? stream_ring_row<uint8_t>(c->hb) : stream_ring_row<uint16_t>(c->hb));
    auto smem_of = [&](int pf) {
        return j.elem == 1 ? stream_smem<uint8_t>(c->hb, c->B, c->q, pf) : stream_smem<uint16_t>(c->hb, c->B, c->q, pf);
    };
    int pf = 2, total = smem_of(pf);
    if (total > 220 * 1024) return false;
    if (const char* e = getenv("RMGPU_STREAM_PF")) {
        pf = std::max(1, atoi(e));
        total = smem_of(pf);
    } else {
        for (int cand = 2; cand <= 12; ++cand) {
            const int t = smem_of(cand);
            if (t > 220 * 1024) break;
            const int occ = std::max(1, std::min(8, (227 * 1024) / (t + 1024)));
            pf = cand;
            total = t;
            if ((long)cand * blk * occ >= 56 * 1024) break;
        }
    }
    c->pf = pf;
    c->smem = total;
    // rows per CTA: enough CTAs for ~2 waves of the resident capacity, long runs for big windows
    const int occ = std::max(1, std::min(8, (227 * 1024) / (total + 1024)));
    const long strips = (long)((j.W + tw - 1) / tw) * j.batch;
    const long target = 148L * occ * 2;
    long splits = std::max(1L, (target + strips - 1) / strips);
    int rh = (int)((j.H + splits - 1) / splits);
    rh = std::max(rh, std::min(j.H, std::max(64, 2 * w1)));
    rh = (rh + 3) / 4 * 4;
    if (const char* e = getenv("RMGPU_STREAM_RH")) {  // tuning hook
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
        *err = j.mode == MODE_MIN ? dispatch_u8_min(j, c.vb, c.hb, c.rh, c.B, c.q, c.pf) : dispatch_u8_max(j, c.vb, c.hb, c.rh, c.B, c.q, c.pf);
    else
        *err = j.mode == MODE_MIN ? dispatch_u16_min(j, c.vb, c.hb, c.rh, c.B, c.q, c.pf) : dispatch_u16_max(j, c.vb, c.hb, c.rh, c.B, c.q, c.pf);
    return true;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

bool encode_input_map(const MorphJob& j, int box_words, int box_rows, CUtensorMap* map) {
    memset(map, 0, sizeof(*map));
    if (getenv("RMGPU_NO_TMA")) return false;
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const size_t row_bytes = (size_t)j.W * j.elem;
    const long rows = (long)j.above + j.H + j.below;
    if (j.sp % 16 || (j.batch > 1 && j.simg % 16) || rows < 1) return false;
    const uint8_t* base = static_cast<const uint8_t*>(j.src) - (ptrdiff_t)j.above * (ptrdiff_t)j.sp;
    if (reinterpret_cast<uintptr_t>(base) & 15) return false;
    cuuint64_t dims[3] = {(row_bytes + 3) / 4, (cuuint64_t)rows, (cuuint64_t)std::max(1, j.batch)};
    cuuint64_t strides[2] = {j.sp, j.batch > 1 ? j.simg : j.sp * (cuuint64_t)rows};
    cuuint32_t box[3] = {(cuuint32_t)box_words, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_output_map(const MorphJob& j, int box_bytes, int box_rows, CUtensorMap* map) {
    memset(map, 0, sizeof(*map));
    if (getenv("RMGPU_NO_TMA")) return false;
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    if (j.dp % 16 || (j.batch > 1 && j.dimg % 16) || (reinterpret_cast<uintptr_t>(j.dst) & 15)) return false;
    cuuint64_t dims[3] = {(cuuint64_t)j.W * j.elem, (cuuint64_t)j.H, (cuuint64_t)std::max(1, j.batch)};
    cuuint64_t strides[2] = {j.dp, j.batch > 1 ? j.dimg : j.dp * (cuuint64_t)j.H};
    cuuint32_t box[3] = {(cuuint32_t)box_bytes, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, j.dst, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

void set_trace(long long* buf, int cta) {
    g_trace = buf;
    g_trace_cta = cta;
}

const char* plan_name(const MorphJob& j) {
    static thread_local char buf[96];
    MorphJob k = j;
    k.src = nullptr;
    k.sp = (size_t)((j.W * j.elem + 15) / 16 * 16);
    Choice c;
    if (!choose(k, &c)) return nullptr;
    snprintf(buf, sizeof(buf), "stream_%s_v%s%d_h%s%d_rh%d_pf%d_smem%dK", j.elem == 1 ? "u8" : "u16",
             c.vb <= 7 ? "d" : "b", c.vb, c.hb <= 7 ? "d" : "b", c.hb, c.rh, c.pf, c.smem / 1024);
    return buf;
}

}  // namespace stream
}  // namespace rmgpu

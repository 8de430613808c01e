// morph_stream.cu -- host side of the shared TMA infrastructure (morph_stream.cuh): tensor-map
// encoding through the driver entry point (cuTensorMapEncodeTiled) for the input / output maps of
// the fused kernels, and the debug-trace hook of the phase kernel (tools/trace_phase.py).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "morph_stream.cuh"

namespace rmgpu {
namespace stream {
long long* g_trace = nullptr;
int g_trace_cta = 0;
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

}  // namespace stream
}  // namespace rmgpu

// kernels.h -- internal launcher interface between the C-ABI (capi.cu) and the
// kernel translation units. Host code only; no torch types anywhere.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace rmgpu {

// One separable rectangle reduction over a pitched image (or row band).
struct MorphJob {
    const void* src = nullptr;  // points at output row 0 of the input
    size_t sp = 0;              // source pitch, bytes
    void* dst = nullptr;
    size_t dp = 0;              // destination pitch, bytes
    int W = 0, H = 0;           // output extent
    int above = 0, below = 0;   // valid input rows before row 0 / after row H-1 (row bands)
    int gx = 0, gy = 0;         // wings (window = 2g+1), already clamped to the valid extent
    int mode = 0;               // Mode (common.cuh)
    int cmode = 0;              // 0 replicate, 1 constant
    uint32_t bval = 0;          // constant border value
    int elem = 1;               // bytes per pixel: 1 (u8) or 2 (u16)
    int batch = 1;              // independent images (gridDim.z)
    size_t simg = 0, dimg = 0;  // bytes between consecutive images (batch > 1)
    cudaStream_t stream = nullptr;
    int algo_h = 0, algo_v = 0;  // rmgpu_algo hints (Auto / Linear / VanHerk); never change results
};

// ---- launch bookkeeping (capi.cu): cached per (kernel, device) so a launch costs no extra
// driver round trips. Sets the dynamic shared-memory limit on first use; returns resident CTAs
// per SM (0 and an error on failure).
int kernel_occupancy(const void* kern, int threads, int smem, cudaError_t* err);
int device_sm_count();
// Planner knob: the rmgpu_debug_set override if any, else the environment variable RMGPU_<NAME>
// (upper-cased), else dflt.
int tune(const char* name, int dflt);

// ---- generic paths (morph_generic.cu): any window, any pitch --------------------------------
bool generic_tile_fits(const MorphJob& j);
cudaError_t launch_generic_tile(const MorphJob& j);
// 1-D pass along rows (uses gx) or columns (uses gy, above, below); any window size.
cudaError_t launch_pass_rows(const MorphJob& j);
cudaError_t launch_pass_cols(const MorphJob& j);
// dst = a - b (wrapping, dispatch.cpp:68), pitched, elem 1 or 2
cudaError_t launch_subtract(const void* a, size_t ap, const void* b, size_t bp, void* dst,
                            size_t dp, int W, int H, int elem, cudaStream_t s);

// ---- shared TMA infrastructure (morph_stream.cu) -----------------------------------------------
namespace stream {
void set_trace(long long* device_buf, int cta);  // debug timeline of the phase kernel (tools/trace_phase.py)
}  // namespace stream

// ---- persistent phase-based fused path (morph_phase.cu), preferred over the streaming one -----
namespace phase {
bool launch(const MorphJob& j, cudaError_t* err);
const char* plan_name(const MorphJob& j);
}  // namespace phase

// ---- register-streaming fused path for small windows (morph_col.cu), preferred over phase ----
namespace col {
bool launch(const MorphJob& j, cudaError_t* err);
const char* plan_name(const MorphJob& j);
}  // namespace col

// ---- K3: vertical and horizontal streaming passes handing over through L2 (morph_sep.cu) ------
namespace sep {
bool applicable(const MorphJob& j);
size_t scratch_bytes(const MorphJob& j);  // 0: no intermediate (one axis has window 1)
cudaError_t run(const MorphJob& j, void* tmp);
const char* plan_name(const MorphJob& j);
// opening (mode MIN first) / closing (MAX first) in three launches; whole images only
bool compound_applicable(const MorphJob& j);
size_t compound_scratch_bytes(const MorphJob& j);
cudaError_t run_compound(const MorphJob& j, void* tmp);
}  // namespace sep

// ---- K4: the separable rectangle in one kernel, intermediate in shared memory (morph_fuse.cu) ----
namespace fuse {
bool launch(const MorphJob& j, cudaError_t* err);  // false: K4 does not take this job
const char* plan_name(const MorphJob& j);
}  // namespace fuse

// ---- transposes (transpose.cu) ---------------------------------------------------------------
cudaError_t launch_transpose(const void* src, size_t sp, void* dst, size_t dp, int W, int H,
                             int elem, cudaStream_t s);
cudaError_t launch_transpose_tiles(void* data, size_t n_tiles, int n, size_t row_stride,
                                   size_t tile_step, int elem, cudaStream_t s);

// ---- generator (generate.cu) -----------------------------------------------------------------
cudaError_t launch_generate(void* dst, size_t pitch, int W, int H, uint64_t seed, uint64_t stream_id,
                            int elem, cudaStream_t s);

}  // namespace rmgpu

// morph_sep_h_u8_min.cu -- K3 horizontal-pass instantiations (u8, min); see morph_sep.cuh.
#include "morph_sep.cuh"

namespace rmgpu {
namespace sep {

cudaError_t launch_h_u8_min(const SepParams& p, int C, int bx, dim3 grid, cudaStream_t s) {
    switch (C * 100 + bx) {
#define RM_H(CC, BB)                                                  \
    case CC * 100 + BB:                                               \
        return launch_hk(hpass_kernel<uint8_t, MODE_MIN, CC, BB>, p, grid, s);
        RM_H(16, 0) RM_H(16, 1) RM_H(16, 2) RM_H(16, 3) RM_H(16, 4) RM_H(16, 5) RM_H(16, 6) RM_H(16, 7) \
        RM_H(16, 8) RM_H(16, 9) RM_H(16, 10) RM_H(16, 11) RM_H(16, 12) RM_H(16, 13) RM_H(16, 14) RM_H(16, 15) \
        RM_H(8, 4) RM_H(8, 5) RM_H(8, 6) RM_H(8, 7) \
        RM_H(16, 36) RM_H(16, 37) RM_H(16, 38) RM_H(16, 39)
#undef RM_H
    }
    return cudaErrorInvalidValue;
}

// two horizontal passes (this mode, then the other) in one sweep: opening / closing
cudaError_t launch_hh_u8_min(const SepParams& p, int C, int bx, dim3 grid, cudaStream_t s) {
    switch (C * 100 + bx) {
#define RM_H(CC, BB)                                                  \
    case CC * 100 + BB:                                               \
        return launch_hk(hpass_kernel<uint8_t, MODE_MIN, CC, BB, 2>, p, grid, s);
        RM_H(16, 0) RM_H(16, 1) RM_H(16, 2) RM_H(16, 3) RM_H(16, 4) RM_H(16, 5) RM_H(16, 6) RM_H(16, 7) \
        RM_H(16, 8) RM_H(16, 9) RM_H(16, 10) RM_H(16, 11) RM_H(16, 12) RM_H(16, 13) RM_H(16, 14) RM_H(16, 15) \
        RM_H(8, 4) RM_H(8, 5) RM_H(8, 6) RM_H(8, 7) \
        RM_H(16, 36) RM_H(16, 37) RM_H(16, 38) RM_H(16, 39)
#undef RM_H
    }
    return cudaErrorInvalidValue;
}

}  // namespace sep
}  // namespace rmgpu

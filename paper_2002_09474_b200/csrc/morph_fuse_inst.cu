// morph_fuse_inst.cu -- K4 instantiations for one (pixel size, mode, block size B), selected at
// build time: build.py compiles this file once per variant with -DFUSE_SZ={1,2} -DFUSE_MAX={0,1}
// -DFUSE_B={12,20} (u8) / {8,12} (u16). Each object holds every horizontal chunk class g mod C of that B
// (+ the u8 short-wing variants 36..39, see sep::h_lane_pass).
#include "morph_fuse.cuh"

#ifndef FUSE_SZ
#define FUSE_SZ 1
#define FUSE_MAX 0
#define FUSE_B 20
#endif

#if FUSE_SZ == 1
#define FUSE_T uint8_t
#define FUSE_TN u8
#else
#define FUSE_T uint16_t
#define FUSE_TN u16
#endif
#if FUSE_MAX
#define FUSE_MODE MODE_MAX
#define FUSE_MN max
#else
#define FUSE_MODE MODE_MIN
#define FUSE_MN min
#endif

#define RM_CAT_(a, b, c, d) a##b##_##c##_b##d
#define RM_CAT(a, b, c, d) RM_CAT_(a, b, c, d)

namespace rmgpu {
namespace fuse {

cudaError_t launch_kernel(const void* kern, const FuseParams& p, dim3 grid, int smem, cudaStream_t s,
                          const CUtensorMap& map, const CUtensorMap& gmap);

// launch_<tn><mode>_b<B>(params, bxs, ...): cudaErrorInvalidValue when bxs has no instantiation
cudaError_t RM_CAT(launch_, FUSE_TN, FUSE_MN, FUSE_B)(const FuseParams& p, int bxs, dim3 grid, int smem,
                                                       cudaStream_t s, const CUtensorMap& map,
                                                       const CUtensorMap& gmap) {
    switch (bxs) {
#define RM_F(X)                                                                                              \
    case X:                                                                                                  \
        return launch_kernel((const void*)fused_kernel<FUSE_T, FUSE_MODE, FUSE_B, X>, p, grid, smem, s, map, \
                             gmap);
        RM_F(0) RM_F(1) RM_F(2) RM_F(3) RM_F(4) RM_F(5) RM_F(6) RM_F(7)
#if FUSE_SZ == 1
        RM_F(8) RM_F(9) RM_F(10) RM_F(11) RM_F(12) RM_F(13) RM_F(14) RM_F(15)
        RM_F(36) RM_F(37) RM_F(38) RM_F(39)
#endif
#undef RM_F
    }
    return cudaErrorInvalidValue;
}

}  // namespace fuse
}  // namespace rmgpu

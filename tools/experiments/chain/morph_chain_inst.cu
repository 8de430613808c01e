// morph_chain_inst.cu -- K5 instantiations; compiled once per (pixel size, mode, stage count, part):
// -DCHAIN_SZ=1|2 -DCHAIN_MAX=0|1 -DCHAIN_NS=2|3 -DCHAIN_PART=0..3 (see build.py). A part is a
// quarter of the horizontal variants (parallel builds).
#include "morph_chain.cuh"

#ifndef CHAIN_SZ
#define CHAIN_SZ 1
#endif
#ifndef CHAIN_MAX
#define CHAIN_MAX 0
#endif
#ifndef CHAIN_NS
#define CHAIN_NS 2
#endif
#ifndef CHAIN_PART
#define CHAIN_PART 0
#endif

namespace rmgpu {
namespace sep {

#define CHAIN_CAT2(a, b, c, d, e) a##b##_##c##_##d##_##e
#define CHAIN_CAT(a, b, c, d, e) CHAIN_CAT2(a, b, c, d, e)
#if CHAIN_SZ == 1
using CT_T = uint8_t;
#define CHAIN_TN u8
#else
using CT_T = uint16_t;
#define CHAIN_TN u16
#endif
#if CHAIN_MAX
#define CHAIN_MN max
#else
#define CHAIN_MN min
#endif
#define CHAIN_FN CHAIN_CAT(launch_chain_, CHAIN_TN, CHAIN_MN, CHAIN_NS, CHAIN_PART)

// grid.x == 0: only report the resident CTAs per SM (cached occupancy query). Returns
// cudaErrorInvalidValue when this part does not hold the variant.
cudaError_t CHAIN_FN(const ChainParams& cp, int var, dim3 grid, cudaStream_t s, int* occ) {
    constexpr int M = CHAIN_MAX ? MODE_MAX : MODE_MIN;
    void (*kern)(const ChainParams) = nullptr;
    switch (var) {
#define RM_CK(CC, BB) \
    case CC * 100 + BB: kern = chain_kernel<CT_T, M, CC, BB, CHAIN_NS>; break;
#if CHAIN_SZ == 1 && CHAIN_NS == 2
#if CHAIN_PART == 0
        RM_CK(16, 0) RM_CK(16, 1) RM_CK(16, 2) RM_CK(16, 3) RM_CK(16, 4) RM_CK(16, 5)
#elif CHAIN_PART == 1
        RM_CK(16, 6) RM_CK(16, 7) RM_CK(16, 8) RM_CK(16, 9) RM_CK(16, 10) RM_CK(16, 11)
#elif CHAIN_PART == 2
        RM_CK(16, 12) RM_CK(16, 13) RM_CK(16, 14) RM_CK(16, 15) RM_CK(8, 4) RM_CK(8, 5)
#else
        RM_CK(8, 6) RM_CK(8, 7) RM_CK(16, 36) RM_CK(16, 37) RM_CK(16, 38) RM_CK(16, 39)
#endif
#elif CHAIN_SZ == 1
#if CHAIN_PART == 0
        RM_CK(8, 4) RM_CK(8, 5) RM_CK(8, 6) RM_CK(8, 7)  // 8-column chunks only (registers)
#endif
#else
#if CHAIN_PART == 0
        RM_CK(8, 0) RM_CK(8, 1)
#elif CHAIN_PART == 1
        RM_CK(8, 2) RM_CK(8, 3)
#elif CHAIN_PART == 2
        RM_CK(8, 4) RM_CK(8, 5)
#else
        RM_CK(8, 6) RM_CK(8, 7)
#endif
#endif
#undef RM_CK
    }
    if (!kern) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    *occ = kernel_occupancy((const void*)kern, CT, 0, &e);
    if (e != cudaSuccess || grid.x == 0) return e;
    kern<<<grid, CT, 0, s>>>(cp);
    return cudaGetLastError();
}

}  // namespace sep
}  // namespace rmgpu
